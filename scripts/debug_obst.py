import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.step import OracleSolver
from oracle.tt import TtTensor, rel_err
from paper_1912_04582_b200.cuda import Context
from paper_1912_04582_b200.problems import obstacle_flow
from paper_1912_04582_b200.tt_batch import TtBatch
p = obstacle_flow((5, 4, 4), hole=2, nv=16, seed=9)
ctx = Context(0)
ctx.setup(p)
rng = np.random.default_rng(1)
f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
f = [(t + t.scaled(0.05 * rng.uniform())).rounded(1e-12) for t in f]
ctx.upload_state(TtBatch.from_list(f))
ctx.step(p.dt, p.eps, p.cap, 1)
phi = ctx.stage("phi")
solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
m = p.mesh
out = {}
for j in range(m.nface):
    want = solver.face_flux(f, j, p.eps, p.cap)
    e = rel_err(phi.full(j), want.to_full())
    g = int(m.face_group[j]); r = int(m.face_right[j])
    kind = "interior" if r >= 0 else p.bcs[g]["kind"]
    print(j, kind, m.face_normal[j].round(4), "err %.3e" % e, tuple(phi.ranks[j]), want.ranks()[1:3])
np.savez("gpurun_out/debug_obst.npz", phi_cores=phi.cores, phi_ranks=phi.ranks, phi_off=phi.offsets)
