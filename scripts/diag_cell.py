"""Stage-by-stage GPU-vs-reference comparison of ONE cell of the full config-4 run
(diagnostics for a parity-block outlier): fluxes of its faces, J, R, new state."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from oracle.tt import rel_err  # noqa: E402
from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.partition import build_part  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

cell = int(sys.argv[1]) if len(sys.argv) > 1 else 15606
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = config(4)
m = p.mesh
ctx = Context(0)
ctx.setup(p)
ctx.step(p.dt, p.eps, p.cap, steps - 1)
prev = ctx.download_state()
ctx.step(p.dt, p.eps, p.cap, 1)
new = ctx.download_state()
owner = np.ones(m.ncell, dtype=np.int32)
owner[cell] = 0
part = build_part(m, owner, 0)
loc = prev.subset(part.local_to_global)
r = ref.RefSolver(p.nv, p.bound, p.gas, part.mesh, p.bcs)
r.set_state(loc)
r.step(p.dt, p.eps, p.cap, cells=np.arange(1, dtype=np.int32))
want = r.state()
print("cell", cell, "ranks before", prev.ranks[cell], "after gpu", new.ranks[cell], "ref", want.ranks[0])
print("state rel err", rel_err(new.full(cell), want.full(0)))
faces = [(fid, s) for fid, s in part.mesh.cell_faces(0)]
print("faces (local id, sign, group, right):", [(f, s, int(part.mesh.face_group[f]), int(part.mesh.face_right[f])) for f, s in faces])
gphi = ctx.stage("phi")
rphi = r.fetch(r.PHI)
for f, s in faces:
    g = int(part.face_global[f])
    a, b = gphi.full(g), rphi.full(f)
    print(f"  phi face {g}: ranks gpu {gphi.ranks[g]} ref {rphi.ranks[f]} rel diff {rel_err(a, b):.3e} "
          f"norm {np.linalg.norm(b):.3e} normal {m.face_normal[g].round(4)} group {int(m.face_group[g])}")
gj, rj = ctx.stage("jr"), r.fetch(r.J)
mac = ctx.macros()
print("  J: ranks gpu", gj.ranks[cell], "ref", rj.ranks[0], "rel diff",
      rel_err(gj.full(cell) * mac[cell, 10], rj.full(0)), "norm", np.linalg.norm(rj.full(0)))
gr, rr = ctx.stage("res"), r.fetch(r.R)
print("  R: ranks gpu", gr.ranks[cell], "ref", rr.ranks[0], "rel diff", rel_err(gr.full(cell), rr.full(0)),
      "norm", np.linalg.norm(rr.full(0)), "||f||", np.linalg.norm(prev.full(cell)))
wd = ctx.wall_densities()
print("  wall densities (first 5):", wd[:5])
