"""|xi_n| estimate of one face normal of config 4: GPU against the compiled reference,
with the h-search diagnostics (best / runner-up Frobenius error, chosen candidate)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from oracle.tt import rel_err  # noqa: E402
from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

faces = [int(v) for v in sys.argv[1:]] or [1195060, 939902]
p = config(4)
nrm = p.mesh.face_normal[faces]
ctx = Context(0)
ctx.set_grid(p.nv, p.bound)
out = ctx.face_factors(nrm, 4, "abs", diag=True)
got, diag = out if isinstance(out, tuple) else (out, None)
r = ref.RefSolver(p.nv, p.bound, p.gas)
want = r.face_factors(nrm, 4, 0)
for i, f in enumerate(faces):
    print("face", f, "normal", nrm[i], "ranks gpu", got.ranks[i], "ref", want.ranks[i], "rel diff E",
          rel_err(got.full(i), want.full(i)))
    if diag is not None:
        d = np.asarray(diag).reshape(len(faces), -1)[i]
        print("   diag [best err2, runner-up err2, choice, min kept sigma^2 ratio]:", d,
              " relative gap", (d[1] - d[0]) / d[0])
