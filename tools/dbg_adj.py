import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import oracle
import paper_2410_10503_b200 as m
np.set_printoptions(linewidth=200, precision=3, suppress=True)
for g in [(8, 8, 4, 12, 1.0), (8, 8, 6, 12, 1.0), (9, 7, 5, 13, 1.0)]:
    geom = m.Geometry(*g)
    op = m.RayTransform(geom)
    orc = oracle.RayTransform(oracle.Geometry(*g))
    for a in range(g[2]):
        y = np.zeros(geom.sino_shape)
        y[a, g[3] // 2] = 1.0
        got, ref = op.adjoint_apply(y), orc.adjoint_apply(y)
        err = np.abs(got - ref).max()
        print(g, "angle", a, "maxerr", err)
        if err > 1e-5:
            print("got\n", got, "\nref\n", ref)
