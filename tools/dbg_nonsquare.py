import sys; sys.path.insert(0, '.')
import numpy as np
import oracle
import paper_2410_10503_b200 as m
m.build_native()
for g in [(19, 41, 64, 61, 1.0), (33, 35, 3, 47, 1.0), (48, 40, 30, 70, 1.0)]:
    geom = m.Geometry(*g)
    op = m.RayTransform(geom)
    orc = oracle.RayTransform(oracle.Geometry(*g))
    x = np.random.default_rng(0).standard_normal(geom.image_shape)
    a, b = op.apply(x), orc.apply(x)
    err = np.abs(a - b).max(axis=1) / (np.abs(b).max() + 1e-30)
    bad = np.nonzero(err > 1e-5)[0]
    print(g, "bad angles", bad.tolist()[:40])
    if len(bad):
        r = bad[0]
        badj = np.nonzero(np.abs(a[r] - b[r]) > 1e-5 * np.abs(b).max())[0]
        print("   row", r, "bad bins", badj.tolist()[:40])
