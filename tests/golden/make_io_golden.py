"""Scene/camera text fixtures written by the REFERENCE's own writers
(ref/scene.py:283-289 save_scene, 340-349 save_cameras), for the I/O parity
tests (tests/test_scene_io.py).  Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from adpsplit import scene as RS  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
rng = np.random.default_rng(7)


def gaussian(k):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    return RS.Gaussian3D(mu=rng.normal(size=3) * 3, scale=np.exp(rng.normal(size=3) - 2), rot=q,
                         opacity=float(rng.uniform(0.01, 0.99)), sh_dc=rng.normal(size=3),
                         sh_rest=tuple(rng.normal(size=3) * 0.1 for _ in range(k)))


def camera(w, h):
    a = rng.normal(size=(3, 3))
    r, _ = np.linalg.qr(a)
    return RS.Camera(r_c2w=r, center=rng.normal(size=3) * 4, f_x=float(rng.uniform(200, 900)),
                     f_y=float(rng.uniform(200, 900)), p_x=w / 2 - 0.5, p_y=h / 2 - 0.5, width=w, height=h)


os.makedirs(OUT, exist_ok=True)
RS.save_scene(RS.Scene(gaussians=[gaussian(0) for _ in range(40)], extent=3.75), os.path.join(OUT, "scene_k0.txt"))
RS.save_scene(RS.Scene(gaussians=[gaussian(3) for _ in range(25)], extent=1.5), os.path.join(OUT, "scene_k3.txt"))
RS.save_cameras([camera(64, 48), camera(33, 17), camera(256, 256)], os.path.join(OUT, "cameras.txt"))
# the reference's own parse of its files, as arrays (what a load must reproduce)
for name in ("scene_k0", "scene_k3"):
    s = RS.load_scene(os.path.join(OUT, f"{name}.txt"))
    k = len(s.gaussians[0].sh_rest)
    np.savez(os.path.join(OUT, f"{name}.npz"), extent=s.extent,
             rec=np.array([[*g.mu, *g.scale, *g.rot, g.opacity, *g.sh_dc,
                            *[c for co in g.sh_rest for c in co]] for g in s.gaussians]), k=k)
cams = RS.load_cameras(os.path.join(OUT, "cameras.txt"))
np.savez(os.path.join(OUT, "cameras.npz"),
         rows=np.array([[*c.r_c2w.ravel(), *c.center, c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height] for c in cams]))
print("wrote", sorted(os.listdir(OUT)))
