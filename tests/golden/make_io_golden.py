"""Scene/camera fixtures for the binary-format tests (tests/test_scene_io.py).

The scenes and cameras are written AND parsed by the reference's own text
I/O (ref/scene.py:283-381, save_scene/load_scene/save_cameras/load_cameras);
the reference's parse is then stored twice: as plain arrays (.npz, what a
load must reproduce) and as this repo's binary v1 files (.bin).  Run in the
build container (the reference is not needed at test time):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from adpsplit import scene as RS  # noqa: E402

from paper_2605_06876_b200 import scene_io as IO  # noqa: E402

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
for f in os.listdir(OUT):
    os.remove(os.path.join(OUT, f))
tmp = tempfile.mkdtemp()
scenes = {"scene_k0": RS.Scene(gaussians=[gaussian(0) for _ in range(40)], extent=3.75),
          "scene_k3": RS.Scene(gaussians=[gaussian(3) for _ in range(25)], extent=1.5)}
for name, sc in scenes.items():
    txt = os.path.join(tmp, f"{name}.txt")
    RS.save_scene(sc, txt)
    s = RS.load_scene(txt)                      # the reference's own parse of its file
    k = len(s.gaussians[0].sh_rest)
    np.savez(os.path.join(OUT, f"{name}.npz"), extent=s.extent,
             rec=np.array([[*g.mu, *g.scale, *g.rot, g.opacity, *g.sh_dc,
                            *[c for co in g.sh_rest for c in co]] for g in s.gaussians]), k=k)
    IO.save_scene_bin(IO.scene_to_arrays(s), os.path.join(OUT, f"{name}.bin"))
ctxt = os.path.join(tmp, "cameras.txt")
RS.save_cameras([camera(64, 48), camera(33, 17), camera(256, 256)], ctxt)
cams = RS.load_cameras(ctxt)
np.savez(os.path.join(OUT, "cameras.npz"),
         rows=np.array([[*c.r_c2w.ravel(), *c.center, c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height] for c in cams]))
IO.save_cameras_bin(cams, os.path.join(OUT, "cameras.bin"))
print("wrote", sorted(os.listdir(OUT)))
