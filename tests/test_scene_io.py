"""Scene/camera files: the v1 text format against
files written and parsed by the reference itself (tests/golden/make_io_golden.py),
and the binary v1 format by exact round trips.  CPU only."""
import os

import numpy as np
import pytest

from paper_2605_06876_b200 import scene_io as IO
from paper_2605_06876_b200.types import InvariantError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _rec(a):
    return np.concatenate([a.mu, a.scale, a.rot, a.opacity[:, None], a.sh_dc, a.sh_rest.reshape(len(a), -1)], axis=1)


@pytest.mark.parametrize("name", ["scene_k0", "scene_k3"])
def test_text_scene_matches_reference(name, tmp_path):
    path = os.path.join(GOLD, f"{name}.txt")
    ref = np.load(os.path.join(GOLD, f"{name}.npz"))
    s = IO.load_scene(path)
    a = IO.scene_to_arrays(s)
    assert a.extent == float(ref["extent"])
    np.testing.assert_array_equal(_rec(a), ref["rec"])        # bit-exact parse
    np.testing.assert_array_equal(_rec(IO.load_scene_arrays(path)), ref["rec"])
    # writing back gives the reference's bytes, from either representation
    IO.save_scene(s, tmp_path / "a.txt")
    IO.save_scene(a, tmp_path / "b.txt")
    orig = open(path).read()
    assert open(tmp_path / "a.txt").read() == orig
    assert open(tmp_path / "b.txt").read() == orig


@pytest.mark.parametrize("name", ["scene_k0", "scene_k3"])
def test_binary_scene_round_trip(name, tmp_path):
    a = IO.load_scene_arrays(os.path.join(GOLD, f"{name}.txt"))
    IO.save_scene_bin(a, tmp_path / "s.bin")
    b = IO.load_scene_bin(tmp_path / "s.bin")
    assert b.extent == a.extent and b.sh_rest.shape == a.sh_rest.shape
    np.testing.assert_array_equal(_rec(b), _rec(a))
    # Scene -> binary -> Scene -> text reproduces the reference's file
    IO.save_scene_bin(IO.load_scene(os.path.join(GOLD, f"{name}.txt")), tmp_path / "s2.bin")
    IO.save_scene(IO.arrays_to_scene(IO.load_scene_bin(tmp_path / "s2.bin")), tmp_path / "s.txt")
    assert open(tmp_path / "s.txt").read() == open(os.path.join(GOLD, f"{name}.txt")).read()


def test_cameras_text_and_binary(tmp_path):
    path = os.path.join(GOLD, "cameras.txt")
    ref = np.load(os.path.join(GOLD, "cameras.npz"))["rows"]
    cams = IO.load_cameras(path)
    rows = np.array([[*c.r_c2w.ravel(), *c.center, c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height] for c in cams])
    np.testing.assert_array_equal(rows, ref)
    IO.save_cameras(cams, tmp_path / "c.txt")
    assert open(tmp_path / "c.txt").read() == open(path).read()
    IO.save_cameras_bin(cams, tmp_path / "c.bin")
    back = IO.load_cameras_bin(tmp_path / "c.bin")
    rows2 = np.array([[*c.r_c2w.ravel(), *c.center, c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height] for c in back])
    np.testing.assert_array_equal(rows2, ref)


def test_text_errors(tmp_path):
    good = open(os.path.join(GOLD, "scene_k0.txt")).read().splitlines()
    cases = {
        "nohdr": (["bogus"] + good[1:], IO.SceneFormatError, "header"),
        "noext": ([good[0], "x 1"] + good[2:], IO.SceneFormatError, "extent"),
        "badext": ([good[0], "extent zz"] + good[2:], IO.SceneFormatError, "bad extent"),
        "nan_tok": (good[:3] + ["1 2 x"] + good[4:], IO.SceneFormatError, "non-numeric"),
        "trunc": (good[:3] + [" ".join(good[3].split()[:13])] + good[4:], IO.SceneFormatError, "truncated"),
        "empty": (good[:2], IO.SceneFormatError, "no Gaussians"),
    }
    for name, (lines, exc, msg) in cases.items():
        p = tmp_path / f"{name}.txt"
        p.write_text("\n".join(lines) + "\n")
        with pytest.raises(exc, match=msg):
            IO.load_scene(p)
        with pytest.raises(exc, match=msg):
            IO.load_scene_arrays(p)
    # invariant violation reported with the line number, as the reference does
    vals = good[4].split()
    vals[10] = "1.5"   # opacity
    p = tmp_path / "inv.txt"
    p.write_text("\n".join(good[:4] + [" ".join(vals)] + good[5:]) + "\n")
    with pytest.raises(InvariantError, match=r":5: Gaussian 2: opacity"):
        IO.load_scene(p)
    with pytest.raises(InvariantError, match=r":5: Gaussian 2: opacity"):
        IO.load_scene_arrays(p)


def test_binary_errors(tmp_path):
    a = IO.load_scene_arrays(os.path.join(GOLD, "scene_k3.txt"))
    IO.save_scene_bin(a, tmp_path / "s.bin")
    raw = (tmp_path / "s.bin").read_bytes()
    (tmp_path / "t.bin").write_bytes(raw[:-8])
    with pytest.raises(IO.SceneFormatError, match="truncated"):
        IO.load_scene_bin(tmp_path / "t.bin")
    (tmp_path / "m.bin").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(IO.SceneFormatError, match="magic"):
        IO.load_scene_bin(tmp_path / "m.bin")
    a.scale[7, 1] = -1.0
    IO.save_scene_bin(a, tmp_path / "i.bin")
    with pytest.raises(InvariantError, match="Gaussian 7: scale"):
        IO.load_scene_bin(tmp_path / "i.bin")
    IO.save_cameras_bin(IO.load_cameras(os.path.join(GOLD, "cameras.txt")), tmp_path / "c.bin")
    with pytest.raises(IO.SceneFormatError, match="truncated"):
        (tmp_path / "c2.bin").write_bytes((tmp_path / "c.bin").read_bytes()[:-1])
        IO.load_cameras_bin(tmp_path / "c2.bin")


def test_ragged_sh_rest_needs_text(tmp_path):
    a = IO.load_scene(os.path.join(GOLD, "scene_k3.txt"))
    g = a.gaussians[0]
    a.gaussians[0] = type(g)(mu=g.mu, scale=g.scale, rot=g.rot, opacity=g.opacity, sh_dc=g.sh_dc, sh_rest=g.sh_rest[:1])
    IO.save_scene(a, tmp_path / "r.txt")
    assert len(IO.load_scene(tmp_path / "r.txt").gaussians[0].sh_rest) == 1   # the text format keeps it
    with pytest.raises(IO.SceneFormatError, match="ragged"):
        IO.save_scene_bin(a, tmp_path / "r.bin")
    with pytest.raises(IO.SceneFormatError, match="ragged"):
        IO.load_scene_arrays(tmp_path / "r.txt")


@pytest.mark.gpu
def test_scene_tensors_on_device(tmp_path):
    import torch
    a = IO.load_scene_arrays(os.path.join(GOLD, "scene_k3.txt"))
    IO.save_scene_bin(a, tmp_path / "s.bin")
    g, extent = IO.scene_tensors(IO.load_scene_bin(tmp_path / "s.bin"), device="cuda:0")
    assert extent == a.extent and g.n == len(a) and g.sh_k == 3
    np.testing.assert_array_equal(g.mu.cpu().numpy(), a.mu.astype(np.float32))
    np.testing.assert_array_equal(g.sh_rest.cpu().numpy(), a.sh_rest.astype(np.float32))
    assert g.mu.device == torch.device("cuda:0")
