"""Binary scene/camera files against fixtures whose
values the reference itself wrote and parsed (tests/golden/make_io_golden.py),
plus exact round trips and the error paths.  CPU only except the device upload."""
import os

import numpy as np
import pytest

from paper_2605_06876_b200 import scene_io as IO
from paper_2605_06876_b200.types import InvariantError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _rec(a):
    return np.concatenate([a.mu, a.scale, a.rot, a.opacity[:, None], a.sh_dc, a.sh_rest.reshape(len(a), -1)], axis=1)


def _cam_rows(cams):
    return np.array([[*c.r_c2w.ravel(), *c.center, c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height] for c in cams])


@pytest.mark.parametrize("name", ["scene_k0", "scene_k3"])
def test_binary_scene_matches_reference_parse(name, tmp_path):
    ref = np.load(os.path.join(GOLD, f"{name}.npz"))
    a = IO.load_scene_bin(os.path.join(GOLD, f"{name}.bin"))
    assert a.extent == float(ref["extent"]) and a.sh_rest.shape[1] == int(ref["k"])
    np.testing.assert_array_equal(_rec(a), ref["rec"])          # bit-exact values
    # SceneArrays -> Scene objects -> binary -> SceneArrays is the identity
    s = IO.arrays_to_scene(a)
    IO.save_scene_bin(s, tmp_path / "s.bin")
    b = IO.load_scene_bin(tmp_path / "s.bin")
    np.testing.assert_array_equal(_rec(b), ref["rec"])
    assert (tmp_path / "s.bin").read_bytes() == open(os.path.join(GOLD, f"{name}.bin"), "rb").read()


def test_binary_cameras_match_reference_parse(tmp_path):
    ref = np.load(os.path.join(GOLD, "cameras.npz"))["rows"]
    cams = IO.load_cameras_bin(os.path.join(GOLD, "cameras.bin"))
    np.testing.assert_array_equal(_cam_rows(cams), ref)
    IO.save_cameras_bin(cams, tmp_path / "c.bin")
    np.testing.assert_array_equal(_cam_rows(IO.load_cameras_bin(tmp_path / "c.bin")), ref)


def test_binary_errors(tmp_path):
    a = IO.load_scene_bin(os.path.join(GOLD, "scene_k3.bin"))
    raw = open(os.path.join(GOLD, "scene_k3.bin"), "rb").read()
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
    a.scale[7, 1] = 1.0
    a.opacity[2] = 1.5
    IO.save_scene_bin(a, tmp_path / "o.bin")
    with pytest.raises(InvariantError, match="Gaussian 2: opacity"):
        IO.load_scene_bin(tmp_path / "o.bin")
    craw = open(os.path.join(GOLD, "cameras.bin"), "rb").read()
    (tmp_path / "c2.bin").write_bytes(craw[:-1])
    with pytest.raises(IO.SceneFormatError, match="truncated"):
        IO.load_cameras_bin(tmp_path / "c2.bin")


def test_ragged_sh_rest_rejected(tmp_path):
    s = IO.arrays_to_scene(IO.load_scene_bin(os.path.join(GOLD, "scene_k3.bin")))
    g = s.gaussians[0]
    s.gaussians[0] = type(g)(mu=g.mu, scale=g.scale, rot=g.rot, opacity=g.opacity, sh_dc=g.sh_dc,
                             sh_rest=g.sh_rest[:1])
    with pytest.raises(IO.SceneFormatError, match="ragged"):
        IO.save_scene_bin(s, tmp_path / "r.bin")


@pytest.mark.gpu
def test_scene_tensors_on_device():
    import torch
    a = IO.load_scene_bin(os.path.join(GOLD, "scene_k3.bin"))
    g, extent = IO.scene_tensors(a, device="cuda:0")
    assert extent == a.extent and g.n == len(a) and g.sh_k == 3
    np.testing.assert_array_equal(g.mu.cpu().numpy(), a.mu.astype(np.float32))
    np.testing.assert_array_equal(g.sh_rest.cpu().numpy(), a.sh_rest.astype(np.float32))
    assert g.mu.device == torch.device("cuda:0")
