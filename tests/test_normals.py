"""Device normals == numpy Generator(PCG64).standard_normal, bit for bit.

The fallback children of ref/adc.py:97 draw rng.normal(size=(k, 3)) per
fallback parent; adps_normals_pcg64 reproduces that slice of the Generator's
stream on the GPU.  CPU tests pin the ziggurat tables and the stream model
(tools/gen_ziggurat.py) against numpy itself; GPU tests compare the device
stream with numpy at sizes up to millions of draws (thousands of wedge and
tail cases) and check the Generator is advanced exactly as numpy would.
"""
import os
import re
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gen_ziggurat as Z  # noqa: E402

HEADER = os.path.join(ROOT, "paper_2605_06876_b200", "csrc", "ziggurat_tables.h")


def _header_tables():
    txt = open(HEADER).read()

    def block(name):
        body = re.search(name + r"\[256\] = \{(.*?)\};", txt, re.S).group(1)
        return [t.strip() for t in body.replace("\n", " ").split(",") if t.strip()]

    ki = [int(t.rstrip("ULL"), 16) for t in block("kZigKi")]
    wi = [float(t) for t in block("kZigWi")]
    fi = [float(t) for t in block("kZigFi")]
    return ki, wi, fi


def test_header_tables_match_numpy():
    ki, wi, fi = Z.find_tables()
    hk, hw, hf = _header_tables()
    assert hk == ki
    assert np.array_equal(np.array(hw).view(np.uint64), np.array(wi).view(np.uint64))
    assert np.array_equal(np.array(hf).view(np.uint64), np.array(fi).view(np.uint64))


@pytest.mark.parametrize("seed", [0, 7, 2024])
def test_stream_model_matches_numpy(seed):
    """The attempt/length model the kernel uses reproduces numpy's stream and state."""
    stats = Z.verify(*_header_tables(), n=60_000, seed=seed)
    assert stats["wedge"] > 0


# ---------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def plan():
    from paper_2605_06876_b200 import operator as op
    return op.Plan("cuda:0")


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 6, 31, 32, 33, 1000, 65_537])
@pytest.mark.parametrize("seed", [0, 1, 12345])
def test_device_normals_small(plan, n, seed):
    rng = np.random.default_rng(seed)
    rng.standard_normal(seed % 5)          # arbitrary position in the stream
    st = rng.bit_generator.state
    want = rng.standard_normal(n)
    out, consumed, status = plan.normals_pcg64(st, n)
    assert status == 0
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))
    ref = np.random.default_rng(seed)
    ref.bit_generator.state = st
    ref.bit_generator.advance(consumed)
    assert ref.bit_generator.state["state"] == rng.bit_generator.state["state"]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [3_000_000, 12_000_000])
def test_device_normals_large(plan, n):
    """Millions of draws: ~1.5% wedge tests and ~1 tail per 4k draws, all exact."""
    rng = np.random.default_rng(n)
    st = rng.bit_generator.state
    want = rng.standard_normal(n)
    out, consumed, status = plan.normals_pcg64(st, n)
    assert status == 0
    got = out.cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])
    ref = np.random.default_rng(0)
    ref.bit_generator.state = st
    ref.bit_generator.advance(consumed)
    assert ref.bit_generator.state["state"] == rng.bit_generator.state["state"]
    assert np.abs(want).max() > 4.0        # the tail was exercised


@pytest.mark.gpu
def test_device_normals_zero(plan):
    rng = np.random.default_rng(3)
    out, consumed, status = plan.normals_pcg64(rng.bit_generator.state, 0)
    assert consumed == 0 and status == 0 and out.numel() == 0
