"""The device BM32 transform against the oracle over its WHOLE domain, bitwise (SURVEY.md
Appendix B; A17).  Every radius input (the 2^23 values of w >> 9) and every angle
index (the 2^24 values of w >> 8) goes through the scalar device functions and their packed
FP32x2 twins (csrc/noise.cuh, via libmppi_probe.so) and through the oracle's own BM32
(oracle/mppi_oracle.cpp).  The low bits the transform ignores are filled with a hash of the
index on both sides.  This closes the gap between the sampled noise tests and the contract:
the device divide and sqrt are hand-refined fast paths without range tests (noise.cuh), and
this sweep shows they return the IEEE results on every input the contract can produce."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1509_01149_b200 import probe_build  # noqa: E402


def words(n, shift):
    """w = (n << shift) | (uint32(n * 0x9E3779B9) >> (32 - shift)), as include/mppi_probe.h states."""
    n = n.astype(np.uint64)
    low = ((n * 0x9E3779B9) & 0xFFFFFFFF) >> (32 - shift)
    return ((n << shift) | low).astype(np.uint32)


def _first_mismatch(a, b, idx):
    bad = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
    if bad.size == 0:
        return None
    i = bad[0]
    return "%d mismatches; first at index %d: gpu %r oracle %r" % (bad.size, idx[i], a[i], b[i])


@pytest.mark.parametrize("packed", [0, 1])
def test_radius_all_inputs_bitwise(oracle, packed):
    count = 1 << 23
    n = np.arange(count, dtype=np.uint64)
    ref = oracle.bm_radius_words(words(n, 9))
    out = torch.empty(count, dtype=torch.float32, device="cuda")
    probe_build.bm32(0, packed, 0, count, out)
    got = out.cpu().numpy()
    msg = _first_mismatch(got, ref, n)
    assert msg is None, msg
    assert np.isfinite(got).all() and got.min() > 0.0
    print("PARITY BM32 radius (packed=%d): %d of %d inputs bitwise equal to the oracle" % (packed, count, count))


@pytest.mark.parametrize("packed", [0, 1])
def test_angle_all_inputs_bitwise(oracle, packed):
    count = 1 << 24
    n = np.arange(count, dtype=np.uint64)
    rs, rc = oracle.bm_angle_words(words(n, 8))
    sn = torch.empty(count, dtype=torch.float32, device="cuda")
    cs = torch.empty(count, dtype=torch.float32, device="cuda")
    probe_build.bm32(1, packed, 0, count, sn, cs)
    gs, gc = sn.cpu().numpy(), cs.cpu().numpy()
    for g, r, name in ((gs, rs, "sin"), (gc, rc, "cos")):
        msg = _first_mismatch(g, r, n)
        assert msg is None, name + ": " + msg
    print("PARITY BM32 angle (packed=%d): %d of %d sin and cos bitwise equal to the oracle" % (packed, count, count))


def test_ragged_subrange_and_odd_packed_count(oracle):
    """A range not starting at 0 with an odd count (the packed probe's last lane pairs with itself)."""
    first, count = (1 << 23) - 1001, 1001
    n = np.arange(first, first + count, dtype=np.uint64)
    ref = oracle.bm_radius_words(words(n, 9))
    for packed in (0, 1):
        out = torch.empty(count, dtype=torch.float32, device="cuda")
        probe_build.bm32(0, packed, first, count, out)
        assert _first_mismatch(out.cpu().numpy(), ref, n) is None
