"""Pins P1 (Philox KAT), P2 (BM32 accuracy and moments) and noise determinism for the
oracle's independent noise generator ("epsilon is
a vector of standard normal Gaussian random variables")."""
import ctypes as C
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_random123_kat(oracle):
    # Random123 known-answer vectors for philox4x32_10 (tests/golden/philox_kat.json)
    with open(os.path.join(GOLDEN, "philox_kat.json")) as f:
        kats = json.load(f)["vectors"]
    for v in kats:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        want = [int(x, 16) for x in v["out"]]
        assert oracle.philox4x32_10(ctr, key).tolist() == want


def test_philox_matches_curand_host_generator(oracle):
    """cuRAND's host-side Philox4_32_10 generator (runs on the CPU, no GPU) at seed 0
    emits the blocks for ctr = (0, 0, j, 0), key = (0, 0): an implementation we did not write."""
    path = None
    try:
        import nvidia.curand
        d = os.path.join(list(nvidia.curand.__path__)[0], "lib")
        path = os.path.join(d, "libcurand.so.10")
        L = C.CDLL(path)
    except Exception:
        pytest.skip("libcurand not loadable")
    g = C.c_void_p()
    assert L.curandCreateGeneratorHost(C.byref(g), 161) == 0  # CURAND_RNG_PSEUDO_PHILOX4_32_10
    assert L.curandSetPseudoRandomGeneratorSeed(g, C.c_ulonglong(0)) == 0
    out = np.zeros(16, np.uint32)
    assert L.curandGenerate(g, out.ctypes.data_as(C.c_void_p), C.c_size_t(16)) == 0
    L.curandDestroyGenerator(g)
    for j in range(4):
        assert out[4 * j:4 * j + 4].tolist() == oracle.philox4x32_10([0, 0, j, 0], [0, 0]).tolist()


def test_bm32_exhaustive_accuracy(oracle):
    """P2: over all 2^23 radius inputs and 2^24 angles, BM32 is within the error bounds
    SURVEY Appendix B states (ln <= 1.65 ulp, r <= 1.5 ulp, |sin/cos err| <= 8.3e-8)."""
    a = oracle.bm_accuracy()
    assert a["ln_ulp"] <= 1.65
    assert a["r_ulp"] <= 1.5
    assert a["sin_err"] <= 8.3e-8 and a["cos_err"] <= 8.3e-8
    # largest possible radius: u1 = 2^-24 -> sqrt(48 ln 2) = 5.7681...
    assert abs(a["max_abs_z"] - np.sqrt(48 * np.log(2))) < 1e-5


def test_bm32_special_inputs(oracle):
    # w = 0 -> u1 = 2^-24 exactly, angle 0 -> z0 = r = sqrt(48 ln 2), z1 = 0
    z = oracle.bm_normals([0, 0, 0, 0])
    assert z[1] == 0.0 and z[3] == 0.0
    assert abs(z[0] - np.sqrt(48 * np.log(2))) < 2e-6
    # angle index 2^22 (w = 2^30) is exactly pi/2: cos term from the o=2 branch -> -0 / +0
    z = oracle.bm_normals([0, 1 << 30, 0, 1 << 30])
    assert abs(z[0]) < 1e-6 and abs(z[1] - np.sqrt(48 * np.log(2))) < 2e-6


def test_noise_moments(oracle):
    """mean within 4 sigma/sqrt(N), covariance identity within 1 % Frobenius."""
    eps = oracle.noise(seed=7, step=3, T=100, K=25000, m=4).reshape(-1, 4).astype(np.float64)
    N = eps.shape[0]
    assert np.all(np.abs(eps.mean(0)) < 4.0 / np.sqrt(N))
    cov = np.cov(eps.T)
    assert np.linalg.norm(cov - np.eye(4)) / np.linalg.norm(np.eye(4)) < 0.01


def test_noise_determinism_and_prefix(oracle):
    """SPEC.md:80-83 scheduling independence; SURVEY A22 rank-sharded streams use the
    global k, so a shard equals the corresponding slice of the full tensor."""
    a = oracle.noise(1, 0, 10, 64, 2)
    b = oracle.noise(1, 0, 10, 64, 2)
    assert np.array_equal(a, b)
    shard = oracle.noise(1, 0, 10, 16, 2, k0=32)
    assert np.array_equal(shard, a[:, 32:48, :])
    # m < 4 keeps the leading components of the same Philox call
    full = oracle.noise(1, 0, 10, 64, 4)
    assert np.array_equal(full[:, :, :2], a)
    # step and seed both change the stream
    assert not np.array_equal(oracle.noise(1, 1, 10, 64, 2), a)
    assert not np.array_equal(oracle.noise(2, 0, 10, 64, 2), a)


def test_noise_counter_mapping(oracle):
    """eps[t][k][j] = z_j(Philox(ctr=(k, t, step_lo, step_hi), key=(seed_lo, seed_hi)))."""
    seed, step = 0x123456789ABCDEF0, 0xFEDCBA9876543210
    eps = oracle.noise(seed, step, 3, 5, 4)
    for t in range(3):
        for k in range(5):
            w = oracle.philox4x32_10([k, t, step & 0xFFFFFFFF, step >> 32],
                                     [seed & 0xFFFFFFFF, seed >> 32])
            assert np.array_equal(eps[t, k], oracle.bm_normals(w))
