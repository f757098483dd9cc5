"""Row (e) with the library's own communicator (mppi_nccl_attach, include/mppi.h): mppi_optimize
runs rollouts -> ncclAllReduce(MIN key) -> weighted sums -> ncclAllReduce(SUM [eta, A]) -> update
on the context stream.  One GPU here, so a single-rank communicator: the collectives are
identities and the result must equal the direct single-GPU step bit for bit (same kernels, same
reduction order).  The cross-rank arithmetic itself is covered by test_gpu_parity's sharding
emulation and test_dist_gloo."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MppiError, from_workload  # noqa: E402


@pytest.mark.parametrize("gather", [1, 0])
@pytest.mark.parametrize("cfg,K,lam", [("C1", 1024, None), ("C4", 65536, None), ("C4", 65536 + 256, 30.0)])
def test_single_rank_nccl_equals_direct(cfg, K, lam, gather):
    """The in-library NCCL step equals the direct single-GPU step bit for bit, with both combines:
    one all-gather of [key, eta, A] records rescaled in rank order (default; one rank: the scale is
    exp(0) = 1 exactly), or MIN of the key + SUM of [eta, A].  At C4 sizes both run the fused
    reduction (lambda = 30: many CTAs carry weight, so the per-CTA rescaling is exercised)."""
    from paper_1509_01149_b200 import _capi as A
    w = get(cfg)
    if lam is not None:
        w.lam = lam
    a = from_workload(w, K=K)
    b = from_workload(w, K=K)
    b.set_option(A.MPPI_OPTION_GATHER_COMBINE, gather)
    b.attach_nccl()
    Ua = torch.tensor(w.U0, device="cuda")
    Ub = Ua.clone()
    for i in range(3):
        a.optimize(w.x0, Ua, w.seed, i)
        b.optimize(w.x0, Ub, w.seed, i)
    torch.cuda.synchronize()
    assert torch.equal(Ua, Ub)
    if K >= 65536:
        assert any("epi_combine" in n for n in a.last_kernels())
        assert any("epi_combine" in n for n in b.last_kernels())
    sa, sb = a.stats(), b.stats()
    assert sa["k_star"] == sb["k_star"] and sa["s_min"] == sb["s_min"] and sa["eta"] == sb["eta"]
    Uh = np.ascontiguousarray(w.U0.copy())
    b.optimize_host(w.x0, Uh, w.seed, 0)
    Ud = torch.tensor(w.U0, device="cuda")
    a.optimize(w.x0, Ud, w.seed, 0)
    assert np.array_equal(Uh, Ud.cpu().numpy())
    a.close()
    b.close()


@pytest.mark.parametrize("cfg,K", [("C2", 4096), ("C4", 65536)])
def test_single_rank_nccl_cost_to_go_equals_direct(cfg, K):
    """NEXT-1 sharded: MIN over the per-step minima and SUM over [eta_t, A] through the library's
    communicator; one rank reproduces the direct cost-to-go step bit for bit."""
    w = get(cfg)
    a = from_workload(w, K=K)
    b = from_workload(w, K=K)
    a.set_weighting(True)
    b.set_weighting(True)
    b.attach_nccl()
    Ua = torch.tensor(w.U0, device="cuda")
    Ub = Ua.clone()
    for i in range(3):
        a.optimize(w.x0, Ua, w.seed, i)
        b.optimize(w.x0, Ub, w.seed, i)
    torch.cuda.synchronize()
    assert torch.equal(Ua, Ub)
    assert a.stats() == b.stats()
    with pytest.raises(MppiError):                  # the split phase is trajectory-only
        b.accumulate()
    a.close()
    b.close()


def test_world2_optimize_needs_communicator():
    w = get("C1")
    m = from_workload(w, K=1024, rank=0, world=2)
    U = torch.tensor(w.U0, device="cuda")
    with pytest.raises(MppiError):
        m.optimize(w.x0, U, w.seed, 0)
    m.close()


def test_double_attach_rejected():
    w = get("C1")
    m = from_workload(w, K=1024)
    m.attach_nccl()
    with pytest.raises(MppiError):
        m.attach_nccl()
    m.close()


@pytest.mark.parametrize("K,lam", [(8192, None), (8192, 30.0), (1 << 19, None), (1 << 19, 1e4)])
def test_gather_combine_emulated_ranks(K, lam):
    """The one-collective combine's arithmetic with G = 2, 4, 8 ranks, emulated on one GPU through
    its split phase (mppi_accumulate_record on every shard, the records stacked in rank order as an
    all-gather delivers them, mppi_apply_gathered on every rank): every rank gets the same bits,
    k* and S_min are the single-GPU ones, U agrees with the single-GPU step to 1e-6 (one-hot and
    dense weights; K = 2^19 puts every shard on the packed kernels)."""
    w = get("C4")
    if lam is not None:
        w.lam = lam
    one = from_workload(w, K=K)
    U1 = torch.tensor(w.U0, device="cuda")
    one.optimize(w.x0, U1, 4, 1)
    s1 = one.stats()
    for G in (2, 4, 8):
        ms = [from_workload(w, K=K, rank=r, world=G) for r in range(G)]
        U = torch.tensor(w.U0, device="cuda")
        for m in ms:
            m.rollout_costs(w.x0, U, 4, 1)
        recs = torch.stack([m.accumulate_record() for m in ms])
        assert recs.shape == (G, ms[0].gather_record_len())
        Us = []
        for m in ms:
            Ur = torch.tensor(w.U0, device="cuda")
            m.apply_gathered(Ur, recs)
            Us.append(Ur)
        torch.cuda.synchronize()
        for Ur in Us[1:]:
            assert torch.equal(Ur, Us[0])
        assert torch.max(torch.abs(Us[0] - U1)).item() <= 1e-6
        st = ms[0].stats()
        assert st["k_star"] == s1["k_star"] and st["s_min"] == s1["s_min"]
        assert st["eta"] == pytest.approx(s1["eta"], rel=1e-5)
        for m in ms:
            m.close()
    one.close()
