"""MPPI_OPTION_RADIUS_TABLE: the packed C5 rollout reads the Box-Muller radius r(w) (SURVEY.md
Appendix B "Radius") from a 2^23-entry table built on the device at create.  The
table equals the oracle's BM32 radius on every input, and the rollout with the table gives the
same noise, costs and key as the rollout computing the radius (and, with the fused reduction,
the same update)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MppiError, _capi as A, from_workload  # noqa: E402


def test_table_equals_oracle_radius_everywhere(oracle):
    w = get("C4")
    m = from_workload(w, K=65536)
    tab = m.radius_table().cpu().numpy()
    m.close()
    n = np.arange(1 << 23, dtype=np.uint64)
    ref = oracle.bm_radius_words((n << 9).astype(np.uint32))
    bad = np.nonzero(tab.view(np.uint32) != ref.view(np.uint32))[0]
    assert bad.size == 0, "first mismatch at n = %d" % bad[0]


def test_no_table_without_the_packed_path():
    w = get("C1")
    m = from_workload(w)
    with pytest.raises(MppiError):
        m.radius_table()
    m.close()


@pytest.mark.parametrize("K,lam", [(65536 + 4, None), (1 << 18, 30.0)])
def test_table_rollout_is_bitwise_computed_radius(K, lam):
    w = get("C4")
    if lam is not None:
        w.lam = lam
    a = from_workload(w, K=K)
    b = from_workload(w, K=K)
    b.set_option(A.MPPI_OPTION_RADIUS_TABLE, 0)
    Ua, Ub = torch.tensor(w.U0, device="cuda"), torch.tensor(w.U0, device="cuda")
    for i in range(2):
        a.optimize(w.x0, Ua, 9, i)
        b.optimize(w.x0, Ub, 9, i)
        assert any("rollout_kernel_x2ILin2ELi2E" in n for n in a.last_kernels()), a.last_kernels()
        assert not any("rollout_kernel_x2ILin2ELi2E" in n for n in b.last_kernels())
        torch.cuda.synchronize()
        assert torch.equal(Ua, Ub) and a.stats() == b.stats()
    # the noise the table kernel wrote for the reduction is K1's (the computed transform)
    ca, ka = a.rollout_costs(w.x0, Ua, 4, 7)
    cb, kb = b.rollout_costs(w.x0, Ub, 4, 7)
    assert torch.equal(ca, cb) and int(ka.item()) == int(kb.item())
    a.close()
    b.close()
