"""The rollouts' slow path (a sample or pair re-run from x0 after its step loop: angle out of the
fast sin/cos range, position beyond the obstacle grid's band or in an overflowing cell; DESIGN.md
§6) is counted by mppi_replay_count.  Results never depend on it; its frequency is performance:
  * a converged controller on C4 (150 optimisation steps from the same x0, trajectories reaching
    past the forest) replays no pair -- the grid band covers them and no cell overflows
    (round 2: six overflowing border cells made 6 % of the warps replay, C4 241 -> 435 us);
  * a start 2 km from the forest forces every rollout through the replay: the count grows by
    one per pair (packed kernel) or per sample (one-sample kernel) and the costs stay bitwise
    equal to the full 50-cylinder search."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402


def test_converged_controller_replays_nothing():
    w = get("C4")
    m = from_workload(w)
    U = torch.tensor(w.U0, device="cuda")
    for i in range(150):
        m.optimize(w.x0, U, w.seed, i)
    n0 = m.replay_count()
    for i in range(150, 170):
        m.optimize(w.x0, U, w.seed, i)
    n = m.replay_count() - n0
    assert any("rollout_kernel_x2" in k for k in m.last_kernels())
    print("replayed pairs over 20 converged steps: %d of %d" % (n, 20 * w.K // 2))
    assert n <= 20 * w.K // 2 * 1e-4


@pytest.mark.parametrize("K,per", [(65536, 2), (4096, 1)])
def test_far_start_replays_every_rollout_with_identical_costs(K, per):
    w = get("C4")
    x0 = np.array(w.x0, np.float32).copy()
    x0[0] = 2000.0                         # 2 km east: beyond the grid's 30-spacing band
    m = from_workload(w, K=K)
    full = from_workload(w, K=K)
    full.set_option(A.MPPI_OPTION_OBSTACLE_GRID, 0)
    U = torch.tensor(w.U0, device="cuda")
    n0 = m.replay_count()
    c, _ = m.rollout_costs(x0, U, 3, 0)
    assert m.replay_count() - n0 == K // per
    c_full, _ = full.rollout_costs(x0, U, 3, 0)
    assert np.array_equal(c.cpu().numpy().view(np.uint32), c_full.cpu().numpy().view(np.uint32))
