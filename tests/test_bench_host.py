"""Host-side logic of bench.py (no GPU): the rollout-variant parser that reads the library's
launched-kernel names (mppi_last_kernels), and the reference arm's JSON line on the oracle."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

# mangled device-function names as cudaFuncGetName returns them
X2 = "_ZN4mppi17rollout_kernel_x2IL%sELb%dELb%dELb%dELb%dEEEvNS_11RolloutArgsINS_15QuadrotorParamsEEE"


@pytest.mark.parametrize("np_,gen,qstep,diag,epi,want", [
    ("in2", 1, 0, 1, 1, "x2-grid-fused-epi"),
    ("in2", 1, 0, 1, 0, "x2-grid-fused"),
    ("in2", 1, 0, 0, 1, "x2-grid-fused-general-epi"),
    ("in2", 1, 1, 1, 1, "x2-grid-fused-ctg-epi"),
    ("in1", 0, 1, 1, 0, "x2-ctg"),
    ("i25", 0, 0, 1, 0, "x2"),
])
def test_variant_of_packed_names(np_, gen, qstep, diag, epi, want):
    names = [X2 % (np_, gen, qstep, diag, epi), "_ZN4mppi18epi_combine_kernelENS_13EpiCombineArgsE"]
    assert bench.variant_of(names) == want


def test_variant_of_scalar_and_empty():
    assert bench.variant_of(["_ZN4mppi12noise_kernelILi4EEEvNS_9NoiseArgsE",
                             "_ZN4mppi14rollout_kernelINS_8CartpoleELb1ELin1ELb0ELb0EEEvNS_11RolloutArgsINS_14CartpoleParamsEEE"]) == "scalar:cartpole"
    assert bench.variant_of(["_ZN4mppi14rollout_kernelINS_9QuadrotorELb1ELin2ELb1ELb0EEEvNS_11RolloutArgsINT_6ParamsEEE"]) \
        == "scalar-grid-fused:quadrotor"
    # ncu's demangled names (the roofline-constant captures) parse to the same variants
    assert bench.variant_of(["void mppi::rollout_kernel<mppi::Racecar, true, 1, true, false>(x)"]) == "scalar-fused:racecar"
    assert bench.variant_of(["void mppi::rollout_kernel_x2<(int)-2, 1, 0, 1, 1>(x)"]) == "x2-grid-fused-epi"
    assert bench.variant_of([]) is None
    assert bench.variant_of(["_ZN4mppi15finalize_kernelENS_12FinalizeArgsE"]) is None


def test_short_names():
    assert bench.short_names(["_ZN4mppi18epi_combine_kernelENS_13EpiCombineArgsE", X2 % ("in2", 1, 0, 1, 1),
                              "plain"]) == ["epi_combine_kernel", "rollout_kernel_x2", "plain"]


def test_reference_arm_json_line():
    """--impl reference: one JSON line with the contract's keys, the GPU arm's workload string,
    the oracle's sample stated, and e2e without host-device copies."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "impl", "cpu_baseline", "e2e"):
        assert key in line
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["workload"].startswith("C1: cartpole K=256 T=50")
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
