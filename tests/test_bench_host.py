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
    assert bench.variant_of(["void mppi::rollout_kernel_x2s<(int)-2, 1, 0, 1, 1>(x)"]) == "x2s-grid-fused-epi"
    assert bench.variant_of([X2.replace("rollout_kernel_x2IL", "rollout_kernel_x2sIL") % ("in2", 1, 0, 1, 1)]) == "x2s-grid-fused-epi"
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


def test_rollout_roofline_arithmetic():
    """achieved = FLOP/ss x K T / time; issue fraction from the instruction count; the ceiling of
    the instruction mix from the FMA-heavy pipe utilisation of the same capture."""
    consts = {"x2-grid-fused-epi:quadrotor": {"flop": 340.0, "inst": 300.0, "dram_bytes": 28.0,
                                              "fmaheavy_pipe_pct": 72.0, "capture": "c5_epi"}}
    r = bench.rollout_roofline("x2-grid-fused-epi", "quadrotor", 1 << 22, 200, 10.0, 74.4, 148, 1965.0,
                               consts, {"stale": False})
    units = (1 << 22) * 200
    assert abs(r["achieved"] - 340.0 * units / 10e-3 / 1e12) < 1e-9
    assert abs(r["frac"] - r["achieved"] / 74.4) < 1e-12
    assert abs(r["issue_frac"] - 300.0 / 32 * units / 10e-3 / (148 * 4 * 1965e6)) < 1e-12
    assert abs(r["frac_ceiling_of_mix"] - r["frac"] / 0.72) < 1e-12
    assert r["traffic"] == 28.0 * units and r["bound"] == "alu"
    # a variant without constants reports no fraction rather than a wrong one
    r = bench.rollout_roofline("scalar:cartpole", "cartpole", 256, 50, 0.01, 74.4, 148, 1965.0, consts, {})
    assert r["frac"] is None and "no ncu constants" in r["note"]


def test_roofline_constants_staleness(tmp_path, monkeypatch):
    """bench.py marks the committed constants stale when the rollout machine code they were keyed
    to is not the library's."""
    import json
    p = tmp_path / "rc.json"
    p.write_text(json.dumps({"source_hash": "0000", "variants": {"v:p": {"flop": 1.0}}}))
    monkeypatch.setattr(bench, "CONSTANTS_PATH", str(p))
    from paper_1509_01149_b200 import build as B
    monkeypatch.setattr(B, "source_hash", lambda lib=None: "1111")
    v, meta = bench.roofline_constants()
    assert v == {"v:p": {"flop": 1.0}} and meta["stale"] is True
    monkeypatch.setattr(B, "source_hash", lambda lib=None: "0000")
    v, meta = bench.roofline_constants()
    assert meta["stale"] is False
