#!/usr/bin/env python
"""bench.py — MPPI rollout timesteps/s (K*T per s) and control-update latency on B200.

One "step" = one full MPPI optimisation (Alg. 1 :356-368): Philox noise -> rollouts
-> [NCCL MIN] -> weights + weighted noise sum -> [NCCL SUM] -> U update, over K_global samples.
Default workload: BASELINE config C5 (quadrotor, 50-cylinder 4 m forest, T=200) at K = 2^22,
strong-scaled over N GPUs (each rank rolls out K/N samples).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5]
  torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1; NCCL over NVLink)

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPPI rollout timesteps/sec (K*T per s)"
UNIT = "K*T/s"

# Roofline numerators per sample-step of each rollout variant (FP32 FLOPs = FADD + FMUL + 2 FFMA +
# 2 FADD2 + 2 FMUL2 + 4 FFMA2 thread-level SASS counters, thread instructions, DRAM bytes), from
# the ncu captures of scripts/gpu_roofline_capture.sh, written with the source hash of the tree
# they measured (profiles/roofline_constants.json, scripts/roofline_constants.py).  bench.py
# recomputes the hash of the library sources and marks the constants stale when they differ.
CONSTANTS_PATH = os.path.join(ROOT, "profiles", "roofline_constants.json")
# the full 50-cylinder search with the noise read from HBM (the v7 packed kernel's ncu count,
# profiles/r1_ncu_full_c5_v7.txt): the effective-rate comparison only, not executed FLOPs
FULL_SEARCH_QUAD_FLOP = 464.56


def roofline_constants():
    """{variant key: {flop, inst, dram_bytes, ...}}, and whether they measured this source tree."""
    try:
        with open(CONSTANTS_PATH) as f:
            doc = json.load(f)
    except Exception:
        return {}, {"file": None, "stale": True}
    cur = None
    try:
        from paper_1509_01149_b200 import build as B
        cur = B.source_hash()
    except Exception:
        pass
    meta = {"file": os.path.relpath(CONSTANTS_PATH, ROOT), "source_hash": doc.get("source_hash"),
            "current_source_hash": cur, "stale": cur is None or cur != doc.get("source_hash"),
            "git_head": doc.get("git_head")}
    return doc.get("variants", {}), meta


def variant_key(variant, plant):
    return variant if (variant and ":" in variant) else "%s:%s" % (variant, plant)


_B = r"(?:\(bool\))?(true|false|1|0)"
_I = r"(?:\(int\))?(-?\d+)"


def _b(v):
    return v in ("1", "true")


def variant_of(kernels):
    """The rollout variant the library's dispatch chose, from the device-function names of the
    last step's launches (mppi_last_kernels, mangled) or an ncu kernel name (demangled):
    rollout_kernel_x2<NP, GEN, QSTEP, DIAG, EPI> -> "x2[-grid][-fused][-general][-ctg][-epi]",
    rollout_kernel<Plant, DIAG, NP, GEN, QSTEP> -> "scalar[-grid][-fused][-general][-ctg]:<plant>"."""
    import re
    for k in kernels:
        mt = re.search(r"rollout_kernel_x2(s?)IL(in?)(\d+)ELb([01])ELb([01])ELb([01])ELb([01])E", k)
        if mt:
            vs = mt.group(1) == "s"
            np_ = -int(mt.group(3)) if mt.group(2) == "in" else int(mt.group(3))
            gen, qstep, diag, epi = (mt.group(i) == "1" for i in range(4, 8))
        else:
            mt = re.search(r"rollout_kernel_x2(s?)<\s*%s,\s*%s,\s*%s,\s*%s,\s*%s\s*>" % (_I, _B, _B, _B, _B), k)
            if mt:
                vs = mt.group(1) == "s"
                np_ = int(mt.group(2))
                gen, qstep, diag, epi = (_b(mt.group(i)) for i in range(3, 7))
        if mt:   # (rollout_kernel_x2s: a v31 small-K variant, folded back into x2 in v32)
            return ("x2" + ("s" if vs else "") + ("-grid" if np_ == -2 else "") + ("-fused" if gen else "") +
                    ("" if diag else "-general") + ("-ctg" if qstep else "") + ("-epi" if epi else ""))
        mt = re.search(r"rollout_kernelINS_\d+([A-Za-z]+)(?:I.*?E)?ELb([01])EL(in?)(\d+)ELb([01])ELb([01])E", k)
        if mt:
            plant = mt.group(1)
            diag = mt.group(2) == "1"
            np_ = -int(mt.group(4)) if mt.group(3) == "in" else int(mt.group(4))
            gen, qstep = mt.group(5) == "1", mt.group(6) == "1"
        else:
            mt = re.search(r"rollout_kernel<\s*mppi::([A-Za-z]+)(?:<[^>]*>)?,\s*%s,\s*%s,\s*%s,\s*%s\s*>" % (_B, _I, _B, _B), k)
            if mt:
                plant = mt.group(1)
                diag, np_, gen, qstep = _b(mt.group(2)), int(mt.group(3)), _b(mt.group(4)), _b(mt.group(5))
        if mt:
            return ("scalar" + ("-grid" if np_ == -2 else "") + ("-fused" if gen else "") +
                    ("" if diag else "-general") + ("-ctg" if qstep else "") + ":" + plant.lower())
        if "rollout_kernel" in k:
            return "scalar"
    return None


def short_names(kernels):
    """_ZN4mppi17rollout_kernel_x2ILin2E... -> rollout_kernel_x2 (the identifier only)."""
    import re
    out = []
    for k in kernels:
        mt = re.match(r"_ZN4mppi(\d+)", k)
        out.append(k[mt.end():mt.end() + int(mt.group(1))] if mt else k)
    return out


def rollout_variant(w, K_loc, fused_reduction=True, m=None):
    """Which rollout kernel bench.py's configuration runs: asked from the library when a context
    that has stepped is given, else predicted (mirrors dispatch_np/fused_noise_applies/epi_applies)."""
    if m is not None:
        v = variant_of(m.last_kernels())
        if v is not None:
            return v
    if w.plant == "quadrotor" and K_loc >= 65536 and w.obstacles is not None and len(w.obstacles) >= 2:
        return "x2-grid-fused-epi" if fused_reduction else "x2-grid-fused"
    return "scalar"

SM_COUNT_B200 = 148
FP32_LANES_PER_SM = 128


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C5")
    p.add_argument("--K", type=int, default=0, help="global samples (default: the config's)")
    p.add_argument("--no-latency", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-probe", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the C3/C4/K-sweep/closed-loop extras")
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                   help="process-group backend for N > 1 (gloo: a CPU-side test of the sharded path "
                        "that lets several ranks share one GPU)")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every 10 ms (pynvml,
    initialised before the region), else nvidia-smi every 200 ms."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []          # (sm_mhz, sm_max_mhz, {reasons})
        self.power = []         # W (NVML)
        self.proc = None
        self.thread = None
        self.stop_flag = threading.Event()
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.sm_max = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.masks = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        except Exception:
            self.nvml = None

    def start(self):
        if self.nvml is not None:
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read_smi, daemon=True)
        self.thread.start()

    def _poll_nvml(self):
        nv = self.nvml
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                try:
                    self.power.append(nv.nvmlDeviceGetPowerUsage(self.handle) / 1000.0)
                except Exception:
                    pass
                self.rows.append((float(sm), float(self.sm_max),
                                  {n for n, m in zip(self.REASONS, self.masks) if bits & m}))
            except Exception:
                pass
            self.stop_flag.wait(0.01)

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS) and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else 0.0,
                                  {self.REASONS[i] for i in range(4) if parts[3 + i].lower() == "active"}))

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.thread.join(timeout=5)
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=5)
        else:
            return None
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [r[0] for r in self.rows]
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
               "reasons": sorted(set().union(*[r[2] for r in self.rows])), "samples": len(self.rows),
               "sm_mhz_min": min(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}
        if self.power:
            out["power_w_median"] = statistics.median(self.power)
            out["power_w_max"] = max(self.power)
        return out


# ----------------------------------------------------------------------------- helpers
HBM_SPEC_GBS = 8000.0   # B200 HBM3e data-sheet bandwidth (SURVEY 8.4 asks for this ratio beside the measured one)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def run_fp32_probe():
    """FFMA / FFMA2 chain probes (TFLOP/s).  bench.py runs them before the warm-up steps, which
    also brings the GPU out of idle before the timed region."""
    try:
        from paper_1509_01149_b200 import probe_build
        return {"ffma_probe_tflops": probe_build.probe(False)[0], "ffma2_probe_tflops": probe_build.probe(True)[0]}
    except Exception as e:  # the probe is context for the denominator, never the product
        return {"probe_error": str(e)[:200]}


def fp32_peak(probe, sm_count, sm_max_mhz):
    derived = sm_count * FP32_LANES_PER_SM * 2 * sm_max_mhz * 1e6 / 1e12
    out = {"derived_tflops": derived, "ffma_probe_tflops": None, "ffma2_probe_tflops": None}
    out.update(probe or {})
    cands = [v for k, v in out.items() if k.endswith("tflops") and v]
    out["peak_tflops"] = max(cands)
    return out


def cpu_baseline(w, steps=1, k_sample=None):
    """The fp64 oracle (as it stands) on this host's cores, on a bounded sample of the workload."""
    import numpy as np
    from oracle import oracle as O
    cores = len(os.sched_getaffinity(0))
    K = k_sample or min(w.K, 1 << 16)
    pb = O.Problem(w.plant, T=w.T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                   obstacles=w.obstacles if w.plant == "quadrotor" else None)
    U = w.U0.astype(np.float64)
    t0 = time.perf_counter()
    for s in range(steps):
        eps = O.noise(w.seed, s, w.T, K, w.m)
        r = O.optimize(pb, w.x0, U, eps, nthreads=cores)
        U = r["U"]
    dt = time.perf_counter() - t0
    # one core (SURVEY §8.4 asks for the single-threaded oracle beside the OpenMP one): the
    # rollouts of a quarter of the sample on one thread
    K1 = max(4, K // 4)
    eps = O.noise(w.seed, 0, w.T, K1, w.m)
    t1 = time.perf_counter()
    O.rollout_costs(pb, w.x0, w.U0.astype(np.float64), eps, nthreads=1)
    d1 = time.perf_counter() - t1
    return {"value": K * w.T * steps / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "%d step(s) of %s at K=%d (of %d), T=%d: noise + rollouts (OpenMP over k) "
                      "+ k-ordered reduction, fp64" % (steps, w.name, K, w.K, w.T),
            "seconds": dt,
            "one_core_rollouts_KT_per_s": K1 * w.T / d1,
            "one_core_sample": "rollouts only (fp64, 1 thread) at K=%d, T=%d" % (K1, w.T)}


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def rollout_roofline(variant, plant, K_loc, T, avg_ms, peak, sm_count, sm_max_mhz, consts, meta):
    """FP32 ALU roofline of one rollout launch: the variant's FLOPs per sample-step (ncu, this
    source tree unless `stale`) x K_loc T / the launch's CUDA-event time; issue-slot fraction from
    the instruction count; `traffic` = ncu DRAM bytes of the same capture scaled to this launch."""
    key = variant_key(variant, plant)
    c = consts.get(key)
    units = K_loc * T
    out = {"kernel": "rollout", "variant": key, "bound": "alu", "unit": "TFLOP/s", "peak": peak,
           "achieved": None, "frac": None, "traffic": None, "avg_ms": avg_ms,
           "constants": dict(meta, capture=(c or {}).get("capture"))}
    if not c or not avg_ms:
        out["note"] = "no ncu constants for %s" % key
        return out
    ach = c["flop"] * units / (avg_ms * 1e-3) / 1e12
    slots = sm_count * 4 * sm_max_mhz * 1e6
    out.update({"achieved": ach, "frac": ach / peak, "flop_per_sample_step": c["flop"],
                "inst_per_sample_step": c["inst"],
                "issue_frac": c["inst"] / 32.0 * units / (avg_ms * 1e-3) / slots,
                "traffic": c["dram_bytes"] * units,
                "algorithmic_bytes_per_launch": None})
    heavy = c.get("fmaheavy_pipe_pct")
    if heavy:
        # the binding pipe: every packed FP32 op and every IMAD (Philox) occupies
        # the FMA-heavy pipe; the same instruction stream with that pipe 100 % busy would execute
        # frac / (heavy / 100) of the FP32 peak -- the ceiling of this instruction mix
        out["pipes_ncu_pct"] = {"fmaheavy": heavy, "fmalite": c.get("fmalite_pipe_pct"),
                                "alu": c.get("alu_pipe_pct"), "issue": c.get("issue_active_pct"),
                                "capture": c.get("capture")}
        out["frac_ceiling_of_mix"] = out["frac"] / (heavy / 100.0)
    return out


def fp32_peak_now(probe, sm_count, sm_max_mhz):
    return fp32_peak(probe, sm_count, sm_max_mhz)["peak_tflops"]


# ----------------------------------------------------------------------------- reference arm
def workload_name(cfg, w, K):
    return "%s: %s K=%d T=%d m=%d nu=%g lambda=%g (K/N per GPU)" % (cfg, w.plant, K, w.T, w.m, w.nu, w.lam)


def run_reference(args, rank, world):
    """--impl reference: the oracle timed on the host cores, same metric/config."""
    if rank != 0:
        return 0
    from mppi_inputs import get
    w = get(args.config)
    w.K = args.K or w.K
    ksamp = min(w.K, 1 << 14)
    for _ in range(args.warmup):
        cpu_baseline(w, steps=1, k_sample=min(ksamp, 1024))
    r = cpu_baseline(w, steps=args.steps, k_sample=ksamp)
    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * r["seconds"] / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            # the GPU arm's workload (same string and sizes); the oracle times a bounded sample
            # of it per step, stated in cpu_baseline.sample
            "config": {"workload": workload_name(args.config, w, w.K), "K": w.K, "T": w.T,
                       "n_obstacles": int(len(w.obstacles)) if w.obstacles is not None else 0,
                       "oracle_sample_K_per_step": ksamp},
            "impl": "reference",
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"], "cpu": lscpu_model()},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- latency
def latency(cfg_name, iters=200, warm=20, K=None):
    import torch
    from mppi_inputs import get
    from paper_1509_01149_b200 import from_workload
    w = get(cfg_name)
    Kx = K or w.K
    m = from_workload(w, K=Kx)
    U = torch.tensor(w.U0, device="cuda")
    for i in range(warm):
        m.optimize(w.x0, U, w.seed, i)
    torch.cuda.synchronize()
    dev, host = [], []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for i in range(iters):
        t0 = time.perf_counter()
        evs[i][0].record()
        m.optimize(w.x0, U, w.seed, warm + i)
        evs[i][1].record()
        u0 = U[0].cpu()                       # control to send to the actuators (4 m bytes D2H)
        host.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    dev = [a.elapsed_time(b) * 1e3 for a, b in evs]
    del u0
    q = lambda xs, p: sorted(xs)[min(len(xs) - 1, int(round(p * (len(xs) - 1))))]
    launches = m.last_launch_count()
    m.close()
    return {"K": Kx, "T": w.T, "plant": w.plant, "device_us_p50": q(dev, 0.5),
            "device_us_p99": q(dev, 0.99), "host_us_p50": q(host, 0.5), "host_us_p99": q(host, 0.99),
            "calls": iters, "kernels_per_call": launches,
            "KT_per_s_at_p50": Kx * w.T / (q(dev, 0.5) * 1e-6)}


def paper_context_latency():
    """The paper's operating point beside our latency: K = 1000 rollouts of the
    cart-pole over a 1 s horizon (T = 50 at 50 Hz, :396), re-optimised every 20 ms (:387) on an
    unnamed GPU (:10, :343).  Context, not a target: the paper prints no timing."""
    r = latency("C1", K=1000)
    r["paper"] = {"K": 1000, "T": 50, "control_period_ms": 20.0, "gpu": "not named",
                  "implied_KT_per_s_floor": 1000 * 50 / 0.020,
                  "cite": "PAPER.md:387 (50 Hz), :396 (1 s horizon), :402-403 (K up to 1000)"}
    r["host_p99_rate_hz"] = 1e6 / r["host_us_p99"]
    r["device_p99_rate_hz"] = 1e6 / r["device_us_p99"]
    return r


def _safe(fn, *a, **k):
    try:
        return fn(*a, **k)
    except Exception as e:          # an extra must not sink the bench line
        return {"error": str(e)[:200]}


# ----------------------------------------------------------------------------- other configs
def throughput(cfg_name, K=None, steps=10, warm=3, cost_to_go=False, sparse=False,
               fused_reduction=True, peak=None, consts=None, meta=None):
    """K*T/s of one config on this GPU (graph replay, CUDA events around `steps` steps), then a
    separate profiled pass of the same number of steps (per-kernel CUDA events) for the rollout's
    FP32 fraction and, where the dense reduction runs as its own kernel, its HBM fraction."""
    import torch
    from mppi_inputs import get
    from paper_1509_01149_b200 import _capi as A, from_workload
    w = get(cfg_name)
    Kx = K or w.K
    m = from_workload(w, K=Kx)
    if cost_to_go:
        m.set_weighting(True)
    if sparse:      # the sparse skip belongs to the separate K3 reduction
        m.set_option(A.MPPI_OPTION_FUSED_REDUCTION, 0)
        m.set_option(A.MPPI_OPTION_SPARSE_REDUCTION, 1)
    if not fused_reduction:
        m.set_option(A.MPPI_OPTION_FUSED_REDUCTION, 0)
    U = torch.tensor(w.U0, device="cuda")
    for i in range(warm):
        m.optimize(w.x0, U, w.seed, i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(steps):
        m.optimize(w.x0, U, w.seed, warm + i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launched = m.last_kernels()
    m.profile_enable(True)          # the profiled pass, after the timed one
    for i in range(steps):
        m.optimize(w.x0, U, w.seed, warm + steps + i)
    kt = m.profile_read()
    m.profile_enable(False)
    m.close()
    kern = {k: v[0] / v[1] for k, v in kt.items() if v[1]}
    tot = sum(v[0] for v in kt.values()) or 1.0
    share = {k: v[0] / tot for k, v in kt.items() if v[1]}
    out = {"plant": w.plant, "K": Kx, "T": w.T, "ms_per_step": ms, "kernel_avg_ms": kern,
           "KT_per_s": Kx * w.T / (ms * 1e-3),
           "weighting": "cost-to-go (PAPER.md:320-322)" if cost_to_go else "trajectory",
           "rollout": variant_of(launched), "kernels": short_names(launched),
           "reduction": ("sparse (all-zero weight blocks skipped, bit-identical)" if sparse else
                         "fused into the rollout" if any("epi_combine" in k for k in launched)
                         else "dense GEMV")}
    out["kernel_share"] = share
    if peak and kern.get("rollout"):
        # the rollout's time in the timed pass: ms/step x its share (as the headline roofline)
        r = rollout_roofline(out["rollout"], w.plant, Kx, w.T, ms * share["rollout"], peak,
                             *_sm(), consts or {}, meta or {})
        out["rollout_fp32"] = {k: r.get(k) for k in ("variant", "achieved", "frac", "issue_frac",
                                                     "flop_per_sample_step", "avg_ms")}
        out["rollout_fp32"]["stale_constants"] = (meta or {}).get("stale")
    if kern.get("wsum") and out["reduction"] == "dense GEMV" and not cost_to_go:
        b = 4.0 * w.T * Kx * w.m + 4.0 * Kx
        pk = measured_peaks()
        out["wsum_hbm_GBps"] = b / (kern["wsum"] * 1e-3) / 1e9
        out["wsum_hbm_frac"] = out["wsum_hbm_GBps"] / pk.get("hbm_gbs", 6650.0)
        out["wsum_hbm_frac_spec"] = out["wsum_hbm_GBps"] / HBM_SPEC_GBS   # also vs the spec
    return out


def _sm():
    import torch
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    return props.multi_processor_count, measured_peaks().get("sm_max_mhz", 1965.0)


def c_abi_closed_loop(steps=200):
    """examples/cartpole_mpc.c (config C2 from plain C through the ABI): control-update wall time
    p50/p99 per mppi_optimize_host call (x0 and U in, the step, U out) and the swing-up result."""
    import shutil
    import tempfile
    from paper_1509_01149_b200 import build as B
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        return {"error": "no C compiler"}
    lib = B.build()
    libdir = os.path.dirname(lib)
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "cartpole_mpc")
        subprocess.run([gcc, "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "cartpole_mpc.c"),
                        "-L", libdir, "-lmppi_b200", "-Wl,-rpath," + libdir, "-lm", "-o", exe], check=True)
        out = subprocess.run([exe, str(steps)], capture_output=True, text=True, timeout=300, check=True).stdout.split()
    val = lambda k: float(out[out.index(k) + 1])
    return {"config": "C2", "steps": steps, "update_us_p50": val("update_us_p50"),
            "update_us_p99": val("update_us_p99"), "final_1_plus_cos_theta": val("1+cos(theta)"),
            "mean_q": val("q"), "api": "mppi_optimize_host from C (examples/cartpole_mpc.c)"}


def closed_loop(cfg_name="C2"):
    """Alg. 1 receding horizon through the public API: optimise (graph),
    send u_0 (D2H), plant step on the host (mppi_plant_step), shift; per-step wall clock."""
    import math as _m
    import numpy as np
    import torch
    from mppi_inputs import get
    from paper_1509_01149_b200 import from_workload
    w = get(cfg_name)
    m = from_workload(w)
    U = torch.tensor(w.U0, device="cuda")
    x = w.x0.copy()
    crashed = 0
    lat, qs = [], []
    for step in range(w.steps):
        t0 = time.perf_counter()
        m.optimize(x, U, w.seed, step)
        u0 = U[0].cpu().numpy()                       # "send to actuators"
        lat.append((time.perf_counter() - t0) * 1e6)
        x, q, crashed = m.plant_step(x, u0, crashed)  # environment step (noise-free)
        m.shift(U, np.zeros(w.m, np.float32))         # PAPER.md:372-375, u_init = 0
        qs.append(q)
    torch.cuda.synchronize()
    m.close()
    srt = sorted(lat)
    return {"config": cfg_name, "plant": w.plant, "K": w.K, "T": w.T, "nu": w.nu, "steps": w.steps,
            "step_us_p50": srt[len(srt) // 2], "step_us_p99": srt[int(0.99 * (len(srt) - 1))],
            "mean_q": float(np.mean(qs)), "final_1_plus_cos_theta": float(1 + _m.cos(x[2])),
            "note": "optimize + u0 D2H per step (host wall clock); host plant step and shift excluded"}


def device_closed_loop(cfg_name="C2"):
    """mppi_closed_loop: the whole receding-horizon loop as one CUDA graph (NEXT-2): the first call
    (graph build + instantiation included) and a second call of the same length (the instantiated
    graph reused, only the changed node arguments updated), wall clock per step."""
    import math as _m
    import torch
    from mppi_inputs import get
    from paper_1509_01149_b200 import from_workload
    w = get(cfg_name)
    m = from_workload(w)
    out = {"config": cfg_name, "steps": w.steps}
    for call in ("first_call", "graph_reused"):
        x = torch.tensor(w.x0, device="cuda")
        U = torch.tensor(w.U0, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xl, ul, ql = m.closed_loop(x, U, w.steps, seed=w.seed)
        el = time.perf_counter() - t0
        out["wall_us_per_step_" + call] = el / w.steps * 1e6
    xs = xl.cpu().numpy()
    m.close()
    out.update({"mean_q": float(ql.mean().item()), "final_1_plus_cos_theta": float(1 + _m.cos(xs[-1, 2]))})
    return out


def fig1_trend(nus=(1.0, 10.0, 100.0, 1000.0, 1500.0), Ks=(12, 100, 1000), seconds=10.0):
    """PAPER.md:388-396 Fig. 1 (values unreadable; the trend is what can be compared): average
    running cost of the cart-pole swing-up over 10 s at 50 Hz, 1 s horizon, for nu x K."""
    import torch
    from mppi_inputs.configs import cartpole
    from paper_1509_01149_b200 import from_workload
    steps = int(round(seconds / 0.02))
    out = {}
    for nu in nus:
        row = {}
        for K in Ks:
            w = cartpole(K, 50, nu, steps=steps)
            m = from_workload(w)
            x = torch.tensor(w.x0, device="cuda")
            U = torch.tensor(w.U0, device="cuda")
            _, _, ql = m.closed_loop(x, U, steps, seed=1)
            row[str(K)] = round(float(ql.mean().item()), 2)
            m.close()
        out[str(nu)] = row
    return {"steps": steps, "T": 50, "mean_running_cost[nu][K]": out}


# ----------------------------------------------------------------------------- main
def main():
    args = parse_args()
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    from mppi_inputs import get
    from paper_1509_01149_b200 import ShardedMPPI, from_workload

    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    w = get(args.config)
    K = args.K or w.K
    m = from_workload(w, K=K, rank=rank, world=world)
    U = torch.tensor(w.U0, device="cuda")
    # NCCL: the library drives both collectives itself on its stream (mppi_nccl_attach); gloo (a
    # CPU-side check of the same sharded path): the split-phase calls + torch.distributed
    lib_nccl = world > 1 and args.backend == "nccl"
    if lib_nccl:
        ok = 1
        try:
            t_attach = time.perf_counter()
            m.attach_nccl()
            print("bench.py: rank %d/%d: mppi_nccl_attach ok (ncclCommInitRank, %.1f ms, K_loc %d)"
                  % (rank, world, 1e3 * (time.perf_counter() - t_attach), m.K_loc), file=sys.stderr)
        except Exception as e:      # still a GPU path: the split phase + torch.distributed NCCL
            print("bench.py: mppi_nccl_attach failed (%s); using ShardedMPPI" % e, file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], device="cuda", dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)     # every rank takes the same path
        lib_nccl = bool(flag.item())
    sh = ShardedMPPI(m) if world > 1 and not lib_nccl else None

    def step(i, Ut):
        if sh is None:
            m.optimize(w.x0, Ut, w.seed, i)
        else:
            sh.optimize(w.x0, Ut, w.seed, i)

    probe = None if args.no_probe else run_fp32_probe()
    for i in range(args.warmup):
        step(i, U)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---- the timed region: the shipped default path (CUDA-graph replay with programmatic edges
    # on one GPU; the library's NCCL step at N > 1), no per-kernel events
    clocks = ClockSampler(dev)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record()
    for i in range(args.steps):
        step(args.warmup + i, U)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    launched = m.last_kernels()     # the kernel sequence of one timed step
    per_step_launches = m.last_launch_count() if sh is None else None
    # ---- the profiled pass: the same number of steps right after, every kernel (and collective)
    # bracketed by CUDA events on the context stream (direct launches)
    pclocks = ClockSampler(dev)
    pclocks.start()
    m.profile_enable(True)
    for i in range(args.steps):
        step(args.warmup + args.steps + i, U)
    ktimes = m.profile_read()
    m.profile_enable(False)
    pclk = pclocks.stop()
    kernel_launches = sum(v[1] for k, v in ktimes.items() if k != "collective")
    launches = per_step_launches * args.steps if per_step_launches else kernel_launches
    coll = ktimes.get("collective", (0.0, 0))
    rank_stats = [float(K // world), ms, coll[0] / max(args.steps, 1), ktimes["rollout"][0] / max(ktimes["rollout"][1], 1)]
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([launches], device="cuda", dtype=torch.int64)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt.item())
        rs = torch.tensor(rank_stats, device="cuda", dtype=torch.float64)
        allrs = [torch.zeros_like(rs) for _ in range(world)]
        dist.all_gather(allrs, rs)
        rank_stats = [r.tolist() for r in allrs]
    else:
        rank_stats = [rank_stats]
    assert torch.isfinite(U).all(), "U diverged"
    value = K * w.T * args.steps / (ms * 1e-3)

    # ---- e2e through the public API from host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Uh = np.ascontiguousarray(w.U0.copy())
        h2d = w.T * w.m * 4 + w.n * 4
        d2h = w.T * w.m * 4
        if sh is None:
            if world > 1:
                dist.barrier()
            for i in range(2):
                m.optimize_host(w.x0, Uh, w.seed, i)
            t0 = time.perf_counter()
            for i in range(args.steps):
                m.optimize_host(w.x0, Uh, w.seed, args.warmup + i)
            el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([el], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t.item())
        else:
            Up = torch.tensor(w.U0).pin_memory()
            Ud = torch.empty_like(U)
            dist.barrier()
            t0 = time.perf_counter()
            for i in range(args.steps):
                Ud.copy_(Up, non_blocking=True)
                sh.optimize(w.x0, Ud, w.seed, args.warmup + i)
                Up.copy_(Ud, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            el = time.perf_counter() - t0
            t = torch.tensor([el], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": K * w.T * args.steps / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * el / args.steps,
               "api": "mppi_optimize_host" if sh is None else "ShardedMPPI.optimize + pinned copies"}

    if rank != 0:
        m.close()
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (rank 0's profiled pass, CUDA events on its stream)
    pk = measured_peaks()
    props = torch.cuda.get_device_properties(dev)
    sm_max = (clk or {}).get("sm_max_mhz") or pk.get("sm_max_mhz", 1965.0)
    consts, cmeta = roofline_constants()
    kern = {k: {"avg_ms": v[0] / v[1] if v[1] else None, "launches": v[1], "share": None}
            for k, v in ktimes.items()}
    tot = sum(v[0] for v in ktimes.values()) or 1.0
    for k, v in ktimes.items():
        kern[k]["share"] = v[0] / tot
    dom = max((k for k in ktimes if k != "collective"), key=lambda k: ktimes[k][0])
    K_loc = K // world
    variant_of_step = variant_of(launched) or rollout_variant(w, K_loc)
    fp = fp32_peak(probe, props.multi_processor_count, sm_max)
    # the rollout's time inside the timed region: the step time x the rollout's share of the
    # step's kernel time (CUDA events of the profiled pass; a share is insensitive to the clock
    # drift between the two passes, and step x share also charges the graph's inter-kernel gaps
    # to the rollout, so it never overstates the rate)
    dom_ms_timed = ms / args.steps * kern[dom]["share"]
    if dom == "rollout":
        roof = rollout_roofline(variant_of_step, w.plant, K_loc, w.T, dom_ms_timed,
                                fp["peak_tflops"], props.multi_processor_count, sm_max, consts, cmeta)
        pr = rollout_roofline(variant_of_step, w.plant, K_loc, w.T, kern["rollout"]["avg_ms"],
                              fp["peak_tflops"], props.multi_processor_count, sm_max, consts, cmeta)
        roof["profiled_pass"] = {"avg_ms": kern["rollout"]["avg_ms"], "achieved": pr["achieved"],
                                 "frac": pr["frac"], "clocks": pclk}
        roof["peak_detail"] = fp
        roof["peak_source"] = ("max(derived %.1f, FFMA probe, FFMA2 probe) TFLOP/s; derived = SMs x 128 "
                               "lanes x 2 x max SM clock (B200_PROFILING.md unit counts)" % fp["derived_tflops"])
        if variant_of_step.startswith("x2-grid-fused"):
            # algorithmic bytes: eps written once (and, with the fused reduction, read back once)
            # plus the costs
            roof["algorithmic_bytes_per_launch"] = ((8.0 if variant_of_step.endswith("-epi") else 4.0)
                                                    * w.m * K_loc * w.T + 4.0 * K_loc)
            if w.plant == "quadrotor":
                eff = FULL_SEARCH_QUAD_FLOP * K_loc * w.T / (dom_ms_timed * 1e-3) / 1e12
                roof["effective_full_search"] = {"tflops": eff, "frac": eff / fp["peak_tflops"],
                                                 "flop_per_sample_step": FULL_SEARCH_QUAD_FLOP}
    else:
        algo = 4.0 * w.T * K_loc * w.m + 4.0 * K_loc if dom == "wsum" else 4.0 * w.T * K_loc * w.m
        peak = pk.get("hbm_gbs", 6650.0)
        ach = algo / (dom_ms_timed * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "algorithmic_bytes_per_launch": algo,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"}
    roof["avg_ms"] = dom_ms_timed
    roof["kernel_timing"] = ("avg_ms = timed-region ms/step x the kernel's share of the step's kernel "
                             "time; the share from CUDA events around each launch on the context "
                             "stream in a profiled pass of the same %d steps right after the timed "
                             "region (which itself runs the default graph path without events); "
                             "profiled_pass gives that pass's own per-launch average" % args.steps)
    # secondary rooflines: the HBM-bound reduction and noise kernels
    extra = {}
    if variant_of_step.endswith("-epi"):
        extra["epi_combine_ms"] = kern["wsum"]["avg_ms"]   # K3 is the per-CTA partial combine
    elif kern["wsum"]["avg_ms"]:
        b = 4.0 * w.T * K_loc * w.m + 4.0 * K_loc
        extra["wsum_hbm_GBps"] = b / (kern["wsum"]["avg_ms"] * 1e-3) / 1e9
        extra["wsum_hbm_frac"] = extra["wsum_hbm_GBps"] / pk.get("hbm_gbs", 6650.0)
        extra["wsum_hbm_frac_spec"] = extra["wsum_hbm_GBps"] / HBM_SPEC_GBS
    if kern["noise"]["avg_ms"]:
        b = 4.0 * w.T * K_loc * w.m
        extra["noise_write_GBps"] = b / (kern["noise"]["avg_ms"] * 1e-3) / 1e9
    roof["secondary"] = extra
    roof["step_share"] = kern[dom]["share"]

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(w)
            cpu["cpu"] = lscpu_model()
        except Exception as e:
            cpu = {"error": str(e)[:200]}

    lat = None
    if not args.no_latency and world == 1:
        lat = {c: latency(c) for c in ("C1", "C2")}
        lat["paper_point_K1000_T50"] = _safe(paper_context_latency)

    extra = None
    if not args.no_extra and world == 1:
        tp = dict(peak=fp["peak_tflops"], consts=consts, meta=cmeta)
        extra = {"configs": {c: throughput(c, **tp) for c in ("C1", "C2", "C3", "C4")},
                 "C5_sweep": [throughput("C5", K=1 << e, steps=5, **tp) for e in (16, 18, 20, 22)],
                 "C5_cost_to_go": throughput("C5", steps=5, cost_to_go=True, **tp),
                 "C5_sparse_reduction": throughput("C5", steps=5, sparse=True, **tp),
                 "C5_separate_reduction": _safe(throughput, "C5", steps=5, fused_reduction=False, **tp),
                 # the dense K x (T m) GEMV as its own kernel at every sweep K: its HBM fraction
                 "C5_sweep_separate_reduction": [_safe(throughput, "C5", K=1 << e, steps=5, fused_reduction=False, **tp)
                                                 for e in (16, 18, 20)],
                 "c_abi_closed_loop": _safe(c_abi_closed_loop),
                 "closed_loop": closed_loop("C2"),
                 "device_closed_loop": device_closed_loop("C2"),
                 "fig1_trend": fig1_trend()}

    if extra and args.config == "C5" and not args.K:
        sep = extra.get("C5_separate_reduction") or {}
        if "wsum_hbm_GBps" in sep:   # the dense K x (T m) GEMV as its own kernel (same workload)
            roof["secondary"]["separate_wsum_ms"] = sep["kernel_avg_ms"]["wsum"]
            roof["secondary"]["separate_wsum_hbm_GBps"] = sep["wsum_hbm_GBps"]
            roof["secondary"]["separate_wsum_hbm_frac"] = sep["wsum_hbm_frac"]
            roof["secondary"]["separate_wsum_hbm_frac_spec"] = sep["wsum_hbm_frac_spec"]
    eps_bytes = 4 * w.T * K_loc * w.m
    multi = None
    if world > 1:
        multi = {"ranks": world, "K_loc": K_loc,
                 "per_rank": [{"rank": i, "K_loc": int(r[0]), "ms_timed_region": r[1],
                               "collective_ms_per_step": r[2], "rollout_avg_ms": r[3]}
                              for i, r in enumerate(rank_stats)],
                 "collectives": ("ncclAllGather of every rank's [key, eta, A] record (%d B per rank) on the "
                                 "library stream, rescaled in rank order (MPPI_OPTION_GATHER_COMBINE; "
                                 "mppi_nccl_attach, ncclCommInitRank over torch's NCCL)" % (4 * (2 + ((w.T * w.m + 2) & ~1)))
                                 if lib_nccl else "torch.distributed all_reduce MIN + SUM (split phase)"),
                 "collective_ms_per_step_max": max(r[2] for r in rank_stats),
                 "communicator": ("library-owned NCCL communicator of %d ranks (mppi_nccl_attach; per-rank "
                                  "init lines on stderr)" % world) if lib_nccl else "torch.distributed process group"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Philox noise, committed 4 m cylinder forest, paper cost weights)",
        "config": {"workload": workload_name(args.config, w, K),
                   "K": K, "K_per_gpu": K_loc, "T": w.T, "n_obstacles": int(len(w.obstacles)),
                   "l2": "inputs larger than L2 (noise %.1f GB per GPU per step)" % (eps_bytes / 1e9),
                   "parallelism": "K-sharded dp%d, %s" % (world, "single GPU" if world == 1 else
                                                          "in-library NCCL: one all-gather of per-rank [key, eta, A] records"
                                                          if lib_nccl else
                                                          "MIN + SUM allreduce via torch.distributed")},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "gpu_launches_note": ("library kernels per step (mppi_last_launch_count) x steps, summed over ranks"
                              if per_step_launches else "kernels of the profiled pass (same steps)"),
        "kernel_sequence": short_names(launched),
        "clocks": clk, "kernels": kern, "latency": lat, "extra": extra, "multi_gpu": multi,
        "device": torch.cuda.get_device_name(dev),
        "backend": args.backend if world > 1 else None,
    }
    print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
