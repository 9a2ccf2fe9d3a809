#!/usr/bin/env python
"""Benchmark: ETD3RKDS steps/s and Tucker fp64 TFLOP/s (% of measured DMMA peak) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kx|reference] [--config C2]

Workload (BASELINE.json configs[1]): 2D Schnakenberg, 2 species,
1024 x 1024 grid, exprk3ds_real (Algorithm 1, Table 1), tau = T/m = 2/6000, synthetic seeded
initial data (inputs.make_problem).  One "step" = one full exprk3ds step of both species
(1 Kronecker-sum action + 10 Tucker operators per species, 3 nonlinearity evaluations).

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on the library's
stream, with a 256 MiB L2 flush (> 126 MB L2) between steps, outside the events.  Per-kernel
CUDA events (kx_set_profiling) over the same timed region give the dominant kernel's
(mode-product GEMM) achieved TFLOP/s for the roofline.  e2e: the same steps through
kx_integrate_host with pinned host buffers (H2D of U, step, D2H of U inside the timed region).
N > 1 (torchrun): independent replicas, one per GPU (weak scaling), barrier + max over ranks.

--impl reference: the CPU oracle (oracle/, numpy fp64) timed on this host's cores on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ETD3RKDS steps/sec and Tucker fp64 TFLOP/s (% DMMA peak) at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kx", choices=["kx", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4"])
    ap.add_argument("--no-extras", action="store_true", help="skip Tucker sweep / e2e / cpu leg")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="sharded mode: producers store straight into the peers' receive buffers "
                         "(CUDA IPC, NCCL only as a barrier), or NCCL all-to-alls")
    ap.add_argument("--no-overlap", action="store_true",
                    help="sharded mode: one exchange per phase instead of term-by-term overlap")
    ap.add_argument("--scheme", default=None, choices=["etd2rkds", "etd3rkds", "exprk3ds_cplx"],
                    help="override the config's scheme (e.g. the complex split, Table 2)")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "sharded"],
                    help="N>1: replicas (independent problems, weak scaling) or slab-sharded "
                         "(one global problem, NCCL all-to-all, strong scaling); auto = sharded "
                         "for the 3D configs, replicas for the 2D ones")
    return ap.parse_args()


SCHEME_OVERRIDE = None


def config_dict(name):
    import inputs
    cfg = dict(inputs.CONFIGS[name])
    if SCHEME_OVERRIDE:
        cfg["scheme"] = SCHEME_OVERRIDE
    return cfg


# -------------------------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.samples.append([x.strip() for x in line.split(",")])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax.append(float(s[1]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(s) > 4 + k and s[4 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# -------------------------------------------------------------------------------- oracle --
class OracleRunner:
    """The CPU oracle's step function on this host's cores, on the bench workload.  The
    phi-bank formation (setup, ~7 TFLOP for C2 in the oracle) is replaced by random dense
    matrices of the same shapes: the per-step cost does not depend on their values."""

    def __init__(self, cfg_name):
        import inputs
        from oracle.etd import Exprk3Bank, exprk3ds_step, etd2rkds_step, Etd2Bank
        from oracle import coeffs
        from oracle.models import g_of
        from oracle.tensor import unvec
        cfg = config_dict(cfg_name)
        self.cfg, self.cfg_name = cfg, cfg_name
        prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
        tau = cfg["T"] / cfg["m"]
        d = cfg["d"]
        rs = np.random.default_rng(0)
        if cfg["scheme"] in ("etd3rkds", "exprk3ds_cplx"):
            variant = "cplx" if cfg["scheme"] == "exprk3ds_cplx" else "real"
            s1, s2 = coeffs.etd3_scheme(1, d, variant), coeffs.etd3_scheme(2, d, variant)
            bank = Exprk3Bank(tau, s1, s2)

            def rnd(n):
                m = rs.uniform(0, 1.0 / n, (n, n))
                return m + 1j * rs.uniform(0, 1.0 / n, (n, n)) if variant == "cplx" else m
            for c in range(2):
                Pc = {}
                for key in [("2", 1), ("3", 1), ("3", 2), ("f", 1), ("f", 2)]:
                    Pc[key] = [[rnd(n) for n in prob.n] for _ in range(s1.nterms)]
                bank.P.append(Pc)
            self.stepf = exprk3ds_step
        else:
            P = [[[rs.uniform(0, 1.0 / n, (n, n)) for n in prob.n]] for _ in range(2)]
            bank = Etd2Bank(tau, P, P, 1.0, 2.0 ** (d - 1))
            self.stepf = etd2rkds_step
        self.bank, self.prob, self.g = bank, prob, g_of(prob.model)
        self.U0 = [unvec(u, prob.n) for u in prob.U0]

    def step(self):
        # every sampled step starts from the initial data (random P would otherwise let the
        # state overflow; the cost of a step does not depend on the values)
        self.stepf(self.U0, 0.0, self.bank, self.prob.A, self.g, self.prob.params)

    def sample(self, seconds):
        """steps/s over >= 1 step and about `seconds` of CPU work."""
        t0 = time.perf_counter()
        k = 0
        while True:
            self.step()
            k += 1
            if time.perf_counter() - t0 >= seconds:
                break
        return k / (time.perf_counter() - t0), k

    @staticmethod
    def cores():
        try:
            from threadpoolctl import threadpool_info
            return max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
        except Exception:
            return os.cpu_count()

    def describe(self, k):
        c = self.cfg
        return (f"{k} oracle {c['scheme']} step(s) of {self.cfg_name} ({c['desc']}), numpy fp64 "
                f"(BLAS matmul per mode product) on {os.cpu_count()} host cores; phi-bank formation "
                f"excluded (random dense P of the same shapes)")


def oracle_sample(cfg_name, seconds, threads=None):
    """(steps_per_s, cores, sample description) of a bounded oracle sample; `threads` limits
    the BLAS thread pool (all host cores and one core)."""
    r = OracleRunner(cfg_name)
    if threads is None:
        v, k = r.sample(seconds)
        return v, r.cores(), r.describe(k)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        v, k = r.sample(seconds)
    return v, threads, r.describe(k).replace(f"on {os.cpu_count()} host cores", f"on {threads} core(s)")


# -------------------------------------------------------------------------------- GPU arm --
_PEAK = None


def load_peak():
    """(fp64 DMMA TFLOP/s sustained, HBM copy GB/s, source) — measured IN THIS JOB by the
    tools/peaks.cu microbenchmark (build/peaks: a 1.5 s sustained mma.sync.m8n8k4.f64 loop on
    every SM, DFMA and copy loops; ~5 s), else the round-1 measurement on this pool.
    MEASURED_PEAKS.json has no fp64 entry."""
    global _PEAK
    if _PEAK is not None:
        return _PEAK
    exe = os.path.join(ROOT, "build", "peaks")
    if os.path.exists(exe):
        try:
            r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
            j = json.loads(r.stdout.strip().splitlines()[-1])
            _PEAK = (float(j["dmma_tflops_sustained"]), float(j["hbm_copy_gbs"]),
                     "measured in this job before the timed region: tools/peaks.cu (build/peaks), "
                     f"fp64 DMMA mma.sync.m8n8k4 on all {j.get('sms')} SMs, "
                     f"{j.get('dmma_sustained_ms', 0):.0f} ms sustained; MEASURED_PEAKS.json has no fp64 entry "
                     "(bf16 sustained x nominal 45/2250 would give 28.0)")
            return _PEAK
        except Exception:
            pass
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r01.json")) as f:
            j = json.load(f)
        _PEAK = (float(j["dmma_tflops_sustained"]), float(j.get("hbm_copy_gbs", 0)),
                 "profiles/peaks_r01.json (tools/peaks.cu on this pool, round 1): fp64 DMMA 1.5 s sustained")
    except Exception:
        _PEAK = (None, None, "unavailable")
    return _PEAK


def hbm_peak():
    """HBM copy bandwidth of this pool (driver-written MEASURED_PEAKS.json), else ours."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"
    except Exception:
        _, h, _src = load_peak()
        return h, "tools/peaks.cu copy kernel (this job)"


def stream_floor(N):
    """Size floor of HBM streaming at N doubles per field (profiles/stream_probe_r02.log, written
    by tools/stream_probe.cu on a B200): the step's elementwise launches at C2 are one fused
    first phase (2 fields read, 4 written) and two D = g(U_s) - G passes (4 read, 2 written);
    returns their summed bytes / summed floor times in GB/s, or None."""
    best = {}
    try:
        with open(os.path.join(ROOT, "profiles", "stream_probe_r02.log")) as f:
            for line in f:
                m = re.match(r"N=(\d+) R=(\d+) W=(\d+) grid=\d+: ([\d.]+) us", line)
                if m:
                    k = (int(m.group(1)), int(m.group(2)), int(m.group(3)))
                    best[k] = min(best.get(k, 1e30), float(m.group(4)))
    except OSError:
        return None
    if (N, 2, 4) not in best or (N, 4, 2) not in best:
        return None
    return 3 * 48.0 * N / (best[(N, 2, 4)] + 2 * best[(N, 4, 2)]) / 1e3


def elementwise_roofline(prof, N=None):
    """Aggregate HBM roofline of the non-GEMM kernels (fused G/F pass, D = g(U_s) - G, ...):
    algorithmic bytes (whole-field reads + writes) / their event-timed duration, next to the
    size floor of a pure streaming kernel of the same traffic at this N."""
    if not prof.get("other_ms") or not prof.get("other_bytes"):
        return None
    peak, src = hbm_peak()
    ach = prof["other_bytes"] / prof["other_ms"] / 1e6
    floor = stream_floor(N) if N else None
    return {"bound": "hbm", "kernels": "g_kronsum (G = g(U), F = K U + G), nonlinearity D = g(U_s) - G",
            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak if peak else None,
            "peak_source": src, "ms_total": prof["other_ms"],
            "size_floor": floor, "frac_of_size_floor": ach / floor if floor else None,
            "size_floor_source": "profiles/stream_probe_r02.log (tools/stream_probe.cu)"}


def load_traffic(cfg_name):
    """DRAM bytes (read + write) of ALL mode-product GEMM launches of one step of this config,
    from one `ncu --set full` capture (profiles/ncu_gemm_r02.json, tools/ncu_gemm_summary.py),
    with the algorithmic operand bytes of the same launches: (traffic, alg_bytes) or (None, None)."""
    p = os.path.join(ROOT, "profiles", "ncu_gemm_r02.json")
    try:
        with open(p) as f:
            st = json.load(f)[cfg_name]["step"]
        return st["dram_bytes"], st.get("alg_bytes")
    except Exception:
        return None, None


def setup_ctx(kx, prob, scheme, tau, stream, ctx=None):
    if ctx is None:
        ctx = kx.Context(0 if stream is None else stream.device.index, stream)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    t0 = time.perf_counter()
    ctx.set_tau(tau, scheme)
    return ctx, time.perf_counter() - t0


def other_configs(kx, torch, stream, steps=10):
    """Secondary workloads reported beside the headline (same timing protocol, fewer steps):
    C3 (3D FitzHugh-Nagumo 128^3, exprk3ds_real), the complex split on C2, and C4 (512^3 on
    this one GPU, 3 timed steps)."""
    import inputs
    out = {}
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    full_steps = steps
    for name, cfg_name, scheme in [("C3_fhn_128^3_etd3rkds_real", "C3", None),
                                   ("C2_schnakenberg_1024^2_exprk3ds_cplx", "C2", "exprk3ds_cplx"),
                                   ("C4_fhn_512^3_etd3rkds_real_1gpu", "C4", None)]:
        steps = 3 if cfg_name == "C4" else full_steps
        cfg = config_dict(cfg_name)
        if scheme:
            cfg["scheme"] = scheme
        prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
        tau = cfg["T"] / cfg["m"]
        ctx, _ = setup_ctx(kx, prob, cfg["scheme"], tau, stream)
        U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
        def run(profiled):
            ctx.set_profiling(profiled)
            for _ in range(3):
                ctx.step(U)
            ctx.sync()
            ctx.set_profiling(profiled)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(steps)]
            with torch.cuda.stream(stream):
                for k in range(steps):
                    flush.fill_(float(k))
                    ev[k][0].record()
                    ctx.step(U)
                    ev[k][1].record()
            torch.cuda.synchronize()
            return sum(a.elapsed_time(b) for a, b in ev) / steps
        ms = run(False)          # plain graph: steps/s
        run(True)                # instrumented pass: GEMM device time
        prof = ctx.profile()
        ctx.set_profiling(False)
        ach = prof["gemm_flops"] / prof["gemm_ms"] / 1e9
        out[name] = {"steps_per_s": round(1e3 / ms, 2), "ms_per_step": round(ms, 4),
                     "gemm_tflops": round(ach, 2)}
        ctx.close()
        del U
        torch.cuda.empty_cache()
    # C1 with many steps per launch (kx_step_n: the small-grid cluster kernel keeps the state in
    # shared memory across steps; one launch, so no L2 flush between its steps)
    cfg = config_dict("C1")
    prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
    ctx, _ = setup_ctx(kx, prob, cfg["scheme"], cfg["T"] / cfg["m"], stream)
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    nsteps = 3000   # the C1 protocol (T = 0.25, m = 3000) in one launch
    ctx.step_n(U, 10)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        ctx.step_n(U, nsteps)
        e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / nsteps
    out["C1_schnakenberg_64^2_etd2rkds_step_n"] = {"steps_per_s": round(1e3 / ms, 1),
                                                   "us_per_step": round(ms * 1e3, 2),
                                                   "launches": 1, "steps_per_launch": nsteps}
    ctx.close()
    return out


def tf32_peak():
    """Dense tf32 tensor peak of this pool: MEASURED_PEAKS.json bf16 sustained x the guide's nominal
    ratio tf32 / bf16 = 1.1 / 2.25 PFLOP/s (B200_PROFILING.md), with the source."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return (float(j["bf16_tflops_sustained"]) * 1.1 / 2.25,
                "MEASURED_PEAKS.json bf16_tflops_sustained x 1.1/2.25 (nominal tf32/bf16 dense)")
    except Exception:
        return 1100.0, "B200_PROFILING.md nominal tf32 dense 1.1 PFLOP/s (MEASURED_PEAKS.json absent)"


def f32_workloads(kx, torch, stream, steps=10):
    """The fp32 variant (the paper's "CUDA single" columns): kx_step_f32 at C2 and
    C3 (same timing protocol: L2 flushed between steps, CUDA events on the library stream) and its
    mode-product GEMM (tcgen05 kind::tf32, three passes) against the tf32 tensor peak."""
    import inputs
    out = {}
    peak, src = tf32_peak()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for cfg_name in ("C2", "C3", "C4"):
        cfg = config_dict(cfg_name)
        prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
        ctx, _ = setup_ctx(kx, prob, cfg["scheme"], cfg["T"] / cfg["m"], stream)
        U = [torch.from_numpy(u.astype("float32")).cuda() for u in prob.U0]
        ctx.step_f32(U, 1 if cfg_name == "C4" else 3)
        ctx.sync()
        nsteps = 3 if cfg_name == "C4" else steps
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nsteps)]
        with torch.cuda.stream(stream):
            for k in range(nsteps):
                flush.fill_(float(k))
                ev[k][0].record()
                ctx.step_f32(U, 1)
                ev[k][1].record()
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / nsteps
        ctx.set_profiling(True)
        ctx.step_f32(U, 1 if cfg_name == "C4" else 5)
        ctx.sync()
        prof = ctx.profile()
        ctx.set_profiling(False)
        alg = prof["gemm_flops"] / prof["gemm_ms"] / 1e9   # (profile over the same number of steps)
        out[cfg_name] = {"workload": cfg["desc"] + " (fp32)", "steps_per_s": round(1e3 / ms, 1),
                         "ms_per_step": round(ms, 4), "gemm_share": round(prof["gemm_ms"] / (prof["gemm_ms"] + prof["other_ms"]), 3),
                         "gemm_tflops_fp32_equiv": round(alg, 1),
                         "gemm_tflops_tensor": round(3 * alg, 1),
                         "gemm_frac_of_tf32_peak": round(3 * alg / peak, 3),
                         "finite": all(bool(torch.isfinite(u).all()) for u in U)}
        ctx.close()
        del U
        torch.cuda.empty_cache()
    # one large Tucker (the GEMM at its best shape)
    n = 4096
    ctx = kx.Context(stream.device.index, stream)
    ctx.set_grid([n, n], 1)
    X = torch.rand(n * n, device="cuda")
    Y = torch.empty_like(X)
    Ls = [torch.rand(n * n, device="cuda") / n] * 2
    ms = _graph_time(torch, stream, lambda: ctx.tucker_f32(X, Y, Ls), 10)
    fl = 2.0 * n * n * 2 * n
    out["tucker_d2_n4096"] = {"ms": round(ms, 4), "tflops_fp32_equiv": round(fl / ms / 1e9, 1),
                              "frac_of_tf32_peak": round(3 * fl / ms / 1e9 / peak, 3)}
    ctx.close()
    out["peak_tf32_tflops"] = round(peak, 1)
    out["peak_source"] = src
    out["method"] = ("tcgen05.mma kind::tf32, A B ~ A_lo B_hi + A_hi B_lo + A_hi B_hi (x = hi + lo, tf32 "
                     "parts), TMA loads, per-k-tile TMEM partials summed round-to-nearest in registers")
    return out


def _graph_time(torch, stream, fn, reps):
    """Best-of-3 device ms per call of fn(), R back-to-back calls captured in a CUDA graph."""
    for _ in range(2):
        fn()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
        for _ in range(reps):
            fn()
    g.replay()
    stream.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        with torch.cuda.stream(stream):
            e0.record()
            g.replay()
            e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        best = ms if best is None else min(best, ms)
    del g
    return best


# batch sizes of the batched sweep: >= ~4 GFLOP per batched Tucker where memory allows
BATCH = {(2, 64): 4096, (2, 128): 512, (2, 256): 64, (2, 512): 16, (2, 1024): 4,
         (3, 64): 32, (3, 128): 4, (3, 256): 1}


def tucker_sweep(kx, torch, stream, budget_s=60.0):
    """Tucker microbenchmark, fp64, dense flops 2 N d n / device time:
      * single: ONE Tucker operator T(X, {L_mu}) on an n^d tensor (its latency);
      * batched: kx_tucker_batched over B independent n^d tensors sharing {L_mu} (throughput:
        one GEMM launch per mode for the whole batch).
    R back-to-back calls are captured in a CUDA graph and replayed between CUDA events (no host
    launch overhead in the number); the larger working sets exceed L2, the small ones are
    L2-resident by nature."""
    single, batched, single_us, batch_of = {}, {}, {}, {}
    t_start = time.perf_counter()
    sizes = [(2, n) for n in (64, 128, 256, 512, 1024, 2048, 4096)] + \
            [(3, n) for n in (64, 128, 256, 512, 1024)]
    for d, n in sizes:
        if time.perf_counter() - t_start > budget_s:
            break
        N = n ** d
        fl = 2.0 * N * n * d
        ctx = kx.Context(stream.device.index, stream)
        ctx.set_grid([n] * d, 1)
        L = torch.rand(n * n, dtype=torch.float64, device="cuda") / n
        Ls = [L] * d
        B = BATCH.get((d, n), 0)
        X = torch.rand(N * max(B, 1), dtype=torch.float64, device="cuda")
        Y = torch.empty_like(X)
        reps = int(min(200, max(3, 2e10 / fl)))
        ms = _graph_time(torch, stream, lambda: ctx.tucker(X[:N], Y[:N], Ls), reps)
        key = f"d{d}_n{n}"
        single[key] = round(fl / ms / 1e9, 2)
        single_us[key] = round(ms * 1e3, 2)
        if B > 1:
            reps = int(min(100, max(3, 2e10 / (fl * B))))
            ms = _graph_time(torch, stream, lambda: ctx.tucker_batched(X, Y, Ls, B), reps)
            batched[key] = round(fl * B / ms / 1e9, 2)
            batch_of[key] = B
        ctx.close()
        del X, Y, L
        torch.cuda.empty_cache()
    return {"single": single, "single_us": single_us, "batched": batched, "batch": batch_of}


def emulate_sharded_p8(kx, torch, stream, c4_one, P=8, steps=3, warm=2):
    """The 8-GPU slab-sharded C4 step emulated on this one GPU (tools/emulate_sharded.py): an
    in-process loopback group runs every rank's kernels back to back with direct peer stores
    between the ranks' buffers; group step / P is the compute one rank does in a real 8-GPU
    step (communication excluded), compared with the single-GPU C4 step / P.  Self-checking:
    three i_d planes of every rank's slab after the warm + timed steps are compared with a
    single-GPU run of the same steps (relative inf-norm)."""
    import inputs
    if not c4_one:
        return None
    cfg = config_dict("C4")
    tau = cfg["T"] / cfg["m"]
    grp, Ug = None, None
    try:
        grp = kx.Group(P, stream=stream)
        for r in range(P):
            pr = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0, slab=(r, P))
            setup_ctx(kx, pr, cfg["scheme"], tau, stream, ctx=grp.ctx[r])
        grp.set_p2p(True)
        Ug = [[torch.from_numpy(u.copy()).cuda() for u in
               inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0, slab=(r, P)).U0]
              for r in range(P)]
        for _ in range(warm):
            grp.step(Ug)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
            for _ in range(steps):
                grp.step(Ug)
            e1.record()
        e1.synchronize()
        per_rank = e0.elapsed_time(e1) / steps / P
        n = cfg["n"]
        plane = n * n
        loc = n // P                       # i_d planes per rank
        picks = [0, loc // 2, loc - 1]
        sample = {(r, c): Ug[r][c].view(loc, plane)[picks].cpu().numpy()
                  for r in range(P) for c in range(2)}
    except Exception as e:   # the emulation is an extra; it never takes the headline down
        return {"error": str(e)[:200]}
    finally:
        if grp is not None:
            grp.close()
        del Ug
        torch.cuda.empty_cache()
    one = c4_one["ms_per_step"]
    out = {"ranks": P, "per_rank_compute_ms": round(per_rank, 3), "single_gpu_ms": one,
           "compute_efficiency": round(one / (P * per_rank), 3),
           "note": "one-GPU emulation (loopback group, direct peer stores): the compute of one "
                   "rank of an 8-GPU C4 step; communication not included"}
    ctx, U = None, None
    try:   # the same warm + timed steps on one GPU, compared at the sampled planes
        prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
        ctx, _ = setup_ctx(kx, prob, cfg["scheme"], tau, stream)
        U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
        del prob
        for _ in range(warm + steps):
            ctx.step(U)
        ctx.sync()
        err, scale = 0.0, 0.0
        for (r, c), got in sample.items():
            ref = U[c].view(n, plane)[[r * loc + k for k in picks]].cpu().numpy()
            err = max(err, float(np.max(np.abs(got - ref))))
            scale = max(scale, float(np.max(np.abs(ref))))
        rel = err / scale
        out["check"] = {"vs": f"single-GPU C4 after the same {warm + steps} steps",
                        "sampled_points": int(sum(v.size for v in sample.values())),
                        "rel_inf_err": rel, "tol": 1e-12, "pass": bool(rel <= 1e-12)}
    except Exception as e:
        out["check"] = {"error": str(e)[:200]}
    finally:
        if ctx is not None:
            ctx.close()
        del U
        torch.cuda.empty_cache()
    return out


def sharded_closed_form_check(kx, torch, stream, cfg, n, rank, world, dist):
    """Correctness of the sharded step at full size, without an oracle run: g = 0 and cosine-mode
    data (an eigenvector of every Neumann Laplacian A_mu, inputs.cosine_mode) make one exprk3ds
    step the scalar recurrence U+ = Re(1 + tau sum_mu lam_mu sum_i eta_i prod_mu
    phi_{l_i}(tau alpha_{i,mu} lam_mu)) U (eq:exprk3 P:586-594 with F = K U, split eq:splitnd3),
    evaluated from the library's own Table 3 coefficients (kx_scheme_coefficients); every
    rank compares its slab, max over ranks."""
    import cmath
    import math
    import inputs
    tau = cfg["T"] / cfg["m"]
    d = cfg["d"]
    ks = (2, 37, 130)[:d]
    delta = 42.1887 if cfg["model"] == "fhn" else 1.0
    length = math.pi if cfg["model"] == "fhn" else 1.0
    A = inputs.laplacian_neumann(n[0], length, delta)
    lams = [inputs.cosine_eigenvalue(n[mu], length, delta, ks[mu]) for mu in range(d)]
    modes = [inputs.cosine_mode(n[mu], ks[mu]) for mu in range(d)]
    ndl = n[-1] // world
    modes[-1] = modes[-1][rank * ndl:(rank + 1) * ndl]          # this rank's i_d block
    x = inputs.kron_vec(modes)
    uid = [kx.nccl_unique_id() if rank == 0 else None]   # a fresh communicator needs a fresh id
    if dist is not None:
        dist.broadcast_object_list(uid, src=0)
    ctx = kx.Context(torch.cuda.current_device(), stream, dist=(uid[0], rank, world))
    try:
        ctx.set_grid(n, 2)
        for c in range(2):
            for mu in range(d):
                ctx.set_direction_matrix(c, mu + 1, A)
        ctx.set_model("none")
        ctx.set_tau(tau, "etd3rkds")
        etas, inner, alphas = kx.scheme_coefficients("etd3rkds", 1, d)

        def phis(ell, z):
            e = cmath.exp(z)
            return [e, (e - 1) / z, (e - 1 - z) / (z * z)][ell]

        split = sum(eta * math.prod(phis(li, tau * al[m] * lams[m]) for m in range(d))
                    for eta, li, al in zip(etas, inner, alphas))
        factor = (1.0 + tau * sum(lams) * split).real
        U = [torch.from_numpy(x.copy()).cuda(), torch.from_numpy(x.copy()).cuda()]
        ctx.step(U)
        ctx.sync()
        got = U[0].cpu().numpy()
        err = float(abs(got - factor * x).max() / abs(factor * x).max())
        if dist is not None:
            t = torch.tensor([err], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            err = float(t.item())
        return {"what": "one sharded step, g = 0, cosine mode (k = %s), scalar recurrence from Table 3" % (ks,),
                "rel_inf_err": err, "tol": 1e-11, "pass": err <= 1e-11}
    except Exception as e:
        return {"error": str(e)[:300]}
    finally:
        ctx.close()


def sharded_tucker(kx, torch, stream, rank, world, dist, sizes=(512, 1024), reps=3):
    """C5 at P GPUs (BASELINE.json configs[4]): one d = 3 Tucker operator on an n^3 tensor slab-
    sharded over the ranks (kx_tucker on NCCL ranks: pack, all-to-all, modes 3..2 on full fibres,
    all-to-all, concatenated-K mode 1), dense flops 2 N d n over the max-over-ranks device time."""
    out = {}
    peak = load_peak()[0] if rank == 0 else None
    for n in sizes:
        N = n ** 3
        uid = [kx.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        ctx = kx.Context(torch.cuda.current_device(), stream, dist=(uid[0], rank, world))
        try:
            ctx.set_grid([n, n, n], 1)
            X = torch.rand(N // world, dtype=torch.float64, device="cuda")
            Y = torch.empty_like(X)
            Ls = [torch.rand(n * n, dtype=torch.float64, device="cuda") / n for _ in range(3)]
            ctx.tucker(X, Y, Ls)
            ctx.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if dist is not None:
                dist.barrier()
            with torch.cuda.stream(stream):
                e0.record()
                for _ in range(reps):
                    ctx.tucker(X, Y, Ls)
                e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            if dist is not None:
                t = torch.tensor([ms], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            tf = 2.0 * N * 3 * n / ms / 1e9
            out[f"d3_n{n}"] = {"ms": round(ms, 3), "tflops": round(tf, 2),
                               "frac_of_P_dmma": round(tf / (world * peak), 3) if peak else None}
            del X, Y, Ls
        except Exception as e:
            out[f"d3_n{n}"] = {"error": str(e)[:200]}
        finally:
            ctx.close()
            torch.cuda.empty_cache()
    return out


def run_kx(args, rank, world, sharded):
    import torch
    import inputs
    from paper_2310_07551_b200 import kx

    torch.cuda.set_device(rank % torch.cuda.device_count())
    stream = torch.cuda.Stream()
    cfg = config_dict(args.config)
    tau = cfg["T"] / cfg["m"]
    dist = None
    if world > 1:
        import torch.distributed as dist
    if sharded:
        uid = [kx.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0, slab=(rank, world))
        ctx = kx.Context(torch.cuda.current_device(), stream, dist=(uid[0], rank, world))
        if args.no_overlap:
            ctx.set_dist_overlap(False)
        ctx.set_grid(prob.n, 2)
        for c in range(2):
            for mu in range(prob.d):
                ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
        ctx.set_model(prob.model, prob.params)
        t0 = time.perf_counter()
        ctx.set_tau(tau, cfg["scheme"])
        phi_s = time.perf_counter() - t0
        exchange = args.exchange
        if args.exchange == "p2p":
            # direct peer stores: every rank maps the others' receive buffers (CUDA IPC); if any
            # rank cannot export or import, every rank falls back to NCCL all-to-alls
            why = ""
            try:
                blob = ctx.ipc_export()
            except Exception as e:
                blob, why = None, f"export: {e}"[:200]
            blobs = [blob]
            if world > 1:
                blobs = [None] * world
                dist.all_gather_object(blobs, blob)
            ok = all(b is not None for b in blobs)
            if ok:
                try:
                    ctx.ipc_import(blobs)
                except Exception as e:
                    ok, why = False, f"import: {e}"[:200]
            if world > 1:
                t = torch.tensor([1 if ok else 0], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                ok = bool(t.item())
            if not ok:
                ctx.set_tau(tau, cfg["scheme"])   # drops any partial peer mapping
                exchange = "nccl (CUDA IPC peer mapping failed" + (f": {why}" if why else " on another rank") + ")"
    else:
        prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=rank)
        ctx, phi_s = setup_ctx(kx, prob, cfg["scheme"], tau, stream)
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")   # 256 MiB
    torch.cuda.synchronize()
    # warm-up (graph capture + replay on one GPU)
    for k in range(args.warmup):
        ctx.step(U, k * tau)
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.reset_counters()

    def timed_pass(profiled):
        """K steps, each bracketed by CUDA events on the library stream, L2 flushed between."""
        ctx.set_profiling(profiled)
        if profiled:       # re-capture the step graph with per-kernel event nodes
            ctx.step(U)
            ctx.sync()
            ctx.set_profiling(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                flush.fill_(float(k))
                evs[k][0].record()
                ctx.step(U, (args.warmup + k) * tau)
                evs[k][1].record()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    # timed region 1 (the headline): the plain step graph, no instrumentation
    clocks = ClockSampler(rank % max(1, torch.cuda.device_count()))
    clocks.start()
    time.sleep(0.3)
    torch.cuda.profiler.start()    # `ncu --profile-from-start off` sees exactly the timed steps
    step_ms = timed_pass(False)
    torch.cuda.profiler.stop()
    clk = clocks.stop()
    cnt = ctx.counters()
    # timed region 2: the same K steps with an event pair around every kernel (the graph's
    # event-record nodes add 4-8% per step, so they are kept out of the headline) -> per-kernel
    # device time of the mode-product GEMMs for the roofline
    prof_step_ms = timed_pass(True)
    prof = ctx.profile()
    ctx.set_profiling(False)
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    prof_ms = sum(prof_step_ms) / len(prof_step_ms)
    ok = all(ctx.check_finite(u) for u in U)
    res = dict(ms=ms, step_ms=step_ms, prof=prof, prof_ms=prof_ms, cnt=cnt, clocks=clk, phi_s=phi_s,
               finite=ok)
    if sharded:
        res["exchange"] = exchange
    # ---- e2e: pinned host state -> device, one step through the public API, device -> host
    if not args.no_extras:
        Uh = [torch.from_numpy(u.copy()).pin_memory() for u in prob.U0]
        e2e_ms = []
        for k in range(args.steps + 1):
            flush.fill_(float(k))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if sharded:
                with torch.cuda.stream(stream):
                    for c in range(2):
                        U[c].copy_(Uh[c], non_blocking=True)
                    ctx.step(U)
                    for c in range(2):
                        Uh[c].copy_(U[c], non_blocking=True)
                stream.synchronize()
            else:
                ctx.integrate_host([u.numpy() for u in Uh], 1)
            if k > 0:    # the first call captures the graph for the host-path buffers
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e = sum(e2e_ms) / len(e2e_ms)
        if world > 1:
            t = torch.tensor([e], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e = float(t.item())
        res["e2e_ms"] = e
        res["e2e_bytes"] = 2 * (prob.N // (world if sharded else 1)) * 8
    ctx.close()
    if sharded and cfg["d"] == 3:   # after the timed context is gone (memory)
        del U
        torch.cuda.empty_cache()
        res["check"] = sharded_closed_form_check(kx, torch, stream, cfg, prob.n, rank, world,
                                                 dist if world > 1 else None)
        res["tucker_sharded"] = sharded_tucker(kx, torch, stream, rank, world, dist if world > 1 else None)
    if not args.no_extras and rank == 0 and not sharded:
        del U, flush
        torch.cuda.empty_cache()
        res["tucker"] = tucker_sweep(kx, torch, stream)
        res["others"] = other_configs(kx, torch, stream)
        try:
            res["f32"] = f32_workloads(kx, torch, stream)
        except Exception as e:   # the fp64 headline must not depend on the fp32 variant
            res["f32"] = {"error": str(e)[:300]}
        if world == 1:
            res["emulated"] = emulate_sharded_p8(kx, torch, stream,
                                                 res["others"].get("C4_fhn_512^3_etd3rkds_real_1gpu"))
    return res, cfg, prob


def child_env(rank, world, port):
    """Environment of a child rank with its own rendezvous on 127.0.0.1:port.  Under torchrun the
    parent's environment says TORCHELASTIC_USE_AGENT_STORE=True (the agent hosts the TCPStore),
    which would make every child a store CLIENT of a server nobody starts on the new port: the
    TORCHELASTIC_* variables are dropped so that the child rank 0 hosts it."""
    env = {k: v for k, v in os.environ.items() if not k.startswith("TORCHELASTIC_")}
    env.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
               LOCAL_RANK=os.environ.get("LOCAL_RANK", str(rank)), NCCL_DEBUG="INFO")
    return env


def sharded_subrun(args, rank, world, timeout_s=480):
    """N > 1 replicas runs also measure the north_star's multi-GPU workload: C4 (512^3)
    slab-sharded over the same GPUs (direct peer stores + NCCL barriers), in child processes
    with their own rendezvous and a timeout, so that a failure there cannot take the headline
    line down.  Every rank joins; rank 0 returns the child's result (or the error)."""
    import socket
    import subprocess
    import torch
    import torch.distributed as dist
    port = [None]
    if rank == 0:
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port[0] = sk.getsockname()[1]
        sk.close()
    dist.broadcast_object_list(port, src=0)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    env = child_env(rank, world, port[0])
    steps = 10
    cmd = [sys.executable, os.path.abspath(__file__), "--gpus", str(world), "--config", "C4",
           "--mode", "sharded", "--steps", str(steps), "--warmup", "3", "--no-extras"]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout_s)
        out = {"rc": r.returncode}
        if rank == 0:
            lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
            if r.returncode == 0 and lines:
                d = json.loads(lines[-1])
                out = {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                       "steps": d["steps"], "warmup": d["warmup"],
                       "n_gpus": d["n_gpus"], "scaling": d["scaling"],
                       "workload": d["config"]["workload"], "parallelism": d["config"]["parallelism"],
                       "exchange": d.get("exchange"), "check": d.get("check"),
                       "tucker_sharded": d.get("tucker_sharded"),
                       "roofline_frac": d["roofline"]["frac"], "clocks": d.get("clocks"),
                       "finite": d.get("finite")}
            else:
                out["error"] = [l for l in r.stderr.strip().splitlines() if "NCCL INFO" not in l][-3:]
            # NCCL communicator evidence (NCCL_DEBUG=INFO on the child ranks)
            info = [l.strip() for l in r.stderr.splitlines() if "NCCL INFO" in l]
            out["nccl_comm_lines"] = [l[-160:] for l in info if "nRanks" in l][:4]
            out["nccl_nvls_lines"] = [l[-160:] for l in info if "NVLS" in l][:3]
    except subprocess.TimeoutExpired:
        out = {"error": f"timeout after {timeout_s} s", "steps": steps}
    dist.barrier()
    return out if rank == 0 else None


def main():
    global SCHEME_OVERRIDE
    args = parse()
    SCHEME_OVERRIDE = args.scheme
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and world == 1:
        print(json.dumps({"error": "run N>1 under torchrun (one process per GPU)"}))
        return 2
    cfg = config_dict(args.config)
    if args.impl == "reference":
        # the oracle on this host's cores (rank 0 only under torchrun; the others exit 0)
        if rank != 0:
            return 0
        runner = OracleRunner(args.config)
        for _ in range(args.warmup):        # untimed warm-up steps
            runner.step()
        per = max(0.5, args.cpu_seconds / max(1, args.steps))
        vals, ks = [], 0
        for _ in range(max(1, args.steps)):   # K timed samples, each >= 1 step
            v, k = runner.sample(per)
            vals.append(v)
            ks += k
        value = statistics.mean(vals)
        cores = runner.cores()
        line = {"metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": f"{args.config}: {cfg['desc']}", "grid": [cfg["n"]] * cfg["d"],
                           "species": 2, "scheme": cfg["scheme"], "parallelism": "single host"},
                "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores,
                                 "kind": "oracle", "sample": runner.describe(ks)},
                "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("nccl")
    sharded = args.mode == "sharded" or (world > 1 and args.mode == "auto" and cfg["d"] == 3)
    if rank == 0:
        load_peak()   # the roofline denominator, measured on this GPU before the timed region
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    res, cfg, prob = run_kx(args, rank, world, sharded)
    extra_sharded = None
    if world > 1 and not sharded and not args.no_extras and args.mode == "auto":
        extra_sharded = sharded_subrun(args, rank, world)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0
    value = (1 if sharded else world) * 1e3 / res["ms"]
    prof = res["prof"]
    peak, hbm, peak_src = load_peak()
    achieved = prof["gemm_flops"] / prof["gemm_ms"] / 1e9 if prof["gemm_ms"] > 0 else None
    launches = res["cnt"]["gemm_launches"] + res["cnt"]["other_launches"]
    gemm_launches = prof["gemm_launches"]
    traffic, traffic_alg = load_traffic(args.config)
    step_flops = res["cnt"]["mode_product_flops"] / max(1, res["cnt"]["steps"])
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"],
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 initial data, FD Neumann Laplacians; inputs/)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "grid": prob.n, "species": 2,
                   "scheme": cfg["scheme"], "tau": cfg["T"] / cfg["m"],
                   "parallelism": ((f"slab-sharded x{world} along i_d ("
                                    + ("direct peer stores over NVLink + NCCL barrier" if args.exchange == "p2p"
                                       else "NCCL all-to-all") + ")") if sharded
                                   else ("replicas" if world > 1 else "single GPU")),
                   "l2": "256 MiB buffer written between timed steps (L2 flushed)"},
        "roofline": {"bound": "tensor", "kernel": "mode-product GEMM (fp64 DMMA mma.sync.m8n8k4)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if (achieved and peak) else None,
                     "traffic": traffic,
                     "traffic_alg": traffic_alg,
                     "traffic_per": "step: the sum over all mode-product GEMM launches of one step "
                                    "(ncu dram__bytes_read.sum + dram__bytes_write.sum; traffic_alg = each "
                                    "operand read once, the output written once)",
                     "peak_source": peak_src,
                     "measured_over": "a second pass of the same K steps with a CUDA-event pair "
                                      "around every kernel (event-record nodes in the step graph)",
                     "gemm_share_of_step": prof["gemm_ms"] / (res["prof_ms"] * args.steps),
                     "instrumented_ms_per_step": res["prof_ms"],
                     "gemm_launches_per_step": gemm_launches / args.steps},
        "elementwise_roofline": elementwise_roofline(prof, int(np.prod(prob.n))),
        "step_tflops": step_flops / res["ms"] / 1e9,
        "gpu_launches": launches,
        "clocks": res["clocks"],
        "phi_bank_setup_s": res["phi_s"],
        "finite": res["finite"],
    }
    if sharded:
        line["exchange"] = res.get("exchange")
        if res.get("check"):
            line["check"] = res["check"]
        if res.get("tucker_sharded"):
            line["tucker_sharded"] = res["tucker_sharded"]
    if "e2e_ms" in res:
        line["e2e"] = {"value": (1 if sharded else world) * 1e3 / res["e2e_ms"], "unit": "steps/s",
                       "h2d_bytes_per_step": res["e2e_bytes"], "d2h_bytes_per_step": res["e2e_bytes"]}
    if "tucker" in res:
        tk = res["tucker"]
        line["tucker_tflops"] = tk["single"]
        line["tucker_single_us"] = tk["single_us"]
        line["tucker_batched_tflops"] = tk["batched"]
        line["tucker_batch_size"] = tk["batch"]
        line["other_workloads"] = res.get("others")
        if res.get("f32"):
            line["fp32_variant"] = res["f32"]
        if res.get("emulated"):
            line["sharded_c4_emulated"] = res["emulated"]
        if peak:
            line["tucker_frac_of_dmma"] = {k: round(v / peak, 3) for k, v in tk["single"].items()}
            line["tucker_batched_frac_of_dmma"] = {k: round(v / peak, 3) for k, v in tk["batched"].items()}
    if not args.no_extras and prob.N <= 64 * 1024 * 1024:
        v, cores, sample = oracle_sample(args.config, args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle",
                                "sample": sample}
        v1, _, sample1 = oracle_sample(args.config, args.cpu_seconds / 2, threads=1)
        line["cpu_baseline_1core"] = {"value": v1, "unit": "steps/s", "cores": 1, "kind": "oracle",
                                      "sample": sample1}
    if extra_sharded is not None:
        c4 = (res.get("others") or {}).get("C4_fhn_512^3_etd3rkds_real_1gpu") or {}
        if extra_sharded.get("ms_per_step") and c4.get("ms_per_step"):
            P = extra_sharded["n_gpus"]
            extra_sharded["one_gpu_ms_per_step"] = c4["ms_per_step"]
            extra_sharded["parallel_efficiency"] = round(c4["ms_per_step"] / (P * extra_sharded["ms_per_step"]), 4)
            extra_sharded["efficiency_def"] = "E(P) = T(1 GPU) / (P T(P)), C4 512^3 step, both measured in this job"
        line["sharded_c4"] = extra_sharded
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
