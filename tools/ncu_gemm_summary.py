"""Summarise `ncu --set full` raw CSV exports of every mode-product GEMM launch of ONE step
(tools/prof_step.py --steps 1, -k regex:gemm_kernel) into profiles/ncu_gemm_r02.json: per launch
duration, DMMA-pipe activity, SM-active fraction, DRAM bytes, L2 hit rate; per step the sums,
next to the algorithmic operand bytes of the same launches (each operand read once, the output
written once: A + B (+ D) + C, from the launch shapes of the step schedule).

    python tools/ncu_gemm_summary.py C2=gpurun_out/raw_C2.csv C3=gpurun_out/raw_C3.csv
"""
import csv
import json
import os
import sys

M = {"time_us": "gpu__time_duration.sum",
     "dmma_active_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
     "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
     "l2_hit_pct": "lts__t_sector_hit_rate.pct",
     "sm_active_cycles": "sm__cycles_active.avg", "elapsed_cycles": "sm__cycles_elapsed.avg"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def alg_bytes(cfg):
    """(name, algorithmic bytes) of every GEMM launch of one step, both species (fp64)."""
    if cfg == "C2":     # d = 2, n = 1024, T = 2: F first (6 terms), U2 (2 seg), D2 first, U3 (4), D3, U+ (4)
        n, N, T = 1024, 1024 ** 2, 2
        first = lambda t: (t * n * n + N + t * N) * 8 * 2
        stage = lambda k: (k * N + k * n * n + 2 * N) * 8 * 2
        return [("F first mode (concat-M 3T)", first(3 * T)), ("U2 stage (concat-K T)", stage(T)),
                ("D2 first mode", first(T)), ("U3 stage (concat-K 2T)", stage(2 * T)),
                ("D3 first mode", first(T)), ("U+ stage (concat-K 2T)", stage(2 * T))]
    if cfg == "C3":     # d = 3, n = 128, T = 3: + middle modes batched over terms
        n, N, T = 128, 128 ** 3, 3
        first = lambda t: (t * n * n + N + t * N) * 8 * 2
        mid = lambda t: (t * n * n + 2 * t * N) * 8 * 2
        stage = lambda k: (k * N + k * n * n + 2 * N) * 8 * 2
        return [("F first mode", first(3 * T)), ("F middle mode", mid(3 * T)), ("U2 stage", stage(T)),
                ("D2 first", first(T)), ("D2 middle", mid(T)), ("U3 stage", stage(2 * T)),
                ("D3 first", first(T)), ("D3 middle", mid(T)), ("U+ stage", stage(2 * T))]
    return None


def main():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out_path = os.path.join(root, "profiles", "ncu_gemm_r02.json")
    out = {"source": "ncu --set full --clock-control none, one step (graph replay), -k regex:gemm_kernel; "
                     "cold L2 per launch (ncu cache control)"}
    for arg in sys.argv[1:]:
        cfg, path = arg.split("=", 1)
        rows = list(csv.reader(open(path)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        hdr, units = rows[hi], rows[hi + 1]
        alg = alg_bytes(cfg)
        launches = []
        for j, r in enumerate(rows[hi + 2:]):
            e = {}
            for k, m in M.items():
                c = hdr.index(m)
                v = float(r[c])
                e[k] = v * SCALE.get(units[c], 1)
            e["dram_bytes"] = e.pop("dram_read") + e.pop("dram_write")
            e["sm_active_frac"] = e.pop("sm_active_cycles") / e.pop("elapsed_cycles")
            if alg and j < len(alg):
                e["what"], e["alg_bytes"] = alg[j]
                e["dram_over_alg"] = round(e["dram_bytes"] / e["alg_bytes"], 2)
            launches.append(e)
        step = {"time_us": sum(e["time_us"] for e in launches),
                "dram_bytes": sum(e["dram_bytes"] for e in launches),
                "dmma_active_pct_time_weighted": sum(e["dmma_active_pct"] * e["time_us"] for e in launches)
                / sum(e["time_us"] for e in launches)}
        if alg:
            step["alg_bytes"] = sum(b for _, b in alg)
            step["dram_over_alg"] = round(step["dram_bytes"] / step["alg_bytes"], 2)
        out[cfg] = {"launches": launches, "step": step}
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps({k: v["step"] for k, v in out.items() if isinstance(v, dict)}, indent=1))


if __name__ == "__main__":
    main()
