"""The paper's own server benchmarks on one B200: Table 5 (2-D Schnakenberg, T = 2, 6000 steps,
N = 2 * 300^2 / 450^2 / 600^2) and Table 7 (3-D FitzHugh-Nagumo, T = 150,
10000 steps, N = 2 * 100^3 / 150^3 / 200^3), exprk3ds_real and exprk3ds_cplx,
fp64.  Wall-clock seconds of the whole integration (phi bank included, in brackets as in the
paper) next to the paper's V100 "CUDA double" column.

    python tools/paper_tables.py [--quick]  > profiles/paper_tables_r01.json
    python tools/paper_tables.py --f32      > profiles/paper_tables_f32_r02.json

--f32: the exprk3ds_real rows in single precision (kx_step_f32, tcgen05 kind::tf32 x 3) next to
the paper's "CUDA single" column (the grids whose extents are multiples of 4: 300^2, 600^2,
100^3, 200^3).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# load every kernel when the CUDA context is created, so that the one-time module loading is
# not charged to whichever table row first launches a given kernel variant
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

# (table, model, d, n, T, steps, scheme, paper V100 CUDA double seconds (phi seconds))
ROWS = [
    ("Table 5", "schnakenberg", 2, 300, 2.0, 6000, "etd3rkds", (7.32, 0.31)),
    ("Table 5", "schnakenberg", 2, 450, 2.0, 6000, "etd3rkds", (16.39, 0.54)),
    ("Table 5", "schnakenberg", 2, 600, 2.0, 6000, "etd3rkds", (26.15, 0.83)),
    ("Table 5", "schnakenberg", 2, 300, 2.0, 6000, "exprk3ds_cplx", (16.33, 0.52)),
    ("Table 5", "schnakenberg", 2, 450, 2.0, 6000, "exprk3ds_cplx", (46.28, 1.01)),
    ("Table 5", "schnakenberg", 2, 600, 2.0, 6000, "exprk3ds_cplx", (89.93, 1.73)),
    ("Table 7", "fhn", 3, 100, 150.0, 10000, "etd3rkds", (57.31, 0.28)),
    ("Table 7", "fhn", 3, 150, 150.0, 10000, "etd3rkds", (251.62, 0.40)),
    ("Table 7", "fhn", 3, 200, 150.0, 10000, "etd3rkds", (685.89, 0.44)),
    ("Table 7", "fhn", 3, 100, 150.0, 10000, "exprk3ds_cplx", (127.47, 0.24)),
    ("Table 7", "fhn", 3, 150, 150.0, 10000, "exprk3ds_cplx", (470.61, 0.33)),
    ("Table 7", "fhn", 3, 200, 150.0, 10000, "exprk3ds_cplx", (1469.11, 0.45)),
]


# (table, model, d, n, T, steps, paper V100 CUDA single seconds (phi seconds)), exprk3ds_real
ROWS_F32 = [
    ("Table 5", "schnakenberg", 2, 300, 2.0, 6000, (4.12, 0.26)),
    ("Table 5", "schnakenberg", 2, 600, 2.0, 6000, (13.17, 0.51)),
    ("Table 7", "fhn", 3, 100, 150.0, 10000, (32.59, 0.22)),
    ("Table 7", "fhn", 3, 200, 150.0, 10000, (321.81, 0.35)),
]


def run(model, d, n, T, steps, scheme, f32=False):
    prob = inputs.make_problem(model, d, n, seed=0)
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    U = [torch.from_numpy(u.astype("float32") if f32 else u.copy()).cuda() for u in prob.U0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.set_tau(T / steps, scheme)
    ctx.sync()
    t_phi = time.perf_counter() - t0
    if f32:
        ctx.step_f32(U, steps)   # the fp32 planes of the bank are formed by the first step
    else:
        ctx.step_n(U, steps)
    ctx.sync()
    total = time.perf_counter() - t0
    finite = all(bool(torch.isfinite(u).all()) for u in U)
    ctx.close()
    return total, t_phi, finite


def main_f32():
    out = {"note": "fp32 (kx_step_f32: tcgen05 kind::tf32, three-pass split) wall-clock seconds of the "
                   "whole exprk3ds_real integration on one B200 (phi bank in brackets) next to the "
                   "paper's V100 CUDA single column (context, other hardware)", "rows": []}
    for table, model, d, n, T, steps, paper in ROWS_F32:
        total, t_phi, finite = run(model, d, n, T, steps, "etd3rkds", f32=True)
        row = {"table": table, "model": model, "N": f"2*{n}^{d}", "T": T, "steps": steps,
               "scheme": "etd3rkds (fp32)", "seconds": round(total, 3), "phi_seconds": round(t_phi, 3),
               "steps_per_s": round(steps / (total - t_phi), 1), "finite": finite,
               "paper_v100_single_seconds": paper[0], "paper_phi_seconds": paper[1],
               "speedup_vs_paper": round(paper[0] / total, 1)}
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


def main():
    if "--f32" in sys.argv:
        return main_f32()
    quick = "--quick" in sys.argv
    out = {"note": "wall-clock seconds of the whole integration on one B200 (phi bank in "
                   "brackets, as the paper's tables); the paper's column is CUDA double on a "
                   "V100 16 GB (context, other hardware)", "rows": []}
    for table, model, d, n, T, steps, scheme, paper in ROWS:
        if quick and steps * n ** d > 6000 * 450 ** 2:
            continue
        total, t_phi, finite = run(model, d, n, T, steps, scheme)
        row = {"table": table, "model": model, "N": f"2*{n}^{d}", "T": T, "steps": steps,
               "scheme": scheme, "seconds": round(total, 3), "phi_seconds": round(t_phi, 3),
               "steps_per_s": round(steps / (total - t_phi), 1), "finite": finite,
               "paper_v100_double_seconds": paper[0], "paper_phi_seconds": paper[1],
               "speedup_vs_paper": round(paper[0] / total, 1)}
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
