"""Paper-protocol convergence on the GPU (Figs. 1/4/5/8):
absolute inf-norm error over both species against a reference exprk3ds_real run with many
steps ("a sufficiently large number of time steps"), at the paper's grids, final
times and step ladders (Figs. 1/4/5/8); prints one JSON object (errors, fitted slopes, steps/s).

    python tools/convergence.py [--quick] [--only fig8] > profiles/convergence_r02.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402


def run(prob, scheme, T, m):
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(T / m, scheme)
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(m):
        ctx.step(U)
    ctx.sync()
    el = time.perf_counter() - t0
    out = [u.cpu().numpy() for u in U]
    ctx.close()
    return out, m / el


# (name, model, d, n, T, reference steps, {scheme: ladder}, paper's printed errors for context)
PROTOCOLS = [
    ("fig1_schnakenberg_n150_T0.25", "schnakenberg", 2, 150, 0.25, 40000,
     {"etd2rkds": [3000, 4000, 5000, 6000], "exprk3ds_real": [1000, 1500, 2000, 2500],
      "exprk3ds_cplx": [1000, 1500, 2000, 2500]},
     {"source": "P:877-916 (Fig. 1, MATLAB, n = 150)",
      "etd2rkds": [4.085e-3, 2.335e-3, 1.509e-3, 1.055e-3],
      "exprk3ds_real": [6.383e-4, 1.771e-4, 7.056e-5, 3.397e-5],
      "exprk3ds_cplx": [7.369e-4, 2.252e-4, 9.593e-5, 4.886e-5]}),
    ("fig4_schnakenberg_n300_T0.25", "schnakenberg", 2, 300, 0.25, 40000,
     {"etd2rkds": [3000, 4000, 5000, 6000], "exprk3ds_real": [1000, 1500, 2000, 2500],
      "exprk3ds_cplx": [1000, 1500, 2000, 2500]}, {"source": "P:1298-1347 (Fig. 4, V100/Xeon, n = 300)"}),
    ("fig5_fhn_n64_T5", "fhn", 3, 64, 5.0, 100000,
     {"etd2rkds": [60000, 65000, 70000, 75000], "exprk3ds_real": [14000, 16000, 18000, 20000],
      "exprk3ds_cplx": [14000, 16000, 18000, 20000]},
     {"source": "P:1551-1586 (Fig. 5, MATLAB, n = 64)",
      "etd2rkds": [2.253e-4, 1.920e-4, 1.655e-4, 1.442e-4],
      "exprk3ds_real": [9.054e-5, 5.997e-5, 4.151e-5, 2.970e-5],
      "exprk3ds_cplx": [9.110e-5, 6.035e-5, 4.177e-5, 2.990e-5]}),
    ("fig8_fhn_n100_T5", "fhn", 3, 100, 5.0, 100000,
     {"etd2rkds": [60000, 65000, 70000, 75000], "exprk3ds_real": [14000, 16000, 18000, 20000],
      "exprk3ds_cplx": [14000, 16000, 18000, 20000]},
     {"source": "P:1919-1925 (protocol), P:1953-2001 (Fig. 8 data, CUDA double, n = 100)",
      "etd2rkds": [5.012e-4, 4.270e-4, 3.682e-4, 3.207e-4],
      "exprk3ds_real": [2.107e-4, 1.378e-4, 9.534e-5, 6.823e-5],
      "exprk3ds_cplx": [2.085e-4, 1.381e-4, 9.557e-5, 6.840e-5]}),
]


def main():
    quick = "--quick" in sys.argv
    fhn_amp = float(sys.argv[sys.argv.index("--fhn-amp") + 1]) if "--fhn-amp" in sys.argv else None
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    out = {"note": "initial data are seeded (SplitMix64, seed 0) while the paper's were unseeded "
                   "U(0,1) draws: compare magnitudes and slopes, not digits"}
    for name, model, d, n, T, mref, ladders, paper in PROTOCOLS:
        if (quick and n > 150) or (only and only not in name):
            continue
        amp = fhn_amp if model == "fhn" else None
        prob = inputs.make_problem(model, d, n, seed=0, amplitude=amp)
        ref, ref_rate = run(prob, "exprk3ds_real", T, mref)
        refmax = float(max(np.max(np.abs(ref[c])) for c in range(2)))
        res = {"reference": {"scheme": "exprk3ds_real", "steps": mref, "steps_per_s": round(ref_rate, 1),
                             "max_abs": refmax}, "paper": paper}
        for scheme, ladder in ladders.items():
            errs, rates = [], []
            for m in ladder:
                o, rate = run(prob, scheme, T, m)
                errs.append(float(max(np.max(np.abs(o[c] - ref[c])) for c in range(2))))
                rates.append(rate)
            slope = float(-np.polyfit(np.log(ladder), np.log(errs), 1)[0])
            res[scheme] = {"steps": ladder, "errors": errs, "relative_errors": [e / refmax for e in errs],
                           "slope": round(slope, 3),
                           "steps_per_s": [round(r, 1) for r in rates]}
        out[name] = res
        print(json.dumps({name: {k: (v.get("slope") if isinstance(v, dict) else None)
                                 for k, v in res.items()}}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
