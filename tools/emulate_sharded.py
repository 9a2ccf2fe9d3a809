"""The slab-sharded step at P = 2, 4, 8 ranks emulated on ONE GPU (an in-process loopback
group: every rank's kernels run one after another on one stream, the exchanges are direct
peer stores into the other ranks' buffers, nothing waits on another rank).  The time of a
group step divided by P is the per-rank compute of a real P-GPU step (communication excluded);
its ratio to the single-GPU step / P is the compute efficiency of the decomposition.

    python tools/emulate_sharded.py [C4|C3] [P ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402


def setup(ctx, prob, cfg):
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(cfg["T"] / cfg["m"], cfg["scheme"])


def timed(fn, steps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    Ps = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    cfg = inputs.CONFIGS[name]
    steps = 3 if name == "C4" else 10
    prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
    one = kx.Context(0)
    setup(one, prob, cfg)
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    t1 = timed(lambda: one.step(U), steps)
    one.close()
    del U
    torch.cuda.empty_cache()
    out = {"config": name, "single_gpu_ms": round(t1, 3), "ranks": {}}
    for P in Ps:
        grp = kx.Group(P)
        for r in range(P):
            pr = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0, slab=(r, P))
            setup(grp.ctx[r], pr, cfg)
        grp.set_p2p(True)
        Ug = []
        for r in range(P):
            pr = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0, slab=(r, P))
            Ug.append([torch.from_numpy(u.copy()).cuda() for u in pr.U0])
        tg = timed(lambda: grp.step(Ug), steps)
        out["ranks"][P] = {"group_step_ms": round(tg, 3), "per_rank_ms": round(tg / P, 3),
                           "compute_efficiency": round(t1 / tg, 3)}
        print(json.dumps({P: out["ranks"][P]}), file=sys.stderr, flush=True)
        grp.close()
        del Ug
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
