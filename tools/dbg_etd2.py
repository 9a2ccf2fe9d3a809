import dataclasses, sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import inputs
from oracle.etd import integrate
from paper_2310_07551_b200 import kx
from test_gpu_f32 import _cast_bank, relerr
for scheme, n in (("etd2rkds", 32), ("etd2rkds", [32, 32]), ("etd3rkds", 32)):
    d = 3 if isinstance(n, int) else 2
    prob = inputs.make_problem("fhn", d, n, seed=3)
    prob = dataclasses.replace(prob, U0=[u.astype(np.float32).astype(np.float64) for u in prob.U0])
    tau = 0.015
    for steps in (1, 5, 20):
        ref, bank = integrate(prob, scheme, T=tau * steps, m=steps, steps=steps)
        p32 = dataclasses.replace(prob, A=[[A.astype(np.float32) for A in Ac] for Ac in prob.A], U0=[u.astype(np.float32) for u in prob.U0])
        r32, _ = integrate(p32, scheme, T=tau * steps, m=steps, steps=steps, bank=_cast_bank(bank))
        for prec in (32, 64):
            ctx = kx.Context(0); ctx.set_grid(prob.n, 2)
            for c in range(2):
                for mu in range(prob.d): ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
            ctx.set_model(prob.model, prob.params); ctx.set_tau(tau, scheme)
            if prec == 32:
                U = [torch.from_numpy(u.astype(np.float32)).cuda() for u in prob.U0]; ctx.step_f32(U, steps)
            else:
                U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]; ctx.step_n(U, steps)
            ctx.sync(); out = [u.cpu().numpy().astype(np.float64) for u in U]; ctx.close()
            e = [relerr(out[c], ref[c]) for c in range(2)]
            diff = np.abs(out[0] - ref[0]).reshape(prob.n[::-1])
            print(scheme, n, steps, prec, "err", e, "o32", [relerr(r32[c], ref[c]) for c in range(2)], "argmax", np.unravel_index(diff.argmax(), diff.shape), "|U|", np.abs(ref[0]).max(), flush=True)
