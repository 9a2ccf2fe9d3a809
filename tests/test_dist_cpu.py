"""Multi-process (gloo, world_size 2 and 4) check of the slab decomposition the library's
distributed step uses, on the CPU with the oracle's local arithmetic.

Each process owns the i_d-slab of every component (layout A) and performs exactly the data
movement of paper_2310_07551_b200/csrc/kx_api.cpp's dist_* phases:
  [A] G = g(U); T1G = U x_1 A_1 + G; peer-pack T1G and U by i_1 block; all_to_all -> layout B
  [B] F_B = T1G_B + sum_{mu=d..2} U_B x_mu A_mu; modes d..2 of every F-term; all_to_all of
      each term (chunk = destination's i_d block) -> peer-major layout A
  [A] stage = U + sum over (term, source rank) of chunk x_1 (scaled P{1})[:, source i_1 block]
  [A] D = g(stage) - G, peer-packed -> [B] D-terms -> [A] next stage ...
The assembled result must equal the unsharded oracle step (exprk3ds_step) to rounding.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
from oracle.etd import exprk3ds_precompute, exprk3ds_step
from oracle.models import g_of
from oracle.tensor import mode_product, unvec


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def a2a(chunks):
    """all_to_all of a list of P equally-shaped numpy chunks (chunk q goes to rank q)."""
    P = len(chunks)
    shape = chunks[0].shape
    send = torch.from_numpy(np.concatenate([c.reshape(-1, order="F") for c in chunks]))
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    m = int(np.prod(shape))
    return [recv[q * m:(q + 1) * m].numpy().reshape(shape, order="F") for q in range(P)]


def to_B(TA, P):
    """layout A (i_d local block, all i_1) -> layout B (all i_d, i_1 local block)."""
    n1l = TA.shape[0] // P
    parts = a2a([np.ascontiguousarray(TA[q * n1l:(q + 1) * n1l]) for q in range(P)])
    return np.concatenate(parts, axis=-1)           # source rank order = i_d order


def to_A_peer(TB, P):
    """layout B -> the peer-major layout A chunks: list over source rank q of
    (i_1 block of q, ..., local i_d block)."""
    ndl = TB.shape[-1] // P
    return a2a([np.ascontiguousarray(TB[..., q * ndl:(q + 1) * ndl]) for q in range(P)])


def stage_concat_k(U_A, terms, P):
    """U + sum over terms (chunks, matrix L1, scale) and source ranks q of
    chunk_q x_1 (scale * L1)[:, q-th i_1 block] — the K-segmented last mode."""
    out = U_A.copy()
    for chunks, L1, scale in terms:
        n1l = L1.shape[0] // P
        for q in range(P):
            blk = (scale * L1)[:, q * n1l:(q + 1) * n1l]
            out = out + mode_product_rect(chunks[q], blk)
    return out


def mode_product_rect(T, L):
    """mode-1 product with a rectangular L (rows: output i_1, cols: this chunk's i_1)."""
    S = np.tensordot(L, T, axes=([1], [0]))
    return S


def dist_exprk3ds_step(U_A, bank, A, g, params, P):
    d = U_A[0].ndim
    s1, s2 = bank.s1, bank.s2
    G = g(0.0, U_A[0], U_A[1], params)
    F_B = []
    for c in range(2):
        T1G = mode_product(U_A[c], A[c][0], 1) + G[c]
        T1G_B, U_B = to_B(T1G, P), to_B(U_A[c], P)
        F = T1G_B
        for mu in range(d, 1, -1):
            F = F + mode_product(U_B, A[c][mu - 1], mu)
        F_B.append(F)

    def terms_B(X_B, Pl):
        """modes d..2 of every term on layout B, sent back peer-major."""
        out = []
        for Pi in Pl:
            W = X_B
            for mu in range(d, 1, -1):
                W = mode_product(W, Pi[mu - 1], mu)
            out.append(to_A_peer(W, P))
        return out

    def D_B_of(stage):
        Gs = g(0.0, stage[0], stage[1], params)
        return [to_B(Gs[c] - G[c], P) for c in range(2)]

    tau = bank.tau
    WF = [{k: terms_B(F_B[c], bank.P[c][k]) for k in [("2", 1), ("3", 1), ("f", 1)]} for c in range(2)]
    U2 = [stage_concat_k(U_A[c], [(WF[c][("2", 1)][i], bank.P[c][("2", 1)][i][0], tau / 3 * s1.etas[i])
                                  for i in range(s1.nterms)], P) for c in range(2)]
    D2 = D_B_of(U2)
    W2 = [terms_B(D2[c], bank.P[c][("3", 2)]) for c in range(2)]
    U3 = [stage_concat_k(U_A[c],
                         [(WF[c][("3", 1)][i], bank.P[c][("3", 1)][i][0], 2 * tau / 3 * s1.etas[i])
                          for i in range(s1.nterms)]
                         + [(W2[c][i], bank.P[c][("3", 2)][i][0], 4 * tau / 3 * s2.etas[i])
                            for i in range(s2.nterms)], P) for c in range(2)]
    D3 = D_B_of(U3)
    W3 = [terms_B(D3[c], bank.P[c][("f", 2)]) for c in range(2)]
    return [stage_concat_k(U_A[c],
                           [(WF[c][("f", 1)][i], bank.P[c][("f", 1)][i][0], tau * s1.etas[i])
                            for i in range(s1.nterms)]
                           + [(W3[c][i], bank.P[c][("f", 2)][i][0], 1.5 * tau * s2.etas[i])
                              for i in range(s2.nterms)], P) for c in range(2)]


def _worker(rank, world, port, model, d, n, tau, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = inputs.make_problem(model, d, n, seed=3)
        bank = exprk3ds_precompute(prob.A, tau)
        g = g_of(model)
        U = [unvec(u, prob.n) for u in prob.U0]
        ndl = n[-1] // world
        U_A = [u[..., rank * ndl:(rank + 1) * ndl].copy() for u in U]
        for _ in range(2):
            U_A = dist_exprk3ds_step(U_A, bank, prob.A, g, prob.params, world)
            U = exprk3ds_step(U, 0.0, bank, prob.A, g, prob.params)
        err = max(np.max(np.abs(U_A[c] - U[c][..., rank * ndl:(rank + 1) * ndl])) / np.max(np.abs(U[c]))
                  for c in range(2))
        q.put((rank, float(err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("schnakenberg", 2, [12, 10], 1e-4, 2),
                                  ("fhn", 3, [8, 6, 4], 0.015, 2),
                                  ("fhn", 3, [8, 5, 8], 0.015, 4)])
def test_slab_decomposition_gloo(case):
    model, d, n, tau, world = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, model, d, n, tau, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err <= 1e-13, (rank, err)


# ---------------------------------------------------------------- direct peer stores --------
def peer_redirect(off, P, rank, chunk, span):
    """Where the library's kx::peer_redirect (kx_internal.h) sends element `off` of a
    peer-packed send buffer: (destination rank, offset in its receive buffer)."""
    slot, within = divmod(off, span)
    q = within // chunk
    return q, slot * span + rank * chunk + (within - q * chunk)


def _p2p_worker(rank, world, port, nslots, nloc, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        chunk = nloc // world
        rs = np.random.default_rng(rank)
        send = rs.standard_normal(nslots * nloc)
        # reference: the exchange the NCCL path performs, per slot an all-to-all of chunks
        ref = np.empty_like(send)
        for s in range(nslots):
            blk = torch.from_numpy(send[s * nloc:(s + 1) * nloc].copy())
            out = torch.empty_like(blk)
            dist.all_to_all_single(out, blk)
            ref[s * nloc:(s + 1) * nloc] = out.numpy()
        # direct stores: every rank scatters its elements to (q, offset); gather what lands here
        allsend = [torch.empty(nslots * nloc, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allsend, torch.from_numpy(send))
        got = np.full_like(send, np.nan)
        for r in range(world):
            src = allsend[r].numpy()
            for off in range(src.size):
                dq, doff = peer_redirect(off, world, r, chunk, nloc)
                if dq == rank:
                    assert np.isnan(got[doff])      # every receive element is written once
                    got[doff] = src[off]
        q.put((rank, bool(np.array_equal(got, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_direct_peer_stores_equal_all_to_all_gloo(world):
    """The direct-peer-store address map writes exactly the receive buffers the slot-wise
    all-to-all produces (each element once)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, 3, 8 * world, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res


# ---------------------------------------------------------------- distributed operators -----
def dist_tucker(X_A, Ls, P):
    """The library's distributed Tucker operator (csrc/kx_dist_ops.cpp): [A] pack by i_1 block
    -> all-to-all -> [B] modes d..2 on full fibres -> all-to-all -> [A] mode 1 as a sum over
    source ranks q of chunk_q x_1 L_1[:, q-th i_1 block] (the concatenated-K GEMM)."""
    d = X_A.ndim
    W = to_B(X_A, P)
    for mu in range(d, 1, -1):
        W = mode_product(W, Ls[mu - 1], mu)
    chunks = to_A_peer(W, P)
    n1l = Ls[0].shape[0] // P
    out = 0.0
    for q in range(P):
        out = out + mode_product_rect(chunks[q], Ls[0][:, q * n1l:(q + 1) * n1l])
    return out


def _tucker_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.tensor import tucker
        N = int(np.prod(n))
        X = unvec(inputs.uniform_sym(11, 0, N), n)
        Ls = [inputs.uniform_sym(12, mu, m * m).reshape(m, m) for mu, m in enumerate(n)]
        ndl = n[-1] // world
        Y_A = dist_tucker(X[..., rank * ndl:(rank + 1) * ndl].copy(), Ls, world)
        ref = tucker(X, Ls)
        err = np.max(np.abs(Y_A - ref[..., rank * ndl:(rank + 1) * ndl])) / np.max(np.abs(ref))
        q.put((rank, float(err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [([12, 10], 2), ([8, 6, 4], 2), ([8, 5, 8], 4), ([4, 3, 2, 4], 2)])
def test_distributed_tucker_gloo(case):
    """The three-phase sharded Tucker operator equals the oracle's T(X, {L_mu}) on
    every rank's slab, world 2 and 4, d = 2..4."""
    n, world = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tucker_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err <= 1e-13, (rank, err)
