"""bench.py's multi-rank plumbing on the CPU (gloo): the child ranks of the sharded C4 sub-run
(bench.sharded_subrun) rendezvous on their own port even when the parents run under torchrun,
whose environment carries TORCHELASTIC_USE_AGENT_STORE=True (the agent hosts the store)."""
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
t = torch.ones(1) * (dist.get_rank() + 1)
dist.all_reduce(t)
print("sum", int(t.item()))
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _parent(rank, world, port, q):
    os.environ["TORCHELASTIC_USE_AGENT_STORE"] = "True"      # as under torchrun (static rdzv)
    os.environ["TORCHELASTIC_RESTART_COUNT"] = "0"
    sys.path.insert(0, ROOT)
    import bench
    env = bench.child_env(rank, world, port)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=120)
    q.put((rank, r.returncode, r.stdout.strip(), r.stderr[-300:]))


@pytest.mark.parametrize("world", [2, 3])
def test_child_ranks_rendezvous_under_torchrun_env(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_parent, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, rc, out, err in res:
        assert rc == 0, (rank, err)
        assert out == f"sum {world * (world + 1) // 2}", (rank, out)


def test_child_env_drops_agent_store(monkeypatch):
    monkeypatch.setenv("TORCHELASTIC_USE_AGENT_STORE", "True")
    sys.path.insert(0, ROOT)
    import bench
    env = bench.child_env(1, 2, 12345)
    assert "TORCHELASTIC_USE_AGENT_STORE" not in env
    assert env["RANK"] == "1" and env["WORLD_SIZE"] == "2" and env["MASTER_PORT"] == "12345"
    assert env["MASTER_ADDR"] == "127.0.0.1"


def test_stream_floor_reads_the_committed_probe():
    """elementwise_roofline.size_floor: the C2 / C3 floors come from profiles/stream_probe_r02.log
    (one R2W4 + two R4W2 launches), between the probe's own per-shape rates; unknown N -> None."""
    sys.path.insert(0, ROOT)
    import bench
    f2, f3 = bench.stream_floor(1 << 20), bench.stream_floor(1 << 21)
    assert 3000 < f2 < 4500 and 4000 < f3 < 6000 and f2 < f3
    assert bench.stream_floor(12345) is None
    r = bench.elementwise_roofline({"other_ms": 1.0, "other_bytes": 1e-3 * f2 * 1e9 * 0.5}, 1 << 20)
    assert abs(r["frac_of_size_floor"] - 0.5) < 1e-9
