"""The N>1 path on CPU: world_size 2 (and 3) over gloo.  Each rank plans its
shard, scans it, and takes its global offset from the all_gather count
exchange (paper_1704_02272_b200/dist.py).  The per-rank scanner here is the C
oracle restricted to the shard's starts -- the host-side plumbing (shard and
halo arithmetic, count exchange, ordering) is what is under test; the GPU
scan_shard itself is checked against whole-text scans in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1704_02272_b200 import dist as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(seed=3):
    rng = np.random.default_rng(seed)
    pats = sorted({bytes(rng.integers(65, 69, size=int(rng.integers(2, 9)), dtype=np.uint8)) for _ in range(40)})
    text = rng.integers(65, 69, size=20000, dtype=np.uint8)
    return pats, text


def _oracle_scanner(pats):
    import oracle

    def scan(shard_bytes, lo, owned):
        recs = oracle.naive_find_all(shard_bytes, pats)
        recs = recs[recs["start"] < owned].copy()
        recs["start"] += lo
        return recs
    return scan


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pats, text = _instance()
        halo = max(len(p) for p in pats) - 1
        shard = D.plan(text.size, world, rank, halo)
        recs, off, total = D.scan_sharded(text, shard, _oracle_scanner(pats))
        allrecs = D.gather_all(recs)
        if rank == 0:
            q.put((off, total, allrecs.tobytes()))
        else:
            q.put((off, total, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_scan_equals_whole_text(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pats, text = _instance()
    want = oracle.naive_find_all(text, pats)
    totals = {r[1] for r in results}
    assert totals == {want.size}
    offs = sorted(r[0] for r in results)
    assert offs[0] == 0 and len(set(offs)) == world
    got = [np.frombuffer(r[2], dtype=want.dtype) for r in results if r[2] is not None][0]
    assert np.array_equal(got, want)


def test_plan_covers_every_start_once():
    for n in (0, 1, 7, 4096, 100003):
        for world in (1, 2, 3, 8):
            shards = [D.plan(n, world, r, 31) for r in range(world)]
            assert sum(s.owned for s in shards) == n
            for a, b in zip(shards, shards[1:]):
                assert a.lo + a.owned == b.lo
            assert all(s.end == min(n, s.lo + s.owned + 31) for s in shards)
    with pytest.raises(ValueError):
        D.plan(10, 2, 0, -1)


def test_reference_arm_under_torchrun():
    # The driver launches `bench.py --impl reference` like the GPU arm
    # (torchrun, N ranks): rank 0 times the compiled reference on the CPU and
    # prints one JSON line; the other ranks exit 0 without a process group or
    # a CUDA context (this container has no GPU).
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-sample-bytes", str(2 << 20)]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    if "unavailable" not in line:
        assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
        assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
