"""The N>1 path on CPU: world_size 2 (and 3) over gloo.  Each rank plans its
shard, scans it, and takes its global offset from the all_gather count
exchange (paper_1704_02272_b200/dist.py).  Without a GPU the per-rank scanner
is the C oracle or the compiled reference restricted to the shard's starts;
the shard and halo arithmetic (the halo from the product library), the global
block text, the count exchange and the ordering are what is under test.  The
GPU scan_shard itself is checked against whole-text scans in
test_gpu_parity.py, bench.py --check compares the rank-order
concatenation with a one-rank scan on the GPU box, and the gpu-marked test
at the end runs two ranks whose scanner is the product itself."""
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


def _workload_worker(rank, world, port, q, per_rank):
    # One global text (workloads: 16 MiB blocks, any range reproducible),
    # each rank generating only its own bytes [lo, end) -- halo included --
    # the halo taken from the product library (hepfac_b200_halo works without
    # a GPU), shards scanned by the compiled reference through the same C ABI
    # and restricted to the rank's starts, offsets from the count exchange.
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1704_02272_b200 import hepfac, workloads
        ref = oracle.ref_library()
        lib = hepfac.lib()
        w = workloads.config("c1")
        t, _ = workloads.build_trie(lib, w, "s1trunc")
        halo = lib.halo(t)
        rt, _ = workloads.build_trie(ref, w, "s1trunc")
        shard = D.plan(per_rank * world, world, rank, halo)
        mine = w.make_text(shard.nbytes, lo=shard.lo)

        def scanner(b, lo, owned):
            recs = ref.scan(rt, b, workers=2)
            recs = recs[recs["start"] < owned].copy()
            recs["start"] += lo
            return recs

        recs, off, total = D.scan_sharded(mine, shard, scanner)
        allrecs = D.gather_all(recs)
        q.put((rank, off, total, halo, allrecs.tobytes() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_sharded_workload_text_with_product_halo():
    import oracle
    ref = oracle.ref_library()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from paper_1704_02272_b200 import hepfac, workloads
    world, per_rank = 3, (11 << 20) + 7  # shard seams inside and across 16 MiB blocks
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_workload_worker, args=(r, world, port, q, per_rank)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = workloads.config("c1")
    rt, _ = workloads.build_trie(ref, w, "s1trunc")
    whole = w.make_text(per_rank * world)
    want = ref.scan(rt, whole, workers=4)
    assert results[0][3] == 31  # longest c1 pattern (32) - 1
    assert {r[2] for r in results} == {want.size}
    assert [r[1] for r in results] == sorted(r[1] for r in results)
    got = np.frombuffer(results[0][4], dtype=want.dtype)
    assert got.tobytes() == want.tobytes() and want.size > 5000


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
    with pytest.raises(ValueError):  # a cyclic trie's unbounded halo
        D.plan(10, 2, 0, D.UNBOUNDED)
    with pytest.raises(ValueError):
        D.plan(10, 2, 0, None)


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


def _gpu_worker(rank, world, port, q, per_rank):
    # As _workload_worker, but every rank scans its shard with the product
    # (hepfac_b200_scan_shard on the GPU); the ranks share one device, the
    # count exchange goes over gloo.  Nothing waits across ranks on the GPU.
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1704_02272_b200 import hepfac, workloads
        lib = hepfac.lib()
        w = workloads.config("c1")
        t, _ = workloads.build_trie(lib, w, "s1trunc")
        shard = D.plan(per_rank * world, world, rank, lib.halo(t))
        mine = w.make_text(shard.nbytes, lo=shard.lo)
        recs, off, total = D.scan_sharded(mine, shard, lambda b, lo, owned: lib.scan_shard(t, b, lo, owned))
        launches = lib.last_scan_stats()["kernel_launches"]
        allrecs = D.gather_all(recs)
        q.put((rank, off, total, launches, allrecs.tobytes() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_sharded_workload_equals_reference():
    # the product's shard scans, placed by the count exchange,
    # concatenate to the reference's whole-text list (scan.cpp:104-111).
    import oracle
    ref = oracle.ref_library()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from paper_1704_02272_b200 import workloads
    world, per_rank = 2, (24 << 20) + 5  # the seam inside a 16 MiB block
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, per_rank)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = workloads.config("c1")
    rt, _ = workloads.build_trie(ref, w, "s1trunc")
    want = ref.scan(rt, w.make_text(per_rank * world), workers=os.cpu_count() or 4)
    assert all(r[3] >= 1 for r in results)  # GPU kernels ran on every rank
    assert {r[2] for r in results} == {want.size}
    got = np.frombuffer(results[0][4], dtype=want.dtype)
    assert got.tobytes() == want.tobytes() and want.size > 5000
