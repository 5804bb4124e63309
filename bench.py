#!/usr/bin/env python
"""PFAC match throughput (Gbps) on B200 -- BASELINE.json metric.

Workload (default): config 3 of BASELINE.json -- 20,000 byte signatures
(len 4-32, sigma 256) over synthetic traffic with one planted occurrence per
4 KiB, scanned with the reference's benchmark trie (stage-1 merged, truncated
at choose_depth, bucket verification: bench.cpp:199-205).  4 GiB of text per
GPU (weak scaling: rank r owns a contiguous shard plus a max_len-1 halo).

  value : device-resident throughput -- text already in HBM, each step one
          launch of the sm_100a scan kernel, timed with CUDA events on the
          engine's stream, max over ranks.
  e2e   : the same scan through the C ABI call hepfac_scan with the shard in
          pinned HOST memory: H2D copy, kernel, D2H of the sorted match list
          and the count exchange (all_gather) inside the timed region.

`--impl reference` times the reference's own CPU matcher (compiled from its
sources into oracle/_ref) with every host thread on a bounded sample.

Launch: python bench.py [--gpus 1] [--steps K] [--warmup W]
        torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PFAC match throughput Gbps (kernel & end-to-end) at 1/2/4/8 B200 vs CPU ref"
UNIT = "Gbps"


def gbps(nbytes: float, seconds: float) -> float:
    return nbytes * 8.0 / seconds / 1e9


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed only; the data path has no collective
# beyond the per-shard count exchange)

class Dist:
    def __init__(self, want_gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.dev = "cuda"
        self.gpu = self.local
        self.oversubscribed = False
        if self.world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            n = torch.cuda.device_count()
            if self.world <= n:
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                # more ranks than GPUs (a --check run on a small box): ranks
                # share devices, so the count exchange goes over gloo; the
                # timings of such a run are not scaling numbers
                self.gpu = self.local % max(1, n)
                self.dev = "cpu"
                self.oversubscribed = True
                torch.cuda.set_device(self.gpu)
                dist.init_process_group("gloo")
            self.pg = dist
        os.environ["HEPFAC_DEVICE"] = str(self.gpu)

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def sync(self):
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.synchronize()
        except Exception:
            pass

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: int) -> int:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.int64, device=self.dev)
        self.pg.all_reduce(t)
        return int(t.item())

    def exclusive_prefix(self, count: int) -> int:
        """K4: exclusive scan of per-shard match counts (all_gather of one u64)."""
        if not self.pg:
            return 0
        import torch
        t = torch.tensor([count], dtype=torch.int64, device=self.dev)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.pg.all_gather(out, t)
        return int(sum(o.item() for o in out[: self.rank]))

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x40: "sw_thermal_slowdown",
               0x80: "hw_thermal_slowdown", 0x100: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------

def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name: str, text_bytes: int):
    """DRAM bytes (read + write) per launch from the committed ncu --set full
    capture of this workload (profiles/ncu_traffic.json), scaled to this
    launch's text size when the capture used a smaller text; None if absent."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f).get(config_name)
    if not d:
        return None
    return int(round(d["dram_bytes"] * text_bytes / d["text_bytes"]))


def make_shard(w, rank: int, world: int, per_gpu: int, halo: int):
    """Rank r owns global starts [r*per_gpu, (r+1)*per_gpu) of one global
    text of world*per_gpu bytes and gets the `halo` bytes after them -- the
    next rank's first bytes."""
    N = per_gpu * world
    lo = rank * per_gpu
    end = min(N, lo + per_gpu + halo)
    text = w.make_text(end - lo, lo=lo)
    return text, lo, per_gpu


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference_gbps(w, trie_state: str, sample: np.ndarray, runs: int = 3):
    """The reference CPU matcher (oracle/_ref, compiled from its sources) on the
    same workload sample: hepfac_run_throughput with every host thread."""
    import oracle
    from paper_1704_02272_b200 import workloads
    ref = oracle.ref_library()
    cores = os.cpu_count() or 1
    if ref is not None:
        t, _ = workloads.build_trie(ref, w, trie_state)
        rep = ref.run_throughput(t, sample, runs=runs, workers=cores)
        # also one worker, on a smaller slice of the same sample
        one = sample[: min(sample.size, 32 << 20)]
        rep["single_worker"] = {"value": round(ref.run_throughput(t, one, runs=runs, workers=1)["gbps"], 4),
                                "sample_bytes": int(one.size)}
        return rep["gbps"], cores, "reference", rep
    # port: the C restatement, one core
    from paper_1704_02272_b200 import hepfac
    lib = hepfac.lib()
    t, _ = workloads.build_trie(lib, w, trie_state)
    tr = oracle.HtriTrie(t.save_bytes())
    t0 = time.perf_counter()
    tr.scan(sample)
    return gbps(sample.size, time.perf_counter() - t0), 1, "port", {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bytes-per-gpu", type=int, default=4 << 30)
    ap.add_argument("--trie", default="s1trunc", choices=["s1trunc", "stage2", "stage1", "full"])
    ap.add_argument("--sigma", type=int, default=256, help="config c4 alphabet size")
    ap.add_argument("--count", type=int, default=0, help="config c5 pattern count")
    ap.add_argument("--cpu-sample-bytes", type=int, default=256 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="default: min(steps, 5), raised to cover >= 4 GiB of text (at most 50)")
    ap.add_argument("--check", action="store_true",
                    help="compare the rank-order concatenation of the shard lists with a one-rank scan (SHA-256)")
    args = ap.parse_args()

    from paper_1704_02272_b200 import hepfac, workloads

    w = workloads.config(args.config, sigma=args.sigma, count=args.count)
    workload_desc = {
        "c1": "1,000 byte patterns len 4-32 over synthetic payload",
        "c2": "DNA {A,C,G,T}: 10k patterns len 8-32 over synthetic genome",
        "c3": "20k Snort-like byte signatures (len 4-32, sigma 256) over synthetic traffic",
        "c4": f"alphabet sweep point sigma={args.sigma}: 10k patterns x len 20",
        "c5": f"pattern-count sweep point n={args.count or 100000}, byte patterns len 4-32",
    }[args.config]

    if args.impl == "reference":
        # Reference arm: rank 0 only, CPU, bounded sample of the same workload.
        # No process group and no CUDA context: the other ranks exit at once.
        if int(os.environ.get("RANK", "0")) != 0:
            return
        times = []
        import oracle
        ref = oracle.ref_library()
        cores = os.cpu_count() or 1
        if ref is None:
            out = {"impl": "reference", "unavailable": "oracle/_ref/libhepfac_ref.so not built"}
            print(json.dumps(out))
            return
        t, _ = workloads.build_trie(ref, w, args.trie)
        sample = w.make_text(args.cpu_sample_bytes)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = ref.scan(t, sample, workers=cores)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        mean = sum(times) / len(times)
        val = gbps(sample.size, mean)
        print(json.dumps({
            "metric": METRIC, "value": round(val, 4), "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": {"workload": f"{args.config}: {workload_desc}", "trie": args.trie,
                                            "sample_bytes": int(sample.size), "matches": int(res.size)},
            "cpu_baseline": {"value": round(val, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                             "cpu_model": cpu_model(),
                             "sample": f"{sample.size >> 20} MiB of the {args.config} text, hepfac_scan "
                                       f"(walk + merge + sort), {cores} workers"},
            "e2e": {"value": round(val, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    d = Dist(args.gpus)
    lib = hepfac.lib()
    if lib.device_count() < 1:
        raise SystemExit("bench.py needs a CUDA device")
    trie, ps = workloads.build_trie(lib, w, args.trie)
    halo = lib.halo(trie)
    text, lo, owned = make_shard(w, d.rank, d.world, args.bytes_per_gpu, halo)
    info = lib.layout_info(trie)

    # ---- value: device-resident kernel throughput ------------------------
    # shard session: starts [lo, lo + owned) of the global text; walks may read the halo
    sess = lib.session(trie, text, offset=lo, owned=owned)
    l2_note = "inputs larger than L2 (text %d MiB/GPU vs 126 MB L2)" % (owned >> 20)
    flush = owned < (256 << 20)
    if flush:
        l2_note = "L2 flushed between timed iterations"
    sess.run(args.warmup, flush)
    d.barrier()
    d.sync()
    with ClockSampler(d.gpu) as clk:
        ms, matches = sess.run(args.steps, flush)
    d.sync()
    d.barrier()
    first_ms, second_ms, kernels_per_scan = sess.kernel_ms(args.steps)
    total_ms = sum(ms)
    max_total_ms = d.max(total_ms)
    all_bytes = owned * d.world
    value = gbps(all_bytes * args.steps, max_total_ms / 1e3)
    mean_launch_s = total_ms / args.steps / 1e3
    sess.close()

    # ---- e2e: hepfac_scan from host memory ---------------------------------
    # pinned (the config-3 contract: "streamed from pinned host memory") and
    # pageable (the reference's normal caller: a std::vector, staged by the
    # library through its pinned ring); H2D, kernels, per-chunk D2H of the
    # sorted list and the count exchange all inside the timed region
    try:
        import torch
        pinned = torch.empty(text.size, dtype=torch.uint8, pin_memory=True)
        host = pinned.numpy()
        host[:] = text
    except Exception:
        host = text
    # at least ~4 GiB of text per rank over the e2e window (5 scans of the
    # 4 GiB contract text; 20 of a 1 GiB config), so one host-side hiccup
    # does not swing a short window (at most 50 scans)
    e2e_steps = args.e2e_steps or max(min(args.steps, 5), min(50, -(-(4 << 30) // max(1, owned))))

    def e2e_run(buf):
        # view=True: the records stay in the library's (pinned) list, as a C
        # caller gets them -- no extra host copy by the Python binding
        r = None
        for _ in range(min(args.warmup, 2)):
            r = None
            r = lib.scan_shard(trie, buf, lo, owned, view=True)
        d.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r = None  # the previous list goes back to the pinned pool first
            r = lib.scan_shard(trie, buf, lo, owned, view=True)
            d.exclusive_prefix(int(r.size))
        d.barrier()
        return r, d.max(time.perf_counter() - t0), lib.last_scan_stats()

    res, e2e_s, stats = e2e_run(host)
    e2e_val = gbps(all_bytes * e2e_steps, e2e_s)
    total_matches = d.sum(int(res.size))
    # the host-link ceiling: a plain pinned H2D copy of up to 1 GiB (torch)
    h2d_ceiling = None
    try:
        import torch
        n = min(text.size, 1 << 30)
        dev = torch.empty(n, dtype=torch.uint8, device="cuda")
        src = pinned[:n]
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.copy_(src, non_blocking=True)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        h2d_ceiling = gbps(n, best / 1e3)
        del dev
    except Exception:
        pass
    res_pg, e2e_pg_s, stats_pg = e2e_run(text)
    e2e_pg_val = gbps(all_bytes * e2e_steps, e2e_pg_s)
    if not (res_pg.shape == res.shape and (res_pg == res).all()):
        raise SystemExit("pageable and pinned hepfac_scan results differ")

    # ---- --check: the rank-order concatenation equals a one-rank scan ---------
    check = None
    if args.check:
        import hashlib
        parts = [res.tobytes()]
        if d.pg:
            parts = [None] * d.world
            d.pg.all_gather_object(parts, res.tobytes())
        if d.rank == 0:
            mine = hashlib.sha256(b"".join(parts)).hexdigest()
            whole = w.make_text(owned * d.world)
            one = lib.scan(trie, whole)
            ref_sha = hashlib.sha256(one.tobytes()).hexdigest()
            check = {"equal": mine == ref_sha, "sha256": mine, "one_rank_sha256": ref_sha,
                     "matches": int(one.size), "global_bytes": int(whole.size),
                     "how": "SHA-256 of the rank-order concatenation of every rank's hepfac_b200_scan_shard list "
                            "vs hepfac_scan of the whole global text on one device"}
            if not check["equal"]:
                print(json.dumps({"check": check}), file=sys.stderr)
        d.barrier()

    # ---- roofline of the dominant kernel ----------------------------------------
    # Pair pipeline: the filter pass reads the text (1 B per start) and is the
    # dominant kernel; the walking pass writes the records (16 B per match).
    # Fused kernel: both in one launch.
    peak, peak_src = measured_hbm_peak()
    pipeline = kernels_per_scan >= 2
    direct = info["filter_mode"] == 5  # pack pass + direct-index scan
    first_s = sum(first_ms) / len(first_ms) / 1e3
    second_s = sum(second_ms) / len(second_ms) / 1e3
    alg_bytes = owned if (pipeline and not direct) else owned + 16 * int(matches)
    dominant_s = first_s + second_s if direct else first_s
    achieved = alg_bytes / dominant_s / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(w.name, owned),
                "peak_source": peak_src,
                "kernel": ("pfac_pack_dna_kernel + pfac_dna_kernel (the whole step)" if direct else
                           "pfac_l2_filter_kernel (filter pass)" if info["filter_mode"] == 4 and pipeline else
                           {2: "pfac_pair_filter_kernel (filter pass)",
                            3: "pfac_pack_symbols_kernel + pfac_symbol_filter_kernel (filter pass)"}
                           .get(kernels_per_scan, "pfac_scan_kernel (fused)")),
                "algorithmic_bytes_per_launch": alg_bytes,
                "per_unit": "1 B text read per start" + ("" if (pipeline and not direct) else " + 16 B per match written"),
                "step_share": round(dominant_s / mean_launch_s, 4)}
    kernels = {"first_pass_ms": round(first_s * 1e3, 4), "second_pass_ms": round(second_s * 1e3, 4),
               "kernels_per_step": kernels_per_scan,
               "whole_step_GBps": round((owned + 16 * int(matches)) / mean_launch_s / 1e9, 2)}

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": d.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(max_total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"{args.config}: {workload_desc}", "patterns": len(ps.to_list()) if d.rank == 0 else None,
                   "text_bytes_per_gpu": owned, "trie": args.trie, "depth_limit": trie.depth_limit(),
                   "trie_nodes": trie.node_count(), "parallelism": f"shard x{d.world} (contiguous starts + "
                   f"{halo} B halo)" + (" [oversubscribed: ranks share GPUs, not a scaling run]"
                                        if d.oversubscribed else ""), "l2": l2_note, "matches_per_gpu": int(matches),
                   "filter": {"k": info["filter_k"], "bits": info["filter_bits"], "paths": info["filter_paths"]}},
        "e2e": {"value": round(e2e_val, 3), "unit": UNIT, "h2d_bytes_per_step": int(text.size),
                "d2h_bytes_per_step": int(res.size) * 16, "steps": e2e_steps, "host_memory": "pinned",
                "device_breakdown_ms": {k: round(stats[k], 3) for k in ("h2d_ms", "kernel_ms", "d2h_ms", "total_ms")},
                "chunks": stats["chunks"], "matches_total": total_matches,
                "h2d_ceiling_Gbps": round(h2d_ceiling, 1) if h2d_ceiling else None},
        "e2e_pageable": {"value": round(e2e_pg_val, 3), "unit": UNIT, "h2d_bytes_per_step": int(text.size),
                         "d2h_bytes_per_step": int(res_pg.size) * 16, "steps": e2e_steps,
                         "host_memory": "pageable (numpy), staged by the library through its pinned ring",
                         "staged": bool(stats_pg["staged"]),
                         "device_breakdown_ms": {k: round(stats_pg[k], 3)
                                                 for k in ("h2d_ms", "kernel_ms", "d2h_ms", "total_ms")},
                         "vs_pinned": round(e2e_pg_val / e2e_val, 4) if e2e_val else None},
        "gpu_launches": args.steps * kernels_per_scan,
        "roofline": roofline,
        "kernels": kernels,
        "clocks": clk.summary(),
    }

    # ---- CPU baseline (rank 0, N=1 only) ------------------------------------
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        sample = np.ascontiguousarray(text[: min(args.cpu_sample_bytes, text.size)])
        g, cores, kind, rep = cpu_reference_gbps(w, args.trie, sample)
        out["cpu_baseline"] = {"value": round(g, 4), "unit": UNIT, "cores": cores, "kind": kind,
                               "cpu_model": cpu_model(),
                               "sample": f"first {sample.size >> 20} MiB of the same text; "
                                         f"hepfac_run_throughput walk-phase mean of 3 runs after 1 warm-up"}
        if "single_worker" in rep:
            sw = rep["single_worker"]
            out["cpu_baseline"]["single_worker"] = {
                "value": sw["value"], "unit": UNIT, "cores": 1,
                "sample": f"first {sw['sample_bytes'] >> 20} MiB of the same text, same timing"}
    if check is not None:
        out["check"] = check
    if d.rank == 0:
        print(json.dumps(out))
    d.close()
    if check is not None and not check["equal"]:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
