#!/usr/bin/env python
"""bench.py -- GCUPS of the SW#db scoring path on BASELINE config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--scale S]

Workload (config.workload): the 20-query sweep (lengths 144..5478) against a synthetic Swiss-Prot-shaped
database (565,928 sequences, ~204 M residues), BLOSUM62, gap open 10 / extend 2, top_k 10.  One *step* is
one full sweep: 20 searches, 8.5e12 cell updates.  GCUPS = sum(query_len x db_residues) / seconds / 1e9
(SPEC.md:353), real residues only (padding is never counted).

  value      the sweep as ONE batch through swb_search_many (N = 1): queries are issued back to back on the stream,
             the queries share database scans as two streams (duo_pipeline_kernel); device time = sum of the per-job CUDA-event
             times the call returns (database already resident in HBM, packed once outside the timed region like the
             reference's load phase).  N > 1: the per-search path below (one all-gather per search).
  e2e        the same batch through the same C-ABI call with HOST buffers: host queries/matrix in, host hits out,
             host<->device copies, host preparation and the final synchronisation inside the timed region (CUDA
             events on the stream the kernels run on plus a barrier; max over ranks).
  single_query  the drop-in run_search path: one swb_search call per query (what include/swsearch/scheduler.hpp
             forwards to), device-timed per search and end to end, with the per-query table.
  roofline   the scan kernels (pipeline_s16_kernel, wavefront_s16_kernel) against the DPX cell-update roofline P_dpx x 2 / 6
             (SURVEY.md 8(d)); P_dpx is measured live by swb_measure_pipe_rates.  The HBM side (packed-database
             stream, 1 byte per residue per search) is reported against MEASURED_PEAKS.json.
  cpu_baseline  the unmodified reference (oracle/_ref/libswref.so, run_search without traceback) on the host
             cores, on a bounded subsample of the same workload (N=1, rank 0 only).

N > 1 (torchrun, one rank per GPU): the same database is sharded by residue count (strong scaling).  The batched
sweep ends with one all-gather of 20 x k packed keys per rank (NCCL); the per-search path has one all-gather of k keys
per search and a device-side merge.  If the batched sweep fails on any rank the per-search numbers are the headline.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

TOP_K = 10
GAPS = (10, 2)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="database size relative to Swiss-Prot (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-workloads", action="store_true", help="skip the config3 / config5_share sub-records")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


# ------------------------------------------------------------------------------------------------------------
# clocks: sampled with NVML while the timed region runs
# ------------------------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.power = [], set(), []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:   # NVML missing: report that instead of inventing numbers
            self.nv = None
            self.err = str(exc)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def start(self):
        if self.nv:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()

    def stop(self):
        self._stop.set()
        if self._thread:
            self._thread.join()
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml unavailable")}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "power_w_max": max(self.power) if self.power else None,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------------------
# CPU reference leg
# ------------------------------------------------------------------------------------------------------------
def cpu_sample(queries, sdb, seed=7, n_seqs=20000, query_ids=(0, 9, 19)):
    """A bounded sample of the workload: a seeded subsample of the database (with one long sequence) and three
    of the twenty queries."""
    rng = np.random.default_rng(seed)
    lens = sdb.lengths()
    pick = rng.choice(sdb.n, size=min(n_seqs, sdb.n), replace=False)
    longs = np.nonzero(lens >= 3000)[0]
    if len(longs):
        pick[0] = longs[len(longs) // 2]
    sub = sdb.subset(np.sort(pick))
    return [queries[i] for i in query_ids if i < len(queries)], sub


def run_cpu_reference(queries, sub, threads, repeats=1):
    """Times the unmodified reference's run_search (compute_alignments=false) on the sample. Returns
    (GCUPS, seconds, kind)."""
    from oracle import pyoracle as po
    from paper_2203_11100_b200 import synth
    b62 = synth.blosum62()
    cells = sum(len(q) for q in queries) * sub.residues
    if po.Ref.available():
        ref = po.Ref()
        h = ref.db_create(po.FlatDb(sub.codes, sub.offsets))
        best = None
        for _ in range(repeats):
            t0 = time.perf_counter()
            for q in queries:
                ref.run_search(h, q, b62, GAPS[0], GAPS[1], worker_count=threads, lane_width=8, chunk_width=64,
                               length_threshold=3000, top_k=TOP_K, cpu_pool_threads=threads)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        ref.db_destroy(h)
        return cells / best / 1e9, best, "reference"
    port = po.Port()      # the C restatement, OpenMP over sequences
    fdb = po.FlatDb(sub.codes, sub.offsets)
    t0 = time.perf_counter()
    for q in queries:
        port.score_all(q, fdb, b62, GAPS[0], GAPS[1])
    dt = time.perf_counter() - t0
    return cells / dt / 1e9, dt, "port"


def describe_sample(queries, sub):
    return (f"{sub.n} sequences ({sub.residues} residues, seeded subsample of the config-2 database incl. one long "
            f"sequence) x queries of length {[len(q) for q in queries]}")


def workload_name(scale):
    base = ("config2: 20-query sweep (len 144-5478) vs synthetic Swiss-Prot-shaped DB (565,928 seqs, ~204M residues), "
            "BLOSUM62, gap 10/2, top_k 10")
    return base if scale == 1.0 else base + f" [DEBUG scale={scale}]"


def main_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    from paper_2203_11100_b200 import synth
    queries, sdb = synth.config2(scale=args.scale)
    qs, sub = cpu_sample(queries, sdb)
    threads = os.cpu_count() or 1
    times = []
    for step in range(args.warmup + args.steps):
        gc, dt, kind = run_cpu_reference(qs, sub, threads)
        if step >= args.warmup:
            times.append(dt)
    cells = sum(len(q) for q in qs) * sub.residues
    sec = float(np.mean(times))
    value = cells / sec / 1e9
    line = {
        "impl": "reference", "metric": "GCUPS", "value": value, "unit": "GCUPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int16 saturating + int32 re-run (CPU)", "data": "synthetic",
        "config": {"workload": workload_name(args.scale), "step": "bounded CPU sample: " + describe_sample(qs, sub)},
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": threads, "kind": kind, "sample": describe_sample(qs, sub)},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))
    return 0


def measure_extra_workload(name, queries, sdb, matrix, gaps, p_dpx, steps, warmup, device_index, stream):
    """One of BASELINE's other single-GPU workloads (configs[2], configs[4]'s per-GPU share), measured like the headline:
    `warmup` untimed sweeps, then `steps` sweeps one query at a time (swb_search, device-timed per search and end to
    end with host buffers) and as one batch (swb_search_many), clocks sampled during the timed region.  Hits of every
    repetition are compared with the first and the planted exact copy must be the top hit."""
    import torch
    from paper_2203_11100_b200 import Database, GapModel
    g = GapModel(*gaps)
    cells = sum(len(q) for q in queries) * sdb.residues
    with Database(sdb.codes, sdb.offsets, device=device_index) as db:
        db.set_stream(stream.cuda_stream)
        info = db.info()
        first = None
        for _ in range(max(warmup, 1)):
            first = [db.search(q, matrix, g, TOP_K)[:2] for q in queries]
            db.search_many(queries, matrix, g, TOP_K)
        for qi, (idx, sc) in enumerate(first):
            if idx[0] != sdb.planted[qi][0]:
                raise SystemExit(f"{name}: query {qi}: top hit {idx[0]} is not the planted exact copy")
        sampler = ClockSampler(device_index)
        torch.cuda.synchronize()
        sampler.start()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        dev_ms, launches, rescored, per_query = 0.0, 0, 0, []
        for _ in range(steps):
            per_query = []
            for q, (fi, fs) in zip(queries, first):
                idx, sc, st = db.search(q, matrix, g, TOP_K)
                if not ((idx == fi).all() and (sc == fs).all()):
                    raise SystemExit(f"{name}: determinism_error in a single search")
                dev_ms += st["ms_total"]
                launches += st["kernel_launches"]
                rescored += st["rescored_i32"]
                per_query.append({"m": len(q), "gcups": len(q) * sdb.residues / (st["ms_total"] * 1e-3) / 1e9, "ms": st["ms_total"],
                                  "rescored_i32": int(st["rescored_i32"])})
        e1.record(stream)
        batch_ms = 0.0
        l0 = db.info()["kernel_launches_total"]
        for _ in range(steps):
            many, ms = db.search_many(queries, matrix, g, TOP_K)
            batch_ms += float(ms.sum())
            for (a, b), (c, e) in zip(many, first):
                if not ((a == c).all() and (b == e).all()):
                    raise SystemExit(f"{name}: determinism_error in the batched sweep")
        e2.record(stream)
        torch.cuda.synchronize()
        batch_launches = db.info()["kernel_launches_total"] - l0
        clocks = sampler.stop()
    roof = p_dpx * 2.0 / 6.0
    single = cells * steps / (dev_ms * 1e-3) / 1e9
    batched = cells * steps / (batch_ms * 1e-3) / 1e9
    return {"workload": name, "metric": "GCUPS", "value": max(single, batched), "unit": "GCUPS",
            "single_query": {"value": single, "e2e": cells * steps / (e0.elapsed_time(e1) * 1e-3) / 1e9, "gpu_launches": launches,
                             "per_query": per_query},
            "batched": {"value": batched, "e2e": cells * steps / (e1.elapsed_time(e2) * 1e-3) / 1e9, "gpu_launches": batch_launches},
            "steps": steps, "warmup": max(warmup, 1), "rescored_i32_per_sweep": rescored // max(steps, 1),
            "roofline": {"bound": "dpx_alu", "peak": roof, "unit": "GCUPS", "frac": max(single, batched) / roof,
                         "frac_single_query": single / roof, "peak_def": "P_dpx x 2 / 6, P_dpx measured live in this run"},
            "db": {k: info[k] for k in ("n_total", "n_groups", "residues", "padded_residues", "n_short", "n_long")},
            "clocks": clocks}


# ------------------------------------------------------------------------------------------------------------
# native leg
# ------------------------------------------------------------------------------------------------------------
def main_native(args):
    import torch
    import torch.distributed as dist
    from paper_2203_11100_b200 import GapModel, measure_pipe_rates, synth
    from paper_2203_11100_b200.dist import ShardedSearch

    rank, local_rank, world = env_rank()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the native path has no CPU fallback")
    # Rehearsal of the N > 1 code path on a box with one GPU (tests only, never a bench value): every rank on device 0,
    # collectives over gloo, because NCCL refuses two ranks on one device.
    rehearsal = os.environ.get("SWB_BENCH_REHEARSAL") == "1"
    if rehearsal:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    if world > 1:
        if rehearsal:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)

    b62 = synth.blosum62()
    gaps = GapModel(*GAPS)
    queries, sdb = synth.config2(scale=args.scale)
    t0 = time.perf_counter()
    engine = ShardedSearch(sdb.codes, sdb.offsets, length_threshold=3000, device_index=local_rank)
    pack_upload_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream(device)
    engine.db.set_stream(stream.cuda_stream)      # all kernels now run on the stream torch's events record on
    info = engine.db.info()

    total_cells = sum(len(q) for q in queries) * sdb.residues     # whole job, all ranks
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else None
    rates = measure_pipe_rates(local_rank, 1.0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    def one_step():
        """One sweep. Returns (device ms summed over searches, kernel ms of the scan, launches, hits, per-query)."""
        dev_ms = scan_ms = 0.0
        launches = 0
        hits, per_query = [], []
        for q in queries:
            idx, sc, st = engine.search(q, b62, gaps, TOP_K)
            dev_ms += st["ms_total"]
            scan_ms += st["ms_scan"]
            launches += st["kernel_launches"]
            hits.append((idx.copy(), sc.copy()))
            per_query.append((len(q), st["ms_total"], st["ms_scan"], st["rescored_i32"], st["chunks_claimed"]))
        return dev_ms, scan_ms, launches, hits, per_query

    first_hits = None
    for _ in range(max(args.warmup, 0)):
        _, _, _, hits, _ = one_step()
        first_hits = first_hits or hits

    # ---- the sweep as one batch (swb_search_many on every rank's shard, ONE all-gather per sweep): the headline -------
    batch = None
    try:
        for _ in range(max(args.warmup, 0)):
            engine.search_many(queries, b62, gaps, TOP_K)
        bsampler = ClockSampler(local_rank)
        barrier()
        bsampler.start()
        launches0 = engine.db.info()["kernel_launches_total"]
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        batch_dev_ms = 0.0
        batch_jobs = None
        for _ in range(args.steps):
            many, ms = engine.search_many(queries, b62, gaps, TOP_K)
            batch_dev_ms += float(ms.sum())
            batch_jobs = ms
            for (a, b), (c, e) in zip(many, first_hits or many):     # determinism check of SPEC.md:377
                if not ((a == c).all() and (b == e).all()):
                    raise RuntimeError("determinism_error: the batched sweep returned a different ranked list")
        b1.record(stream)
        barrier()
        batch = {"ok": 1.0, "dev_ms": batch_dev_ms, "e2e_ms": b0.elapsed_time(b1), "clocks": bsampler.stop(),
                 "launches": engine.db.info()["kernel_launches_total"] - launches0,
                 "per_query_ms": [float(x) for x in batch_jobs]}
    except Exception as exc:      # keep the per-search numbers below as the headline, say why
        if world == 1:
            raise
        batch = {"ok": 0.0, "dev_ms": 0.0, "e2e_ms": 0.0, "clocks": None, "launches": 0, "per_query_ms": [], "error": repr(exc)}
    if world > 1:
        # all ranks agree on whether the batched sweep counts; times are the max over ranks, launches the sum
        flag = torch.tensor([batch["ok"]], dtype=torch.float64, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        bt = torch.tensor([batch["dev_ms"], batch["e2e_ms"]], dtype=torch.float64, device=device)
        dist.all_reduce(bt, op=dist.ReduceOp.MAX)
        bl = torch.tensor([batch["launches"]], dtype=torch.int64, device=device)
        dist.all_reduce(bl)
        batch["dev_ms"], batch["e2e_ms"], batch["launches"] = float(bt[0]), float(bt[1]), int(bl.item())
        if float(flag.item()) < 1.0:
            batch = None

    sampler = ClockSampler(local_rank)
    barrier()
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    dev_ms = scan_ms = 0.0
    launches = 0
    per_query = None
    for _ in range(args.steps):
        d, s, l, hits, per_query = one_step()
        dev_ms += d
        scan_ms += s
        launches += l
        if first_hits is None:
            first_hits = hits
        for (a, b), (c, e) in zip(hits, first_hits):       # determinism check of SPEC.md:377
            if not ((a == c).all() and (b == e).all()):
                raise SystemExit("determinism_error: a repetition returned a different ranked list")
    ev1.record(stream)
    barrier()
    clocks = sampler.stop()
    e2e_ms = ev0.elapsed_time(ev1)

    t = torch.tensor([dev_ms, e2e_ms, scan_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms, scan_ms = (float(x) for x in t.cpu())
    if world > 1:
        lt = torch.tensor([launches], dtype=torch.int64, device=device)
        dist.all_reduce(lt)
        launches = int(lt.item())

    if rank == 0:
        steps = max(args.steps, 1)
        value = total_cells * steps / (dev_ms * 1e-3) / 1e9
        e2e = total_cells * steps / (e2e_ms * 1e-3) / 1e9
        # planted exact copies must be the top hit of every query (cheap sanity on the full size)
        for qi, (idx, sc) in enumerate(first_hits):
            if args.scale == 1.0 and world == 1 and idx[0] != sdb.planted[qi][0]:
                raise SystemExit(f"query {qi}: top hit {idx[0]} is not the planted exact copy")
        p_dpx = rates["viaddmnmx_s16x2"]                      # 1e9 thread-instructions/s, all SMs
        roof = p_dpx * 2.0 / 6.0 * world                      # GCUPS: 6 DPX instr per 2 cells
        scan_gcups = total_cells * steps / (scan_ms * 1e-3) / 1e9
        hbm_peak = peaks["hbm_gbs"] if peaks else 6650.0
        db_stream_gbs = sdb.residues * len(queries) * steps / (scan_ms * 1e-3) / 1e9
        # DRAM bytes per launch come from an ncu --set full capture (profiles/traffic.json, written by
        # tools/traffic_from_ncu.py), stamped with the hash of the kernel sources it was taken from: a capture of other
        # kernels than the ones timed here is not quoted
        traffic, traffic_note = None, "profiles/traffic.json missing"
        tfile = ROOT / "profiles" / "traffic.json"
        if tfile.exists():
            from paper_2203_11100_b200.build import kernel_source_hash
            traffic = json.loads(tfile.read_text())
            if traffic.get("kernel_source_sha256") != kernel_source_hash():
                traffic_note = (f"stale: profiles/traffic.json was captured from kernel sources {str(traffic.get('kernel_source_sha256'))[:12]}, "
                                f"this run's are {kernel_source_hash()[:12]}")
                traffic = None
            else:
                traffic_note = "ncu capture of these kernel sources (hash matches)"
        single = {"value": value, "e2e": e2e, "unit": "GCUPS", "ms_per_step": e2e_ms / steps, "gpu_launches": launches,
                  "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                  "scan_kernel_gcups": scan_gcups,
                  # host time per search that the device does not hide: (end-to-end - device) / searches
                  "host_overhead_us_per_search": (e2e_ms - dev_ms) * 1e3 / (steps * len(queries)),
                  "api": "swb_search, one call per query (what swsearch::run_search forwards to)" +
                         ("" if world == 1 else " + one all-gather of k keys per search"),
                  "per_query": [{"m": m, "gcups": m * sdb.residues / (ms * 1e-3) / 1e9, "ms": ms, "scan_ms": sms,
                                 "rescored_i32": int(r), "units": int(u)} for (m, ms, sms, r, u) in per_query]}
        # bytes copied per sweep.  One search at a time: matrix + query + the wavefront kernel's unit tables up, k keys +
        # counters down, per query.  Batched: per shared scan the matrix, the queries and a 32-byte tile descriptor per
        # tile of the longer stream up; k keys per query down (queries left out of the scans copy as single searches do).
        h2d_single = int(sum(len(q) + 2304 + 9 * (info["n_groups"] + 1) for q in queries))
        d2h_single = int(len(queries) * (TOP_K * 8 + 16))
        h2d, d2h = h2d_single, d2h_single
        if batch:
            from paper_2203_11100_b200 import batch_plan
            scan_of, stream_of = batch_plan(sdb.lengths(), [len(q) for q in queries], sm_count=rates["sm_count"],
                                            shard_rank=rank, shard_count=world)
            h2d, d2h = 0, int(len(queries) * TOP_K * 8)
            for sc in sorted(set(int(x) for x in scan_of)):
                members = [i for i in range(len(queries)) if scan_of[i] == sc]
                if sc < 0:
                    h2d += sum(len(queries[i]) + 2304 + 9 * (info["n_groups"] + 1) for i in members)
                    continue
                tiles = [sum((len(queries[i]) + 31) // 32 for i in members if stream_of[i] == half) for half in (0, 1)]
                h2d += 2304 + sum((len(queries[i]) + 15) // 16 * 16 for i in members) + 32 * max(tiles)
        hbm_def = "packed-database stream: 1 byte per residue per search / scan-kernel time"
        if batch:
            n_scans = len(set(int(x) for x in scan_of if x >= 0))
            n_single = sum(1 for x in scan_of if x < 0)
            # a shared scan reads the packed database twice (once per half of a group), whatever the number of queries
            db_stream_gbs = sdb.residues / world * (2 * n_scans + n_single) * steps / (batch["dev_ms"] * 1e-3) / 1e9
            hbm_def = "packed-database stream: 2 bytes per residue per shared scan (+ 1 per single search) / device time"
        if batch:
            head_value = total_cells * steps / (batch["dev_ms"] * 1e-3) / 1e9
            head_e2e = total_cells * steps / (batch["e2e_ms"] * 1e-3) / 1e9
            head_ms, head_launches, head_clocks = batch["e2e_ms"] / steps, batch["launches"], batch["clocks"]
            api = ("swb_search_many, one call per sweep (the queries share one database scan as two streams)" if world == 1 else
                   "swb_search_many on every rank's shard + one all-gather of the sweep's keys per rank")
            kernel = "duo_pipeline_kernel (shared scan of the batch)"
        else:
            head_value, head_e2e, head_ms, head_launches, head_clocks = value, e2e, e2e_ms / steps, launches, clocks
            api = single["api"]
            kernel = "pipeline_s16_kernel + wavefront_s16_kernel (tall groups, short queries)"
        line = {
            "metric": "GCUPS", "value": head_value, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "s16x2 (packed int16 DPX) + int32 re-run", "data": "synthetic",
            "config": {"workload": workload_name(args.scale), "parallelism": f"db-shard x{world}", "api": api,
                       "l2": "inputs larger than L2: the 207 MB packed database is streamed once per scan vs 126 MB L2; "
                             "consecutive scans use different queries",
                       "db": {k: info[k] for k in ("n_total", "n_local", "n_groups", "residues", "padded_residues", "device_bytes")},
                       "pack_upload_s_outside_timing": pack_upload_s},
            "e2e": {"value": head_e2e, "unit": "GCUPS", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "cold_first_search_incl_pack_upload_s": pack_upload_s},
            "gpu_launches": head_launches,
            "clocks": head_clocks,
            "roofline": {"bound": "dpx_alu", "kernel": kernel,
                         "achieved": head_value, "peak": roof,
                         "unit": "GCUPS", "frac": head_value / roof,
                         "peak_def": "P_dpx x 2 / 6 (SURVEY 8(d): 6 DPX instructions per two cells), P_dpx = measured "
                                     "VIADDMNMX.S16x2 thread-instr/s (live, this run); the two-stream kernel issues 3.5 ALU-pipe "
                                     "instructions per two cells and the others 4.5, so frac can exceed 1",
                         # the same pipe rate over the ALU-pipe instructions the kernel actually issues per two cells
                         "peak_executed_mix": p_dpx * 2.0 / (3.5 if batch else 4.5) * world,
                         "frac_executed_mix": head_value / (p_dpx * 2.0 / (3.5 if batch else 4.5) * world),
                         "p_dpx_ginst_per_s": p_dpx, "pipe_rates": rates,
                         "traffic": traffic.get("dram_bytes") if traffic else None, "traffic_detail": traffic, "traffic_note": traffic_note,
                         "hbm": {"bound": "hbm", "achieved": db_stream_gbs, "peak": hbm_peak, "unit": "GB/s",
                                 "frac": db_stream_gbs / hbm_peak,
                                 "peak_src": "MEASURED_PEAKS.json" if peaks else "fallback",
                                 "def": hbm_def}},
            "single_query": single,
        }
        line["single_query"]["h2d_bytes_per_step"], line["single_query"]["d2h_bytes_per_step"] = h2d_single, d2h_single
        if rehearsal:
            line["rehearsal"] = "all ranks on device 0, collectives over gloo: exercises the N > 1 code path, not a bench value"
        if batch:
            line["batched_per_query_ms"] = [{"m": len(q), "ms": ms} for q, ms in zip(queries, batch["per_query_ms"])]
            line["single_query"]["clocks"] = clocks
        if world == 1 and args.scale == 1.0 and not args.no_extra_workloads:
            # BASELINE configs[2] and configs[4] (one GPU's share) next to the headline, same run, same clocks protocol
            engine.close()
            q3, db3, _ = synth.config3()
            line["config3"] = measure_extra_workload(
                "config3: long-sequence pool -- the 9 queries >= 3005 vs only the config-2 entries >= 3000 residues "
                f"({db3.n} seqs, {db3.residues} residues), BLOSUM62 10/2", q3, db3, b62, GAPS, p_dpx, args.steps, args.warmup,
                local_rank, stream)
            q5, db5 = synth.config5_share()
            line["config5_share"] = measure_extra_workload(
                "config5_share: one GPU's 1/8 share of the TrEMBL-shaped DB (350,000 seqs, ~125M residues), BLOSUM50 12/2, "
                "queries 144..9000 (planted copies of the two longest leave int16: int32 re-run)", q5, db5, synth.blosum50(),
                (12, 2), p_dpx, args.steps, args.warmup, local_rank, stream)
        if world == 1 and not args.no_cpu_baseline:
            qs, sub = cpu_sample(queries, sdb)
            threads = os.cpu_count() or 1
            gc, dt, kind = run_cpu_reference(qs, sub, threads)
            line["cpu_baseline"] = {"value": gc, "unit": "GCUPS", "cores": threads, "kind": kind,
                                    "sample": describe_sample(qs, sub), "seconds": dt}
        print(json.dumps(line))
    engine.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    a = parse_args()
    sys.exit(main_reference(a) if a.impl == "reference" else main_native(a))
