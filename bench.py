#!/usr/bin/env python
"""Benchmark: rows/s reordered + PHC-scored by prefixopt::ggr on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one full `ggr()` (GgrConfig defaults: dictionary encoding, greedy
group recursion, leaf fallbacks, whole-table fallback competition and the
PHC of the emitted schedule) over one synthetic table.

N = 1: BASELINE config C2 (Amazon-products shape, 1M rows x 6 columns,
~0.75 GB of cell bytes; the configuration BASELINE.json's metric is quoted
on), po_ggr on one GPU. Inputs are larger than L2 (126 MB): no flush.

N > 1 (torchrun, one rank per GPU): config C4, the north star's 100M-row x
8 table, split N ways (strong scaling): rank r generates and holds its
contiguous row range and the ranks solve ONE table together through
po_ggr_sharded over NCCL (global dictionary sample sort, replicated
value-group tables from exchanged contributions, distributed leaf sort;
csrc/shard.cu); value = total rows / max-over-ranks time. --config / --rows
override the table, --sharded forces the sharded path at N=1, --transport
host runs the collectives host-staged over gloo (ranks may share a GPU).

  value   whole-job rows/s with the table resident in HBM (device buffers)
  e2e     the same call through the C ABI with pinned HOST buffers: the
          arena+offsets H2D copy and the schedule D2H copy are inside every
          step; two calls in flight (--e2e-inflight) so one step's copy
          overlaps another's solve

--impl reference times the reference C++ implementation (oracle/_ref, the
unmodified prefixopt headers compiled from /root/reference; the CPU port in
oracle/ when _ref is absent) on the host cores: the whole C2 table per step
(a 200K-row prefix of C4 under N > 1).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "rows/sec reordered+PHC-scored (1/2/4/8 B200) & HBM roofline %, vs CPU ref"
UNIT = "rows/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        # started well before the timed region; only samples whose timestamp
        # falls inside [mark_start, mark_end] are kept
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(1.0)
        except OSError:
            self.proc = None
        return self

    def mark_start(self):
        import datetime
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        import datetime
        self.t1 = datetime.datetime.now()

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        import datetime
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f")
            except ValueError:
                ts = None
            if ts is not None and self.t0 is not None and self.t1 is not None and \
                    not (self.t0 - datetime.timedelta(milliseconds=25) <= ts <= self.t1):
                continue
            try:
                sm.append(float(f[2]))
                mx = max(mx, float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "samples every 20 ms inside the timed region"}


def cpu_reference_rows_per_s(table, fds, sample_rows: int, kind: str):
    """Reference prefixopt::ggr on the first `sample_rows` rows; rows/s from the
    reference's own SolveStats.wall_ms (excludes building its Table)."""
    from oracle.pyoracle import available, oracle
    from paper_2403_05821_b200 import GgrConfig, Table
    if kind == "reference" and not available("reference"):
        kind = "port"
    m = table.field_count()
    n = min(sample_rows, table.row_count())
    offs = table.offsets[: n * m + 1].copy()
    sub = Table.from_arena(table.field_names, table.arena[: int(offs[-1]) or 1], offs, n)
    res = oracle(kind).ggr(sub, fds, GgrConfig())
    secs = res.stats.wall_ms / 1e3
    return n / secs, secs, kind, n, res


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2403_05821_b200 import gen
    cfg_id = args.config if args.config is not None else (4 if world > 1 else 2)
    # the whole table when one core finishes it in well under a minute (C2),
    # else a bounded row prefix of it (C4's 100M rows: 200K rows per step)
    full = gen.CONFIGS[cfg_id].rows
    sample = args.ref_rows if args.ref_rows is not None else (full if full <= 1_000_000 else 200_000)
    table = gen.generate(cfg_id, n_rows=sample)
    fds = gen.fds(cfg_id)
    # untimed warm-up steps on a small prefix (page-in, allocator); the timed
    # steps run the reference on the whole configured table
    for _ in range(args.warmup):
        cpu_reference_rows_per_s(table, fds, min(sample, 20_000), "reference")
    rates, secs_total, kind = [], 0.0, "reference"
    for _ in range(args.steps):
        r, secs, kind, n, _res = cpu_reference_rows_per_s(table, fds, sample, "reference")
        rates.append(r)
        secs_total += secs
    value = args.steps * sample / secs_total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": gen.CONFIGS[cfg_id].name, "rows_per_step": sample,
                   "sample": (f"the whole {gen.CONFIGS[cfg_id].name} table"
                              if sample >= gen.CONFIGS[cfg_id].rows else
                              f"first {sample} rows of {gen.CONFIGS[cfg_id].name}"),
                   "parallelism": "single-thread CPU (the reference has no threads)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind,
                         "sample": f"{sample} rows of {gen.CONFIGS[cfg_id].name} (warm-up: "
                                   "20K-row prefix), GgrConfig defaults, wall time from "
                                   "SolveStats.wall_ms"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    # one GPU per rank (the host transport may put several ranks on one GPU)
    torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
    if world > 1:
        import torch.distributed as dist
        if args.transport == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    import paper_2403_05821_b200 as po
    from paper_2403_05821_b200 import gen
    from paper_2403_05821_b200._abi import PO_LOC_DEVICE, PO_LOC_HOST, cuda_lib
    from paper_2403_05821_b200.dist import shard_range

    lib = cuda_lib()
    sharded = world > 1 or args.sharded
    # N = 1: C2 (the headline metric's config); N > 1: C4, the north star's
    # 100M-row table, split N ways (strong scaling)
    cfg_id = args.config if args.config is not None else (4 if world > 1 else 2)
    t0 = time.time()
    n_total = args.rows if args.rows is not None else gen.CONFIGS[cfg_id].rows
    lo, hi = shard_range(n_total, world, rank) if sharded else (0, n_total)
    table = gen.generate(cfg_id, n_rows=hi - lo, row_begin=lo)
    n, m = table.row_count(), table.field_count()
    cell_bytes = table.cell_bytes
    log(f"[rank {rank}] generated {gen.CONFIGS[cfg_id].name} rows [{lo}, {hi}): "
        f"{cell_bytes/1e9:.3f} GB in {time.time()-t0:.1f}s")
    fds = gen.fds(cfg_id)
    fd_idx = [[table.require_field(x) for x in g] for g in fds]
    cfg = po.GgrConfig()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    d_arena = torch.from_numpy(table.arena).to("cuda")
    d_offs = torch.from_numpy(table.offsets.view(np.int64)).to("cuda")
    dview = table.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
    d_rows = torch.empty(n, dtype=torch.int64, device="cuda")
    d_orders = torch.empty(n * m, dtype=torch.int32, device="cuda")

    comm = None
    if sharded:
        from paper_2403_05821_b200.dist import ggr_sharded_into, host_comm, nccl_comm
        comm = nccl_comm(rank, world) if args.transport == "nccl" else host_comm()

    def step_device():
        if sharded:
            r = ggr_sharded_into(comm, dview, fd_idx, cfg, 0, 0, sp, out_location=None)
            return r[4], r[5]
        return po.ggr_into(dview, fd_idx, cfg, 0, 0, PO_LOC_DEVICE, d_rows, d_orders, sp)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if args.transport == "nccl" else "cpu")
        dist.all_reduce(t)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if args.transport == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 0)):
        phc, st = step_device()
    barrier()
    l0 = lib.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        clk.mark_start()
        ev0.record(stream)
        marks = []
        for _ in range(args.steps):
            phc, st = step_device()
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            marks.append(e)
        ev1.record(stream)
        barrier()
        clk.mark_end()
    launches_total = lib.kernel_launch_count() - l0  # our kernels inside the timed region
    launches = launches_total // max(args.steps, 1)
    ms = ev0.elapsed_time(ev1) / args.steps
    per = [ev0.elapsed_time(marks[0])] + [a.elapsed_time(b) for a, b in zip(marks, marks[1:])]
    log(f"[rank {rank}] per-step ms: " + " ".join(f"{x:.2f}" for x in per))
    ms = max_over_ranks(ms)
    value = n_total / (ms / 1e3)
    total_cell_bytes = int(sum_over_ranks(cell_bytes))
    log(f"[rank {rank}] device-resident: {ms:.3f} ms/step, phc={phc}, stats={st}")

    # per-kernel CUDA-event profile of the same step (separate pass)
    lib.profile_enable(1)
    lib.profile_report()
    for _ in range(args.prof_steps):
        step_device()
    torch.cuda.synchronize()
    prof = lib.profile_report()
    lib.profile_enable(0)
    prof_steps = max(args.prof_steps, 1)
    # leaf launches only ("scope:" entries wrap other launches); the total is
    # the device time under any launch ("busy:", the union of the intervals)
    kern = sorted(((v[1] / prof_steps, k, v[0] / prof_steps) for k, v in prof.items()
                   if not k.startswith(("scope:", "busy:"))), reverse=True)
    total_kernel_ms = prof.get("busy:", (1, sum(x[0] for x in kern) * prof_steps))[1] / prof_steps
    for ms_k, k, cnt in kern[:12]:
        log(f"   {k:28s} {ms_k:8.3f} ms/step  {cnt:6.1f} launches  "
            f"({100*ms_k/max(total_kernel_ms,1e-9):5.1f}% of kernel time)")

    # roofline of the dominant kernel: the top kernel by time when its
    # algorithmic bytes are defined, else the HBM-streaming dictionary kernel.
    # k_hash_probe (K1 + K2a) must read every cell byte and its offset pair
    # once: S + 8*(n*m+1) per launch over all its launches of a step (the
    # 4-byte id it writes per cell is an intermediate of this design and is
    # not counted)
    peak, peak_kind = peaks()
    alg = {"k_hash_probe": cell_bytes + 8 * (n * m + 1)}
    top = kern[0][1] if kern else "k_hash_probe"
    dom = top if top in alg else "k_hash_probe"
    dom_ms = prof.get(dom, (1, 0.0))[1] / prof_steps  # all launches of one step
    dom_bytes = alg[dom]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():  # dram bytes per launch from the committed ncu --set full capture
        try:
            tj = json.loads(tfile.read_text())
            if tj.get("workload") == gen.CONFIGS[cfg_id].name and n == tj.get("rows"):
                traffic = tj.get("kernels", {}).get(dom)
        except (ValueError, OSError):
            traffic = None
    # whole-pipeline figure on SURVEY.md §8d's B_alg = S_row + 8m + 4 + m per row
    b_alg = cell_bytes + n * (8 * m + 4 + m)

    # e2e: pinned host inputs and outputs through the C ABI every step (large
    # shards are page-locked in place instead of copied)
    registered = []
    if cell_bytes > (4 << 30):
        from cuda.bindings import runtime as rt
        for arr in (table.arena, table.offsets):
            rt.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
            registered.append(arr.ctypes.data)
        h_arena, h_offs = table.arena, table.offsets
    else:
        h_arena = torch.from_numpy(table.arena).pin_memory()
        h_offs = torch.from_numpy(table.offsets.view(np.int64)).pin_memory()
    hview = table.view(PO_LOC_HOST, arena=h_arena, offsets=h_offs)
    h_rows = torch.empty(n, dtype=torch.int64).pin_memory()
    h_orders = torch.empty(n * m, dtype=torch.int32).pin_memory()

    def step_e2e():
        if sharded:
            r = ggr_sharded_into(comm, hview, fd_idx, cfg, 0, 0, sp, out_location=PO_LOC_HOST)
            return r[4], r[5]
        return po.ggr_into(hview, fd_idx, cfg, 0, 0, PO_LOC_HOST, h_rows, h_orders, sp)

    inflight = 1 if sharded else max(1, args.e2e_inflight)
    if inflight == 1:
        for _ in range(max(1, args.warmup // 2)):
            step_e2e()
    barrier()
    # Calls in flight: P host threads, each with its own stream and output
    # buffers, take the steps round-robin, so one step's table copy (PCIe)
    # overlaps another step's solve (SMs); every step still copies its whole
    # table in and its schedule out. Device time from an event before the
    # first step to the last stream's completion.
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_e = time.perf_counter()
    if inflight == 1:
        e0.record(stream)
        for _ in range(args.steps):
            phc_e2e, _st = step_e2e()
        e1.record(stream)
    else:
        import threading
        streams = [torch.cuda.Stream() for _ in range(inflight)]
        outs = [(torch.empty(n, dtype=torch.int64).pin_memory(),
                 torch.empty(n * m, dtype=torch.int32).pin_memory()) for _ in range(inflight)]
        results, errors = [], []

        def worker(j, nsteps):
            try:
                torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
                for _ in range(j, nsteps, inflight):
                    results.append(po.ggr_into(hview, fd_idx, cfg, 0, 0, PO_LOC_HOST, outs[j][0],
                                               outs[j][1], streams[j].cuda_stream))
            except Exception as ex:  # pragma: no cover
                errors.append(ex)

        def run(nsteps):
            ths = [threading.Thread(target=worker, args=(j, nsteps)) for j in range(inflight)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            if errors:
                raise errors[0]

        # warm-up in the same configuration: the block cache then holds the
        # buffers of every call in flight (no cudaMalloc in the timed steps)
        run(max(2, args.warmup // 2) * inflight)
        torch.cuda.synchronize()
        results.clear()
        t_e = time.perf_counter()
        e0.record(stream)
        for st_ in streams:
            st_.wait_event(e0)
        run(args.steps)
        for st_ in streams:
            done = torch.cuda.Event()
            done.record(st_)
            stream.wait_event(done)
        e1.record(stream)
        phc_e2e = results[-1][0]
        if any(r[0] != phc_e2e for r in results):
            raise RuntimeError("pipelined e2e steps disagree")
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    wall_e2e = (time.perf_counter() - t_e) * 1e3 / args.steps
    h2d = int(sum_over_ranks(table.arena.nbytes + table.offsets.nbytes))
    d2h = int(n_total * 8 + n_total * m * 4 + 8 * world)
    if registered:
        from cuda.bindings import runtime as rt
        for ptr in registered:
            rt.cudaHostUnregister(ptr)
    if phc_e2e != phc:
        raise RuntimeError(f"e2e PHC {phc_e2e} != device-resident PHC {phc}")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            rate, secs, kind, ns, res = cpu_reference_rows_per_s(
                table, fds, args.cpu_rows if args.cpu_rows is not None else n, "reference")
            cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": kind,
                   "sample": f"first {ns} rows of {gen.CONFIGS[cfg_id].name}, GgrConfig "
                             f"defaults, {secs:.1f} s single-threaded (SolveStats.wall_ms)"}
            log(f"[rank 0] CPU reference ({kind}) on {ns} rows: {secs:.2f}s -> {rate:.0f} rows/s")
        except Exception as ex:  # pragma: no cover
            log(f"[rank 0] CPU baseline failed: {ex}")

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": gen.CONFIGS[cfg_id].name if not sharded else
                       f"{gen.CONFIGS[cfg_id].name} split {world} ways "
                       f"({n_total} rows, ~{n_total // world} per GPU)",
                       "rows": n_total, "rows_per_gpu": n_total // world, "fields": m,
                       "cell_bytes": total_cell_bytes,
                       "ggr_config": "defaults (4/2/100000, fds on)",
                       "tokenizer": "char", "scoring": "value_only",
                       "l2": "inputs (arena+offsets) larger than the 126 MB L2; no flush",
                       "parallelism": (f"dp{world}: one table row-range sharded, "
                                       f"{'NCCL' if args.transport == 'nccl' else 'host-staged gloo'}"
                                       " (po_ggr_sharded)") if sharded else "single GPU"},
            "phc": int(phc),
            "solve_stats": {"recursive_calls": st.recursive_calls,
                            "candidates_examined": st.candidates_examined,
                            "max_depth": st.max_depth},
            "e2e": {"value": n_total / (ms_e2e / 1e3), "unit": UNIT,
                    "cell_bytes_per_s": total_cell_bytes / (ms_e2e / 1e3),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": ms_e2e, "host_wall_ms_per_step": wall_e2e,
                    "calls_in_flight": inflight},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_step": dom_bytes,
                         "kernel_ms_per_step": dom_ms, "peak_source": peak_kind,
                         "top_kernel": {"name": top, "ms_per_step": kern[0][0] if kern else None,
                                        "share": (kern[0][0] / total_kernel_ms) if kern else None},
                         "pipeline_b_alg_frac": (b_alg / (ms / 1e3) / 1e9) / peak},
            "cell_bytes_per_s": value * total_cell_bytes / n_total,
            "kernels_ms_per_step": {k: round(v, 4) for v, k, _ in kern[:16]},
            "kernel_ms_total": round(total_kernel_ms, 4),
            "cpu_baseline": cpu,
            "gpu_launches": int(launches_total),
            "gpu_launches_per_step": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE config (default: 2 at N=1, 4 split N ways at N>1)")
    ap.add_argument("--transport", choices=["nccl", "host"], default="nccl",
                    help="collectives of the sharded solver: NCCL (one GPU per rank) or "
                         "host-staged over gloo (ranks may share a GPU; for testing)")
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-rows", type=int, default=None,
                    help="rows of the CPU baseline sample (default: the whole table)")
    ap.add_argument("--ref-rows", type=int, default=None,
                    help="rows per reference step (default: the whole configured table)")
    ap.add_argument("--prof-steps", type=int, default=3)
    ap.add_argument("--e2e-inflight", type=int, default=2,
                    help="e2e calls in flight (host threads with their own streams; 1 = serial)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded solver even at N=1 (NCCL, world size 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
