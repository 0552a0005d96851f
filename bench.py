#!/usr/bin/env python
"""Benchmark: multiple-precision CSR SpMV on B200 (arXiv 1411.2377 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--op ax]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...      (the CPU oracle, timed as it stands)

A "step" is one application y = A x (or A^T x) of the whole hot path over the
config's synthetic matrix: (N>1: NCCL all-gather of x, then) the SpMV kernel
over the rank's row block.  Inputs are resident in HBM when the timed region
starts.  Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MP SpMV nnz/s and limb-MACs/s per GPU at p=128..1024 bits; % roofline"
UNIT = "MP-nnz/s"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--op", default="ax", choices=["ax", "atx"])
    ap.add_argument("--impl", default="mpsp", choices=["mpsp", "reference"])
    ap.add_argument("--exchange", default="window", choices=["window", "allgather"],
                    help="x exchange for N > 1 (dist.py)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--p", type=int, default=None,
                    help="override the config's precision (e.g. 2048: the paper's solver precision)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    return ap.parse_args()


def algorithmic(meta, nrows):
    """Algorithmic bytes / limb-MACs of one application:
    A once (4L+8 B/nnz), x read once and y written once (4L+4 B/elem each),
    int32 rowptr; limb-MACs = nnz * L^2."""
    L = meta["p"] // 32
    nnz = meta["nnz"]
    n = meta["n"]
    bytes_ = nnz * (4 * L + 8) + n * (4 * L + 4) + nrows * (4 * L + 4) + 4 * (nrows + 1)
    return bytes_, nnz * L * L


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=3)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def workload_name(args):
    """`C2 ax`, or `C2@p2048 ax` with a precision override."""
    return f"{args.config}{'' if args.p is None else f'@p{args.p}'} {args.op}"


def cpu_baseline(d, op, seconds, rows_cap=None):
    """The oracle as it stands on the host cores over a bounded row sample."""
    from oracle import run_parallel
    n = d["n"]
    rng = np.random.default_rng(12345)
    order = rng.permutation(n)
    lens = np.diff(d["rowptr"]) if op == "ax" else np.bincount(d["colidx"], minlength=n)
    # estimate cost: ~4 us per nnz per core at p<=1024, aim at `seconds` of work
    cores = run_parallel.n_cores()
    target_nnz = int(seconds * cores * 2.5e5 * (256 / max(d["p"], 256)) ** 0.5)
    cum = np.cumsum(lens[order])
    k = int(np.searchsorted(cum, target_nnz)) + 1
    rows = np.sort(order[:max(1, min(k, n))])
    if op == "ax":
        _, wall, used = run_parallel.spmv_rows_parallel(
            d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            d["x_limbs"], d["x_exps"], d["x_signs"], rows)
    else:  # A^T rows through the oracle's transpose of the sampled columns
        import oracle
        t0 = time.perf_counter()
        oracle.spmv_t_cols(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
                           d["x_limbs"], d["x_exps"], d["x_signs"], rows[:2000])
        wall, used = time.perf_counter() - t0, 1
        rows = rows[:2000]
    nnz = int(lens[rows].sum())
    return {"value": nnz / wall, "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": f"{len(rows)} of {n} rows ({nnz} nnz) of {d['cfg']} {op}, "
                      f"{wall:.1f} s wall on {used} processes"}


def run_reference(args):
    """--impl reference: the CPU oracle timed as it stands, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gen
    d = gen.make(args.config, seed=args.seed, p=args.p)
    times, nnzs, cb = [], [], None
    for step in range(args.warmup + args.steps):
        cb = cpu_baseline(d, args.op, seconds=max(1.0, 60.0 / (args.warmup + args.steps)))
        if step >= args.warmup:
            nnz = int(cb["sample"].split("(")[1].split(" nnz")[0])
            nnzs.append(nnz)
            times.append(nnz / cb["value"])
    value = sum(nnzs) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * d["meta"]["nnz"] / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": f"u32 limbs (p={d['p']})",
            "data": "synthetic",
            "config": {"workload": workload_name(args), **d["meta"]},
            "cpu_baseline": {**cb, "value": value},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "each step is a bounded row sample of the workload; ms_per_step extrapolates "
                    "the sampled rate to the full matrix"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import __graft_entry__
    __graft_entry__.build()
    import gen
    from paper_1411_2377_b200 import CSR, MPVec, launch_count, imad_bench
    from paper_1411_2377_b200.dist import block_range, allgather_x, needed_window, WindowExchange

    t0 = time.perf_counter()
    d = gen.make(args.config, seed=args.seed, p=args.p)
    t_gen = time.perf_counter() - t0
    n, p = d["n"], d["p"]
    L = p // 32
    rb, re = block_range(n, world, rank)
    t0 = time.perf_counter()
    A = CSR(p, d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], rows=(rb, re),
            transpose=(args.op == "atx"))
    t_create = time.perf_counter() - t0
    info = A.info()
    nnz_local = info["nnz"] if args.op == "ax" else info["nnz_t"]
    x_full_host = (d["x_limbs"], d["x_exps"], d["x_signs"])
    x_local = MPVec.from_host(d["x_limbs"][rb:re], d["x_exps"][rb:re], d["x_signs"][rb:re], device=dev)
    x_full = MPVec.from_host(*x_full_host, device=dev) if world == 1 else None
    X = None
    if world > 1 and args.exchange == "window":
        win = needed_window(d["rowptr"], d["colidx"], rb, re, transpose=(args.op == "atx"))
        X = WindowExchange(n, L, win, device=dev)
        v = X.local_view()                 # x_local lives in the exchange buffer
        v.limbs.copy_(x_local.limbs); v.exps.copy_(x_local.exps); v.signs.copy_(x_local.signs)
        x_local = v
    y = MPVec.empty(re - rb, L, device=dev)
    f = A.spmv if args.op == "ax" else A.spmv_t
    stream = torch.cuda.current_stream(dev)

    bytes_alg_full, macs_full = algorithmic(d["meta"], n)
    ws_bytes = bytes_alg_full / world
    flush = ws_bytes < 2 * L2_BYTES
    flush_buf = torch.empty(int(2 * L2_BYTES), dtype=torch.uint8, device=dev) if flush else None

    # events created up front: the host work between a step's first event and
    # its launch stays minimal (the GPU would idle through it)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.warmup + args.steps)]
    it_ev = iter(evs)

    def step(ev0=None, ev1=None):
        if world == 1:
            xf = x_full
        elif X is not None:
            xf = X.exchange(x_local)
        else:
            xf = allgather_x(x_local, n)
        ev0 = ev0 or torch.cuda.Event(enable_timing=True)
        ev1 = ev1 or torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        f(xf, out=y, stream=stream)
        ev1.record(stream)
        return ev0, ev1

    for _ in range(args.warmup):
        if flush:
            flush_buf.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    lc0 = launch_count()
    kern_ms = []
    step_ms = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        s0, s1, e0_, e1_ = next(it_ev)
        if flush:
            flush_buf.zero_()          # outside the step events: L2 cold for each step
        s0.record(stream)
        k0, k1 = step(e0_, e1_)
        s1.record(stream)
        kern_ms.append((k0, k1))
        step_ms.append((s0, s1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = launch_count() - lc0
    clocks = sampler.stop() if sampler else None
    kt = [a.elapsed_time(b) for a, b in kern_ms]
    st = [a.elapsed_time(b) for a, b in step_ms]
    t_total = torch.tensor([sum(st), sum(kt)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_total, op=dist.ReduceOp.MAX)
    total_ms, kern_total_ms = float(t_total[0]), float(t_total[1])
    ms_per_step = total_ms / args.steps
    nnz_all = d["meta"]["nnz"]
    value = nnz_all / (ms_per_step * 1e-3)

    # ---- e2e through the C ABI with host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        xl_h = torch.from_numpy(d["x_limbs"].view(np.int32)).pin_memory()
        xe_h = torch.from_numpy(d["x_exps"]).pin_memory()
        xs_h = torch.from_numpy(d["x_signs"]).pin_memory()
        yl_h = torch.empty((re - rb, L), dtype=torch.int32).pin_memory()
        ye_h = torch.empty((re - rb,), dtype=torch.int32).pin_memory()
        ys_h = torch.empty((re - rb,), dtype=torch.uint8).pin_memory()
        hx = (xl_h.numpy().view(np.uint32), xe_h.numpy(), xs_h.numpy())
        hy = (yl_h.numpy().view(np.uint32), ye_h.numpy(), ys_h.numpy())
        fh = A.spmv_host if args.op == "ax" else A.spmv_t_host
        ksteps = max(2, min(args.steps, 5))
        fh(*hx, out=hy)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            fh(*hx, out=hy)
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0]) * 1e3 / ksteps
        e2e = {"value": nnz_all / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(n * (4 * L + 5)) * world,
               "d2h_bytes_per_step": int(n * (4 * L + 5)),
               "ms_per_step": e2e_ms,
               "note": "mpsp_spmv_host on pinned host buffers: H2D of x, kernel, D2H of y, sync"}

    if rank != 0:
        A.close()
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant (only) kernel
    kern_avg_s = kern_total_ms * 1e-3 / args.steps
    bytes_local, macs_local = algorithmic(dict(d["meta"], nnz=nnz_local), re - rb)
    ib = imad_bench()
    import json as _json
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = _json.load(open(pk))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    int_peak = ib["limb_macs_per_s"]
    t_mem = bytes_local / (hbm_peak * 1e9)
    t_int = macs_local / int_peak
    if t_int >= t_mem:
        roof = {"bound": "alu", "achieved": macs_local / kern_avg_s / 1e12, "peak": int_peak / 1e12,
                "unit": "Tlimb-MAC/s",
                "peak_source": "mpsp_imad_bench: measured sustained Comba IMAD.WIDE rate, this run"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_local / kern_avg_s / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # DRAM bytes per launch of the dominant kernel from the committed ncu
    # --set full capture of this workload (tools/traffic_from_ncu.py)
    roof["traffic"] = None
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tj) and world == 1:
        rec = json.load(open(tj)).get(workload_name(args))
        if rec:
            roof["traffic"] = rec["traffic_bytes"]
            roof["traffic_source"] = f"profiles/{rec['summary'] or rec['report']} ({rec['kernel']})"
            roof["algorithmic_bytes"] = bytes_local
    thr = int(os.environ.get("MPSP_LONG_T", "192"))
    sell = f"spmv_sell_cp<{L}>" if L == 32 and os.environ.get("MPSP_CP", "1") != "0" else f"spmv_sell<{L}>"
    if L > 32:
        sell = f"spmv_wide<{L // 32}> (warp per row, limbs across lanes)"
        thr = 1 << 62
    roof["kernel"] = (sell if d["meta"]["max_row"] <= thr or args.op == "atx" else
                      f"{sell} + spmv_wrow<{L}> (concurrent streams, fork/join timed as one)")
    roof["kernel_ms"] = kern_avg_s * 1e3
    roof["t_roof_ms"] = max(t_mem, t_int) * 1e3
    roof["frac_of_t_roof"] = max(t_mem, t_int) / kern_avg_s
    roof["hbm_achieved_gbs"] = bytes_local / kern_avg_s / 1e9
    roof["macs_achieved_T"] = macs_local / kern_avg_s / 1e12
    # the algorithmic count is the schoolbook L^2 per nnz; the
    # short product with its exactness certificate executes fewer (DESIGN.md
    # "Product"), so frac can exceed 1: also report the IMAD pipe's own load
    # (p > 1024, spmv_wide's short product: the hi columns, diagonal chunks
    # included, plus the three top lo columns: L^2/2 + 19L)
    ex_per = (L * L - (L - 3) * (L - 2) // 2 if L >= 4 else L * L) if L <= 32 else L * L // 2 + 19 * L
    roof["executed_macs_per_nnz"] = ex_per
    roof["frac_executed"] = (nnz_local * ex_per / kern_avg_s) / int_peak

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(d, args.op, args.cpu_seconds)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": f"u32 limbs (p={p})",
        "data": "synthetic",
        "config": {"workload": workload_name(args), "n": n, "nnz": nnz_all, "p": p,
                   "max_row": d["meta"]["max_row"], "seed": args.seed,
                   "parallelism": f"row-block x{world}" + (
                       "" if world == 1 else (" + NCCL all-gather of x" if X is None else
                                              " + NCCL P2P needed-window exchange of x")),
                   "l2": "flushed between steps (2x L2 memset outside step events)" if flush
                   else "inputs larger than L2"},
        "limb_macs_per_s": macs_full / (ms_per_step * 1e-3),
        "kernel_ms_per_step": kern_total_ms / args.steps,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "imad_bench": ib,
        "paper_context": {
            "value": 1.79e6, "unit": "MP-nnz/s (lower bound, derived)",
            "note": "arXiv 1411.2377 reports no SpMV rate; BASELINE.md section 2 derives >= 2 nnz "
                    "per BiCG iteration time: epb3 (n=84617, nnz=463625), p=2048, Intel Core i7 "
                    "920, 1 thread, MPFR 3.0.1 (PAPER.md:160-166, 440-444, 463). Context only: "
                    "other precision, matrix and hardware."},
        "setup_s": {"generate": t_gen, "create": t_create},
    }
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(s + "\n")
    A.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
