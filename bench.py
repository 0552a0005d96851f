#!/usr/bin/env python
"""Benchmark: multiple-precision CSR SpMV on B200 (arXiv 1411.2377 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--op ax]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...      (the CPU oracle, timed as it stands)

A "step" is one application y = A x (or A^T x) of the whole hot path over the
config's synthetic matrix: (N>1: the x exchange, then) the SpMV kernels over
the rank's row block.  Inputs are resident in HBM when the timed region
starts.  Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".

The headline is BASELINE.json's largest config (C5 A x).  At N = 1 the same
line also carries:
  parity      - the GPU result of the headline workload compared limb by limb
                with the oracle's whole result vector (computed on all host
                cores for cpu_baseline; nothing is discarded);
  per_config  - every BASELINE config and operation (C1..C5 x {A x, A^T x}
                where BASELINE asks), each timed here (K steps, CUDA events on
                the launching stream), with its roofline fraction, executed-MAC
                pipe load, clocks, oracle throughput and whole-vector parity.
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
# the operations BASELINE.json asks for per config
OPS = {"C1": ("ax", "atx"), "C2": ("ax", "atx"), "C3": ("ax",), "C4": ("ax", "atx"), "C5": ("ax",)}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--op", default="ax", choices=["ax", "atx"])
    ap.add_argument("--impl", default="mpsp", choices=["mpsp", "reference"])
    ap.add_argument("--exchange", default="auto", choices=["auto", "window", "allgather"],
                    help="x exchange for N > 1 (dist.py); auto: window unless it spans > n/2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--p", type=int, default=None,
                    help="override the config's precision (e.g. 2048: the paper's solver precision)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / parity leg")
    ap.add_argument("--no-per-config", action="store_true", help="skip the per_config block")
    ap.add_argument("--cpu-seconds", type=float, default=30.0,
                    help="bound on the oracle's expected wall time for cpu_baseline/parity; a "
                         "larger workload is checked on a row sample")
    ap.add_argument("--ref-seconds", type=float, default=240.0,
                    help="--impl reference: whole-workload steps if (K+W) steps fit this bound")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    return ap.parse_args(argv)


def algorithmic(meta, nrows, nnz=None):
    """Algorithmic bytes / limb-MACs of one application:
    A once (4L+8 B/nnz), x read once and y written once (4L+4 B/elem each),
    int32 rowptr; limb-MACs = nnz * L^2 (schoolbook count)."""
    L = meta["p"] // 32
    nnz = meta["nnz"] if nnz is None else nnz
    n = meta["n"]
    bytes_ = nnz * (4 * L + 8) + n * (4 * L + 4) + nrows * (4 * L + 4) + 4 * (nrows + 1)
    return bytes_, nnz * L * L


def executed_macs_per_nnz(L):
    """Limb-MACs the kernels execute per nnz: the short
    product with an exactness certificate forms L^2 - (L-2)(L-1)/2 at L >= 4
    (columns L-2 .. 2L-2); p > 1024 (spmv_wide) the hi columns plus three lo
    columns, L^2/2 + 19L."""
    if L > 32:
        return L * L // 2 + 19 * L
    return L * L - (L - 2) * (L - 1) // 2 if L >= 4 else L * L


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


def make_config(args, d, world, exchange=None, flush=None):
    """The `config` dict - identical for the GPU arm and the reference arm."""
    m = d["meta"]
    if flush is None:
        flush = algorithmic(m, m["n"])[0] / world < 2 * L2_BYTES
    par = f"row-block x{world}"
    if world > 1:
        par += {"allgather": " + NCCL all-gather of x (one packed record per element)",
                "window": " + NCCL P2P needed-window exchange of x"}.get(exchange, "")
    return {"workload": workload_name(args), "n": m["n"], "nnz": m["nnz"], "p": m["p"],
            "max_row": m["max_row"], "seed": args.seed, "parallelism": par,
            "l2": ("flushed between steps (2x L2 memset outside step events)" if flush
                   else "inputs larger than L2")}


# ---------------------------------------------------------------- the oracle
def oracle_args(d):
    return (d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            d["x_limbs"], d["x_exps"], d["x_signs"])


def est_oracle_seconds(d, nnz, cores):
    """~1.6 / 1.8 / 2.3 / 4.5 us per nnz per core at p = 128 / 256 / 512 / 1024
    (SURVEY 8(d) plus the round-1 C5 measurement), + 0.6 us per row."""
    us = {128: 1.6, 256: 1.8, 512: 2.3, 1024: 4.5}.get(d["p"], 4.5 * (d["p"] / 1024) ** 1.6)
    return (nnz * us + 0.6 * d["n"]) * 1e-6 / max(1, cores)


def oracle_run(d, op, seconds, T=None):
    """The oracle as it stands on all host cores (oracle/run_parallel.py).

    The whole workload when its expected wall time fits `seconds`, else a
    random row (column) sample.  Returns (rows or None for all, packed result,
    cpu_baseline dict)."""
    from oracle import run_parallel
    n = d["n"]
    cores = run_parallel.n_cores()
    lens = np.diff(d["rowptr"]) if op == "ax" else np.bincount(d["colidx"], minlength=n)
    nnz_all = int(lens.sum())
    rows = None
    if est_oracle_seconds(d, nnz_all, cores) > seconds:
        frac = seconds / est_oracle_seconds(d, nnz_all, cores)
        rng = np.random.default_rng(12345)
        order = rng.permutation(n)
        k = int(np.searchsorted(np.cumsum(lens[order]), frac * nnz_all)) + 1
        rows = np.sort(order[:max(1, min(k, n))])
    t_tr = 0.0
    if op == "ax":
        out, wall, used = run_parallel.spmv_parallel(*oracle_args(d), rows=rows)
    else:
        out, wall, used, t_tr = run_parallel.spmv_t_parallel(*oracle_args(d), cols=rows, T=T)
    nnz = nnz_all if rows is None else int(lens[rows].sum())
    nr = n if rows is None else len(rows)
    what = "rows" if op == "ax" else "columns (rows of A^T)"
    cb = {"value": nnz / wall, "unit": UNIT, "cores": used, "kind": "oracle",
          "sample": (f"{'all ' if rows is None else ''}{nr} of {n} {what} ({nnz} nnz) of "
                     f"{d['cfg']}{'' if d['p'] == _spec_p(d) else '@p' + str(d['p'])} {op}, "
                     f"{wall:.2f} s wall on {used} processes"
                     + (f" (+{t_tr:.2f} s for oracle.transpose_np, not timed)" if op == "atx" else ""))}
    return rows, out, cb


def _spec_p(d):
    import gen
    return gen.configs.SPEC[d["cfg"]]["p"]


def parity_of(got, want, rows=None):
    gl, ge, gs = got
    if rows is not None:
        gl, ge, gs = gl[rows], ge[rows], gs[rows]
    wl, we, ws = want
    gl = np.asarray(gl).reshape(wl.shape)
    bad = np.any(gl != wl, axis=1) | (ge != we) | (gs != ws)
    return {"rows": int(len(we)), "mismatches": int(bad.sum()),
            "checked": "whole vector, limbs + exponent + sign vs oracle" if rows is None
                       else "row sample (whole vector exceeds --cpu-seconds), limbs + exponent + sign"}


# ------------------------------------------------------------ reference arm
def ref_exchange(args, d, world):
    """The exchange the GPU arm's DistCSR resolves to (same rule, all ranks'
    windows), so both arms print the same config."""
    if world == 1:
        return None
    from paper_1411_2377_b200.dist import block_range, choose_exchange, needed_window
    wins = [needed_window(d["rowptr"], d["colidx"], *block_range(d["n"], world, r),
                          transpose=(args.op == "atx")) for r in range(world)]
    return choose_exchange(args.exchange, wins, d["n"])


def run_reference(args):
    """--impl reference: the CPU oracle timed as it stands, rank 0 only.  Each
    step computes the whole workload when (K + W) steps fit --ref-seconds
    (C5: ~6 s per step on 16 cores), else the same bounded row sample every
    step; the config dict is the GPU arm's."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gen
    from oracle import run_parallel
    d = gen.make(args.config, seed=args.seed, p=args.p)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    op = args.op
    cores = run_parallel.n_cores()
    n = d["n"]
    lens = np.diff(d["rowptr"]) if op == "ax" else np.bincount(d["colidx"], minlength=n)
    per_step = max(0.5, args.ref_seconds / max(1, args.warmup + args.steps))
    T = run_parallel.transposed(*oracle_args(d)[:6]) if op == "atx" else None
    times, nnzs, cb = [], [], None
    for step in range(args.warmup + args.steps):
        rows, _, cb = oracle_run(d, op, per_step, T=T)
        if step >= args.warmup:
            nnz = int(lens.sum()) if rows is None else int(lens[rows].sum())
            nnzs.append(nnz)
            times.append(nnz / cb["value"])
    value = sum(nnzs) / sum(times)
    whole = "all " in cb["sample"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": f"u32 limbs (p={d['p']})",
            "data": "synthetic",
            "config": make_config(args, d, world, exchange=ref_exchange(args, d, world)),
            "cpu_baseline": {**cb, "value": value},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": ("each step computes the whole workload" if whole else
                     "each step is the same bounded row sample of the workload; ms_per_step is "
                     "the sample's wall time")}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def time_steps(f, x, y, stream, steps, warmup, flush_buf):
    """K timed applications (CUDA events on the launching stream, L2 flushed
    outside the events when flush_buf is given); returns per-step ms."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for _ in range(warmup):
        if flush_buf is not None:
            flush_buf.zero_()
        f(x, out=y, stream=stream)
    torch.cuda.synchronize()
    for e0, e1 in evs:
        if flush_buf is not None:
            flush_buf.zero_()
        e0.record(stream)
        f(x, out=y, stream=stream)
        e1.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def pow2_fraction(d, op):
    """Fraction of A's stored entries whose mantissa is exactly 2^(p-1) (at
    p = 1024 the kernels form no product for a warp of such entries, DESIGN.md
    "Product"; an upper bound of the skipped share - the whole warp must
    qualify).  0 below p = 1024."""
    if d["p"] != 1024 or len(d["limbs"]) == 0:
        return 0.0
    lm = np.asarray(d["limbs"]).reshape(-1, d["p"] // 32)
    f = (lm[:, -1] == np.uint32(0x80000000)) & ~np.any(lm[:, :-1], axis=1)
    return float(f.mean())


def roofline(meta, nrows, nnz, kern_s, int_peak, hbm_peak, peak_src, skip=0.0):
    """Roofline of one application: t_roof = max(bytes/HBM,
    nnz L^2 / P_int); frac = t_roof / t_kernel (= achieved / peak of the
    binding resource)."""
    L = meta["p"] // 32
    bytes_, macs = algorithmic(meta, nrows, nnz)
    t_mem = bytes_ / (hbm_peak * 1e9)
    t_int = macs / int_peak
    if t_int >= t_mem:
        r = {"bound": "alu", "achieved": macs / kern_s / 1e12, "peak": int_peak / 1e12,
             "unit": "Tlimb-MAC/s",
             "peak_source": "mpsp_imad_bench: measured sustained limb-MAC rate, this run, the "
                            "faster of the Comba (IMAD.WIDE) and operand-scanning (IMAD + IMAD.HI) "
                            "forms, per-lane operands"}
    else:
        r = {"bound": "hbm", "achieved": bytes_ / kern_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
             "peak_source": peak_src}
    r["frac"] = r["achieved"] / r["peak"]
    r["kernel_ms"] = kern_s * 1e3
    r["t_roof_ms"] = max(t_mem, t_int) * 1e3
    r["hbm_achieved_gbs"] = bytes_ / kern_s / 1e9
    r["macs_achieved_T"] = macs / kern_s / 1e12
    r["algorithmic_bytes"] = bytes_
    ex = executed_macs_per_nnz(L) * (1.0 - skip)
    r["executed_macs_per_nnz"] = ex
    if skip:
        r["power_of_two_entries"] = skip
    r["frac_executed"] = (nnz * ex / kern_s) / int_peak     # the IMAD pipe's own load
    return r


def kernel_names(d, op, L):
    sell = f"spmv_sell_cp<{L}>" if L == 32 and os.environ.get("MPSP_CP", "1") != "0" else f"spmv_sell<{L}>"
    if L > 32:
        return f"spmv_wide<{L // 32}> (warp per row, limbs across lanes)"
    thr = int(os.environ.get("MPSP_LONG_T", "256"))
    lens = np.diff(d["rowptr"]) if op == "ax" else np.bincount(d["colidx"], minlength=d["n"])
    if int(lens.max(initial=0)) <= thr:
        return sell
    return f"{sell} + spmv_wrow<{L}> (concurrent streams, fork/join timed as one)"


def per_config_block(args, dev, stream, flush_buf, int_peak, hbm_peak, peak_src, headline):
    """Every BASELINE config x operation, timed in this run, with parity."""
    import torch
    import gen
    from oracle import run_parallel
    from paper_1411_2377_b200 import CSR, MPVec
    out = {}
    for cfg in ("C1", "C2", "C3", "C4", "C5"):
        ops = OPS[cfg]
        d = gen.make(cfg, seed=args.seed)
        L = d["p"] // 32
        n = d["n"]
        A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
                transpose=("atx" in ops))
        info = A.info()
        x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device=dev)
        y = MPVec.empty(n, L, device=dev)
        T = run_parallel.transposed(*oracle_args(d)[:6]) if "atx" in ops and not args.no_cpu else None
        for op in ops:
            key = f"{cfg} {op}"
            if headline is not None and key == headline["key"]:
                out[key] = headline["entry"]
                continue
            f = A.spmv if op == "ax" else A.spmv_t
            nnz = info["nnz"] if op == "ax" else info["nnz_t"]
            ws = algorithmic(d["meta"], n, nnz)[0]
            fb = flush_buf if ws < 2 * L2_BYTES else None
            sampler = ClockSampler(torch.cuda.current_device())
            sampler.start()
            time.sleep(0.2)
            ms = time_steps(f, x, y, stream, max(args.steps, 10), max(args.warmup, 3), fb)
            clocks = sampler.stop()
            kern_s = statistics.median(ms) * 1e-3
            r = roofline(d["meta"], n, nnz, kern_s, int_peak, hbm_peak, peak_src,
                         pow2_fraction(d, op))
            e = {"kernel_ms_median": statistics.median(ms), "kernel_ms_min": min(ms),
                 "kernel_ms_mean": sum(ms) / len(ms), "steps": len(ms),
                 "value": nnz / kern_s, "unit": UNIT, "limb_macs_per_s": nnz * L * L / kern_s,
                 "nnz": nnz, "n": n, "p": d["p"], "max_row": int(d["meta"]["max_row"]),
                 "bound": r["bound"], "frac": r["frac"], "t_roof_ms": r["t_roof_ms"],
                 "frac_executed": r["frac_executed"], "hbm_achieved_gbs": r["hbm_achieved_gbs"],
                 "kernel": kernel_names(d, op, L),
                 "l2": "flushed between steps" if fb is not None else "inputs larger than L2",
                 "clocks": clocks}
            if not args.no_cpu:
                got = y.to_host()
                rows, want, cb = oracle_run(d, op, args.cpu_seconds, T=T)
                e["parity"] = parity_of(got, want, rows)
                e["cpu_baseline"] = cb
            out[key] = e
        A.close()
        del d, A, x, y, T
        torch.cuda.empty_cache()
    return out


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
    __graft_entry__.build()          # file-locked: one rank compiles, the others wait
    import gen
    from paper_1411_2377_b200 import CSR, MPVec, launch_count, imad_bench
    from paper_1411_2377_b200.dist import DistCSR, block_range

    t0 = time.perf_counter()
    d = gen.make(args.config, seed=args.seed, p=args.p)
    t_gen = time.perf_counter() - t0
    n, p = d["n"], d["p"]
    L = p // 32
    tr = args.op == "atx"
    rb, re = block_range(n, world, rank)
    t0 = time.perf_counter()
    exchange = None
    D = None
    if world == 1:
        A = CSR(p, d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], transpose=tr)
        info = A.info()
        nnz_local = info["nnz"] if args.op == "ax" else info["nnz_t"]
        x_full = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device=dev)
    else:
        D = DistCSR(p, d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], transpose=tr,
                    exchange=args.exchange, device=dev)
        exchange = D.xchg[tr].mode
        D.xchg[tr].set_local(d["x_limbs"][rb:re], d["x_exps"][rb:re], d["x_signs"][rb:re])
        nnz_local = sum((h.info()["nnz"] if not tr else h.info()["nnz_t"]) for h, _, _, _ in D.parts[tr])
        A = x_full = None
    t_create = time.perf_counter() - t0
    y = MPVec.empty(re - rb, L, device=dev)
    stream = torch.cuda.current_stream(dev)
    if D is None:
        f = A.spmv if args.op == "ax" else A.spmv_t
        apply = lambda: f(x_full, out=y, stream=stream)          # noqa: E731
    else:
        apply = lambda: D.apply(None, out=y, transpose=tr, stream=stream)   # noqa: E731

    bytes_alg_full, macs_full = algorithmic(d["meta"], n)
    ws_bytes = bytes_alg_full / world
    flush = ws_bytes < 2 * L2_BYTES
    need_flush_buf = flush or (world == 1 and rank == 0 and not args.no_per_config)
    flush_buf = torch.empty(int(2 * L2_BYTES), dtype=torch.uint8, device=dev) if need_flush_buf else None
    step_flush = flush_buf if flush else None

    # events created up front: the host work between a step's first event and
    # its launch stays minimal (the GPU would idle through it)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]

    def step(ev0, ev1):
        # N > 1: the exchange and the kernels interleave (interior rows overlap
        # the transfers), so the "kernel" events bracket the whole application
        ev0.record(stream)
        apply()
        ev1.record(stream)

    for _ in range(args.warmup):
        if step_flush is not None:
            step_flush.zero_()
        step(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    lc0 = launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for s0, s1, k0, k1 in evs:
        if step_flush is not None:
            step_flush.zero_()         # outside the step events: L2 cold for each step
        s0.record(stream)
        step(k0, k1)
        s1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = launch_count() - lc0
    clocks = sampler.stop() if sampler else None
    kt = [k0.elapsed_time(k1) for _, _, k0, k1 in evs]
    st = [s0.elapsed_time(s1) for s0, s1, _, _ in evs]
    t_total = torch.tensor([sum(st), sum(kt)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_total, op=dist.ReduceOp.MAX)
    total_ms, kern_total_ms = float(t_total[0]), float(t_total[1])
    ms_per_step = total_ms / args.steps
    nnz_all = d["meta"]["nnz"]
    value = nnz_all / (ms_per_step * 1e-3)
    y_host = y.to_host() if rank == 0 else None

    # ---- e2e through the public API with host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        xb = (0, n) if world == 1 else (rb, re)
        xl_h = torch.from_numpy(np.ascontiguousarray(d["x_limbs"][xb[0]:xb[1]]).view(np.int32)).pin_memory()
        xe_h = torch.from_numpy(np.ascontiguousarray(d["x_exps"][xb[0]:xb[1]])).pin_memory()
        xs_h = torch.from_numpy(np.ascontiguousarray(d["x_signs"][xb[0]:xb[1]])).pin_memory()
        yl_h = torch.empty((re - rb, L), dtype=torch.int32).pin_memory()
        ye_h = torch.empty((re - rb,), dtype=torch.int32).pin_memory()
        ys_h = torch.empty((re - rb,), dtype=torch.uint8).pin_memory()
        hx = (xl_h.numpy().view(np.uint32), xe_h.numpy(), xs_h.numpy())
        hy = (yl_h.numpy().view(np.uint32), ye_h.numpy(), ys_h.numpy())
        if D is None:
            fh = A.spmv_host if args.op == "ax" else A.spmv_t_host

            def e2e_step():
                fh(*hx, out=hy)
        else:
            v = D.xchg[tr].local_view()

            def e2e_step():
                v.limbs.copy_(xl_h, non_blocking=True)
                v.exps.copy_(xe_h, non_blocking=True)
                v.signs.copy_(xs_h, non_blocking=True)
                D.apply(None, out=y, transpose=tr, stream=stream)
                yl_h.copy_(y.limbs, non_blocking=True)
                ye_h.copy_(y.exps, non_blocking=True)
                ys_h.copy_(y.signs, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
        ksteps = max(2, min(args.steps, 5))
        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            e2e_step()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0]) * 1e3 / ksteps
        if rank == 0:
            assert all(np.array_equal(a, b) for a, b in zip(hy, y_host)), \
                "e2e result differs from the device-resident result"
        e2e = {"value": nnz_all / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(n * (4 * L + 5)),
               "d2h_bytes_per_step": int(n * (4 * L + 5)),
               "ms_per_step": e2e_ms,
               "note": ("mpsp_spmv_host on pinned host buffers: H2D of x, kernels, D2H of y "
                        "(row chunks overlapped with the kernels), sync" if world == 1 else
                        "per rank: H2D of the own x block, exchange + kernels (DistCSR.apply), "
                        "D2H of the own y block, sync; bytes summed over ranks")}

    if rank != 0:
        (A or D).close()
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel(s) (one fork/join launch group per step)
    kern_avg_s = kern_total_ms * 1e-3 / args.steps
    ib = imad_bench()
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if peaks else "B200_PROFILING.md fallback"
    int_peak = ib["limb_macs_per_s"]
    roof = roofline(d["meta"], re - rb, nnz_local, kern_avg_s, int_peak, hbm_peak, peak_src,
                    pow2_fraction(d, args.op))
    # DRAM bytes per launch of the dominant kernel from the committed ncu
    # --set full capture of this workload (tools/traffic_from_ncu.py)
    roof["traffic"] = None
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tj) and world == 1:
        rec = json.load(open(tj)).get(workload_name(args))
        if rec:
            roof["traffic"] = rec["traffic_bytes"]
            src = rec["summary"] or rec["report"]
            src = src if src.startswith("profiles/") else f"profiles/{src}"
            roof["traffic_source"] = f"{src} ({rec['kernel']})"
    roof["kernel"] = kernel_names(d, args.op, L)
    roof["frac_of_t_roof"] = roof["t_roof_ms"] / roof["kernel_ms"]

    cpu = parity = None
    if not args.no_cpu and world == 1:
        rows, want, cpu = oracle_run(d, args.op, args.cpu_seconds)
        parity = parity_of(y_host, want, rows)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": f"u32 limbs (p={p})",
        "data": "synthetic",
        "config": make_config(args, d, world, exchange, flush),
        "exchange": None if D is None else {
            "kind": exchange, "bytes_in_rank0": D.xchg[tr].bytes_in,
            "interior_rows_rank0": D.interior_rows(tr), "rows_rank0": re - rb,
            "note": "one (4L+4)-byte record per x element; interior rows overlap the transfers"},
        "limb_macs_per_s": macs_full / (ms_per_step * 1e-3),
        "kernel_ms_per_step": kern_total_ms / args.steps,
        "roofline": roof,
        "parity": parity,
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
    (A or D).close()
    del A, D, x_full, y
    if world == 1 and not args.no_per_config and args.p is None:
        key = f"{args.config} {args.op}"
        head = {"key": key, "entry": {
            "kernel_ms_median": statistics.median(kt), "kernel_ms_min": min(kt),
            "kernel_ms_mean": sum(kt) / len(kt), "steps": len(kt), "value": nnz_local / kern_avg_s,
            "unit": UNIT, "limb_macs_per_s": nnz_local * L * L / kern_avg_s, "nnz": nnz_local,
            "n": n, "p": p, "max_row": int(d["meta"]["max_row"]), "bound": roof["bound"],
            "frac": roof["frac"], "t_roof_ms": roof["t_roof_ms"],
            "frac_executed": roof["frac_executed"], "hbm_achieved_gbs": roof["hbm_achieved_gbs"],
            "kernel": roof["kernel"], "l2": line["config"]["l2"], "clocks": clocks,
            "parity": parity, "cpu_baseline": cpu, "note": "the headline measurement above"}}
        del d
        t0 = time.perf_counter()
        line["per_config"] = per_config_block(args, dev, stream, flush_buf, int_peak, hbm_peak,
                                              peak_src, head)
        line["per_config_s"] = time.perf_counter() - t0
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(s + "\n")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
