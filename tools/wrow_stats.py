"""Warp-row chain statistics (tuning; needs a -DMPSP_WSTATS build):

    python paper_1411_2377_b200/_build.py --name=v_wstats.so -DMPSP_WSTATS
    python tools/wrow_stats.py --lib v_wstats.so --cfgs C4

One application per config through the C ABI, then the counters of
wchain.cuh: passes, fast commits, failing steps by outcome (one-binade up /
down, dominant product, exact adder), zero-accumulator absorptions - per
32-step block of the warp rows.
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="v_wstats.so")
    ap.add_argument("--cfgs", default="C4")
    a = ap.parse_args()
    import numpy as np
    import torch
    import gen
    dev = torch.device("cuda:0")
    P = ctypes.c_void_p
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1411_2377_b200", a.lib))
    lib.mpsp_csr_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int64, P, P, P, P, P,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32]
    lib.mpsp_spmv.argtypes = [P] * 8
    lib.mpsp_spmv_t.argtypes = [P] * 8
    st = (ctypes.c_ulonglong * 8)()
    names = ["passes", "commits", "fails", "up", "down", "dominant", "exact", "absorb"]
    for c in a.cfgs.split(","):
        cfg, op = (c.split(":") + ["ax"])[:2]
        d = gen.make(cfg, seed=0)
        p, n = d["p"], d["n"]
        L = p // 32
        keep = [np.ascontiguousarray(d[k]) for k in ("rowptr", "colidx", "limbs", "exps", "signs")]
        h = P()
        rc = lib.mpsp_csr_create(ctypes.byref(h), p, n, *[k.ctypes.data_as(P) for k in keep], 0, n,
                                 1 if op == "atx" else 0)
        assert rc == 0, rc
        xl = torch.from_numpy(np.ascontiguousarray(d["x_limbs"]).view(np.int32).reshape(-1)).to(dev)
        xe = torch.from_numpy(np.ascontiguousarray(d["x_exps"]).astype(np.int32)).to(dev)
        xs = torch.from_numpy(np.ascontiguousarray(d["x_signs"]).astype(np.uint8)).to(dev)
        yl = torch.empty(n * L, dtype=torch.int32, device=dev)
        ye = torch.empty(n, dtype=torch.int32, device=dev)
        ys = torch.empty(n, dtype=torch.uint8, device=dev)
        lib.mpsp_debug_wrow_stats(st)
        f = lib.mpsp_spmv_t if op == "atx" else lib.mpsp_spmv
        rc = f(h, P(xl.data_ptr()), P(xe.data_ptr()), P(xs.data_ptr()), P(yl.data_ptr()),
               P(ye.data_ptr()), P(ys.data_ptr()), P(0))
        torch.cuda.synchronize()
        assert rc == 0, rc
        lib.mpsp_debug_wrow_stats(st)
        v = dict(zip(names, list(st)))
        blocks = max(1, v["commits"] + v["fails"] - (v["passes"] - v["commits"]))
        print(f"{cfg}:{op} " + " ".join(f"{k}={x}" for k, x in v.items())
              + f"  passes/commit={v['passes'] / max(1, v['commits']):.3f}"
              + f"  fails/commit={v['fails'] / max(1, v['commits']):.3f}", flush=True)


if __name__ == "__main__":
    main()
