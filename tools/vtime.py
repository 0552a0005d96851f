"""Time several builds of the library side by side in ONE process (tuning).

    python tools/vtime.py --libs libmpsp.so,v1.so,v2.so --cfgs C2,C2:atx,C4 [--steps 20]

Each config is generated once; every library (paper_1411_2377_b200/<name>,
built by `python -m paper_1411_2377_b200._build --name=<name> -D...`) gets its
own handle through the C ABI and is timed with CUDA events (L2 flushed between
steps when the working set fits in L2), rounds interleaved across the libraries
so clock drift hits all of them alike.  Every variant's y must equal the first
library's bit for bit (the first is normally the default build, whose parity
the GPU tests establish).  Prints one line per (config, library).
"""
from __future__ import annotations

import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="libmpsp.so")
    ap.add_argument("--cfgs", default="C2")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch
    import gen
    dev = torch.device("cuda:0")
    P = ctypes.c_void_p
    libs = []
    loaded = {}
    for spec in a.libs.split(","):
        # "lib.so" or "lib.so@ENV=V;ENV2=V2" (environment set around that variant's calls)
        name = spec
        lname, _, envs = spec.partition("@")
        env = dict(kv.split("=", 1) for kv in envs.split(";") if kv)
        if lname not in loaded:
            loaded[lname] = ctypes.CDLL(os.path.join(ROOT, "paper_1411_2377_b200", lname))
        L = loaded[lname]
        L.mpsp_csr_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int64, P, P, P, P, P,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32]
        for f in ("mpsp_spmv", "mpsp_spmv_t"):
            getattr(L, f).argtypes = [P] * 8
        L.mpsp_destroy.argtypes = [P]
        libs.append((name, L, env))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for c in a.cfgs.split(","):
        cfg, op = (c.split(":") + ["ax"])[:2]
        cfg, _, pp = cfg.partition("@")            # "C2@2048": the config at another p
        d = gen.make(cfg, seed=0, p=int(pp) if pp else None)
        p, n = d["p"], d["n"]
        Lm = p // 32
        hp = lambda arr: np.ascontiguousarray(arr).ctypes.data_as(P)
        keep = [np.ascontiguousarray(d[k]) for k in ("rowptr", "colidx", "limbs", "exps", "signs")]
        xl = torch.from_numpy(np.ascontiguousarray(d["x_limbs"]).view(np.int32).reshape(-1)).to(dev)
        xe = torch.from_numpy(np.ascontiguousarray(d["x_exps"]).astype(np.int32)).to(dev)
        xs = torch.from_numpy(np.ascontiguousarray(d["x_signs"]).astype(np.uint8)).to(dev)
        nnz = int(d["rowptr"][-1])
        res = []
        handles = []
        for name, L, env in libs:
            h = P()
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)             # create-time knobs (MPSP_LONG_T, MPSP_CHUNKS)
            rc = L.mpsp_csr_create(ctypes.byref(h), p, n, *[k.ctypes.data_as(P) for k in keep],
                                   0, n, 1 if op == "atx" else 0)
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
            assert rc == 0, (name, rc)
            y = (torch.empty(n * Lm, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
                 torch.empty(n, dtype=torch.uint8, device=dev))
            f = L.mpsp_spmv if op == "ax" else L.mpsp_spmv_t
            args = [h, P(xl.data_ptr()), P(xe.data_ptr()), P(xs.data_ptr()),
                    P(y[0].data_ptr()), P(y[1].data_ptr()), P(y[2].data_ptr()), P(st)]
            handles.append((name, L, h, f, args, y, env))
        times = {name: [] for name, *_ in handles}
        for _ in range(a.rounds):
            for name, L, h, f, args, y, env in handles:
                saved = {k: os.environ.get(k) for k in env}
                os.environ.update(env)
                for _ in range(3):
                    assert f(*args) == 0
                torch.cuda.synchronize()
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(a.steps)]
                for e0, e1 in evs:
                    flush.zero_()
                    e0.record()
                    f(*args)
                    e1.record()
                torch.cuda.synchronize()
                for k, v in saved.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
                times[name] += [x.elapsed_time(z) for x, z in evs]
        ref = handles[0][5]
        for name, L, h, f, args, y, env in handles:
            same = all(torch.equal(u, v) for u, v in zip(y, ref))
            t = times[name]
            print(f"{cfg}:{op} {name:24s} median {statistics.median(t) * 1e3:9.2f} us  "
                  f"min {min(t) * 1e3:9.2f} us  MP-nnz/s {nnz / statistics.median(t) / 1e-3:.3e}  "
                  f"same_as_first={same}", flush=True)
            L.mpsp_destroy(h)
        del handles, xl, xe, xs, d, keep
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
