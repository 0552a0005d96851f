"""Host-link probe for the e2e leg (tuning; run under gpurun).

    python tools/e2e_probe.py [--cfg C5] [--chunks 8,16,32]

Times (wall clock, synchronous) on the config's x / y sizes: a pinned H2D
alone, a pinned D2H alone, both at once on two streams, and mpsp_spmv_host
for handles created with each MPSP_CHUNKS value (the row-chunk pipeline of
mpsp_api.cpp).  Every handle's y must equal the first one's bit for bit.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C5")
    ap.add_argument("--chunks", default="8,16,32")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--small", default="0,1", help="MPSP_E2E_SMALL values to time")
    a = ap.parse_args()
    import numpy as np
    import torch
    import gen
    from paper_1411_2377_b200 import CSR
    dev = torch.device("cuda:0")
    d = gen.make(a.cfg, seed=0)
    n, L = d["n"], d["p"] // 32
    nb = n * (4 * L + 5)
    hbuf = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hbuf2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
    dbuf = torch.empty(nb, dtype=torch.uint8, device=dev)
    dbuf2 = torch.empty(nb, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def wall(f):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / a.reps

    def both():
        with torch.cuda.stream(s1):
            dbuf.copy_(hbuf, non_blocking=True)
        with torch.cuda.stream(s2):
            hbuf2.copy_(dbuf2, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    h2d = wall(lambda: dbuf.copy_(hbuf, non_blocking=True))
    d2h = wall(lambda: hbuf2.copy_(dbuf2, non_blocking=True))
    bi = wall(both)
    print(f"{a.cfg}: {nb / 1e6:.0f} MB each way: H2D {h2d:.2f} ms ({nb / h2d / 1e6:.1f} GB/s), "
          f"D2H {d2h:.2f} ms ({nb / d2h / 1e6:.1f} GB/s), both at once {bi:.2f} ms", flush=True)
    del dbuf, dbuf2
    hx = tuple(np.ascontiguousarray(d[k]) for k in ("x_limbs", "x_exps", "x_signs"))
    xl = torch.from_numpy(hx[0].view(np.int32)).pin_memory()
    xe = torch.from_numpy(hx[1]).pin_memory()
    xs = torch.from_numpy(hx[2]).pin_memory()
    hx = (xl.numpy().view(np.uint32), xe.numpy(), xs.numpy())
    first = None
    for c in a.chunks.split(","):
        os.environ["MPSP_CHUNKS"] = c
        A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"])
        yl = torch.empty((n, L), dtype=torch.int32).pin_memory()
        ye = torch.empty((n,), dtype=torch.int32).pin_memory()
        ys = torch.empty((n,), dtype=torch.uint8).pin_memory()
        hy = (yl.numpy().view(np.uint32), ye.numpy(), ys.numpy())
        for small in a.small.split(","):
            os.environ["MPSP_E2E_SMALL"] = small       # read per call
            hy[0][:] = 0
            ms = wall(lambda: A.spmv_host(*hx, out=hy))
            if first is None:
                first = tuple(v.copy() for v in hy)
            same = all(np.array_equal(u, v) for u, v in zip(first, hy))
            print(f"  MPSP_CHUNKS={c} MPSP_E2E_SMALL={small}: spmv_host {ms:.2f} ms  "
                  f"same_as_first={same}", flush=True)
        A.close()


if __name__ == "__main__":
    main()
