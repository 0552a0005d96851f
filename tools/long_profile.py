#!/usr/bin/env python
"""Debug timeline of the long-row kernel (CTA 0): builds libmpsp_dbg.so with
-DMPSP_LONG_PROFILE, runs one C4 A.x and prints per-chunk producer/consumer
clock64() spans.  Diagnostics only (not part of the product path)."""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1411_2377_b200 import _build
out = os.path.join(ROOT, "paper_1411_2377_b200", "build", "libmpsp_dbg.so")
objs = []
for src in _build.SOURCES:
    o = os.path.join(_build.BUILD, "dbg_" + src + ".o")
    subprocess.run([_build.nvcc(), *_build.ARCH, *_build.FLAGS, "-DMPSP_LONG_PROFILE", "-c",
                    os.path.join(_build.CSRC, src), "-o", o], check=True)
    objs.append(o)
subprocess.run([_build.nvcc(), *_build.ARCH, "-shared", "--cudart", "shared", "-o", out, *objs], check=True)
import paper_1411_2377_b200._lib as L
L.LIB_PATH = out
lib = L.lib()
import numpy as np, torch, gen
from paper_1411_2377_b200 import CSR, MPVec
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
d = gen.make(cfg)
A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"])
x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"])
for _ in range(2):
    A.spmv(x)
torch.cuda.synchronize()
n = 260
buf = (ctypes.c_longlong * (n * 6))()
lib.mpsp_debug_long_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
print("rc", lib.mpsp_debug_long_profile(buf, n))
t = np.array(buf[:], dtype=np.int64).reshape(n, 6)
t0 = t[0, 0]
for c in list(range(0, 12)) + list(range(100, 106)) + list(range(200, 212)):
    if c < n and t[c, 0]:
        print(c, (t[c, :4] - t0).tolist(), "prod", t[c, 1] - t[c, 0], "cons", t[c, 3] - t[c, 2], "rare steps", t[c, 4], "rare lanes", t[c, 5] & 0xFFFFF, "stale row-steps", t[c, 5] >> 20)
valid = t[:, 0] > 0
print("total rare steps", t[:, 4].sum(), "of", int(valid.sum()) * 24, "stale row-steps", (t[:, 5] >> 20).sum(), "of", int(valid.sum()) * 24 * 8)
print("avg prod", np.mean((t[:, 1] - t[:, 0])[valid]), "avg cons", np.mean((t[:, 3] - t[:, 2])[t[:, 2] > 0]))
