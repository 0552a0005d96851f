#!/usr/bin/env python
"""Debug: build libmpsp_chk.so with -DMPSP_LONG_CHECK and report the first
step where the long-row consumer diverges from a reference chain."""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1411_2377_b200 import _build
out = os.path.join(ROOT, "paper_1411_2377_b200", "build", "libmpsp_chk.so")
objs = []
for src in _build.SOURCES:
    o = os.path.join(_build.BUILD, "chk_" + src + ".o")
    subprocess.run([_build.nvcc(), *_build.ARCH, *_build.FLAGS, "-DMPSP_LONG_CHECK", "-c",
                    os.path.join(_build.CSRC, src), "-o", o], check=True)
    objs.append(o)
subprocess.run([_build.nvcc(), *_build.ARCH, "-shared", "--cudart", "shared", "-o", out, *objs], check=True)
import paper_1411_2377_b200._lib as Lb
Lb.LIB_PATH = out
lib = Lb.lib()
import numpy as np, torch, gen
from paper_1411_2377_b200 import CSR, MPVec
p = int(sys.argv[1]) if len(sys.argv) > 1 else 32
op = sys.argv[2] if len(sys.argv) > 2 else "atx"
d = gen.stress(p, seed=0) if len(sys.argv) <= 3 else gen.make(sys.argv[3], n=20000, p=p)
A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], transpose=True)
x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"])
y = A.spmv(x) if op == "ax" else A.spmv_t(x)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 64)()
lib.mpsp_debug_long_check.argtypes = [ctypes.c_void_p]
lib.mpsp_debug_long_check(buf)
v = list(buf)
names = ["cta", "lane", "step", "info", "eu", "E0", "S0", "z0", "Ecur", "Scur", "Eref", "Sref", "q0", "Et"]
print({n: (v[i] if i not in (4, 5, 8, 10, 13) else ctypes.c_int32(v[i]).value) for i, n in enumerate(names)})
L = p // 32
print("Sc  ", [hex(v[16 + i]) for i in range(min(L, 8))])
print("Sref", [hex(v[24 + i]) for i in range(min(L, 8))])
print("Qup ", [hex(v[32 + i]) for i in range(min(L, 8))])
print("M   ", [hex(v[40 + i]) for i in range(min(L, 8))])
