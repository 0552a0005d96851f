"""Helpers shared by the GPU tests: run the CUDA path (through the C ABI) and
the oracle on the same seeded inputs and compare bitwise."""
import numpy as np

import oracle


def oracle_args(d):
    return (d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            d["x_limbs"], d["x_exps"], d["x_signs"])


def oracle_full(d, op):
    f = oracle.spmv if op == "ax" else oracle.spmv_t
    return f(*oracle_args(d))


def oracle_rows(d, op, rows):
    """Packed oracle result for the listed rows (A x) or columns (A^T x)."""
    if op == "ax":
        vals = oracle.spmv_rows(*oracle_args(d), rows)
    else:
        vals = oracle.spmv_t_cols(*oracle_args(d), rows)
    return oracle.pack_vec(vals, d["p"])


def gpu_run(d, op, rows=None, device="cuda:0"):
    from paper_1411_2377_b200 import CSR, MPVec
    A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            rows=rows, transpose=(op == "atx"))
    x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device=device)
    y = A.spmv(x) if op == "ax" else A.spmv_t(x)
    out = y.to_host()
    A.close()
    return out


def assert_same(got, want, label=""):
    gl, ge, gs = got
    wl, we, ws = want
    gl = np.asarray(gl).reshape(wl.shape)
    bad = np.flatnonzero(np.any(gl != wl, axis=1) | (ge != we) | (gs != ws))
    if len(bad):
        i = bad[0]
        raise AssertionError(
            f"{label}: {len(bad)} of {len(we)} results differ; first at {i}: "
            f"got (s={gs[i]}, e={ge[i]}, m={[hex(v) for v in gl[i][::-1]]}) "
            f"want (s={ws[i]}, e={we[i]}, m={[hex(v) for v in wl[i][::-1]]})")
