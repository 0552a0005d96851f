"""GPU tests of the C ABI contract and of invariants the CUDA path must obey
(SURVEY.md 4 T2/T4/T5'): error codes, ownership, host-buffer entry points,
row-range handles, determinism, identity/permutation/scaling/negation and
explicit zeros - all bit-exact."""
import ctypes

import numpy as np
import pytest

import gen
from gpu_util import assert_same, gpu_run, oracle_full

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    import __graft_entry__
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    __graft_entry__.build()


def _csr(d, **kw):
    from paper_1411_2377_b200 import CSR
    return CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], **kw)


def _x(d):
    from paper_1411_2377_b200 import MPVec
    return MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")


def test_notrans_alias_misaligned():
    import torch
    from paper_1411_2377_b200 import MPVec, MpspError
    from paper_1411_2377_b200 import _lib
    d = gen.make("C1", n=200)
    A = _csr(d)
    x = _x(d)
    with pytest.raises(MpspError) as e:
        A.spmv_t(x)
    assert e.value.name == "MPSP_E_NOTRANS"
    # aliasing: y's limbs on top of x's limbs
    y = MPVec(x.limbs, torch.empty_like(x.exps), torch.empty_like(x.signs))
    with pytest.raises(MpspError) as e:
        A.spmv(x, out=y)
    assert e.value.name == "MPSP_E_ALIAS"
    # misaligned limbs pointer
    buf = torch.zeros(d["n"] * 4 + 1, dtype=torch.int32, device="cuda:0")
    y = MPVec.empty(d["n"], 4)
    rc = _lib.lib().mpsp_spmv(A._h, buf.data_ptr() + 4, x.exps.data_ptr(), x.signs.data_ptr(),
                              y.limbs.data_ptr(), y.exps.data_ptr(), y.signs.data_ptr(), None)
    assert rc == _lib.ERROR_CODES["MPSP_E_ARG"]
    # host pointer passed to the device entry point
    hx = np.zeros((d["n"], 4), np.uint32)
    rc = _lib.lib().mpsp_spmv(A._h, hx.ctypes.data, x.exps.data_ptr(), x.signs.data_ptr(),
                              y.limbs.data_ptr(), y.exps.data_ptr(), y.signs.data_ptr(), None)
    assert rc == _lib.ERROR_CODES["MPSP_E_ARG"]
    A.close()


def test_handle_owns_copies_and_host_entry_points():
    d = gen.make("C1", n=500, seed=5)
    want = oracle_full(d, "ax")
    want_t = oracle_full(d, "atx")
    keep = {k: d[k].copy() for k in ("limbs", "exps", "signs", "colidx")}
    A = _csr(d, transpose=True)
    d["limbs"][:] = 0xFFFFFFFF                    # mutate inputs after create
    d["exps"][:] = 7
    x = _x(d)
    assert_same(A.spmv(x).to_host(), want, "after mutating host inputs")
    assert_same(A.spmv_host(d["x_limbs"], d["x_exps"], d["x_signs"]), want, "spmv_host")
    assert_same(A.spmv_t_host(d["x_limbs"], d["x_exps"], d["x_signs"]), want_t, "spmv_t_host")
    info = A.info()
    assert info["nnz"] == len(keep["colidx"]) and info["nnz_t"] == len(keep["colidx"])
    assert info["max_row"] == 8
    A.close()
    A.close()                                     # idempotent


@pytest.mark.parametrize("op", ["ax", "atx"])
def test_row_range_handles_concatenate(op):
    """T5': G row-range handles over the full x == the full result (no NCCL)."""
    d = gen.make("C4", n=6000, seed=7)
    full = gpu_run(d, op)
    n = d["n"]
    for G in (2, 3, 8):
        blk = (n + G - 1) // G
        parts = [gpu_run(d, op, rows=(min(r * blk, n), min((r + 1) * blk, n))) for r in range(G)]
        cat = tuple(np.concatenate([p_[i] for p_ in parts]) for i in range(3))
        assert_same(cat, full, f"G={G} {op}")


def test_determinism_repeated_application():
    d = gen.make("C3", n=8000, seed=9)
    A = _csr(d)
    x = _x(d)
    r0 = A.spmv(x).to_host()
    for _ in range(5):
        assert_same(A.spmv(x).to_host(), r0, "repeat")
    A.close()


def test_identity_permutation_scaling_negation():
    p = 256
    L = p // 32
    n = 3000
    d = gen.make("C3", n=n, p=p, seed=11)
    one = np.zeros((n, L), np.uint32)
    one[:, -1] = 0x80000000
    # identity
    ident = dict(p=p, n=n, rowptr=np.arange(n + 1, dtype=np.int64),
                 colidx=np.arange(n, dtype=np.int32), limbs=one, exps=np.ones(n, np.int32),
                 signs=np.zeros(n, np.uint8), x_limbs=d["x_limbs"], x_exps=d["x_exps"],
                 x_signs=d["x_signs"])
    y = gpu_run(ident, "ax")
    assert_same(y, (d["x_limbs"], d["x_exps"], d["x_signs"]), "identity")
    # permutation
    perm = np.random.default_rng(1).permutation(n).astype(np.int32)
    P = dict(ident, colidx=perm)
    assert_same(gpu_run(P, "ax"), (d["x_limbs"][perm], d["x_exps"][perm], d["x_signs"][perm]), "perm")
    # 2^k scaling and negation of A
    base = gpu_run(d, "ax")
    nz = np.any(base[0] != 0, axis=1)
    for k in (-7, 3):
        ds = dict(d, exps=d["exps"] + k)
        want = (base[0], np.where(nz, base[1] + k, 0).astype(np.int32), base[2])
        assert_same(gpu_run(ds, "ax"), want, f"2^{k} scaling")
    dn = dict(d, signs=(1 - d["signs"]).astype(np.uint8))
    want = (base[0], base[1], np.where(nz, 1 - base[2], 0).astype(np.uint8))
    assert_same(gpu_run(dn, "ax"), want, "negation")


def test_explicit_zeros_change_nothing():
    """Insert explicit zero entries (junk sign/exp) into every row."""
    d = gen.make("C1", n=400, seed=12)
    base = gpu_run(d, "ax")
    n, L = d["n"], d["p"] // 32
    rp, ci = d["rowptr"], d["colidx"]
    rows, cols, li, ex, sg = [], [], [], [], []
    rng = np.random.default_rng(3)
    for i in range(n):
        existing = set(ci[rp[i]:rp[i + 1]].tolist())
        extra = [c for c in rng.choice(n, 6, replace=False).tolist() if c not in existing][:3]
        ent = [(c, d["limbs"][k], d["exps"][k], d["signs"][k]) for k, c in
               zip(range(rp[i], rp[i + 1]), ci[rp[i]:rp[i + 1]])]
        ent += [(c, np.zeros(L, np.uint32), rng.integers(-99, 99), rng.integers(0, 2)) for c in extra]
        ent.sort(key=lambda t: t[0])
        for c, l_, e_, s_ in ent:
            rows.append(i); cols.append(c); li.append(l_); ex.append(e_); sg.append(s_)
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rowptr[1:])
    dz = dict(d, rowptr=rowptr, colidx=np.array(cols, np.int32), limbs=np.array(li, np.uint32),
              exps=np.array(ex, np.int32), signs=np.array(sg, np.uint8))
    assert_same(gpu_run(dz, "ax"), base, "explicit zeros")


def test_empty_matrix_and_empty_rows():
    from paper_1411_2377_b200 import CSR, MPVec
    p, L, n = 128, 4, 70
    rowptr = np.zeros(n + 1, np.int64)
    A = CSR(p, rowptr, np.zeros(0, np.int32), np.zeros((0, L), np.uint32), np.zeros(0, np.int32),
            np.zeros(0, np.uint8), transpose=True)
    xl = np.zeros((n, L), np.uint32)
    xl[:, -1] = 0x80000000
    x = MPVec.from_host(xl, np.ones(n, np.int32), np.ones(n, np.uint8))
    for y in (A.spmv(x), A.spmv_t(x)):
        yl, ye, ys = y.to_host()
        assert not yl.any() and not ye.any() and not ys.any()
    A.close()
    # n = 0
    A = CSR(p, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros((0, L), np.uint32),
            np.zeros(0, np.int32), np.zeros(0, np.uint8))
    y = A.spmv(MPVec.empty(0, L))
    assert y.n == 0
    A.close()


def test_launch_counter_counts_kernels():
    from paper_1411_2377_b200 import launch_count
    d = gen.make("C1", n=100)
    A = _csr(d)
    x = _x(d)
    c0 = launch_count()
    for _ in range(3):
        A.spmv(x)
    assert launch_count() - c0 >= 3
    A.close()


@pytest.mark.parametrize("cfg,n,op", [("C5", 4900, "ax"), ("C2", 5000, "ax"), ("C2", 5000, "atx"),
                                      ("C3", 3000, "ax")])
def test_needed_window_suffices(cfg, n, op):
    """Emulated G-rank run on one GPU: each rank's x buffer holds the global x
    only inside its needed window (dist.needed_window) and junk everywhere
    else; the concatenated row blocks must equal the 1-GPU result, i.e. the
    kernels never read x outside the window the exchange fills.  Compared
    with the oracle (and the 1-GPU CUDA result), not with the CUDA path alone."""
    import torch
    from paper_1411_2377_b200 import MPVec
    from paper_1411_2377_b200.dist import block_range, needed_window
    d = gen.make(cfg, n=n, seed=13)
    n = d["n"]
    full = oracle_full(d, op)
    assert_same(gpu_run(d, op), full, f"{cfg} 1-GPU {op}")
    rng = np.random.default_rng(5)
    for G in (2, 4, 8):
        parts = []
        for r in range(G):
            rb, re = block_range(n, G, r)
            lo, hi = needed_window(d["rowptr"], d["colidx"], rb, re, transpose=(op == "atx"))
            xl = rng.integers(0, 2 ** 32, size=d["x_limbs"].shape, dtype=np.uint32)
            xe = rng.integers(-2 ** 20, 2 ** 20, size=n).astype(np.int32)
            xs = rng.integers(0, 2, size=n).astype(np.uint8)
            xl[:, -1] |= np.uint32(0x80000000)
            xl[lo:hi], xe[lo:hi], xs[lo:hi] = d["x_limbs"][lo:hi], d["x_exps"][lo:hi], d["x_signs"][lo:hi]
            A = _csr(d, rows=(rb, re), transpose=(op == "atx"))
            x = MPVec.from_host(xl, xe, xs, device="cuda:0")
            y = (A.spmv_t if op == "atx" else A.spmv)(x)
            torch.cuda.synchronize()
            parts.append(y.to_host())
            A.close()
        cat = tuple(np.concatenate([p_[i] for p_ in parts]) for i in range(3))
        assert_same(cat, full, f"{cfg} G={G} {op}")


@pytest.mark.parametrize("exchange", ["window", "allgather"])
def test_distcsr_single_rank_nccl(exchange):
    """DistCSR over a 1-rank NCCL group (the N > 1 code path: window
    all-gather at setup, the exchange, the local handle) equals CSR.spmv."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_1411_2377_b200 import MPVec
    from paper_1411_2377_b200.dist import DistCSR
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    d = gen.make("C5", n=2500, seed=14)
    want = oracle_full(d, "ax")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        D = DistCSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
                    exchange=exchange, device="cuda:0")
        x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")
        y = D.apply(x)
        torch.cuda.synchronize()
        assert_same(y.to_host(), want, f"DistCSR {exchange}")
        D.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [32, 64, 128, 256, 1024, 2048])
def test_vec_pack_unpack_records(p):
    """mpsp_vec_pack / mpsp_vec_unpack (the x-exchange records, csrc/xchg.cu):
    record i = (L limbs, (sign << 31) | (exp & 0x7fffffff)), built here with
    numpy; unpack restores the vector bit for bit."""
    import torch
    from paper_1411_2377_b200 import MPVec
    from paper_1411_2377_b200.dist import LibPacker
    L = p // 32
    rng = np.random.default_rng(p)
    n = 3001
    xl = rng.integers(0, 2 ** 32, size=(n, L), dtype=np.uint32)
    xe = rng.integers(-(2 ** 29), 2 ** 29 + 1, size=n).astype(np.int32)
    xs = rng.integers(0, 2, size=n).astype(np.uint8)
    v = MPVec.from_host(xl, xe, xs, device="cuda:0")
    rec = torch.zeros((n, L + 1), dtype=torch.int32, device="cuda:0")
    P = LibPacker(L)
    P.pack(v, rec)
    want = np.zeros((n, L + 1), np.uint32)
    want[:, :L] = xl
    want[:, L] = (xs.astype(np.uint32) << 31) | (xe.view(np.uint32) & np.uint32(0x7fffffff))
    torch.cuda.synchronize()
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), want)
    w = MPVec.empty(n, L, device="cuda:0")
    P.unpack(rec, w)
    torch.cuda.synchronize()
    gl, ge, gs = w.to_host()
    assert np.array_equal(gl, xl) and np.array_equal(ge, xe) and np.array_equal(gs, xs)


@pytest.mark.parametrize("cfg,n,op", [("C5", 4900, "ax"), ("C2", 5000, "ax"), ("C2", 5000, "atx"),
                                      ("C4", 6000, "ax")])
def test_interior_boundary_split_emulated(cfg, n, op):
    """DistCSR's overlap split, emulated for G ranks on one GPU: each rank's
    rows are cut into boundary / interior / boundary row-range handles
    (dist.interior_mask / interior_run); the interior rows run with x valid
    ONLY inside the own block (junk elsewhere - as while the exchange is in
    flight), the boundary rows with x valid inside the needed window.  The
    concatenation must equal the oracle's result."""
    import torch
    from paper_1411_2377_b200 import MPVec
    from paper_1411_2377_b200.dist import block_range, interior_mask, interior_run, needed_window
    d = gen.make(cfg, n=n, seed=21)
    n = d["n"]
    tr = op == "atx"
    want = oracle_full(d, op)
    rng = np.random.default_rng(9)

    def junk_x(valid):
        xl = rng.integers(0, 2 ** 32, size=d["x_limbs"].shape, dtype=np.uint32)
        xe = rng.integers(-2 ** 20, 2 ** 20, size=n).astype(np.int32)
        xs = rng.integers(0, 2, size=n).astype(np.uint8)
        xl[:, -1] |= np.uint32(0x80000000)
        a, b = valid
        xl[a:b], xe[a:b], xs[a:b] = d["x_limbs"][a:b], d["x_exps"][a:b], d["x_signs"][a:b]
        return MPVec.from_host(xl, xe, xs, device="cuda:0")

    for G in (2, 4, 8):
        parts, n_inner = [], 0
        for r in range(G):
            rb, re = block_range(n, G, r)
            a, b = interior_run(interior_mask(d["rowptr"], d["colidx"], rb, re, transpose=tr))
            win = needed_window(d["rowptr"], d["colidx"], rb, re, transpose=tr)
            y = MPVec.empty(re - rb, d["p"] // 32, device="cuda:0")
            x_own, x_win = junk_x((rb, re)), junk_x(win)
            for c0, c1, inner in ((rb, rb + a, False), (rb + a, rb + b, True), (rb + b, re, False)):
                if c1 <= c0:
                    continue
                A = _csr(d, rows=(c0, c1), transpose=tr)
                ys = MPVec(y.limbs[c0 - rb:c1 - rb], y.exps[c0 - rb:c1 - rb], y.signs[c0 - rb:c1 - rb])
                (A.spmv_t if tr else A.spmv)(x_own if inner else x_win, out=ys)
                torch.cuda.synchronize()
                A.close()
                n_inner += (c1 - c0) if inner else 0
            parts.append(y.to_host())
        cat = tuple(np.concatenate([p_[i] for p_ in parts]) for i in range(3))
        assert_same(cat, want, f"{cfg} G={G} {op} interior/boundary")
        if cfg in ("C5", "C2"):
            assert n_inner > n // 2            # banded / stencil blocks are mostly interior


@pytest.mark.parametrize("small", ["1", "0"])
@pytest.mark.parametrize("chunks", ["1", "3", "7"])
@pytest.mark.parametrize("cfg,n,op", [("C5", 4900, "ax"), ("C3", 3000, "ax"), ("C2", 5000, "atx"),
                                      ("C1", 700, "ax"), ("C4", 4000, "atx")])
def test_row_chunks_device_and_host_pipeline(cfg, n, op, chunks, small, monkeypatch):
    """Row-chunked layout (rows length-sorted within C contiguous chunks,
    env MPSP_CHUNKS forcing C on small matrices) and the host-buffer
    pipeline of mpsp_spmv_host (per chunk: H2D of x up to the chunk's window
    end, the chunk's kernels, D2H of its y rows, on three streams; the
    exponent / sign arrays batched (MPSP_E2E_SMALL=1, default) or per chunk)
    - both bit-exact against the oracle, from pinned and pageable host
    buffers."""
    import torch
    monkeypatch.setenv("MPSP_CHUNKS", chunks)
    monkeypatch.setenv("MPSP_E2E_SMALL", small)
    d = gen.make(cfg, n=n, seed=31)
    want = oracle_full(d, op)
    A = _csr(d, transpose=(op == "atx"))
    x = _x(d)
    assert_same((A.spmv if op == "ax" else A.spmv_t)(x).to_host(), want, f"device chunks={chunks}")
    f = A.spmv_host if op == "ax" else A.spmv_t_host
    assert_same(f(d["x_limbs"], d["x_exps"], d["x_signs"]), want, f"host pageable chunks={chunks}")
    L = d["p"] // 32
    hx = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
          for a in (d["x_limbs"].view(np.int32), d["x_exps"], d["x_signs"])]
    hx[0] = hx[0].view(np.uint32)
    hy = (torch.empty((d["n"], L), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
          torch.empty(d["n"], dtype=torch.int32).pin_memory().numpy(),
          torch.empty(d["n"], dtype=torch.uint8).pin_memory().numpy())
    for _ in range(2):
        f(*hx, out=hy)
        assert_same(hy, want, f"host pinned chunks={chunks}")
    A.close()


@pytest.mark.parametrize("cfg,n,op,G", [("C5", 4900, "ax", 2), ("C5", 4900, "ax", 4),
                                        ("C2", 5000, "atx", 3), ("C3", 3000, "ax", 2)])
def test_distcsr_apply_emulated_ranks(cfg, n, op, G, monkeypatch):
    """DistCSR itself for G ranks emulated in one process on one GPU: each
    rank's object (interior / boundary row-range handles, apply() ordering:
    interior kernels launched before finish(), boundary kernels after, output
    slices) is built with the rank / world size patched in and an exchange
    stand-in that fills the needed window at finish() and junk before - so an
    interior kernel that read outside the own block, or a boundary kernel run
    before the exchange, would show.  Concatenated blocks vs the oracle."""
    import torch
    from paper_1411_2377_b200 import MPVec
    from paper_1411_2377_b200 import dist as D
    d = gen.make(cfg, n=n, seed=23)
    n = d["n"]
    tr = op == "atx"
    want = oracle_full(d, op)
    L = d["p"] // 32
    xfull = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")

    class FakeX:
        def __init__(self, n_, L_, window, group=None, device=None, mode="auto", packer=None):
            self.rb, self.re = D.block_range(n_, G, rank[0])
            self.win = window
            self.mode, self.bytes_in = "window", 0
            g = torch.Generator(device="cpu").manual_seed(rank[0])
            junk = torch.randint(-2 ** 31, 2 ** 31 - 1, (n_, L_), generator=g, dtype=torch.int32)
            junk[:, -1] |= -2 ** 31                     # normalised junk
            self.x = MPVec(junk.cuda(), torch.zeros(n_, dtype=torch.int32, device="cuda"),
                           torch.zeros(n_, dtype=torch.uint8, device="cuda"))

        def local_view(self):
            return MPVec(self.x.limbs[self.rb:self.re], self.x.exps[self.rb:self.re],
                         self.x.signs[self.rb:self.re])

        def start(self, stream=None):
            return []

        def finish(self, works, stream=None):
            lo, hi = self.win
            for dst, src in ((self.x.limbs, xfull.limbs), (self.x.exps, xfull.exps),
                             (self.x.signs, xfull.signs)):
                dst[lo:hi].copy_(src[lo:hi])
            return self.x

        def close(self):
            pass

    rank = [0]
    monkeypatch.setattr(D, "XExchange", FakeX)
    monkeypatch.setattr(D.dist, "get_world_size", lambda group=None: G)
    monkeypatch.setattr(D.dist, "get_rank", lambda group=None: rank[0])
    monkeypatch.setattr(D.dist, "get_backend", lambda group=None: "nccl")
    parts, inner = [], 0
    for r in range(G):
        rank[0] = r
        Dc = D.DistCSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
                       transpose=tr, device="cuda:0")
        rb, re = Dc.rows
        xl = MPVec(xfull.limbs[rb:re].clone(), xfull.exps[rb:re].clone(), xfull.signs[rb:re].clone())
        y = Dc.apply(xl, transpose=tr)
        torch.cuda.synchronize()
        parts.append(y.to_host())
        inner += Dc.interior_rows(tr)
        Dc.close()
    cat = tuple(np.concatenate([p_[i] for p_ in parts]) for i in range(3))
    assert_same(cat, want, f"DistCSR {cfg} G={G} {op}")
    if cfg in ("C5", "C2"):
        assert inner > n // 2
