// Host-side fuzz driver of the CSR builder (validation, transpose, row
// binning, row chunks, repack) through mpsp_debug_host_build, for builds with
// AddressSanitizer / UndefinedBehaviorSanitizer (tests/test_host_sanitizers.py;
// SURVEY.md 4 T6).  No GPU: the debug entry point never touches CUDA.
//   host_builder_fuzz [iterations] [seed]
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "mpsp.h"

static uint64_t g_state = 1;
static uint64_t rnd() {                       // SplitMix64
  uint64_t z = (g_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static int64_t rr(int64_t lo, int64_t hi) { return lo + (int64_t)(rnd() % (uint64_t)(hi - lo + 1)); }

struct Csr {
  int p = 0;
  int64_t n = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<uint32_t> limbs;
  std::vector<int32_t> exps;
  std::vector<uint8_t> signs;
};

static Csr random_csr(int p, int64_t n, int64_t maxlen, bool full_rows = true) {
  Csr a;
  a.p = p;
  a.n = n;
  const int L = p / 32;
  a.rowptr.assign((size_t)n + 1, 0);
  std::vector<uint8_t> used((size_t)n, 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t len = rnd() % 5 == 0 ? 0 : rr(0, std::min<int64_t>(maxlen, n));
    if (full_rows && rnd() % 50 == 0) len = n;   // a full row
    std::vector<int32_t> cs;
    if (len == n) {
      for (int64_t j = 0; j < n; ++j) cs.push_back((int32_t)j);
    } else {
      for (int64_t t = 0; t < len; ++t) {
        const int32_t j = (int32_t)rr(0, n - 1);
        if (!used[(size_t)j]) { used[(size_t)j] = 1; cs.push_back(j); }
      }
      for (int32_t j : cs) used[(size_t)j] = 0;
      std::sort(cs.begin(), cs.end());
    }
    for (int32_t j : cs) {
      a.col.push_back(j);
      const int kind = (int)(rnd() % 10);
      for (int l = 0; l < L; ++l) a.limbs.push_back(kind == 0 ? 0u : (uint32_t)rnd());
      if (kind != 0) a.limbs[a.limbs.size() - 1] |= 0x80000000u;
      a.exps.push_back(kind == 0 ? (int32_t)rnd() : (int32_t)rr(-(1 << 29), 1 << 29));  // zero: junk exp
      a.signs.push_back((uint8_t)(rnd() & 1));
    }
    a.rowptr[(size_t)i + 1] = (int64_t)a.col.size();
  }
  return a;
}

static int build(const Csr& a, int64_t rb, int64_t re, uint32_t flags, int64_t out[12]) {
  return mpsp_debug_host_build(a.p, a.n, a.rowptr.data(), a.col.empty() ? nullptr : a.col.data(),
                               a.limbs.empty() ? nullptr : a.limbs.data(),
                               a.exps.empty() ? nullptr : a.exps.data(),
                               a.signs.empty() ? nullptr : a.signs.data(), rb, re, flags, out);
}

#define CHECK(c, ...) do { if (!(c)) { std::fprintf(stderr, __VA_ARGS__); std::fprintf(stderr, "\n"); return 1; } } while (0)

int main(int argc, char** argv) {
  const int iters = argc > 1 ? std::atoi(argv[1]) : 200;
  g_state = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
  const int ps[] = {32, 64, 128, 256, 512, 1024, 2048};
  const int64_t ns[] = {0, 1, 2, 5, 33, 100, 700, 3000};
  int64_t out[12];
  for (int it = 0; it < iters; ++it) {
    const int p = ps[rnd() % 7];
    const int64_t n = ns[rnd() % 8];
    const char* lt[] = {"0", "1", "31", "64", "200"};
    const char* ch[] = {"1", "2", "5"};
    setenv("MPSP_LONG_T", lt[rnd() % 5], 1);
    setenv("MPSP_CHUNKS", ch[rnd() % 3], 1);
    Csr a = random_csr(p, n, rnd() % 3 == 0 ? 40 : 6);
    const int64_t rb = n ? rr(0, n) : 0, re = n ? rr(rb, n) : 0;
    const uint32_t flags = (rnd() & 1) ? MPSP_WITH_TRANSPOSE : 0u;
    int rc = build(a, rb, re, flags, out);
    CHECK(rc == MPSP_OK, "iteration %d: valid input rejected (%d), p=%d n=%lld", it, rc, p, (long long)n);
    CHECK(out[0] == a.rowptr[(size_t)re] - a.rowptr[(size_t)rb], "iteration %d: nnz %lld", it, (long long)out[0]);
    CHECK(out[1] >= out[0] && out[4] >= 1, "iteration %d: stored %lld < nnz", it, (long long)out[1]);
    // the same input twice: identical device arrays
    int64_t out2[12];
    rc = build(a, rb, re, flags, out2);
    CHECK(rc == MPSP_OK && out2[5] == out[5] && out2[11] == out[11], "iteration %d: not deterministic", it);
    // invalid inputs keep their error codes
    if (a.col.size() >= 2 && n >= 2) {
      Csr b = a;
      b.col[0] = (int32_t)n;                  // column out of range
      CHECK(build(b, 0, n, 0, out2) == MPSP_E_CSR, "iteration %d: col range", it);
      b = a;
      int64_t r = -1;
      for (int64_t i = 0; i < n && r < 0; ++i) if (b.rowptr[(size_t)i + 1] - b.rowptr[(size_t)i] >= 2) r = i;
      if (r >= 0) {
        const int64_t k = b.rowptr[(size_t)r];
        b.col[(size_t)k + 1] = b.col[(size_t)k];   // duplicate column
        CHECK(build(b, 0, n, 0, out2) == MPSP_E_UNSORTED, "iteration %d: unsorted", it);
      }
      b = a;
      b.limbs[(size_t)(p / 32) - 1] = 0x00000001u;   // unnormalised nonzero
      CHECK(build(b, 0, n, 0, out2) == MPSP_E_VALUE, "iteration %d: value", it);
      b = a;
      b.limbs[(size_t)(p / 32) - 1] |= 0x80000000u;
      b.exps[0] = (1 << 29) + 1;                     // exponent out of range
      CHECK(build(b, 0, n, 0, out2) == MPSP_E_VALUE, "iteration %d: exp", it);
      b = a;
      b.rowptr[1] = b.rowptr[2] + 1;                 // non-monotone
      CHECK(build(b, 0, n, 0, out2) == MPSP_E_CSR, "iteration %d: rowptr", it);
    }
    CHECK(build(a, 0, n + 1, 0, out2) == MPSP_E_ARG, "iteration %d: range", it);
    CHECK(mpsp_debug_host_build(48, n, a.rowptr.data(), nullptr, nullptr, nullptr, nullptr, 0, 0, 0,
                                out2) == MPSP_E_PREC, "iteration %d: precision", it);
  }
  // a part large enough for the default row chunks (>= 131072 short rows)
  unsetenv("MPSP_CHUNKS");
  unsetenv("MPSP_LONG_T");
  Csr big = random_csr(256, 140000, 6, false);
  int rc = build(big, 0, big.n, MPSP_WITH_TRANSPOSE, out);
  CHECK(rc == MPSP_OK && out[4] == 2 && out[10] == 2, "large part: rc %d chunks %lld/%lld", rc,
        (long long)out[4], (long long)out[10]);
  std::printf("host builder fuzz ok: %d iterations\n", iters);
  return 0;
}
