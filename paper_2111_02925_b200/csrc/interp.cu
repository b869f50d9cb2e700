// libsz3g -- SZ3-Interp (NEXT-4): the multilevel interpolation predictor of PAPER.md P:852-853 ("Both
// linear interpolation and cubic spline interpolation are included", "constant coefficients"), with
// linear-scaling quantisation and reconstruction.  Definition: oracle/DEFINITION.md
// I1-I6; readings G30-G33.
//
// The method is level-serial: a pass (s, d) predicts its targets from donors that earlier passes have
// already RECONSTRUCTED, so passes run in plan order, one launch each, while the targets of one pass are
// independent of one another (their donors are even multiples of s along d) and run fully in parallel:
//   k_interp_anchor   the anchor (0,0,0) stored as an outlier; eb_abs / status; x'[0] = x[0]
//   k_interp_rows<T, DEC, KIND>  the default: level s by rows of its sub-grid (three launches per level,
//                     one warp per row; see the comment above the kernel)
//   k_interp_pass<T, DEC>  (-DSZ3G_IP_ROWS=0) one thread per target of pass (s, d): donors from x' at -3s, -s,
//                     +s, +3s along d, cubic / linear / copy (I3), then O8-O10 (compress: code, x', outlier
//                     append warp-aggregated) or the recovery (decompress: x' for code != 0)
//   k_interp_scatter  decompress: outlier values into x' before the passes
//   k_interp_final    outlier-capacity status
// The histogram (O11) is the standalone sz3g_histogram over the finished codes.  Arithmetic is the
// definition's, op for op (fp64, explicit __d*_rn, no contraction): bit-exact against the oracle.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>

#include "../../include/sz3g.h"
#include "ptx.cuh"
#include "tile.cuh"

using namespace sz3g;

namespace {

std::atomic<uint64_t> g_ip_launches{0};

struct IpArgs {
  uint64_t n[3];          // extents
  uint64_t st[3];         // element strides (n1 n2, n2, 1)
  uint64_t first[3], step[3], cnt[3];   // the pass's targets along each axis
  uint64_t s;             // stride of the level
  int d;                  // axis of the pass
  uint32_t R;
  int eb_mode;
  double eb;
  const double* d_minmax;
  double* d_eb_abs;
  int32_t* d_status;
  uint64_t gofs;          // dim0_offset * n1 * n2
  uint64_t cap;
};

__device__ __forceinline__ bool ip_consts(const IpArgs& a, Consts& K) {
  return make_consts(a.eb_mode, a.eb, a.d_minmax, 0.0, K);
}

// I3, op for op: u = b + c, v = a + e, p = (9 u - v) * 0.0625 | (b + c) * 0.5 | b
__device__ __forceinline__ double ip_predict(double a, double b, double c, double e, int m) {
  if (m == 2) return __dmul_rn(__dsub_rn(__dmul_rn(9.0, __dadd_rn(b, c)), __dadd_rn(a, e)), 0.0625);
  if (m == 1) return __dmul_rn(__dadd_rn(b, c), 0.5);
  return b;
}

template <typename T>
__global__ void k_interp_anchor(const T* __restrict__ x, T* __restrict__ xp, uint16_t* __restrict__ codes,
                                uint64_t* __restrict__ oidx, T* __restrict__ oval,
                                unsigned long long* __restrict__ ocount, IpArgs a) {
  Consts K;
  const bool ok = ip_consts(a, K);
  if (!ok && a.d_status) atomicOr(a.d_status, (int)SZ3G_STATUS_BAD_RANGE);
  if (a.d_eb_abs) *a.d_eb_abs = ok ? K.eb_abs : __longlong_as_double(0x7ff8000000000000ll);
  codes[0] = 0;
  xp[0] = x[0];
  const unsigned long long pos = atomicAdd(ocount, 1ull);
  if (pos < a.cap) {
    oidx[pos] = a.gofs;
    oval[pos] = x[0];
  }
}

template <typename T, bool DEC>
__global__ void __launch_bounds__(256) k_interp_pass(const T* __restrict__ x, T* __restrict__ xp,
                                                     uint16_t* __restrict__ codes, uint64_t* __restrict__ oidx,
                                                     T* __restrict__ oval, unsigned long long* __restrict__ ocount,
                                                     IpArgs a) {
  __shared__ Consts s_k;
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    Consts K;
    s_ok = ip_consts(a, K);
    s_k = K;
  }
  SZ3G_SYNCTHREADS();
  if (!s_ok) return;
  const Consts K = s_k;
  const uint64_t sd = a.s * a.st[a.d];
  const uint64_t nd = a.n[a.d];
  const uint64_t t2 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  for (uint64_t t0 = blockIdx.z; t0 < a.cnt[0]; t0 += gridDim.z)
    for (uint64_t t1 = blockIdx.y; t1 < a.cnt[1]; t1 += gridDim.y) {
      const bool live = t2 < a.cnt[2];
      const uint64_t i0 = a.first[0] + t0 * a.step[0], i1 = a.first[1] + t1 * a.step[1];
      const uint64_t i2 = a.first[2] + (live ? t2 : 0) * a.step[2];
      const uint64_t e = i0 * a.st[0] + i1 * a.st[1] + i2 * a.st[2];
      const uint64_t id = a.d == 0 ? i0 : (a.d == 1 ? i1 : i2);
      const int m = (id >= 3 * a.s && id + 3 * a.s < nd) ? 2 : (id + a.s < nd ? 1 : 0);
      bool is_out = false;
      if (live) {
        const uint16_t cin = DEC ? codes[e] : (uint16_t)1;
        if (cin != 0) {
          const double b = to_d<T>(xp[e - sd]);
          const double c = m >= 1 ? to_d<T>(xp[e + sd]) : 0.0;
          const double av = m == 2 ? to_d<T>(xp[e - 3 * sd]) : 0.0;
          const double ev = m == 2 ? to_d<T>(xp[e + 3 * sd]) : 0.0;
          const double p = ip_predict(av, b, c, ev, m);
          if (DEC) {
            // I6: x' = (T)(p + twoeb (code - R)), the product rounded first (no contraction)
            const double q = (double)((int)cin - (int)a.R);
            xp[e] = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, q)));
          } else {
            // I5 = O8-O10 (the exact definition; magic rint valid for |t| < 2^51, larger |t| or NaN fail
            // the radius test exactly as in O8)
            const T xv = x[e];
            const double xd = to_d<T>(xv);
            const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
            const double sm = __dadd_rn(t, RINT_MAGIC);
            const double q = __dsub_rn(sm, RINT_MAGIC);
            const T y = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, q)));
            const bool ok = fabs(t) < (double)a.R && fabs(q) < (double)a.R &&
                            fabs(__dsub_rn(to_d<T>(y), xd)) <= K.eb_abs;
            codes[e] = ok ? (uint16_t)(__double2loint(sm) + (int)a.R) : (uint16_t)0;
            xp[e] = ok ? y : xv;
            is_out = !ok;
          }
        }
      }
      if (!DEC) {   // warp-aggregated outlier append (warp-uniform loop trip: t0, t1 shared by the block)
        const uint32_t bal = __ballot_sync(0xffffffffu, is_out);
        if (bal) {
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(ocount, (unsigned long long)__popc(bal));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (is_out) {
            const unsigned long long pos = base + __popc(bal & ((1u << lane) - 1u));
            if (pos < a.cap) {
              oidx[pos] = a.gofs + e;
              oval[pos] = x[e];
            }
          }
        }
      }
    }
}

// ------------------------------------------------------------------------------------------------
// Level s = 1 passes, one thread per PAIR of columns (k even, k + 1) of a row holding targets: the pass's
// target in the pair is predicted and quantised (or recovered) exactly as in k_interp_pass, and the pair
// is written back whole -- the other element's x' (and code) rewritten unchanged -- so every store covers
// full sectors instead of every other element (the stride-2 stores of the per-target kernel doubled the
// DRAM traffic through partial-sector read-modify-writes).  Pass axis d: 2 -> rows (i, j) all, target
// k + 1; 1 -> rows (i, j odd), target k; 0 -> rows (i odd, j even), target k.
template <typename T, bool DEC, int D>
__global__ void __launch_bounds__(256) k_interp_pairs(const T* __restrict__ x, T* __restrict__ xp,
                                                      uint16_t* __restrict__ codes, uint64_t* __restrict__ oidx,
                                                      T* __restrict__ oval, unsigned long long* __restrict__ ocount,
                                                      IpArgs a) {
  __shared__ Consts s_k;
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    Consts K;
    s_ok = ip_consts(a, K);
    s_k = K;
  }
  SZ3G_SYNCTHREADS();
  if (!s_ok) return;
  const Consts K = s_k;
  const uint64_t n0 = a.n[0], n1 = a.n[1], n2 = a.n[2];
  const uint64_t np = (n2 + 1) / 2;                       // pairs per row
  const uint64_t m = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  // rows of the pass: D = 2: every (i, j); D = 1: (i, j odd); D = 0: (i odd, j even)
  const uint64_t ni = D == 0 ? n0 / 2 : n0, nj = D == 2 ? n1 : (n1 / 2 + (D == 0 ? n1 % 2 : 0));
  for (uint64_t rr = blockIdx.y; rr < ni * nj; rr += gridDim.y) {
    const uint64_t ti = rr / nj, tj = rr - ti * nj;
    const uint64_t i = D == 0 ? 2 * ti + 1 : ti;
    const uint64_t j = D == 2 ? tj : (D == 1 ? 2 * tj + 1 : 2 * tj);
    const bool live = m < np;
    const uint64_t k0 = 2 * (live ? m : 0);
    const uint64_t kt = D == 2 ? k0 + 1 : k0;             // the target column
    const bool has_t = live && kt < n2;
    const bool has_pair = live && k0 + 1 < n2;
    const uint64_t re = (i * n1 + j) * n2;
    const uint64_t e = re + kt;
    bool is_out = false;
    T xnew = T(0), xold = T(0);
    uint16_t cnew = 0;
    if (has_t) {
      const uint64_t eo = re + (D == 2 ? k0 : k0 + 1);   // the pair's other element (no target of this pass)
      const uint64_t id = D == 0 ? i : (D == 1 ? j : kt);
      const uint64_t nd = D == 0 ? n0 : (D == 1 ? n1 : n2);
      const uint64_t sd = D == 0 ? n1 * n2 : (D == 1 ? n2 : 1);
      const int mth = (id >= 3 && id + 3 < nd) ? 2 : (id + 1 < nd ? 1 : 0);
      const double b = to_d<T>(xp[e - sd]);
      const double c = mth >= 1 ? to_d<T>(xp[e + sd]) : 0.0;
      const double av = mth == 2 ? to_d<T>(xp[e - 3 * sd]) : 0.0;
      const double ev = mth == 2 ? to_d<T>(xp[e + 3 * sd]) : 0.0;
      const double p = ip_predict(av, b, c, ev, mth);
      if (has_pair) xold = xp[eo];
      if (DEC) {
        const uint16_t cin = codes[e];
        xnew = cin != 0 ? from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, (double)((int)cin - (int)a.R)))) : xp[e];
      } else {
        const T xv = x[e];
        const double xd = to_d<T>(xv);
        const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
        const double sm = __dadd_rn(t, RINT_MAGIC);
        const double q = __dsub_rn(sm, RINT_MAGIC);
        const T y = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, q)));
        const bool ok = fabs(t) < (double)a.R && fabs(q) < (double)a.R && fabs(__dsub_rn(to_d<T>(y), xd)) <= K.eb_abs;
        cnew = ok ? (uint16_t)(__double2loint(sm) + (int)a.R) : (uint16_t)0;
        xnew = ok ? y : xv;
        is_out = !ok;
      }
    }
    // the whole pair back (the even column first): both values of a pair are this thread's
    if (has_t) {
      if (has_pair) {
        const T lo = D == 2 ? xold : xnew, hi = D == 2 ? xnew : xold;
        xp[re + k0] = lo;
        xp[re + k0 + 1] = hi;
        if (!DEC) codes[e] = cnew;
      } else {
        xp[e] = xnew;
        if (!DEC) codes[e] = cnew;
      }
    }
    if (!DEC) {
      const uint32_t bal = __ballot_sync(0xffffffffu, is_out);
      if (bal) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ocount, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (is_out) {
          const unsigned long long pos = base + __popc(bal & ((1u << lane) - 1u));
          if (pos < a.cap) {
            oidx[pos] = a.gofs + e;
            oval[pos] = x[e];
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Level s by rows of its sub-grid (the multiples of s; coordinates ic, jc, kc).  Pass (s,2) stays inside a
// row (i, j), passes (s,0) and (s,1) touch only even columns: a row with jc odd (KIND 1) holds the (s,1)
// targets at its even columns (donors: the rows jc -+ 1, -+ 3, final once KIND 2 has run) and the (s,2)
// targets at its odd columns (donors: the row's own even columns, just computed); a row with ic odd and
// jc even (KIND 2) the (s,0) targets at its even columns (donors: planes ic -+ 1, -+ 3, coarser levels)
// and (s,2); a row with ic, jc even (KIND 0) only (s,2).  Launched KIND 2, 0, 1: the plan order (s,0),
// (s,1), (s,2) up to targets that do not depend on one another.  One warp per row, lane l on the column
// pair (kc0 + 2l, kc0 + 2l + 1) of a 64-column segment; the (s,2) donors of a segment reach two even
// columns into the next segment, so the even columns are computed (or loaded) one segment ahead, and
// every load is issued one segment before its use.  At s = 1 every row leaves whole -- x' and codes as
// pairs, the even column's value and code rewritten unchanged on KIND 0 rows -- so no store is a
// partial sector; the three kinds run as separate launches, so no launch reads a sector another warp of
// it stores.  The prediction and quantisation are k_interp_pass's, op for op: bit-identical to the
// per-pass schedule.
#ifndef SZ3G_IP_ROWS
#define SZ3G_IP_ROWS 2   // 1: level 1 by rows, coarser levels by k_interp_pass; 2: every level by rows
#endif
constexpr int IR_WARPS = 8;
#ifndef SZ3G_IR_MINB
#define SZ3G_IR_MINB 4   // __launch_bounds__ minimum blocks per SM of the row kernels (c5 A/B, compress /
                         // decompress ms: 1 -> 37.6 / 25.8, 4 -> 30.6 / 22.4, 6 -> 32.9 / 24.3, 8 -> 41.9 / 24.5)
#endif

// O8-O10 of one target (k_interp_pass): code (0 = outlier) and x' (x for an outlier)
template <typename T>
__device__ __forceinline__ bool ip_quant(T xv, double p, const Consts& K, uint32_t R, uint16_t& code, T& y) {
  const double xd = to_d<T>(xv);
  const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
  const double sm = __dadd_rn(t, RINT_MAGIC);
  const double q = __dsub_rn(sm, RINT_MAGIC);
  const T yy = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, q)));
  const bool ok = fabs(t) < (double)R && fabs(q) < (double)R && fabs(__dsub_rn(to_d<T>(yy), xd)) <= K.eb_abs;
  code = ok ? (uint16_t)(__double2loint(sm) + (int)R) : (uint16_t)0;
  y = ok ? yy : xv;
  return ok;
}

template <typename T>
__device__ __forceinline__ void ip_append(bool is_out, uint64_t e, T xv, unsigned long long* ocount, uint64_t* oidx,
                                          T* oval, const IpArgs& a, int lane) {
  const uint32_t bal = __ballot_sync(0xffffffffu, is_out);
  if (bal) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(ocount, (unsigned long long)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (is_out) {
      const unsigned long long pos = base + __popc(bal & ((1u << lane) - 1u));
      if (pos < a.cap) {
        oidx[pos] = a.gofs + e;
        oval[pos] = xv;
      }
    }
  }
}

template <typename T, bool DEC, int KIND>
__global__ void __launch_bounds__(IR_WARPS * 32, SZ3G_IR_MINB) k_interp_rows(const T* __restrict__ x, T* __restrict__ xp,
                                                               uint16_t* __restrict__ codes,
                                                               uint64_t* __restrict__ oidx, T* __restrict__ oval,
                                                               unsigned long long* __restrict__ ocount, IpArgs a) {
  __shared__ Consts s_k;
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    Consts K;
    s_ok = ip_consts(a, K);
    s_k = K;
  }
  SZ3G_SYNCTHREADS();
  if (!s_ok) return;
  const Consts K = s_k;
  const uint64_t n0 = a.n[0], n1 = a.n[1], n2 = a.n[2], S = a.s;
  // the level's sub-grid (the multiples of s): coordinates ic, jc, kc; extents m0, m1, m2
  const uint64_t m0 = (n0 - 1) / S + 1, m1 = (n1 - 1) / S + 1, m2 = (n2 - 1) / S + 1;
  const int lane = threadIdx.x & 31;
  // rows of this launch: KIND 1 (ic, jc odd); KIND 2 (ic odd, jc even); KIND 0 (ic even, jc even)
  const uint64_t nj = KIND == 1 ? m1 / 2 : (m1 + 1) / 2;
  const uint64_t ni = KIND == 1 ? m0 : (KIND == 2 ? m0 / 2 : (m0 + 1) / 2);
  const uint64_t nrows = ni * nj;
  const uint64_t nseg = (m2 + 63) / 64;
  const bool p12 = m2 > 1;                            // pass (s,2) has targets
  const bool base_al = (reinterpret_cast<uintptr_t>(xp) % (2 * sizeof(T))) == 0 &&
                       (reinterpret_cast<uintptr_t>(codes) % 4) == 0;
  // the loads of one segment (issued one segment before their use): the even column's inputs -- its
  // (1,1) donors and x (odd rows), or its final x' and code (even rows) -- and the odd column's x (compress)
  // or code (decompress)
  struct Ld {
    T b, c, av, ev, xe, xo;
    uint16_t ce, co;
  };
  for (uint64_t r = (uint64_t)blockIdx.x * IR_WARPS + (threadIdx.x >> 5); r < nrows;
       r += (uint64_t)gridDim.x * IR_WARPS) {
    const uint64_t ti = r / nj;
    const uint64_t ic = KIND == 1 ? ti : 2 * ti + (KIND == 2 ? 1 : 0), jc = 2 * (r - ti * nj) + (KIND == 1 ? 1 : 0);
    const uint64_t re = (ic * S * n1 + jc * S) * n2;
    const bool vec = S == 1 && (re & 1) == 0 && base_al;   // pairs 2 sizeof(T)-byte / 4-byte (codes) aligned
    // the even column's pass: (s,1) along j (KIND 1) or (s,0) along i (KIND 2), cubic / linear / copy
    // (the I3 conditions i_d >= 3s, i_d + 3s < n_d, i_d + s < n_d on the sub-grid: c >= 3, c + 3 < m, c + 1 < m)
    constexpr bool COMP = KIND != 0;
    const uint64_t sd = S * (KIND == 1 ? n2 : n1 * n2), id = KIND == 1 ? jc : ic, nd = KIND == 1 ? m1 : m0;
    const int mj = (id >= 3 && id + 3 < nd) ? 2 : (id + 1 < nd ? 1 : 0);
    // row pointers and 32-bit column offsets (the host keeps n2 < 2^31): the segment loop's address
    // arithmetic was half of its instructions with 64-bit element indices
    const uint32_t m2u = (uint32_t)m2, S32 = (uint32_t)S;
    const T* xr = DEC ? nullptr : x + re;
    T* pr = xp + re;
    uint16_t* cr = codes + re;
    const T* pm1 = COMP ? pr - sd : pr;
    const T* pp1 = COMP ? pr + sd : pr;
    const T* pm3 = COMP ? pr - 3 * sd : pr;
    const T* pp3 = COMP ? pr + 3 * sd : pr;
    auto load = [&](uint32_t sg) {
      Ld L;
      L.b = L.c = L.av = L.ev = L.xe = L.xo = T(0);
      L.ce = L.co = 0;
      const uint32_t kc = 64u * sg + 2u * lane;
      if (kc >= m2u) return L;
      const uint32_t off = kc * S32;
      if (COMP) {
        L.b = pm1[off];
        if (mj >= 1) L.c = pp1[off];
        if (mj == 2) {
          L.av = pm3[off];
          L.ev = pp3[off];
        }
        if (DEC) L.ce = cr[off];
        else L.xe = xr[off];
      } else {
        L.xe = pr[off];
        if (!DEC) L.ce = cr[off];
      }
      if (p12 && kc + 1 < m2u) {
        if (DEC) L.co = cr[off + S32];
        else L.xo = xr[off + S32];
      }
      return L;
    };
    // the even column's x' and code from its loads (KIND 1 / 2: passes (s,1) / (s,0); KIND 0: as loaded)
    auto even_col = [&](uint32_t sg, const Ld& L, T& xe, uint16_t& ce, bool& out) {
      const uint32_t kc = 64u * sg + 2u * lane;
      out = false;
      xe = L.xe;
      ce = L.ce;
      if (!COMP || kc >= m2u) return;
      const double p = ip_predict(to_d<T>(L.av), to_d<T>(L.b), to_d<T>(L.c), to_d<T>(L.ev), mj);
      if (DEC) {
        xe = L.ce != 0 ? from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, (double)((int)L.ce - (int)a.R)))) : pr[kc * S32];
      } else {
        out = !ip_quant<T>(L.xe, p, K, a.R, ce, xe);
      }
    };
    Ld l_cur = load(0), l_nxt = load(1);
    T xe_cur, xe_nxt, xe_prev = T(0);
    uint16_t ce_cur, ce_nxt;
    bool out_cur, out_nxt;
    even_col(0, l_cur, xe_cur, ce_cur, out_cur);
    const uint32_t nseg32 = (uint32_t)nseg;
    for (uint32_t sg = 0; sg < nseg32; sg++) {
      const Ld l_nn = load(sg + 2);
      even_col(sg + 1, l_nxt, xe_nxt, ce_nxt, out_nxt);
      const uint32_t kc = 64u * sg + 2u * lane, ke = kc * S32, ko = ke + S32;
      // (s,2) donors of ko: ke - 2s, ke, ke + 2s, ke + 4s (lanes l - 1, l, l + 1, l + 2 or the next
      // segment); every lane takes part in every shuffle
      const T dn1 = __shfl_up_sync(0xffffffffu, xe_cur, 1);
      const T up1 = __shfl_down_sync(0xffffffffu, xe_cur, 1), nx0 = __shfl_sync(0xffffffffu, xe_nxt, 0);
      const T up2 = __shfl_down_sync(0xffffffffu, xe_cur, 2), nx1 = __shfl_sync(0xffffffffu, xe_nxt, 1);
      const T dm2 = lane == 0 ? xe_prev : dn1;
      const T dp2 = lane == 31 ? nx0 : up1;
      const T dp4 = lane == 31 ? nx1 : (lane == 30 ? nx0 : up2);
      xe_prev = __shfl_sync(0xffffffffu, xe_cur, 31);
      T xo = T(0);
      uint16_t co = 0;
      bool out_o = false;
      const bool has_o = p12 && kc + 1 < m2u;
      if (has_o) {
        const int mk = (kc + 1 >= 3 && kc + 4 < m2u) ? 2 : (kc + 2 < m2u ? 1 : 0);
        const double p = ip_predict(to_d<T>(dm2), to_d<T>(xe_cur), to_d<T>(dp2), to_d<T>(dp4), mk);
        if (DEC) {
          xo = l_cur.co != 0 ? from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, (double)((int)l_cur.co - (int)a.R))))
                             : pr[ko];
        } else {
          out_o = !ip_quant<T>(l_cur.xo, p, K, a.R, co, xo);
        }
      }
      // the row's pair back, whole
      if (kc < m2u) {
        if (has_o && vec) {
          if (sizeof(T) == 4) {
            float2 v;
            v.x = (float)xe_cur;
            v.y = (float)xo;
            *reinterpret_cast<float2*>(pr + ke) = v;
          } else {
            double2 v;
            v.x = (double)xe_cur;
            v.y = (double)xo;
            *reinterpret_cast<double2*>(pr + ke) = v;
          }
          if (!DEC) *reinterpret_cast<uint32_t*>(cr + ke) = (uint32_t)ce_cur | ((uint32_t)co << 16);
        } else {
          if (COMP || S == 1) {   // KIND 0 at s > 1: the even column is unchanged and no sector is whole anyway
            pr[ke] = xe_cur;
            if (!DEC) cr[ke] = ce_cur;
          }
          if (has_o) {
            pr[ko] = xo;
            if (!DEC) cr[ko] = co;
          }
        }
      }
      if (!DEC) {
        if (COMP) ip_append<T>(out_cur, re + ke, l_cur.xe, ocount, oidx, oval, a, lane);
        ip_append<T>(out_o, re + ko, l_cur.xo, ocount, oidx, oval, a, lane);
      }
      l_cur = l_nxt;
      l_nxt = l_nn;
      xe_cur = xe_nxt;
      ce_cur = ce_nxt;
      out_cur = out_nxt;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Level s = 1 fused (its three passes hold 7/8 of the targets): one CTA per tile of 2 planes (i0 even,
// i0 + 1) x L1_TJ rows x L1_TK columns, in shared memory with a halo of 2 even coordinates along j and k
// (the -+1, -+3 donors).  Pass (1,0) targets (i odd, j and k even) are computed over the whole halo box
// (redundantly with the neighbour tiles: the same inputs, the same IEEE operations, the same x'),
// pass (1,1) targets (j odd, k even) over the tile's rows and the box's columns, pass (1,2) targets
// (k odd) over the tile; the (1,0) donors (level >= 2 points of planes i0 - 2 .. i0 + 4) come from x'
// in global memory, every other donor from the box.  Work is split as one warp per row, lanes along k,
// so a row's global loads and stores are contiguous.  The tile's x' and codes leave as full rows (the
// level >= 2 points' values and codes rewritten unchanged), so no write is a partial sector.  Same
// prediction and quantisation as k_interp_pass, op for op: bit-identical to the per-pass schedule.
constexpr int L1_TJ = 16, L1_TK = 128, L1_BJ = L1_TJ + 6, L1_BK = L1_TK + 6, L1_WARPS = 16;

// box buffers: x' as fp64 (every donor is read up to four times: one conversion when it is written instead
// of one per read), x as T, codes
template <typename T>
struct L1Smem {
  static constexpr size_t box = 2ull * L1_BJ * L1_BK;
  static constexpr size_t off_x = box * sizeof(double);
  static constexpr size_t off_c = off_x + box * sizeof(T);
  static constexpr size_t total = off_c + box * sizeof(uint16_t);
};

template <typename T, bool DEC>
__global__ void __launch_bounds__(L1_WARPS * 32) k_interp_l1(const T* __restrict__ x, T* __restrict__ xp,
                                                             uint16_t* __restrict__ codes, uint64_t* __restrict__ oidx,
                                                             T* __restrict__ oval, unsigned long long* __restrict__ ocount,
                                                             IpArgs a) {
  extern __shared__ __align__(16) uint8_t l1sm[];
  double* sE = reinterpret_cast<double*>(l1sm);                         // x' of the box [2][BJ][BK], fp64
  T* sX = reinterpret_cast<T*>(l1sm + L1Smem<T>::off_x);               // x of the box (compress)
  uint16_t* sC = reinterpret_cast<uint16_t*>(l1sm + L1Smem<T>::off_c);  // codes of the box
  __shared__ Consts s_k;
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    Consts K;
    s_ok = ip_consts(a, K);
    s_k = K;
  }
  const int n0 = (int)a.n[0], n1 = (int)a.n[1], n2 = (int)a.n[2];
  const int I0 = 2 * (int)blockIdx.z, J0 = L1_TJ * (int)blockIdx.y, K0 = L1_TK * (int)blockIdx.x;
  const int jb = J0 - 2, kb = K0 - 2;   // box origin (even)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int klo = kb < 0 ? -kb : 0, khi = min(L1_BK, n2 - kb);   // valid box columns [klo, khi)
  // (1) the box, one warp per row (row base pointers, 32-bit column offsets)
  for (int r = warp; r < 2 * L1_BJ; r += L1_WARPS) {
    const int bi = r / L1_BJ, bj = r - bi * L1_BJ, i = I0 + bi, j = jb + bj;
    if (i >= n0 || j < 0 || j >= n1) continue;
    const uint64_t re = ((uint64_t)i * (uint64_t)n1 + (uint64_t)j) * (uint64_t)n2 + (uint64_t)(int64_t)kb;
    const int ro = r * L1_BK;
    if (DEC) {
      const uint16_t* cr = codes + re;
      for (int bk = klo + lane; bk < khi; bk += 32) {
        const uint16_t c = cr[bk];
        sC[ro + bk] = c;
        if (c == 0) sE[ro + bk] = to_d<T>(xp[re + bk]);   // an outlier's scattered value
      }
    } else {
      const T* xr = x + re;
      for (int bk = klo + lane; bk < khi; bk += 32) sX[ro + bk] = xr[bk];
    }
    if (((i | j) & 1) == 0) {   // level >= 2 points (all coordinates even): final x' and codes
      const int k0 = klo + (klo & 1);
      for (int bk = k0 + 2 * lane; bk < khi; bk += 64) {
        sE[ro + bk] = to_d<T>(xp[re + bk]);
        if (!DEC) sC[ro + bk] = codes[re + bk];
      }
    }
  }
  SZ3G_SYNCTHREADS();
  if (!s_ok) return;
  const Consts K = s_k;
  const double Rd = (double)a.R;
  // one target at box offset o: quantise (compress) or recover (decompress); returns "own outlier"
  auto target = [&](int o, double p, bool own) -> bool {
    if (DEC) {
      const uint16_t c = sC[o];
      if (c != 0) sE[o] = to_d<T>(from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, (double)((int)c - (int)a.R)))));
      return false;
    }
    const T xv = sX[o];
    const double xd = to_d<T>(xv);
    const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
    const double sm = __dadd_rn(t, RINT_MAGIC);
    const double qd = __dsub_rn(sm, RINT_MAGIC);
    const double yd = to_d<T>(from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, qd))));
    const bool ok = fabs(t) < Rd && fabs(qd) < Rd && fabs(__dsub_rn(yd, xd)) <= K.eb_abs;
    sE[o] = ok ? yd : xd;
    if (own) sC[o] = ok ? (uint16_t)(__double2loint(sm) + (int)a.R) : (uint16_t)0;
    return own && !ok;
  };
  auto append = [&](bool is_out, uint64_t e, int o) {   // warp-aggregated outlier append (all lanes call)
    if (DEC) return;
    const uint32_t bal = __ballot_sync(0xffffffffu, is_out);
    if (!bal) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(ocount, (unsigned long long)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (is_out) {
      const unsigned long long pos = base + __popc(bal & ((1u << lane) - 1u));
      if (pos < a.cap) {
        oidx[pos] = a.gofs + e;
        oval[pos] = sX[o];
      }
    }
  };
  const uint64_t p1 = (uint64_t)n1 * n2;
  constexpr int NKE = L1_BK / 2;   // even box columns: 0, 2, .., L1_BK - 2
  // (2) pass (1,0): plane I0 + 1, even rows and columns of the box; donors at i -+ 1 (plane I0 in the box,
  // plane I0 + 2 in global x'), i -+ 3 (global)
  if (I0 + 1 < n0) {
    const int i = I0 + 1;
    const int m = (i >= 3 && i + 3 < n0) ? 2 : (i + 1 < n0 ? 1 : 0);
    for (int r = warp; r < L1_BJ / 2; r += L1_WARPS) {
      const int bj = 2 * r, j = jb + bj;
      const bool rowok = j >= 0 && j < n1;
      const uint64_t re = rowok ? ((uint64_t)i * (uint64_t)n1 + (uint64_t)j) * (uint64_t)n2 + (uint64_t)(int64_t)kb : 0;
      const int ro = (L1_BJ + bj) * L1_BK, ro0 = bj * L1_BK;
      const bool ownrow = j >= J0 && j < J0 + L1_TJ;
      for (int h0 = 0; h0 < NKE; h0 += 32) {
        const int bk = 2 * (h0 + lane);
        const bool live = rowok && h0 + lane < NKE && bk >= klo && bk < khi;
        bool out = false;
        uint64_t e = 0;
        if (live) {
          e = re + (uint64_t)bk;
          const double bv = sE[ro0 + bk];
          const double cv = m >= 1 ? to_d<T>(xp[e + p1]) : 0.0;
          const double av = m == 2 ? to_d<T>(xp[e - 3 * p1]) : 0.0;
          const double ev = m == 2 ? to_d<T>(xp[e + 3 * p1]) : 0.0;
          out = target(ro + bk, ip_predict(av, bv, cv, ev, m), ownrow && bk >= 2 && bk < 2 + L1_TK);
        }
        append(out, e, ro + bk);
      }
    }
  }
  SZ3G_SYNCTHREADS();
  // (3) pass (1,1): both planes, odd rows of the tile, even columns of the box; donors in the box
  for (int r = warp; r < L1_TJ; r += L1_WARPS) {   // L1_TJ / 2 odd rows x 2 planes
    const int bi = r / (L1_TJ / 2), bj = 3 + 2 * (r % (L1_TJ / 2)), i = I0 + bi, j = jb + bj;
    const bool rowok = i < n0 && j < n1;
    const uint64_t re = rowok ? ((uint64_t)i * (uint64_t)n1 + (uint64_t)j) * (uint64_t)n2 + (uint64_t)(int64_t)kb : 0;
    const int m = (j >= 3 && j + 3 < n1) ? 2 : (j + 1 < n1 ? 1 : 0);
    const int ro = (bi * L1_BJ + bj) * L1_BK;
    for (int h0 = 0; h0 < NKE; h0 += 32) {
      const int bk = 2 * (h0 + lane);
      const bool live = rowok && h0 + lane < NKE && bk >= klo && bk < khi;
      bool out = false;
      uint64_t e = 0;
      const int o = ro + bk;
      if (live) {
        e = re + (uint64_t)bk;
        const double bv = sE[o - L1_BK];
        const double cv = m >= 1 ? sE[o + L1_BK] : 0.0;
        const double av = m == 2 ? sE[o - 3 * L1_BK] : 0.0;
        const double ev = m == 2 ? sE[o + 3 * L1_BK] : 0.0;
        out = target(o, ip_predict(av, bv, cv, ev, m), bk >= 2 && bk < 2 + L1_TK);
      }
      append(out, e, o);
    }
  }
  SZ3G_SYNCTHREADS();
  // (4) pass (1,2): the tile's rows, odd columns; donors in the box
  for (int r = warp; r < 2 * L1_TJ; r += L1_WARPS) {
    const int bi = r / L1_TJ, bj = 2 + r % L1_TJ, i = I0 + bi, j = jb + bj;
    const bool rowok = i < n0 && j < n1;
    const uint64_t re = rowok ? ((uint64_t)i * (uint64_t)n1 + (uint64_t)j) * (uint64_t)n2 + (uint64_t)(int64_t)kb : 0;
    const int ro = (bi * L1_BJ + bj) * L1_BK;
    for (int h0 = 0; h0 < L1_TK / 2; h0 += 32) {
      const int bk = 3 + 2 * (h0 + lane), k = kb + bk;
      const bool live = rowok && k < n2;
      bool out = false;
      uint64_t e = 0;
      const int o = ro + bk;
      if (live) {
        e = re + (uint64_t)bk;
        const int m = (k >= 3 && k + 3 < n2) ? 2 : (k + 1 < n2 ? 1 : 0);
        const double bv = sE[o - 1];
        const double cv = m >= 1 ? sE[o + 1] : 0.0;
        const double av = m == 2 ? sE[o - 3] : 0.0;
        const double ev = m == 2 ? sE[o + 3] : 0.0;
        out = target(o, ip_predict(av, bv, cv, ev, m), true);
      }
      append(out, e, o);
    }
  }
  SZ3G_SYNCTHREADS();
  // (5) the tile's rows out: x' (and the codes, compressing), level >= 2 points rewritten unchanged
  for (int r = warp; r < 2 * L1_TJ; r += L1_WARPS) {
    const int bi = r / L1_TJ, tj = r % L1_TJ, i = I0 + bi, j = J0 + tj;
    if (i >= n0 || j >= n1) continue;
    const uint64_t re = ((uint64_t)i * (uint64_t)n1 + (uint64_t)j) * (uint64_t)n2 + (uint64_t)K0;
    const int ro = (bi * L1_BJ + tj + 2) * L1_BK + 2;
    const int kend = min(L1_TK, n2 - K0);
    T* xr = xp + re;
    uint16_t* cr = codes + re;
    for (int tk = lane; tk < kend; tk += 32) {
      xr[tk] = from_d<T>(sE[ro + tk]);
      if (!DEC) cr[tk] = sC[ro + tk];
    }
  }
}

template <typename T>
__global__ void k_interp_scatter(const uint64_t* __restrict__ idx, const T* __restrict__ val, uint64_t n,
                                 const unsigned long long* __restrict__ d_n, uint64_t base, uint64_t N,
                                 T* __restrict__ xo) {
  const uint64_t cnt = d_n ? min((uint64_t)*d_n, n) : n;
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < cnt; o += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = idx[o] - base;
    if (e < N) xo[e] = val[o];
  }
}

__global__ void k_interp_final(const unsigned long long* ocount, uint64_t cap, int32_t* status) {
  if (*ocount > cap) atomicOr(status, (int)SZ3G_STATUS_OUTLIER_OVERFLOW);
}

uint64_t top_stride(const uint64_t n[3]) {
  const uint64_t m = std::max(n[0], std::max(n[1], n[2]));
  uint64_t S = 1;
  while (2 * S < m) S *= 2;
  return m > 1 ? S : 0;
}

// I2: the targets of pass (s, d) along each axis
bool pass_geometry(IpArgs& a, uint64_t s, int d) {
  a.s = s;
  a.d = d;
  for (int ax = 0; ax < 3; ax++) {
    a.first[ax] = ax == d ? s : 0;
    a.step[ax] = ax >= d ? 2 * s : s;
    a.cnt[ax] = a.first[ax] < a.n[ax] ? (a.n[ax] - 1 - a.first[ax]) / a.step[ax] + 1 : 0;
  }
  return a.cnt[0] && a.cnt[1] && a.cnt[2];
}

int ip_validate(const sz3g_grid* g, const sz3g_params* p) {
  if (!g || !p) return SZ3G_EINVAL;
  if (g->dtype != SZ3G_F32 && g->dtype != SZ3G_F64) return SZ3G_EUNSUPPORTED;
  if (g->ndim < 1 || g->ndim > 3) return SZ3G_EUNSUPPORTED;
  if (!g->dims[0] || !g->dims[1] || !g->dims[2]) return SZ3G_EINVAL;
  if (p->block_size != 6) return SZ3G_EUNSUPPORTED;
  if (p->radius < 1 || p->radius > 32768) return SZ3G_ERANGE;
  if (p->eb_mode != SZ3G_EB_ABS && p->eb_mode != SZ3G_EB_REL_RANGE) return SZ3G_EINVAL;
  if (!(p->eb > 0.0) || !(p->eb < 1e308)) return SZ3G_EINVAL;
  return SZ3G_OK;
}

IpArgs base_args(const sz3g_grid* g, const sz3g_params* p, const double* d_minmax) {
  IpArgs a;
  memset(&a, 0, sizeof(a));
  for (int ax = 0; ax < 3; ax++) a.n[ax] = g->dims[ax];
  a.st[0] = a.n[1] * a.n[2];
  a.st[1] = a.n[2];
  a.st[2] = 1;
  a.R = p->radius;
  a.eb_mode = (int)p->eb_mode;
  a.eb = p->eb;
  a.d_minmax = d_minmax;
  a.gofs = g->dim0_offset * a.n[1] * a.n[2];
  return a;
}

#ifndef SZ3G_IP_PAIRS
#define SZ3G_IP_PAIRS 1   // level 1 by the pair kernels: 1 = decompression only (c5: 26.5 vs 33.2 ms), 2 = also
                          // compression (c5: 58.8 vs 43.8 ms: its stores of x and codes interleave with the
                          // other warps' donor loads of the same sectors; not understood yet), 0 = never
#endif
#ifndef SZ3G_IP_L1
#define SZ3G_IP_L1 0   // 1: level 1 in the fused tile kernel (bit-exact; c5 compress 52.4 / decompress 42.9 ms against
                       // 43.7 / 26.5 for the per-pass kernels: the five phases of a tile are serialised by block
                       // barriers with two CTAs per SM, so their load latencies are not hidden; kept for A/B)
#endif

template <typename T, bool DEC>
int run_passes(IpArgs a, const T* x, T* xp, uint16_t* codes, uint64_t* oidx, T* oval, unsigned long long* ocount,
               cudaStream_t st, int& nl) {
  const uint64_t S = top_stride(a.n);
  for (uint64_t s = S; s >= 1; s /= 2) {
    if (s == 1 && SZ3G_IP_L1 && (a.n[0] + 1) / 2 <= 65535 && (a.n[1] + L1_TJ - 1) / L1_TJ <= 65535 &&
        a.n[0] < (1ull << 31) && a.n[1] < (1ull << 31) && a.n[2] < (1ull << 31)) {
      const dim3 grid((unsigned)((a.n[2] + L1_TK - 1) / L1_TK), (unsigned)((a.n[1] + L1_TJ - 1) / L1_TJ),
                      (unsigned)((a.n[0] + 1) / 2));
      auto kern = k_interp_l1<T, DEC>;
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L1Smem<T>::total) !=
          cudaSuccess)
        return SZ3G_ECUDA;
      kern<<<grid, L1_WARPS * 32, L1Smem<T>::total, st>>>(x, xp, codes, oidx, oval, ocount, a);
      nl++;
      break;
    }
    if (SZ3G_IP_ROWS && (s == 1 || SZ3G_IP_ROWS > 1) && a.n[2] < (1ull << 31)) {
      // level s by rows of its sub-grid: (s,0) + (s,2), then (s,2), then (s,1) + (s,2)
      pass_geometry(a, s, 2);   // a.s = s (the row kernels read the extents, s and the constants)
      const uint64_t m0 = (a.n[0] - 1) / s + 1, m1 = (a.n[1] - 1) / s + 1, m2 = (a.n[2] - 1) / s + 1;
      const uint64_t rows[3] = {((m0 + 1) / 2) * ((m1 + 1) / 2), m0 * (m1 / 2), (m0 / 2) * ((m1 + 1) / 2)};
      const bool run[3] = {m2 > 1, m1 > 1, m0 > 1};
      for (int kind : {2, 0, 1}) {
        if (!rows[kind] || !run[kind]) continue;
        const unsigned g = (unsigned)std::min<uint64_t>((rows[kind] + IR_WARPS - 1) / IR_WARPS, 1u << 20);
        if (kind == 2) k_interp_rows<T, DEC, 2><<<g, IR_WARPS * 32, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
        else if (kind == 0) k_interp_rows<T, DEC, 0><<<g, IR_WARPS * 32, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
        else k_interp_rows<T, DEC, 1><<<g, IR_WARPS * 32, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
        nl++;
      }
      if (s == 1) break;
      continue;
    }
    if (s == 1 && SZ3G_IP_PAIRS && (DEC || SZ3G_IP_PAIRS > 1)) {   // level 1: pair kernels (full-sector stores)
      const uint64_t np = (a.n[2] + 1) / 2;
      for (int d = 0; d < 3; d++) {
        if (!pass_geometry(a, s, d)) continue;
        const uint64_t rows = d == 2 ? a.n[0] * a.n[1] : (d == 1 ? a.n[0] * (a.n[1] / 2) : (a.n[0] / 2) * ((a.n[1] + 1) / 2));
        const dim3 grid((unsigned)((np + 255) / 256), (unsigned)std::min<uint64_t>(rows, 65535));
        if (d == 0) k_interp_pairs<T, DEC, 0><<<grid, 256, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
        else if (d == 1) k_interp_pairs<T, DEC, 1><<<grid, 256, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
        else k_interp_pairs<T, DEC, 2><<<grid, 256, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
        nl++;
      }
      break;
    }
    for (int d = 0; d < 3; d++) {
      if (!pass_geometry(a, s, d)) continue;
      const dim3 grid((unsigned)((a.cnt[2] + 255) / 256), (unsigned)std::min<uint64_t>(a.cnt[1], 65535),
                      (unsigned)std::min<uint64_t>(a.cnt[0], 65535));
      k_interp_pass<T, DEC><<<grid, 256, 0, st>>>(x, xp, codes, oidx, oval, ocount, a);
      nl++;
    }
    if (s == 1) break;
  }
  return SZ3G_OK;
}

int ip_check(int nl) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return SZ3G_ECUDA;
  g_ip_launches.fetch_add((uint64_t)nl, std::memory_order_relaxed);
  return SZ3G_OK;
}

}  // namespace

uint64_t sz3g_interp_launch_count_internal() { return g_ip_launches.load(); }

extern "C" {

int sz3g_interp_compress(const sz3g_grid* grid, const sz3g_params* params, const void* x, const double* d_minmax,
                         uint16_t* codes, void* xprime, uint64_t* outlier_idx, void* outlier_val, uint64_t outlier_cap,
                         unsigned long long* d_outlier_count, int64_t* hist, double* d_eb_abs, int32_t* d_status,
                         sz3g_stream_t stream) {
  int rc = ip_validate(grid, params);
  if (rc) return rc;
  if (!x || !codes || !xprime || !outlier_idx || !outlier_val || outlier_cap < 1 || !d_outlier_count || !d_status)
    return SZ3G_EINVAL;
  if (params->eb_mode == SZ3G_EB_REL_RANGE && !d_minmax) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  IpArgs a = base_args(grid, params, d_minmax);
  a.d_eb_abs = d_eb_abs;
  a.d_status = d_status;
  a.cap = outlier_cap;
  int nl = 0;
  if (grid->dtype == SZ3G_F32) {
    k_interp_anchor<float><<<1, 1, 0, st>>>((const float*)x, (float*)xprime, codes, outlier_idx, (float*)outlier_val,
                                            d_outlier_count, a);
    nl++;
    a.d_eb_abs = nullptr;
    a.d_status = nullptr;
    rc = run_passes<float, false>(a, (const float*)x, (float*)xprime, codes, outlier_idx, (float*)outlier_val,
                             d_outlier_count, st, nl);
    if (rc) return rc;
  } else {
    k_interp_anchor<double><<<1, 1, 0, st>>>((const double*)x, (double*)xprime, codes, outlier_idx,
                                             (double*)outlier_val, d_outlier_count, a);
    nl++;
    a.d_eb_abs = nullptr;
    a.d_status = nullptr;
    rc = run_passes<double, false>(a, (const double*)x, (double*)xprime, codes, outlier_idx, (double*)outlier_val,
                              d_outlier_count, st, nl);
    if (rc) return rc;
  }
  k_interp_final<<<1, 1, 0, st>>>(d_outlier_count, outlier_cap, d_status);
  nl++;
  rc = ip_check(nl);
  if (rc) return rc;
  if (hist) {
    const uint64_t N = grid->dims[0] * grid->dims[1] * grid->dims[2];
    return sz3g_histogram(codes, N, params->radius, hist, stream);
  }
  return SZ3G_OK;
}

int sz3g_interp_decompress(const sz3g_grid* grid, const sz3g_params* params, const double* d_minmax,
                           const uint16_t* codes, const uint64_t* outlier_idx, const void* outlier_val,
                           uint64_t n_outliers, const unsigned long long* d_outlier_count, void* x_out,
                           sz3g_stream_t stream) {
  int rc = ip_validate(grid, params);
  if (rc) return rc;
  if (!codes || !x_out || (n_outliers > 0 && (!outlier_idx || !outlier_val))) return SZ3G_EINVAL;
  if (params->eb_mode == SZ3G_EB_REL_RANGE && !d_minmax) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  IpArgs a = base_args(grid, params, d_minmax);
  const uint64_t N = a.n[0] * a.n[1] * a.n[2];
  int nl = 0;
  uint16_t* cw = const_cast<uint16_t*>(codes);   // read-only in the decompress instantiation
  if (grid->dtype == SZ3G_F32) {
    if (n_outliers) {
      k_interp_scatter<float><<<(unsigned)std::min<uint64_t>((n_outliers + 255) / 256, 4096), 256, 0, st>>>(
          outlier_idx, (const float*)outlier_val, n_outliers, d_outlier_count, a.gofs, N, (float*)x_out);
      nl++;
    }
    rc = run_passes<float, true>(a, nullptr, (float*)x_out, cw, nullptr, nullptr, nullptr, st, nl);
    if (rc) return rc;
  } else {
    if (n_outliers) {
      k_interp_scatter<double><<<(unsigned)std::min<uint64_t>((n_outliers + 255) / 256, 4096), 256, 0, st>>>(
          outlier_idx, (const double*)outlier_val, n_outliers, d_outlier_count, a.gofs, N, (double*)x_out);
      nl++;
    }
    rc = run_passes<double, true>(a, nullptr, (double*)x_out, cw, nullptr, nullptr, nullptr, st, nl);
    if (rc) return rc;
  }
  return ip_check(nl);
}

}  // extern "C"
