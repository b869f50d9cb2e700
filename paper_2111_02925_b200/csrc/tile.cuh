// Per-tile device routines of the block-regression path (Lemma 1, prediction and
// linear-scaling quantisation P:156 / P:406-409, recover P:403), shared by the plain and the
// TMA-pipelined kernels.
//
// Work decomposition: a TILE is 6 x 6 x 96 elements (dims 0,1,2) = 16 regression blocks along the
// fastest dimension.  One warp owns one tile; lane l owns block l/2 and the three k-columns
// 3(l&1) .. 3(l&1)+2 of it, i.e. tile columns 3l .. 3l+2 -> two lanes per block, the block
// reduction is one shfl.xor(1), and a lane's shared-memory reads (stride 3 words) are
// bank-conflict free.  Elements outside the grid read as 0 (TMA zero fill / predicated loads),
// which leaves the moments of clipped edge blocks exact.
//
// The arithmetic is oracle/DEFINITION.md O5-O10 + D with these device-side choices:
//   * moments (O4) are summed in a fixed tree order (tolerance-checked, not bit-exact: G13);
//   * the Lemma's divisions use reciprocals (beta within the 1e-12 block-scale tolerance);
//   * everything from the coefficient codes on is op-for-op the definition (bit-exact):
//     rint via the 1.5*2^52 add/sub (exact ties-to-even for |t| < 2^51), explicit __d*_rn
//     intrinsics so nothing is contracted into an FMA, fma only where O7 writes one.
#pragma once
#include <cstdint>

#ifndef SZ3G_DEC_UNROLL
#define SZ3G_DEC_UNROLL 1   // unroll of the decompress column loop (A/B tuning)
#endif

namespace sz3g {

constexpr int DEC_UNROLL = SZ3G_DEC_UNROLL;
#ifndef SZ3G_QKU
#define SZ3G_QKU 1   // unroll of the quantise loop over a lane's three columns (A/B)
#endif
constexpr int QKU = SZ3G_QKU;
constexpr int BS = 6;                          // regression block size B (north_star: 6x6x6)
constexpr int TK = 96;                         // tile extent along dim 2 (16 blocks)
constexpr int TROWS = BS * BS;                 // rows (i,j) per tile
constexpr int TILE_ELEMS = TK * TROWS;         // 3456
constexpr int HWIN = 8192;                     // shared-memory histogram window (bins)
constexpr double RINT_MAGIC = 6755399441055744.0;  // 1.5 * 2^52
constexpr double I2D_MAGIC = 4503599627370496.0;   // 2^52

struct Consts {
  double eb_abs, twoeb, inv2eb, w0, ws, inv_w0, inv_ws;
  double vc, vthr;  // fast verify: |t - q| + vc*|x| <= vthr  implies  |(T)(p + 2eb q) - x| <= eb
  double kS_mul, kS_add;  // fp32 fast path: kS = kS_mul * S + kS_add (see fast32_consts)
  float inv2eb32, c32, k1;
  int fast32;             // fl32(1/(2eb)) is a normal fp32 number: the fp32 fast path applies
};

struct Geo {
  uint64_t n0, n1, n2;
  uint32_t NB0, NB1, NB2, NT2;   // blocks per dim; NT2 = tiles along dim 2 = ceil(NB2/16)
  uint64_t ntiles;
  uint64_t gofs;                 // dim0_offset * n1 * n2 (outlier indices are global)
  uint64_t mNT2, mNB1;           // floor(2^40 / d) + 1: x / d = (x * m) >> 40 exactly for x, d < 2^19
};

// O1/O2 on device: same operations as the definition (IEEE division for the constants).
// `uround` is the fast-verify roundoff constant of T (2^-24 + 1.12e-16 for f32, 2.3e-16 for f64).
__device__ __forceinline__ bool make_consts(int eb_mode, double eb, const double* d_minmax, double uround, Consts& K) {
  double eb_abs = eb;
  if (eb_mode == 1) eb_abs = __dmul_rn(eb, __dsub_rn(d_minmax[1], d_minmax[0]));
  if (!(isfinite(eb_abs) && eb_abs > 0.0)) return false;
  K.eb_abs = eb_abs;
  K.twoeb = __dmul_rn(2.0, eb_abs);
  K.inv2eb = __ddiv_rn(1.0, K.twoeb);
  K.w0 = __ddiv_rn(eb_abs, 2.0);
  K.ws = __ddiv_rn(eb_abs, 2.0 * BS);
  K.inv_w0 = __ddiv_rn(1.0, K.w0);
  K.inv_ws = __ddiv_rn(1.0, K.ws);
  // Fast verify (O9 without forming x'): for |t| < 32768, q = rint(t), y = fl(p + fl(2eb q)),
  //   |r/(2eb) - t| <= 3.4e-16 |t|  (r = x - p),   |x - y| <= 2eb (|t - q| + 1.5e-11) + 1.2e-16 |y|,
  //   |(T)y - y| <= 2^-24 |y| (f32; 0 for f64),  |d| <= |(T)y - x| (1 + 1.2e-16),  |y| <= |x| + 1.01 eb,
  // hence  |t - q| + c |x| <= 0.5 - 1e-10 - 1.02 c eb  with  c = 1.01 uround / (2 eb)  implies  |d| <= eb.
  // (t - q is exact: Sterbenz.)  Elements failing the test take the exact O9 path.  For f32 with a
  // huge eb, (T)y could overflow to inf: the fast test is disabled there.
  K.vc = 1.01 * uround / K.twoeb;
  K.vthr = (uround > 1e-12 && eb_abs > 1e30) ? -1.0 : 0.5 - 1e-10 - 1.02 * K.vc * eb_abs;
  // fp32 fast path constants (f32 data; see fast32_consts): kS = 2.52 u S / eb + 1.2e-11 + 1e-43,
  // evaluated as kS_mul * S + kS_add with the multiplier rounded up.  The fast path needs
  // fl32(1/(2eb)) to be a normal fp32 number (relative error <= u): otherwise it is switched off.
  const double u = 5.9604644775390625e-08;
  K.kS_mul = __ddiv_ru(2.52 * u, eb_abs) * (1.0 + 1e-15);
  K.kS_add = 1.2e-11 + 1e-43;
  K.inv2eb32 = __double2float_rn(K.inv2eb);
  K.fast32 = (K.inv2eb > 2.4e-38 && K.inv2eb < 8.5e37) ? 1 : 0;
  K.c32 = __double2float_ru(K.vc);
  K.k1 = __double2float_ru(2.1 * u);
  return true;
}

template <typename T> __device__ __forceinline__ double to_d(T v);
template <> __device__ __forceinline__ double to_d<float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double to_d<double>(double v) { return v; }
template <typename T> __device__ __forceinline__ T from_d(double v);
template <> __device__ __forceinline__ float from_d<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double from_d<double>(double v) { return v; }

// 6/(m+1) and 2/(m-1) for block extents m = 1..6 (Lemma 1 factors; index 0/1 unused slots = 0)
__constant__ double c_lemma[7][2] = {{0, 0},       {3.0, 0.0},       {2.0, 2.0},      {1.5, 1.0},
                                     {1.2, 2.0 / 3}, {1.0, 0.5}, {6.0 / 7, 0.4}};

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

#ifndef SZ3G_X2
#define SZ3G_X2 1   // packed fp32x2 arithmetic in the fp32 fast path (FFMA2 / FADD2, sm_100a)
#endif
// packed fp32 pairs (sm_100a FFMA2 / FADD2): each lane is the IEEE round-to-nearest result of the
// scalar operation, so a pair computes exactly what two scalar instructions would
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lane_of(uint64_t v, int h) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return h ? hi : lo;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// unconditional shared-memory add of a 0/1 register (red.shared, no return value): no branch and no
// convergence region around it (a predicated +1 is turned into a warp-collective ATOMS.POPC.INC)
__device__ __forceinline__ void red_smem_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

struct TileCoord {
  uint32_t a, b, c;  // block-row index along dim0, dim1; tile index along dim2
};

// tile index -> coordinates.  Multiply-shift division: with m = floor(2^40/d) + 1, (x*m) >> 40 =
// floor(x/d) for x < 2^21 and d < 2^19 (the error x(m - 2^40/d)/2^40 < 2^-19 < 1/d); the host falls
// back to plain division (m = 0) outside that range.
__device__ __forceinline__ uint32_t fdiv(uint32_t x, uint32_t d, uint64_t m) {
  return m ? (uint32_t)(((uint64_t)x * m) >> 40) : x / d;
}

__device__ __forceinline__ TileCoord decode_tile(uint64_t t64, const Geo& g) {
  const uint32_t t = (uint32_t)t64;
  TileCoord tc;
  const uint32_t r = fdiv(t, g.NT2, g.mNT2);
  tc.c = t - r * g.NT2;
  tc.a = fdiv(r, g.NB1, g.mNB1);
  tc.b = r - tc.a * g.NB1;
  return tc;
}

template <typename T>
struct CompressOut {
  uint16_t* codes;              // global codes (used when codes are not staged in smem)
  int32_t* coef;                // [NB][4]
  double* coef_raw;             // nullable
  uint64_t* oidx;
  T* oval;
  uint64_t cap;
  unsigned long long* ocount;
  unsigned long long* hist;     // nullable (int64 bins, accumulated)
  const double* beta_in;        // two-pass mode: [NB][4] beta from the analyze pass (else nullptr)
};

// Shared-memory histogram state of one CTA.
struct HistSmem {
  uint32_t* win;   // HWIN bins, window [lo, lo + HWIN)
  uint32_t* zero;  // bin 0 (outliers)
  uint32_t* dummy; // 32 per-lane sink slots for non-counted elements
  uint32_t lo;
  uint32_t nwin;   // bins actually used (min(2R, HWIN))
  uint32_t W;      // fast-path acceptance |q| < W: every accepted code lies in the window
};


// ------------------------------------------------------------------------------------------
// Compress, in pieces.  A tile's input is addressed as xs[i*si + j*sj + k] (k in [0,96)): either a
// shared-memory stage (si = 576, sj = 96; zero outside the grid) or the global field (IN_SMEM =
// false: loads predicated on the grid bounds).  Codes go to cs[i*ci + j*cj + k] likewise.  A warp
// handles the tile's i-planes [i0, i0 + P): P = 6 for one warp per tile, P = 6/G when a group of G
// warps shares a tile (the partial moments are then summed across the group through shared memory).
// ------------------------------------------------------------------------------------------
struct LaneGeom {
  int h, kcol;        // half of the block (0/1), first tile column of this lane
  uint32_t kb;        // block index along dim 2
  int m0, m1, m2;     // block extents (m2 = 0: no block for this lane)
  bool kv0, kv1, kv2; // validity of the lane's three columns
  __device__ __forceinline__ bool kv(int kk) const { return kk == 0 ? kv0 : (kk == 1 ? kv1 : kv2); }
};

// FULL: the tile lies inside the grid, so every block is 6x6x6 (constants fold)
template <bool FULL = false>
__device__ __forceinline__ LaneGeom lane_geom(const TileCoord tc, const Geo& g) {
  const int lane = threadIdx.x & 31;
  LaneGeom L;
  const int bl = lane >> 1;
  L.h = lane & 1;
  L.kb = tc.c * 16u + (uint32_t)bl;
  L.kcol = 6 * bl + 3 * L.h;
  if (FULL) {
    L.m0 = L.m1 = L.m2 = BS;
    L.kv0 = L.kv1 = L.kv2 = true;
    return L;
  }
  L.m0 = (int)umin64(BS, g.n0 - (uint64_t)tc.a * BS);
  L.m1 = (int)umin64(BS, g.n1 - (uint64_t)tc.b * BS);
  L.m2 = (L.kb < g.NB2) ? (int)umin64(BS, g.n2 - (uint64_t)L.kb * BS) : 0;
  L.kv0 = 3 * L.h + 0 < L.m2;
  L.kv1 = 3 * L.h + 1 < L.m2;
  L.kv2 = 3 * L.h + 2 < L.m2;
  return L;
}

// every element of the tile lies inside the grid (warp-uniform)
__device__ __forceinline__ bool tile_full(const TileCoord tc, const Geo& g) {
  return (uint64_t)(tc.a + 1) * BS <= g.n0 && (uint64_t)(tc.b + 1) * BS <= g.n1 && (uint64_t)(tc.c + 1) * TK <= g.n2;
}

// Running min / max of the valid elements a lane has seen (a0 fused into the analyze pass).  NaN
// never replaces a value (fmin/fmax); the analyze kernel detects NaN from the block sums instead.
template <typename T>
struct MinMax {
  T lo, hi;
  __device__ __forceinline__ void init() {
    lo = sizeof(T) == 4 ? (T)__int_as_float(0x7f800000) : (T)__longlong_as_double(0x7ff0000000000000ll);
    hi = -lo;
  }
  __device__ __forceinline__ void add(T v) {
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
};

// O4 partial moments of the lane's three columns over rows j in [j0, j0+PJ), all six i-planes (fp64).
// Row sums S = f0+f1+f2 and the lane-local k-weighted sum f1 + 2 f2 first; per plane i
// P_i = sum_j S, Q_i = sum_j j S, Z_i = sum_j (f1 + 2 f2); Vz includes the lane's column offset 3h.
// MM: also fold the valid elements into `mm` (FULL: every element of the tile is valid); the sums do
// not depend on MM, so beta is bit-identical with and without it.
template <typename T, bool IN_SMEM, int PJ, bool MM = false, bool FULL = false>
__device__ __forceinline__ void moments_partial(const T* __restrict__ xs, uint64_t si, uint64_t sj, int j0,
                                                const LaneGeom& L, double V[4], MinMax<T>* mm = nullptr) {
  double V0 = 0.0, Vx = 0.0, Vy = 0.0, Vz = 0.0;
  double di = 0.0;
#pragma unroll 1
  for (int i = 0; i < BS; i++, di += 1.0) {
    double Ps = 0.0, Q = 0.0, Z = 0.0;
    const T* plane = IN_SMEM ? xs + (uint32_t)(i * BS * TK + j0 * TK + L.kcol) : xs + (uint64_t)i * si + (uint64_t)j0 * sj + L.kcol;
#pragma unroll
    for (int jj = 0; jj < PJ; jj++) {
      const int j = j0 + jj;
      const T* row = IN_SMEM ? plane + jj * TK : plane + (uint64_t)jj * sj;
      double f0, f1, f2;
      const bool rv = (i < L.m0) && (j < L.m1);
      if (IN_SMEM) {
        const T v0 = row[0], v1 = row[1], v2 = row[2];
        if (MM) {
          if (FULL || (rv && L.kv0)) mm->add(v0);
          if (FULL || (rv && L.kv1)) mm->add(v1);
          if (FULL || (rv && L.kv2)) mm->add(v2);
        }
        f0 = to_d<T>(v0); f1 = to_d<T>(v1); f2 = to_d<T>(v2);
      } else {
        const T v0 = (rv && L.kv0) ? row[0] : T(0);
        const T v1 = (rv && L.kv1) ? row[1] : T(0);
        const T v2 = (rv && L.kv2) ? row[2] : T(0);
        if (MM) {
          if (rv && L.kv0) mm->add(v0);
          if (rv && L.kv1) mm->add(v1);
          if (rv && L.kv2) mm->add(v2);
        }
        f0 = to_d<T>(v0); f1 = to_d<T>(v1); f2 = to_d<T>(v2);
      }
      const double S = (f0 + f1) + f2;
      const double Kw = fma(2.0, f2, f1);
      Ps += S;
      Q = fma((double)j, S, Q);
      Z += Kw;
    }
    V0 += Ps;
    Vx = fma(di, Ps, Vx);
    Vy += Q;
    Vz += Z;
  }
  V[0] = V0;
  V[1] = Vx;
  V[2] = Vy;
  V[3] = fma(3.0 * L.h, V0, Vz);
}

// O5 (Lemma 1; extent-1 axis -> slope 0, G2) from the full block moments.  The fused
// compress kernel and the two-pass analyze kernel both call this one function, so their beta are
// bit-identical.
template <bool FULL = false>
__device__ __forceinline__ void block_beta(const double V[4], const LaneGeom& L, double beta[4]) {
  beta[0] = beta[1] = beta[2] = beta[3] = 0.0;
  if (FULL) {  // 6x6x6 block: Nb = 216, 6/(m+1) = 6/7, 2/(m-1) = 2/5 (same values as the table path)
    const double invNb = 1.0 / 216.0;
    const double sc = (6.0 / 7.0) * invNb;
#pragma unroll
    for (int d = 0; d < 3; d++) beta[d + 1] = sc * fma(V[d + 1], 0.4, -V[0]);
    beta[0] = V[0] * invNb - (2.5 * beta[1] + 2.5 * beta[2] + 2.5 * beta[3]);
  } else if (L.m2 > 0) {
    const double Nb = (double)(L.m0 * L.m1 * L.m2);
    const double invNb = __drcp_rn(Nb);
    const int md[3] = {L.m0, L.m1, L.m2};
#pragma unroll
    for (int d = 0; d < 3; d++) {
      if (md[d] > 1) {
        const double sc = c_lemma[md[d]][0] * invNb;
        const double inner = fma(V[d + 1], c_lemma[md[d]][1], -V[0]);
        beta[d + 1] = sc * inner;
      }
    }
    beta[0] = V[0] * invNb - ((L.m0 - 1) * 0.5 * beta[1] + (L.m1 - 1) * 0.5 * beta[2] + (L.m2 - 1) * 0.5 * beta[3]);
  }
}

// O6 (coefficient codes; bins eb/2, eb/12, G1; zero-predictor fallback): codes and the decoded
// coefficients (bit-exact).
__device__ __forceinline__ void block_codes(const double beta[4], const Consts& K, int32_t cc[4], double bh[4]) {
  // rint by the 1.5*2^52 add/sub (exact for |u| < 2^51; larger, Inf or NaN fail the range test)
  double r[4], sm[4];
  bool bad = false;
#pragma unroll
  for (int d = 0; d < 4; d++) {
    sm[d] = __dadd_rn(beta[d] * (d == 0 ? K.inv_w0 : K.inv_ws), RINT_MAGIC);
    r[d] = __dsub_rn(sm[d], RINT_MAGIC);
    bad |= !(fabs(r[d]) <= 2147483647.0);
  }
  // (double)c == r exactly when c is representable, so b^ = c * w needs no int->fp conversion
#pragma unroll
  for (int d = 0; d < 4; d++) {
    cc[d] = bad ? 0 : __double2loint(sm[d]);
    bh[d] = bad ? 0.0 : __dmul_rn(r[d], d == 0 ? K.w0 : K.ws);
  }
}

// O5 + O6
template <bool FULL = false>
__device__ __forceinline__ void block_coefs(const double V[4], const LaneGeom& L, const Consts& K, double beta[4],
                                            int32_t cc[4], double bh[4]) {
  block_beta<FULL>(V, L, beta);
  block_codes(beta, K, cc, bh);
}

template <typename T>
__device__ __forceinline__ void write_coefs(const CompressOut<T>& o, const TileCoord tc, const Geo& g,
                                            const LaneGeom& L, const int32_t cc[4], const double beta[4]) {
  if (L.m2 > 0 && L.h == 0) {
    const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
    reinterpret_cast<int4*>(o.coef)[bid] = make_int4(cc[0], cc[1], cc[2], cc[3]);
    if (o.coef_raw) {
      reinterpret_cast<double2*>(o.coef_raw)[2 * bid] = make_double2(beta[0], beta[1]);
      reinterpret_cast<double2*>(o.coef_raw)[2 * bid + 1] = make_double2(beta[2], beta[3]);
    }
  }
}

// Exact O7-O10 for one element (the definition, fp64): code, or 0 for an outlier.
template <typename T>
__device__ __forceinline__ uint32_t exact_code(T xv, double p, const Consts& K, uint32_t R) {
  const double xd = to_d<T>(xv);
  const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
  const double sm = __dadd_rn(t, RINT_MAGIC);
  const double q = __dsub_rn(sm, RINT_MAGIC);
  const double y = __dadd_rn(p, __dmul_rn(K.twoeb, q));
  const double d = __dsub_rn(to_d<T>(from_d<T>(y)), xd);
  return (fabs(q) < (double)R && fabs(d) <= K.eb_abs) ? (uint32_t)(__double2loint(sm) + (int)R) : 0u;
}

// Per-block constants of the fp32 fast path (f32 data), evaluated in the SCALED domain: with the
// coefficients a_d = fl32(b^_d * inv2eb) and inv32 = fl32(inv2eb),
//   P32 = fma32(a1, i, fma32(a2, j, fma32(a3, k, a0))),   t32 = fma32(x, inv32, -P32),
// r = rint(t32), e = t32 - r (exact).  Against the definition's t = fl64(fl64(x - p) * inv2eb):
//   |t32 - t| <= E = k1 |t32| + kS,   k1 = 2.1 u,   kS = 2.52 u S / eb + 1.2e-11 + 1e-43
// with u = 2^-24, S = |b0| + 5 (|b1| + |b2| + |b3|) >= |p| (i, j, k <= 5): the t32 rounding (u |t32|),
// the rounding of inv32 (u |x| / 2eb <= u S / 2eb + u |t|), four roundings in P32 (4.001 u S / 2eb) and
// fp32 subnormal absolute errors (<= 2e-44); derivation in DESIGN.md 4.  The fp64 fast-verify term
// c |x| is bounded per block too: |x| <= S + 2eb |t| (1 + 1e-15) and |t| <= |t32| + E, so
// c |x| <= c S + c2e (|t32| + E) with c2e = 2.01 eb c.  Accept the fp32 result when
//   |t32 - r| + (k1 + c2e (1 + k1)) |t32| <= vthr - kS (1 + c2e) - c S   (one-sided fp32 margins):
// then t lies within E of t32, strictly inside r's rounding interval, so rint(t) = r, and the fp64
// fast-verify condition |t - q| + c |x| <= vthr holds, so x' passes O9.
struct Fast32 {
  float a0, a1, a2, a3;  // decoded coefficients scaled by 1/(2eb), rounded to fp32
  float k1, thr;         // |e| + k1 |t32| <= thr
  float pad0, pad1;
};

__device__ __forceinline__ Fast32 fast32_consts(const double bh[4], const Consts& K) {
  Fast32 F;
  F.a0 = __double2float_rn(__dmul_rn(bh[0], K.inv2eb));
  F.a1 = __double2float_rn(__dmul_rn(bh[1], K.inv2eb));
  F.a2 = __double2float_rn(__dmul_rn(bh[2], K.inv2eb));
  F.a3 = __double2float_rn(__dmul_rn(bh[3], K.inv2eb));
  const double u = 5.9604644775390625e-08;
  const double S = (fabs(bh[0]) + 5.0 * (fabs(bh[1]) + fabs(bh[2]) + fabs(bh[3]))) * (1.0 + 1e-15);
  const double kS = __fma_ru(K.kS_mul, S, K.kS_add);             // >= 2.52 u S / eb + ...
  const double c2e = 2.01 * K.eb_abs * K.vc;                       // 2 eb c with margin
  F.k1 = __double2float_ru((2.1 * u + c2e * (1.0 + 2.2 * u)) * (1.0 + 1e-12));
  const double thr = (K.vthr - kS * (1.0 + c2e) - K.vc * S * (1.0 + 1e-12)) * (1.0 - 4.0 * u);
  F.thr = (K.fast32 && thr > 0.0) ? __double2float_rd(thr) : -1.0f;
  F.pad0 = F.pad1 = 0.0f;
  return F;
}

// O7-O11 over rows j in [j0, j0+PJ), all six i-planes: per (j, k) column six independent elements
// (i = 0..5).  f32 data take the fp32 fast path above (no conversions, full-rate pipe); f64 data
// the fp64 fast verify of make_consts.  Both round with a BIASED magic M = 1.5 * 2^(p-1) + R, so the
// low 16 bits of the rounded sum's bit pattern are the code R + q itself (0x4B400000 and 2^51 are
// multiples of 2^16) and the histogram address is one multiply-add of that word.  An element is
// accepted when the fast test certifies it AND |q| < W (W = min(R, HWIN/2): its code lies in the smem
// window); every other valid element (near a half-integer, radius or verify outlier, out-of-window
// code, non-finite input, huge offsets) gets code 0 and a per-lane sink as histogram address, and
// the column then takes the exact definition (rare): exact code, histogram update by atomics, and
// outliers flagged for rare_path().  FULL tiles skip every validity predicate.  Returns whether this
// lane produced an outlier.
template <typename T, bool IN_SMEM, bool HIST, bool FULL, int PJ, bool SLAB>
__device__ __forceinline__ bool quantize_rows(const T* __restrict__ xs, uint64_t si, uint64_t sj,
                                              uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj, int j0,
                                              const LaneGeom& L, const double bh[4], const Fast32& F,
                                              const Consts& K, const uint32_t R, const HistSmem& hs,
                                              unsigned long long* __restrict__ ghist) {
  const int lane = threadIdx.x & 31;
  constexpr bool F32 = sizeof(T) == 4;
  const uint32_t win_base = HIST ? (uint32_t)__cvta_generic_to_shared(hs.win) : 0u;
  const uint32_t sink = HIST ? (uint32_t)__cvta_generic_to_shared(hs.dummy) + 4u * lane : 0u;
  // &win[code - lo] = 4 * word + hb  (32-bit shared addresses, wrap-around arithmetic)
  const uint32_t hb = win_base - 4u * ((F32 ? 0x4B400000u : 0u) + hs.lo);
  const uint32_t W = HIST ? hs.W : R;
  if (IN_SMEM) { si = BS * TK; sj = TK; }             // shared stage: compile-time strides
  if (SLAB) { ci = PJ * TK; cj = TK; }                // codes: this warp's slab [i][jj][k]
  const float inv2eb32 = K.inv2eb32;
  const float M32 = 12582912.0f + (float)R;           // 1.5 * 2^23 + R (exact)
  const float Wf = (float)W;
  const double M64 = RINT_MAGIC + (double)R;          // 1.5 * 2^52 + R (exact)
  const double Wd = (double)W;
  bool has_out = false;
#ifndef SZ3G_IPAIR_REG
#define SZ3G_IPAIR_REG 1
#endif
#if SZ3G_X2
  // the packed (i, i + 1) plane indices: immediates (re-created in uniform registers for every column,
  // 6 UMOV per 6 elements) or, with SZ3G_IPAIR_REG, register pairs (a runtime zero, R >> 31 with
  // R <= 32768, keeps the compiler from folding them back into immediates)
  const float zf = SZ3G_IPAIR_REG ? (float)(R >> 31) : 0.0f;
  uint64_t ipair[3];
#pragma unroll
  for (int q = 0; q < 3; q++) ipair[q] = pack2(zf + (float)(2 * q), zf + (float)(2 * q + 1));
#endif
  // columns (j, k) visited with incremental pointers and fp32 counters (no per-iteration division)
  const T* xrow = xs + (IN_SMEM ? (uint32_t)(j0 * TK + L.kcol) : (uint64_t)j0 * sj + L.kcol);
  uint16_t* crow = cs + (SLAB ? (uint32_t)L.kcol : (uint64_t)j0 * cj + L.kcol);
  float fj = (float)j0;
#pragma unroll 1
  for (int jj = 0; jj < PJ; jj++, fj += 1.0f) {
    const int j = j0 + jj;
    const T* xcol = xrow;
    uint16_t* ccol = crow;
    float fk = (float)(3 * L.h);
#pragma unroll QKU
    for (int kk = 0; kk < 3; kk++, xcol++, ccol++, fk += 1.0f) {
    const bool cv = FULL || ((j < L.m1) && L.kv(kk));
    T xv[BS];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const bool valid = FULL || (cv && i < L.m0);
      if (IN_SMEM || FULL) xv[i] = xcol[i * si];
      else xv[i] = valid ? xcol[i * si] : T(0);
    }
    uint32_t code[BS];   // low 16 bits = the code (0: not accepted)
    uint32_t haddr[BS];
    bool need = false;   // some valid element the fast test cannot decide -> exact definition below
    if (F32 && SZ3G_X2) {
      // the same IEEE operations on pairs of elements (i, i+1): packed FFMA2 / FADD2, per-lane rn
      const float base32 = __fmaf_rn(F.a2, fj, __fmaf_rn(F.a3, fk, F.a0));
#pragma unroll
      for (int i = 0; i < BS; i += 2) {
        const uint64_t x2 = pack2((float)xv[i], (float)xv[i + 1]);
        const uint64_t nP = fma2(pack2(-F.a1, -F.a1), ipair[i >> 1], pack2(-base32, -base32));
        const uint64_t t2 = fma2(x2, pack2(inv2eb32, inv2eb32), nP);   // -P exact: P(i = 0) = base32
        const uint64_t s2 = add2(t2, pack2(M32, M32));
        const uint64_t r2 = sub2(s2, pack2(M32, M32));
        const uint64_t e2 = sub2(t2, r2);                                // exact
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int ii = i + h;
          const bool valid = FULL || (cv && ii < L.m0);
          const float t32 = lane_of(t2, h), e = lane_of(e2, h), r = lane_of(r2, h);
          const float v = __fmaf_rn(F.k1, fabsf(t32), fabsf(e));
          const bool ok = (v <= F.thr) && (fabsf(r) < Wf);
          const uint32_t w = __float_as_uint(lane_of(s2, h));
          code[ii] = ok ? w : 0u;
          haddr[ii] = (ok && valid) ? 4u * w + hb : sink;
          need |= valid && !ok;
        }
      }
    } else if (F32) {
      const float base32 = __fmaf_rn(F.a2, fj, __fmaf_rn(F.a3, fk, F.a0));
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = FULL || (cv && i < L.m0);
        const float P = i == 0 ? base32 : __fmaf_rn(F.a1, (float)i, base32);   // a1 finite: i = 0 exact
        const float t32 = __fmaf_rn((float)xv[i], inv2eb32, -P);
        const float s32 = __fadd_rn(t32, M32);
        const float r = __fsub_rn(s32, M32);
        const float e = __fsub_rn(t32, r);                    // exact
        const float v = __fmaf_rn(F.k1, fabsf(t32), fabsf(e));
        const bool ok = (v <= F.thr) && (fabsf(r) < Wf);
        const uint32_t w = __float_as_uint(s32);
        code[i] = ok ? w : 0u;
        haddr[i] = (ok && valid) ? 4u * w + hb : sink;
        need |= valid && !ok;
      }
    } else {
      const double base = __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * L.h + kk), bh[0]));
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = FULL || (cv && i < L.m0);
        const double xd = to_d<T>(xv[i]);
        const double p = __fma_rn(bh[1], (double)i, base);
        const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
        const double sm = __dadd_rn(t, M64);
        const double q = __dsub_rn(sm, M64);
        const double v = __fma_rn(K.vc, fabs(xd), fabs(__dsub_rn(t, q)));   // fast verify (make_consts)
        const bool ok = (v <= K.vthr) && (fabs(q) < Wd);
        const uint32_t w = (uint32_t)__double2loint(sm);
        code[i] = ok ? w : 0u;
        haddr[i] = (ok && valid) ? 4u * w + hb : sink;
        need |= valid && !ok;
      }
    }
    if (__any_sync(0xffffffffu, need)) {
      const double base = __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * L.h + kk), bh[0]));
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = FULL || (cv && i < L.m0);
        if (valid && code[i] == 0u) {
          const uint32_t c = exact_code<T>(xv[i], __fma_rn(bh[1], (double)i, base), K, R);
          code[i] = c;
          if (c == 0u) has_out = true;   // counted in bin 0 by rare_path
          else if (HIST) {
            if (c - hs.lo < hs.nwin) atomicAdd(&hs.win[c - hs.lo], 1u);
            else atomicAdd(&ghist[c], 1ull);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const bool valid = FULL || (cv && i < L.m0);
      if (valid) ccol[i * ci] = (uint16_t)code[i];
      if (HIST) red_smem_add(haddr[i], 1u);   // O11 (sink for elements not counted here)
    }
    }
    xrow += IN_SMEM ? (uint64_t)TK : sj;
    crow += cj;
  }
  return has_out;
}

// Rare path (warp-uniform entry): outliers of rows [j0, j0+PJ) -> (global index, value) with a
// warp-aggregated append, and their count into bin 0.
template <typename T, bool HIST, int PJ>
__device__ __forceinline__ void rare_path_lanes(const T* __restrict__ xs, uint64_t si, uint64_t sj,
                                          const uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj, int j0,
                                          int cs_j0, const LaneGeom& L, bool has_out, const TileCoord tc,
                                          const Geo& g, const CompressOut<T>& o, const HistSmem& hs) {
  const int lane = threadIdx.x & 31;
  if (!__any_sync(0xffffffffu, has_out)) return;
  const int j1 = min(j0 + PJ, L.m1);
  uint32_t nout = 0;
  if (has_out) {
    for (int j = j0; j < j1; j++)
      for (int kk = 0; kk < 3; kk++) {
        if (!L.kv(kk)) continue;
        for (int i = 0; i < L.m0; i++) nout += (cs[i * ci + (j - cs_j0) * cj + L.kcol + kk] == 0u) ? 1u : 0u;
      }
  }
  uint32_t incl = nout;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long basepos = 0;
  if (lane == 31) {
    basepos = atomicAdd(o.ocount, (unsigned long long)total);
    if (HIST) atomicAdd(hs.zero, total);
  }
  basepos = __shfl_sync(0xffffffffu, basepos, 31);
  unsigned long long pos = basepos + (incl - nout);
  if (nout) {
    const uint64_t gbase =
        g.gofs + ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)L.kb * BS + 3 * L.h;
    for (int j = j0; j < j1; j++)
      for (int kk = 0; kk < 3; kk++) {
        if (!L.kv(kk)) continue;
        for (int i = 0; i < L.m0; i++) {
          if (cs[i * ci + (j - cs_j0) * cj + L.kcol + kk] != 0) continue;
          if (pos < o.cap) {
            o.oidx[pos] = gbase + ((uint64_t)i * g.n1 + j) * g.n2 + kk;
            o.oval[pos] = xs[i * si + j * sj + L.kcol + kk];
          }
          pos++;
        }
      }
  }
}

// Row-ordered rare path (ROW, the kernel instances for small radii, where outliers are common): the list is written row piece by row piece: for
// every (j, i) the warp's outliers of that 96-column row piece take consecutive slots (ballot per column
// of the lanes' three), so the list's stores are coalesced and the decompressor's scatter of
// consecutive entries hits the same few sectors at once (round 1 appended each lane's outliers as one
// run across six planes: on an outlier-heavy field the scatter wrote every sector many times apart).
template <typename T, bool HIST, int PJ>
__device__ __forceinline__ void rare_path_rows(const T* __restrict__ xs, uint64_t si, uint64_t sj,
                                          const uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj, int j0,
                                          int cs_j0, const LaneGeom& L, bool has_out, const TileCoord tc,
                                          const Geo& g, const CompressOut<T>& o, const HistSmem& hs) {
  const int lane = threadIdx.x & 31;
  if (!__any_sync(0xffffffffu, has_out)) return;
  const int j1 = min(j0 + PJ, L.m1);   // m0, m1: the tile's block row, the same for every lane
  uint32_t nout = 0;
  if (has_out) {
    for (int j = j0; j < j1; j++)
      for (int kk = 0; kk < 3; kk++) {
        if (!L.kv(kk)) continue;
        for (int i = 0; i < L.m0; i++) nout += (cs[i * ci + (j - cs_j0) * cj + L.kcol + kk] == 0u) ? 1u : 0u;
      }
  }
  uint32_t total = nout;
#pragma unroll
  for (int off = 16; off; off >>= 1) total += __shfl_xor_sync(0xffffffffu, total, off);
  unsigned long long pos = 0;
  if (lane == 0) {
    pos = atomicAdd(o.ocount, (unsigned long long)total);
    if (HIST) atomicAdd(hs.zero, total);
  }
  pos = __shfl_sync(0xffffffffu, pos, 0);
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t gbase =
      g.gofs + ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)L.kb * BS + 3 * L.h;
  for (int j = j0; j < j1; j++)
    for (int i = 0; i < L.m0; i++)
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        const bool f = has_out && L.kv(kk) && cs[i * ci + (j - cs_j0) * cj + L.kcol + kk] == 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (f) {
          const unsigned long long p = pos + __popc(bal & lt);
          if (p < o.cap) {
            o.oidx[p] = gbase + ((uint64_t)i * g.n1 + j) * g.n2 + kk;
            o.oval[p] = xs[i * si + j * sj + L.kcol + kk];
          }
        }
        pos += __popc(bal);
      }
}

// Rare path (warp-uniform entry): outliers of rows [j0, j0+PJ) -> (global index, value), their count into
// bin 0.  ROW selects the row-ordered append; the default keeps each lane's outliers as one run (its
// code does not disturb the register allocation of the hot quantise loop: the row-ordered one, in the
// same kernel, cost the c5 quantise kernel 3% through register moves in that loop).
template <typename T, bool HIST, int PJ, bool ROW = false>
__device__ __forceinline__ void rare_path(const T* __restrict__ xs, uint64_t si, uint64_t sj,
                                          const uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj, int j0,
                                          int cs_j0, const LaneGeom& L, bool has_out, const TileCoord tc,
                                          const Geo& g, const CompressOut<T>& o, const HistSmem& hs) {
  if (ROW) rare_path_rows<T, HIST, PJ>(xs, si, sj, cs, ci, cj, j0, cs_j0, L, has_out, tc, g, o, hs);
  else rare_path_lanes<T, HIST, PJ>(xs, si, sj, cs, ci, cj, j0, cs_j0, L, has_out, tc, g, o, hs);
}

// One warp compresses a whole tile (plain kernel).  BETA: the block coefficients come from the
// analyze pass (o.beta_in) instead of the moments.
template <typename T, bool IN_SMEM, bool HIST, bool FULL, bool BETA = false>
__device__ __forceinline__ void compress_tile(const T* __restrict__ xs, uint64_t si, uint64_t sj,
                                              uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj,
                                              const TileCoord tc, const Geo& g, const Consts& K,
                                              const uint32_t R, const CompressOut<T>& o, const HistSmem& hs) {
  const LaneGeom L = lane_geom<FULL>(tc, g);
  double V[4], beta[4], bh[4];
  int32_t cc[4];
  if (BETA) {
    beta[0] = beta[1] = beta[2] = beta[3] = 0.0;
    if (L.m2 > 0) {
      const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
      const double2 b01 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid);
      const double2 b23 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid + 1);
      beta[0] = b01.x; beta[1] = b01.y; beta[2] = b23.x; beta[3] = b23.y;
    }
    block_codes(beta, K, cc, bh);
  } else {
    moments_partial<T, IN_SMEM, BS>(xs, si, sj, 0, L, V);
#pragma unroll
    for (int d = 0; d < 4; d++) V[d] += __shfl_xor_sync(0xffffffffu, V[d], 1);
    block_coefs<FULL>(V, L, K, beta, cc, bh);
  }
  write_coefs(o, tc, g, L, cc, beta);
  const Fast32 F = fast32_consts(bh, K);
  const bool has_out =
      quantize_rows<T, IN_SMEM, HIST, FULL, BS, false>(xs, si, sj, cs, ci, cj, 0, L, bh, F, K, R, hs, o.hist);
  rare_path<T, HIST, BS>(xs, si, sj, cs, ci, cj, 0, 0, L, has_out, tc, g, o, hs);
}

// One warp analyzes a whole tile (a0 + a2 + a3): moments and min/max of the valid elements, beta of
// its 16 blocks (same functions, same order as the fused compress path: bit-identical beta).
// Returns whether a block sum is NaN (a NaN element, or infinities of both signs).
template <typename T, bool IN_SMEM, bool FULL>
__device__ __forceinline__ bool analyze_tile(const T* __restrict__ xs, uint64_t si, uint64_t sj, const TileCoord tc,
                                             const Geo& g, double* __restrict__ beta_out, MinMax<T>& mm) {
  const LaneGeom L = lane_geom<FULL>(tc, g);
  double V[4], beta[4];
  moments_partial<T, IN_SMEM, BS, true, FULL>(xs, si, sj, 0, L, V, &mm);
#pragma unroll
  for (int d = 0; d < 4; d++) V[d] += __shfl_xor_sync(0xffffffffu, V[d], 1);
  block_beta<FULL>(V, L, beta);
  if (L.m2 > 0 && L.h == 0) {
    const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
    reinterpret_cast<double2*>(beta_out)[2 * bid] = make_double2(beta[0], beta[1]);
    reinterpret_cast<double2*>(beta_out)[2 * bid + 1] = make_double2(beta[2], beta[3]);
  }
  return L.m2 > 0 && V[0] != V[0];
}

// ------------------------------------------------------------------------------------------
// Decompress (recover): x' = (T)(p + twoeb*(c - R)) for c != 0, 0 for c == 0 (outlier values
// are scattered afterwards) over rows j in [j0, j0+PJ), all six i-planes.  Codes are read from
// cs[i*ci + j*cj + k] (shared stage or global, predicated); x' goes to a shared row slab laid out
// [i][jj][k] for a TMA store of box {96, PJ, 6} (OUT_SMEM) or straight to global xo[i*oi + j*oj + k].
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void decode_coefs(const int4 cc, const Consts& K, double bh[4]) {
  bh[0] = __dmul_rn((double)cc.x, K.w0);
  bh[1] = __dmul_rn((double)cc.y, K.ws);
  bh[2] = __dmul_rn((double)cc.z, K.ws);
  bh[3] = __dmul_rn((double)cc.w, K.ws);
}

template <typename T, bool IN_SMEM, bool OUT_SMEM, bool FULL, int PJ>
__device__ __forceinline__ void decompress_rows(const uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj,
                                                T* __restrict__ xo, uint64_t oi, uint64_t oj, int j0,
                                                const LaneGeom& L, const double bh[4], const Consts& K,
                                                const uint32_t R) {
  if (IN_SMEM) { ci = BS * TK; cj = TK; }
  const double cR = __dadd_rn(I2D_MAGIC, (double)R);  // exact: 2^52 + R
#pragma unroll DEC_UNROLL
  for (int jk = 0; jk < 3 * PJ; jk++) {
    const int jj = jk / 3, kk = jk - 3 * jj, j = j0 + jj;
    const bool cv = FULL || ((j < L.m1) && L.kv(kk));
    const double base = __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * L.h + kk), bh[0]));
    const uint16_t* ccol = cs + (IN_SMEM ? (uint32_t)(j * TK + L.kcol + kk) : (uint64_t)j * cj + L.kcol + kk);
    T* ocol = xo + (OUT_SMEM ? (uint32_t)(jj * TK + L.kcol + kk) : (uint64_t)j * oj + L.kcol + kk);
    uint32_t c[BS];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const bool valid = FULL || (cv && i < L.m0);
      if (IN_SMEM || FULL) c[i] = ccol[i * ci];
      else c[i] = valid ? ccol[i * ci] : 0u;
    }
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const bool valid = FULL || (cv && i < L.m0);
      const double p = __fma_rn(bh[1], (double)i, base);
      // (double)(c - R) exactly, without an int->fp conversion: hi/lo = 2^52 + c, minus 2^52 + R
      const double qd = __dsub_rn(__hiloint2double(0x43300000, (int)c[i]), cR);
      const double y = __dadd_rn(p, __dmul_rn(K.twoeb, qd));
      const T xv = c[i] ? from_d<T>(y) : T(0);
      if (OUT_SMEM) ocol[i * (PJ * TK)] = xv;
      else if (valid) ocol[i * oi] = xv;
    }
  }
}

}  // namespace sz3g
