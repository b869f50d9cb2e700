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

namespace sz3g {

constexpr int BS = 6;                          // regression block size B (north_star: 6x6x6)
constexpr int TK = 96;                         // tile extent along dim 2 (16 blocks)
constexpr int TROWS = BS * BS;                 // rows (i,j) per tile
constexpr int TILE_ELEMS = TK * TROWS;         // 3456
constexpr int HWIN = 8192;                     // shared-memory histogram window (bins)
constexpr double RINT_MAGIC = 6755399441055744.0;  // 1.5 * 2^52
constexpr double I2D_MAGIC = 4503599627370496.0;   // 2^52

struct Consts {
  double eb_abs, twoeb, inv2eb, w0, ws, inv_w0, inv_ws;
};

struct Geo {
  uint64_t n0, n1, n2;
  uint32_t NB0, NB1, NB2, NT2;   // blocks per dim; NT2 = tiles along dim 2 = ceil(NB2/16)
  uint64_t ntiles;
  uint64_t gofs;                 // dim0_offset * n1 * n2 (outlier indices are global)
};

// O1/O2 on device: same operations as the definition (IEEE division for the constants).
__device__ __forceinline__ bool make_consts(int eb_mode, double eb, const double* d_minmax, Consts& K) {
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

// unconditional shared-memory add of a 0/1 register (red.shared, no return value): no branch and no
// convergence region around it (a predicated +1 is turned into a warp-collective ATOMS.POPC.INC)
__device__ __forceinline__ void red_smem_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

struct TileCoord {
  uint32_t a, b, c;  // block-row index along dim0, dim1; tile index along dim2
};

__device__ __forceinline__ TileCoord decode_tile(uint64_t t, const Geo& g) {
  TileCoord tc;
  tc.c = (uint32_t)(t % g.NT2);
  uint64_t r = t / g.NT2;
  tc.b = (uint32_t)(r % g.NB1);
  tc.a = (uint32_t)(r / g.NB1);
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
};

// Shared-memory histogram state of one CTA.
struct HistSmem {
  uint32_t* win;   // HWIN bins, window [lo, lo + HWIN)
  uint32_t* zero;  // bin 0 (outliers)
  uint32_t* dummy; // 32 per-lane sink slots for non-counted elements
  uint32_t lo;
  uint32_t nwin;   // bins actually used (min(2R, HWIN))
};

// every element of the tile lies inside the grid (warp-uniform)
__device__ __forceinline__ bool tile_full(const TileCoord tc, const Geo& g) {
  return (uint64_t)(tc.a + 1) * BS <= g.n0 && (uint64_t)(tc.b + 1) * BS <= g.n1 && (uint64_t)(tc.c + 1) * TK <= g.n2;
}

// ------------------------------------------------------------------------------------------
// Compress one tile.  `xs` + (si, sj) address the tile's input: element (i,j,k) of the tile at
// xs[i*si + j*sj + k] (k in [0,96)); it is either a shared-memory stage (si = 576, sj = 96, all
// 3456 entries valid, zero outside the grid) or the global field itself (IN_SMEM = false: loads
// are predicated on the grid bounds).  Codes go to `cs` + (ci, cj) likewise (shared staging
// buffer or the global code array).
// ------------------------------------------------------------------------------------------
template <typename T, bool IN_SMEM, bool HIST, bool FULL>
__device__ __forceinline__ void compress_tile(const T* __restrict__ xs, uint64_t si, uint64_t sj,
                                              uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj,
                                              const TileCoord tc, const Geo& g, const Consts& K,
                                              const uint32_t R, const CompressOut<T>& o, const HistSmem& hs) {
  const int lane = threadIdx.x & 31;
  const int bl = lane >> 1, h = lane & 1;
  const uint32_t kb = tc.c * 16u + (uint32_t)bl;          // block index along dim 2
  const int m0 = (int)umin64(BS, g.n0 - (uint64_t)tc.a * BS);
  const int m1 = (int)umin64(BS, g.n1 - (uint64_t)tc.b * BS);
  const int m2 = (kb < g.NB2) ? (int)umin64(BS, g.n2 - (uint64_t)kb * BS) : 0;
  const int kcol = 6 * bl + 3 * h;                        // first tile column of this lane
  // validity of the lane's three columns
  const bool kv0 = 3 * h + 0 < m2, kv1 = 3 * h + 1 < m2, kv2 = 3 * h + 2 < m2;

  // ---------------- O4: moments V0, Vx, Vy, Vz (fp64).  Row sums S = f0+f1+f2 and the lane's
  // k-weighted sum K = f1 + 2 f2 first, then P_i = sum_j S, Q_i = sum_j j S, Z_i = sum_j K.
  double V0 = 0.0, Vx = 0.0, Vy = 0.0, Vz = 0.0;
#pragma unroll 1
  for (int i = 0; i < BS; i++) {
    double P = 0.0, Q = 0.0, Z = 0.0;
#pragma unroll
    for (int j = 0; j < BS; j++) {
      const T* row = xs + i * si + j * sj + kcol;
      double f0, f1, f2;
      if (IN_SMEM) {
        f0 = to_d<T>(row[0]); f1 = to_d<T>(row[1]); f2 = to_d<T>(row[2]);
      } else {
        const bool rv = (i < m0) && (j < m1);
        f0 = (rv && kv0) ? to_d<T>(row[0]) : 0.0;
        f1 = (rv && kv1) ? to_d<T>(row[1]) : 0.0;
        f2 = (rv && kv2) ? to_d<T>(row[2]) : 0.0;
      }
      const double S = (f0 + f1) + f2;
      const double Kw = fma(2.0, f2, f1);
      P += S;
      Q = fma((double)j, S, Q);
      Z += Kw;
    }
    V0 += P;
    Vx = fma((double)i, P, Vx);
    Vy += Q;
    Vz += Z;
  }
  Vz = fma(3.0 * h, V0, Vz);
  V0 += __shfl_xor_sync(0xffffffffu, V0, 1);
  Vx += __shfl_xor_sync(0xffffffffu, Vx, 1);
  Vy += __shfl_xor_sync(0xffffffffu, Vy, 1);
  Vz += __shfl_xor_sync(0xffffffffu, Vz, 1);

  // ---------------- O5: Lemma 1; extent-1 axis -> slope 0 (G2)
  const bool blk_ok = m2 > 0 && m0 > 0 && m1 > 0;
  double beta[4] = {0.0, 0.0, 0.0, 0.0};
  if (blk_ok) {
    const double Nb = (double)(m0 * m1 * m2);
    const double invNb = __drcp_rn(Nb);
    const double Vd[3] = {Vx, Vy, Vz};
    const int md[3] = {m0, m1, m2};
#pragma unroll
    for (int d = 0; d < 3; d++) {
      if (md[d] > 1) {
        const double sc = c_lemma[md[d]][0] * invNb;
        const double inner = fma(Vd[d], c_lemma[md[d]][1], -V0);
        beta[d + 1] = sc * inner;
      }
    }
    beta[0] = V0 * invNb - ((m0 - 1) * 0.5 * beta[1] + (m1 - 1) * 0.5 * beta[2] + (m2 - 1) * 0.5 * beta[3]);
  }
  // ---------------- O6: coefficient codes (bins eb/2, eb/12; G1), zero predictor fallback
  int32_t cc[4];
  {
    double r[4];
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 4; d++) {
      r[d] = rint(beta[d] * (d == 0 ? K.inv_w0 : K.inv_ws));
      bad |= !(fabs(r[d]) <= 2147483647.0);
    }
#pragma unroll
    for (int d = 0; d < 4; d++) cc[d] = bad ? 0 : __double2int_rn(r[d]);
  }
  const double bh0 = __dmul_rn((double)cc[0], K.w0);
  const double bh1 = __dmul_rn((double)cc[1], K.ws);
  const double bh2 = __dmul_rn((double)cc[2], K.ws);
  const double bh3 = __dmul_rn((double)cc[3], K.ws);
  const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + kb;
  if (blk_ok && h == 0) {
    reinterpret_cast<int4*>(o.coef)[bid] = make_int4(cc[0], cc[1], cc[2], cc[3]);
    if (o.coef_raw) {
      reinterpret_cast<double2*>(o.coef_raw)[2 * bid] = make_double2(beta[0], beta[1]);
      reinterpret_cast<double2*>(o.coef_raw)[2 * bid + 1] = make_double2(beta[2], beta[3]);
    }
  }

  // ---------------- O7-O11 per element, branch-free: 18 independent elements per j (3 k-columns x
  // 6 i-planes) so the fp64 chains interleave.  FULL tiles (every element inside the grid) skip all
  // validity predicates.  The histogram takes one red.shared per element at the code clamped into
  // the smem window; codes outside it (and outliers, code 0) are detected from the lane's running
  // min / max code and corrected by the rare slow path below, which also appends the outliers.
  //
  // ok = |q| < R && |x' - x| <= eb is O8-O9 exactly: for |t| < 2^51, q = rint(t) and |t| >= R implies
  // |rint(t)| >= R (R integer, rint monotone); for |t| >= 2^51, NaN or Inf, |q| < R is false.  The
  // verify compare uses <=, which agrees with !(> eb) whenever |q| < R (then d is finite or +-Inf).
  const double Rd = (double)R;
  const uint32_t win_base = (uint32_t)__cvta_generic_to_shared(hs.win) - 4u * hs.lo;  // &win[c - lo] = base + 4c
  const uint32_t sink = HIST ? (uint32_t)__cvta_generic_to_shared(hs.dummy) + 4u * lane : 0u;
  const uint32_t wlo = hs.lo, whi = hs.lo + hs.nwin - 1u;
  uint32_t cmin = 0xffffffffu, cmax = 0u;
#pragma unroll 1
  for (int jk = 0; jk < 3 * BS; jk++) {
    const int j = jk / 3, kk = jk - 3 * j;
    const bool cv = FULL || ((j < m1) && (kk == 0 ? kv0 : (kk == 1 ? kv1 : kv2)));
    T xv[BS];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const bool valid = FULL || (cv && i < m0);
      if (IN_SMEM || FULL) xv[i] = xs[i * si + j * sj + kcol + kk];
      else xv[i] = valid ? xs[i * si + j * sj + kcol + kk] : T(0);
    }
    // O7 hoisted: base = fma(b2, j, fma(b3, k, b0)), p = fma(b1, i, base)
    const double base = __fma_rn(bh2, (double)j, __fma_rn(bh3, (double)(3 * h + kk), bh0));
    uint32_t code[BS];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const double xd = to_d<T>(xv[i]);
      const double p = __fma_rn(bh1, (double)i, base);
      // O8: t = (x - p) * inv2eb ; q = rint(t) (1.5*2^52 trick, ties-to-even)
      const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
      const double sm = __dadd_rn(t, RINT_MAGIC);
      const double q = __dsub_rn(sm, RINT_MAGIC);
      // O9: x' = (T)(p + twoeb*q), verify |x' - x| <= eb
      const double y = __dadd_rn(p, __dmul_rn(K.twoeb, q));
      const double d = __dsub_rn(to_d<T>(from_d<T>(y)), xd);
      const bool ok = (fabs(q) < Rd) && (fabs(d) <= K.eb_abs);
      code[i] = ok ? (uint32_t)(__double2loint(sm) + (int)R) : 0u;   // O10
    }
#pragma unroll
    for (int i = 0; i < BS; i++) {
      const bool valid = FULL || (cv && i < m0);
      const uint32_t c = code[i];
      if (valid) cs[i * ci + j * cj + kcol + kk] = (uint16_t)c;
      if (FULL) {
        cmin = min(cmin, c);
        cmax = max(cmax, c);
      } else if (valid) {
        cmin = min(cmin, c);
        cmax = max(cmax, c);
      }
      if (HIST) {  // O11
        const uint32_t cw = min(max(c, wlo), whi);
        red_smem_add(FULL ? win_base + 4u * cw : (valid ? win_base + 4u * cw : sink), FULL ? 1u : (valid ? 1u : 0u));
      }
    }
  }

  // ---------------- slow path (rare): outliers -> (global index, value), warp-aggregated append;
  // histogram correction for codes outside the window [wlo, whi] (counted at the clamped bin).
  const bool has_out = cmin == 0u;
  const bool has_spill = HIST && (cmin < wlo || cmax > whi);
  if (__any_sync(0xffffffffu, has_out || has_spill)) {
    uint32_t nout = 0;
    if (has_out || has_spill) {
      for (int j = 0; j < m1; j++)
        for (int kk = 0; kk < 3; kk++) {
          if (!(kk == 0 ? kv0 : (kk == 1 ? kv1 : kv2))) continue;
          for (int i = 0; i < m0; i++) {
            const uint32_t c = cs[i * ci + j * cj + kcol + kk];
            nout += (c == 0u) ? 1u : 0u;
            if (HIST && c != 0u && (c < wlo || c > whi)) {
              atomicSub(&hs.win[min(max(c, wlo), whi) - wlo], 1u);
              atomicAdd(&o.hist[c], 1ull);
            }
          }
        }
    }
    uint32_t incl = nout;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total) {
      unsigned long long basepos = 0;
      if (lane == 31) {
        basepos = atomicAdd(o.ocount, (unsigned long long)total);
        if (HIST && wlo > 0u) {  // outliers were counted at the clamped bin wlo
          atomicSub(&hs.win[0], total);
          atomicAdd(hs.zero, total);
        }
      }
      basepos = __shfl_sync(0xffffffffu, basepos, 31);
      unsigned long long pos = basepos + (incl - nout);
      if (nout) {
        const uint64_t gbase =
            g.gofs + ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)kb * BS + 3 * h;
        for (int j = 0; j < m1; j++)
          for (int kk = 0; kk < 3; kk++) {
            if (!(kk == 0 ? kv0 : (kk == 1 ? kv1 : kv2))) continue;
            for (int i = 0; i < m0; i++) {
              if (cs[i * ci + j * cj + kcol + kk] != 0) continue;
              if (pos < o.cap) {
                o.oidx[pos] = gbase + ((uint64_t)i * g.n1 + j) * g.n2 + kk;
                o.oval[pos] = xs[i * si + j * sj + kcol + kk];
              }
              pos++;
            }
          }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Decompress one tile (recover): x' = (T)(p + twoeb*(c - R)) for c != 0, 0 for c == 0
// (outlier values are scattered afterwards).  Codes read from cs + (ci, cj) (smem stage or
// global, predicated), x' written to xo + (oi, oj) (smem staging or global, predicated).
// ------------------------------------------------------------------------------------------
template <typename T, bool IN_SMEM, bool OUT_SMEM>
__device__ __forceinline__ void decompress_tile(const uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj,
                                                T* __restrict__ xo, uint64_t oi, uint64_t oj, const TileCoord tc,
                                                const Geo& g, const Consts& K, const uint32_t R,
                                                const int32_t* __restrict__ coef) {
  const int lane = threadIdx.x & 31;
  const int bl = lane >> 1, h = lane & 1;
  const uint32_t kb = tc.c * 16u + (uint32_t)bl;
  const int m0 = (int)umin64(BS, g.n0 - (uint64_t)tc.a * BS);
  const int m1 = (int)umin64(BS, g.n1 - (uint64_t)tc.b * BS);
  const int m2 = (kb < g.NB2) ? (int)umin64(BS, g.n2 - (uint64_t)kb * BS) : 0;
  const int kcol = 6 * bl + 3 * h;
  int4 cc = make_int4(0, 0, 0, 0);
  const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + kb;
  if (m2 > 0) cc = __ldg(reinterpret_cast<const int4*>(coef) + bid);
  const double bh0 = __dmul_rn((double)cc.x, K.w0);
  const double bh1 = __dmul_rn((double)cc.y, K.ws);
  const double bh2 = __dmul_rn((double)cc.z, K.ws);
  const double bh3 = __dmul_rn((double)cc.w, K.ws);
  const double cR = __dadd_rn(I2D_MAGIC, (double)R);  // exact: 2^52 + R
#pragma unroll 1
  for (int j = 0; j < BS; j++) {
#pragma unroll
    for (int kk = 0; kk < 3; kk++) {
      const bool kv = (3 * h + kk < m2) && (j < m1);
      const double base = __fma_rn(bh2, (double)j, __fma_rn(bh3, (double)(3 * h + kk), bh0));
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = kv && (i < m0);
        uint32_t c;
        if (IN_SMEM) c = cs[i * ci + j * cj + kcol + kk];
        else c = valid ? cs[i * ci + j * cj + kcol + kk] : 0u;
        const double p = __fma_rn(bh1, (double)i, base);
        // (double)(c - R) exactly, without an int->fp conversion: hi/lo = 2^52 + c, minus 2^52 + R
        const double qd = __dsub_rn(__hiloint2double(0x43300000, (int)c), cR);
        const double y = __dadd_rn(p, __dmul_rn(K.twoeb, qd));
        const T xv = c ? from_d<T>(y) : T(0);
        if (OUT_SMEM || valid) xo[i * oi + j * oj + kcol + kk] = xv;
      }
    }
  }
}

}  // namespace sz3g
