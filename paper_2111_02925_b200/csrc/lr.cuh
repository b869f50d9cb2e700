// libsz3g -- SZ3-LR (NEXT-4): the composite Lorenzo / regression predictor, "predicts data using the
// better result in between based on blockwise error estimation".  Definition:
// oracle/DEFINITION.md L1-L7 (readings DESIGN G26-G29):
//   L1 q = rint(x * inv2eb) (0 and unusable if |x * inv2eb| >= 2^50 or x is not finite);
//   L2 delta = block-local first-order 3D Lorenzo residual of q (zero outside the block);
//   L3 Lorenzo code R + delta if |delta| < R and x' = (T)(twoeb * q) is within eb, else an outlier;
//   L4 regression codes O7-O10 from the analyze pass's beta;
//   L5 the block takes the predictor with the smaller sum of |code - R| (outliers count R; ties ->
//      regression);  L6 flag per block, coefficient codes 0 for Lorenzo blocks;
//   L7 decompression: outliers scattered first, Lorenzo blocks rebuild q by an exact integer
//      recurrence, x' = (T)(twoeb * q).
// Included by sz3g.cu inside its anonymous namespace (KArgs, TileWalk, histogram helpers, rare_path).
//
// Compression: one warp per 6x6x96 tile (16 blocks, 2 lanes per block, 3 columns per lane, as every
// tile routine of this library).  Each lane walks its 108 elements plane by plane, row by row: the
// regression code by the definition's fp64 arithmetic (exact_code), q by the magic-number rint, and the
// Lorenzo residual as three differences -- along k within the lane plus one shuffle from the block's
// other lane, along j against the previous row (registers), along i against the previous plane (6 rows
// x 3 columns of int64 in registers).  Both codes go to two shared code slabs; after the two lanes of a
// block have summed their costs the chosen codes are emitted (global store, shared histogram window,
// outliers through rare_path).  TMA kernel: W self-fed warps per CTA, each with a private 2-stage ring
// of tiles (as k_analyze_tma).

constexpr double LR_QMAX = 1125899906842624.0;   // 2^50 (L1)
constexpr int LR_HW = 4096;                       // histogram window (bins) of the LR kernels

// L1 for one element: q as an exact double (|q| < 2^50) and whether it is usable
__device__ __forceinline__ double lr_prequant(double xd, const Consts& K, bool& ok) {
  const double t = __dmul_rn(xd, K.inv2eb);
  ok = fabs(t) < LR_QMAX;
  const double q = __dsub_rn(__dadd_rn(t, RINT_MAGIC), RINT_MAGIC);   // rint, ties to even (|t| < 2^51)
  return ok ? q : 0.0;
}

// Where a tile's Lorenzo codes live: a u16 slab, or (TMA kernel) the lane's own element slots of the
// tile stage, each overwritten once its x has been read (a lane only ever reads its own elements of the
// stage; outlier values then come from the field in global memory).
struct LrSlabL {
  uint16_t* s16;
  uint32_t* s32;   // non-null: the code of element s is s32[s * w]
  int w;
  __device__ __forceinline__ void put(uint32_t s, uint32_t c) const {
    if (s32) s32[s * w] = c;
    else s16[s] = (uint16_t)c;
  }
  __device__ __forceinline__ uint16_t get(uint32_t s) const { return s32 ? (uint16_t)s32[s * w] : s16[s]; }
};

// ox / osi / osj: where the outliers' values are read (the stage, or the field when the stage holds codes)
template <typename T, bool IN_SMEM, bool FULL, bool TMA_OUT>
__device__ __forceinline__ void lr_emit(const T* __restrict__ ox, uint64_t osi, uint64_t osj, uint16_t* sR,
                                        const LrSlabL& sL, uint32_t costR, uint32_t costL, const int32_t cc[4],
                                        uint64_t bid, const LaneGeom& L, const TileCoord tc, const Geo& g,
                                        const CompressOut<T>& o, uint8_t* __restrict__ flags, const HistSmem& hs,
                                        const CUtensorMap* tm_c);

// One warp, one tile.  xs: the tile (shared stage, si = 576, sj = 96, zero outside the grid) or the
// field (IN_SMEM = false, predicated loads).  sR / sL: the warp's two code slabs [i][j][k] (6 x 6 x 96).
template <typename T, bool IN_SMEM, bool FULL, bool TMA_OUT>
__device__ __forceinline__ void lr_compress_tile_exact(const T* __restrict__ xs, uint64_t si, uint64_t sj, uint16_t* sR,
                                                 const LrSlabL& sL, const TileCoord tc, const Geo& g, const Consts& K,
                                                 uint32_t R, const CompressOut<T>& o, uint8_t* __restrict__ flags,
                                                 const HistSmem& hs, const CUtensorMap* tm_c) {
  const LaneGeom L = lane_geom<FULL>(tc, g);
  const int h = L.h;
  double beta[4] = {0.0, 0.0, 0.0, 0.0}, bh[4];
  int32_t cc[4];
  const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
  if (L.m2 > 0) {
    const double2 b01 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid);
    const double2 b23 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid + 1);
    beta[0] = b01.x; beta[1] = b01.y; beta[2] = b23.x; beta[3] = b23.y;
  }
  block_codes(beta, K, cc, bh);
  const double dR = (double)R;
  uint32_t costR = 0, costL = 0;
  int64_t pdj[BS][3];   // j-differences of the previous plane, per row
#pragma unroll
  for (int j = 0; j < BS; j++) pdj[j][0] = pdj[j][1] = pdj[j][2] = 0;
  for (int i = 0; i < BS; i++) {
    int64_t pdk[3] = {0, 0, 0};   // k-differences of the previous row
#pragma unroll
    for (int j = 0; j < BS; j++) {
      int64_t q[3];
      uint32_t cr[3];
      bool ok[3], valid[3];
      double xd[3], qd[3];
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        valid[kk] = FULL || (i < L.m0 && j < L.m1 && L.kv(kk));
        const uint64_t off = (uint64_t)i * si + (uint64_t)j * sj + L.kcol + kk;
        const T xv = (IN_SMEM || valid[kk]) ? xs[off] : T(0);
        xd[kk] = to_d<T>(xv);
        const double p = __fma_rn(bh[1], (double)i, __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * h + kk), bh[0])));
        cr[kk] = valid[kk] ? exact_code<T>(xv, p, K, R) : R;
        qd[kk] = lr_prequant(xd[kk], K, ok[kk]);
        if (!valid[kk]) { ok[kk] = false; qd[kk] = 0.0; }   // outside the block: q = 0
        q[kk] = (int64_t)__double2ll_rn(qd[kk]);
      }
      // L2 as three differences: k (the block's left lane supplies column 3h - 1), j, i
      int64_t left = __shfl_up_sync(0xffffffffu, q[2], 1);
      if (h == 0) left = 0;
      const int64_t dk[3] = {q[0] - left, q[1] - q[0], q[2] - q[1]};
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        const int64_t dj = dk[kk] - pdk[kk];
        const int64_t delta = dj - pdj[j][kk];
        pdk[kk] = dk[kk];
        pdj[j][kk] = dj;
        uint32_t cl = 0;
        if (ok[kk] && delta > -(int64_t)R && delta < (int64_t)R) {
          const T xr = from_d<T>(__dmul_rn(K.twoeb, qd[kk]));
          if (fabs(__dsub_rn(to_d<T>(xr), xd[kk])) <= K.eb_abs) cl = (uint32_t)((int64_t)R + delta);
        }
        if (!valid[kk]) cl = R;
        costR += cr[kk] ? (uint32_t)fabs((double)cr[kk] - dR) : R;
        costL += cl ? (uint32_t)fabs((double)cl - dR) : R;
        const uint32_t s = (uint32_t)(i * (BS * TK) + j * TK + L.kcol + kk);
        sR[s] = (uint16_t)cr[kk];
        sL.put(s, cl);
      }
    }
  }
  lr_emit<T, IN_SMEM, FULL, TMA_OUT>(xs, si, sj, sR, sL, costR, costL, cc, bid, L, tc, g, o, flags, hs, tm_c);
}

// L5 + L6 for one tile whose regression / Lorenzo codes are in the slabs sR / sL: the lanes of
// Lorenzo blocks copy their codes over sR, then every valid element's final code is read once
// (histogram, outliers through rare_path) and the tile leaves with one TMA store of sR (TMA_OUT) or
// element stores.  With TMA_OUT the caller waits for the store's reads before sR is written again.
template <typename T, bool IN_SMEM, bool FULL, bool TMA_OUT>
__device__ __forceinline__ void lr_emit(const T* __restrict__ ox, uint64_t osi, uint64_t osj, uint16_t* sR,
                                        const LrSlabL& sL, uint32_t costR, uint32_t costL, const int32_t cc[4],
                                        uint64_t bid, const LaneGeom& L, const TileCoord tc, const Geo& g,
                                        const CompressOut<T>& o, uint8_t* __restrict__ flags, const HistSmem& hs,
                                        const CUtensorMap* tm_c) {
  const int h = L.h;
  SZ3G_SYNCWARP();
  // L5: the block's two lanes sum their costs
  costR += __shfl_xor_sync(0xffffffffu, costR, 1);
  costL += __shfl_xor_sync(0xffffffffu, costL, 1);
  const bool useL = costL < costR;
  if (L.m2 > 0 && h == 0) {
    reinterpret_cast<int4*>(o.coef)[bid] = useL ? make_int4(0, 0, 0, 0) : make_int4(cc[0], cc[1], cc[2], cc[3]);
    flags[bid] = useL ? 1 : 0;
  }
  if (useL) {
#pragma unroll 1
    for (int i = 0; i < BS; i++)
#pragma unroll
      for (int j = 0; j < BS; j++)
#pragma unroll
        for (int kk = 0; kk < 3; kk++) {
          const uint32_t s = (uint32_t)(i * (BS * TK) + j * TK + L.kcol + kk);
          sR[s] = sL.get(s);
        }
  }
  bool has_out = false;
  const uint64_t gbase = ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)tc.c * TK;
  // histogram as in quantize_rows: one unconditional shared reduction per element into the window (or
  // the lane's sink), which the hardware aggregates per address within the warp; codes outside the
  // window (rare) go to the global bins
  const uint32_t hb = (uint32_t)__cvta_generic_to_shared(hs.win) - 4u * hs.lo;
  const uint32_t sink = (uint32_t)__cvta_generic_to_shared(hs.dummy) + 4u * (threadIdx.x & 31);
  const bool hist = o.hist != nullptr;
#pragma unroll 1
  for (int i = 0; i < BS; i++)
#pragma unroll
    for (int j = 0; j < BS; j++)
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        const bool valid = FULL || (i < L.m0 && j < L.m1 && L.kv(kk));
        const uint32_t code = sR[(uint32_t)(i * (BS * TK) + j * TK + L.kcol + kk)];
        if (!TMA_OUT && valid) o.codes[gbase + ((uint64_t)i * g.n1 + j) * g.n2 + L.kcol + kk] = (uint16_t)code;
        const bool inwin = valid && code != 0u && code - hs.lo < hs.nwin;
        if (hist) {
          red_smem_add(inwin ? hb + 4u * code : sink, 1u);
          if (valid && code != 0u && !inwin) atomicAdd(&o.hist[code], 1ull);
        }
        has_out |= valid && code == 0u;
      }
  SZ3G_SYNCWARP();
  if (TMA_OUT) {
    ptx::fence_proxy_async_smem();
    SZ3G_SYNCWARP();
    if ((threadIdx.x & 31) == 0) {
      ptx::tma_store_3d(tm_c, sR, (int)(tc.c * TK), (int)(tc.b * BS), (int)(tc.a * BS));
      ptx::bulk_commit();
    }
  }
  if (o.hist) rare_path<T, true, BS>(ox, osi, osj, sR, BS * TK, TK, 0, 0, L, has_out, tc, g, o, hs);
  else rare_path<T, false, BS>(ox, osi, osj, sR, BS * TK, TK, 0, 0, L, has_out, tc, g, o, hs);
  SZ3G_SYNCWARP();
}

// The exact definitions for one element, out of line (the fast routine's rare fallback)
struct LrExact {
  uint32_t cr;   // regression code (O7-O10)
  int32_t q;     // L1 q (0 if unusable or beyond the int32 residual range)
  bool lv;       // Lorenzo-usable: q usable and (T)(twoeb q) within eb
  bool big;      // |q| >= 2^26: the tile needs the int64 routine
};
template <typename T>
__device__ __noinline__ LrExact lr_exact_elem(T xv, double b0, double b1, double b2, double b3, int i, int j, int k,
                                             const Consts& K, uint32_t R, bool want_cr, bool want_l) {
  LrExact r{0u, 0, false, false};
  if (want_cr) r.cr = exact_code<T>(xv, __fma_rn(b1, (double)i, __fma_rn(b2, (double)j, __fma_rn(b3, (double)k, b0))), K, R);
  if (want_l) {
    bool okq;
    const double xd = to_d<T>(xv);
    const double qd = lr_prequant(xd, K, okq);
    r.big = okq && fabs(qd) >= 67108864.0;
    r.q = (okq && !r.big) ? (int32_t)qd : 0;
    r.lv = okq && fabs(__dsub_rn(to_d<T>(from_d<T>(__dmul_rn(K.twoeb, qd))), xd)) <= K.eb_abs;
  }
  return r;
}

// The fast routine: the tile's (j, k) columns with the six i-planes in registers (as quantize_rows).
// Regression codes by the library's certified fast test (fp32 scaled domain for f32 data, the fp64
// fast verify for f64; make_consts / fast32_consts), the exact definition for the rest (warp vote).
// Lorenzo: L1 + L3's bound check are the SAME test with a zero predictor (q = rint(x inv2eb), x' =
// (T)(0 + twoeb q) = (T)(twoeb q)), so the zero-coefficient constants certify q and the bound; the
// |t| < 2^22 guard keeps the fp32 magic rounding exact.  Residuals in int32: usable while every |q| <
// 2^26 (|delta| < 2^29); a tile with a larger q (or a fallback q beyond that) is redone by
// lr_compress_tile_exact (returns false).
template <typename T, bool IN_SMEM, bool FULL, bool TMA_OUT>
__device__ __forceinline__ bool lr_compress_tile_fast(const T* __restrict__ xs, uint64_t si, uint64_t sj, uint16_t* sR,
                                                      const LrSlabL& sL, const T* __restrict__ ox, uint64_t osi,
                                                      uint64_t osj, const TileCoord tc, const Geo& g, const Consts& K,
                                                      uint32_t R, const CompressOut<T>& o, uint8_t* __restrict__ flags,
                                                      const HistSmem& hs, const CUtensorMap* tm_c) {
  constexpr bool F32 = sizeof(T) == 4;
  const LaneGeom L = lane_geom<FULL>(tc, g);
  const int h = L.h;
  double beta[4] = {0.0, 0.0, 0.0, 0.0}, bh[4];
  int32_t cc[4];
  const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
  if (L.m2 > 0) {
    const double2 b01 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid);
    const double2 b23 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid + 1);
    beta[0] = b01.x; beta[1] = b01.y; beta[2] = b23.x; beta[3] = b23.y;
  }
  block_codes(beta, K, cc, bh);
  const Fast32 F = fast32_consts(bh, K);
  const double zero[4] = {0.0, 0.0, 0.0, 0.0};
  const Fast32 F0 = fast32_consts(zero, K);
  const float inv2eb32 = K.inv2eb32;
  const float M32 = 12582912.0f;                 // 1.5 * 2^23
  const float Rf = (float)R;
  const int iR = (int)R;
  if (IN_SMEM) { si = BS * TK; sj = TK; }
  uint32_t costR = 0, costL = 0;
  bool big = false;
  int32_t Dp[3][BS];   // k-differences of the previous row
#pragma unroll
  for (int kk = 0; kk < 3; kk++)
#pragma unroll
    for (int i = 0; i < BS; i++) Dp[kk][i] = 0;
#pragma unroll 1
  for (int j = 0; j < BS; j++) {
    int32_t q[3][BS];
    uint32_t cr[3][BS];
    bool lv[3][BS];   // Lorenzo-usable: q certified (or exact) and x' = (T)(twoeb q) within eb
    const float fj = (float)j;
#pragma unroll
    for (int kk = 0; kk < 3; kk++) {
      const bool cv = FULL || ((j < L.m1) && L.kv(kk));
      T xv[BS];
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = FULL || (cv && i < L.m0);
        const uint64_t off = (uint64_t)i * si + (uint64_t)j * sj + L.kcol + kk;
        xv[i] = (IN_SMEM || FULL || valid) ? xs[off] : T(0);
      }
      bool need = false;
      if (F32) {
        const float base32 = __fmaf_rn(F.a2, fj, __fmaf_rn(F.a3, (float)(3 * h + kk), F.a0));
#pragma unroll
        for (int i = 0; i < BS; i++) {
          const bool valid = FULL || (cv && i < L.m0);
          const float x32 = (float)xv[i];
          // regression (fast32_consts: certified rint and bound)
          const float P = i == 0 ? base32 : __fmaf_rn(F.a1, (float)i, base32);
          const float t32 = __fmaf_rn(x32, inv2eb32, -P);
          const float r = __fsub_rn(__fadd_rn(t32, M32), M32);
          const float e = __fsub_rn(t32, r);
          const bool ok = __fmaf_rn(F.k1, fabsf(t32), fabsf(e)) <= F.thr && fabsf(r) < Rf;
          cr[kk][i] = ok ? (uint32_t)((int)r + iR) : 0u;
          need |= valid && !ok;
          // Lorenzo prequantisation (zero predictor)
          const float tL = __fmul_rn(x32, inv2eb32);
          const float sLm = __fadd_rn(tL, M32);
          const float rL = __fsub_rn(sLm, M32);
          const float eL = __fsub_rn(tL, rL);
          const bool okL = __fmaf_rn(F0.k1, fabsf(tL), fabsf(eL)) <= F0.thr && fabsf(tL) < 4194304.0f;
          q[kk][i] = okL ? (int32_t)rL : 0;
          lv[kk][i] = okL;
          need |= valid && !okL;
        }
      } else {
        const double base = __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * h + kk), bh[0]));
#pragma unroll
        for (int i = 0; i < BS; i++) {
          const bool valid = FULL || (cv && i < L.m0);
          const double xd = to_d<T>(xv[i]);
          const double p = __fma_rn(bh[1], (double)i, base);
          const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
          const double rq = __dsub_rn(__dadd_rn(t, RINT_MAGIC), RINT_MAGIC);
          const bool ok = __fma_rn(K.vc, fabs(xd), fabs(__dsub_rn(t, rq))) <= K.vthr && fabs(rq) < (double)R;
          cr[kk][i] = ok ? (uint32_t)((int)rq + iR) : 0u;
          need |= valid && !ok;
          const double tL = __dmul_rn(xd, K.inv2eb);
          const double rL = __dsub_rn(__dadd_rn(tL, RINT_MAGIC), RINT_MAGIC);
          const bool okL = __fma_rn(K.vc, fabs(xd), fabs(__dsub_rn(tL, rL))) <= K.vthr && fabs(tL) < 67108864.0;
          q[kk][i] = okL ? (int32_t)rL : 0;
          lv[kk][i] = okL;
          need |= valid && !okL;
        }
      }
      if (__any_sync(0xffffffffu, need)) {   // the exact definitions (rare; out of line: small hot loop)
#pragma unroll
        for (int i = 0; i < BS; i++) {
          const bool valid = FULL || (cv && i < L.m0);
          if (valid && (cr[kk][i] == 0u || !lv[kk][i])) {
            const LrExact ex = lr_exact_elem<T>(xv[i], bh[0], bh[1], bh[2], bh[3], i, j, 3 * h + kk, K, R,
                                                cr[kk][i] == 0u, !lv[kk][i]);
            if (cr[kk][i] == 0u) cr[kk][i] = ex.cr;
            if (!lv[kk][i]) {
              big |= ex.big;
              q[kk][i] = ex.q;
              lv[kk][i] = ex.lv;
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = FULL || (cv && i < L.m0);
        if (!valid) { q[kk][i] = 0; lv[kk][i] = false; cr[kk][i] = R; }
      }
    }
    // L2: k-difference (the block's left lane supplies column 3h - 1), j-difference, i-difference
    int32_t left[BS];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      left[i] = __shfl_up_sync(0xffffffffu, q[2][i], 1);
      if (h == 0) left[i] = 0;
    }
#pragma unroll
    for (int kk = 0; kk < 3; kk++) {
      const bool cv = FULL || ((j < L.m1) && L.kv(kk));
      int32_t Eprev = 0;
#pragma unroll
      for (int i = 0; i < BS; i++) {
        const bool valid = FULL || (cv && i < L.m0);
        const int32_t D = q[kk][i] - (kk == 0 ? left[i] : q[kk - 1][i]);
        const int32_t E = D - Dp[kk][i];
        Dp[kk][i] = D;
        const int32_t delta = E - Eprev;
        Eprev = E;
        uint32_t cl = (lv[kk][i] && delta > -iR && delta < iR) ? (uint32_t)(delta + iR) : 0u;
        if (!valid) cl = R;
        const uint32_t c = cr[kk][i];
        costR += c ? (uint32_t)abs((int)c - iR) : R;
        costL += cl ? (uint32_t)abs((int)cl - iR) : R;
        const uint32_t sidx = (uint32_t)(i * (BS * TK) + j * TK + L.kcol + kk);
        sR[sidx] = (uint16_t)c;
        sL.put(sidx, cl);
      }
    }
  }
  if (__any_sync(0xffffffffu, big)) return false;
  lr_emit<T, IN_SMEM, FULL, TMA_OUT>(ox, osi, osj, sR, sL, costR, costL, cc, bid, L, tc, g, o, flags, hs, tm_c);
  return true;
}

// xs / si / sj: the tile (stage or field); xg: the tile in the field (global strides).  With sL in the
// stage the exact fallback reads the field (the stage may already hold codes).
template <typename T, bool IN_SMEM, bool FULL, bool TMA_OUT>
__device__ __forceinline__ void lr_compress_tile(const T* __restrict__ xs, uint64_t si, uint64_t sj, const T* __restrict__ xg,
                                                 uint16_t* sR, const LrSlabL& sL, const TileCoord tc, const Geo& g,
                                                 const Consts& K, uint32_t R, const CompressOut<T>& o,
                                                 uint8_t* __restrict__ flags, const HistSmem& hs, const CUtensorMap* tm_c) {
#ifndef SZ3G_LR_FAST
#define SZ3G_LR_FAST 1   // the certified fp32 routine first, the exact one for tiles with |q| >= 2^26
#endif
  const bool in_stage = sL.s32 != nullptr;
  if (SZ3G_LR_FAST && lr_compress_tile_fast<T, IN_SMEM, FULL, TMA_OUT>(
                          xs, si, sj, sR, sL, in_stage ? xg : xs, in_stage ? g.n1 * g.n2 : si, in_stage ? g.n2 : sj,
                          tc, g, K, R, o, flags, hs, tm_c))
    return;
  if (in_stage || !IN_SMEM)
    lr_compress_tile_exact<T, false, FULL, TMA_OUT>(xg, g.n1 * g.n2, g.n2, sR, sL, tc, g, K, R, o, flags, hs, tm_c);
  else
    lr_compress_tile_exact<T, IN_SMEM, FULL, TMA_OUT>(xs, si, sj, sR, sL, tc, g, K, R, o, flags, hs, tm_c);
}

template <typename T, int W, int D>
struct LrSmem {
  static constexpr size_t stage_bytes = sizeof(T) * TILE_ELEMS;
  static constexpr size_t slab_bytes = sizeof(uint16_t) * TILE_ELEMS;   // regression (then final) codes
  static constexpr size_t off_slab = (size_t)W * D * stage_bytes;
  static constexpr size_t off_hist = off_slab + (size_t)W * slab_bytes;
  static constexpr size_t off_bar = off_hist + sizeof(uint32_t) * (LR_HW + 36);
  static constexpr size_t off_k = off_bar + (size_t)W * D * sizeof(uint64_t);
  static constexpr size_t total = off_k + sizeof(Consts) + 16;
};

// Persistent, W self-fed warps per CTA (each with a private D-stage TMA ring, as k_analyze_tma).
template <typename T, int W, int D>
__global__ void __launch_bounds__(W * 32, 1)
    k_lr_compress_tma(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_c,
                      const T* __restrict__ x, KArgs a, CompressOut<T> o, uint8_t* __restrict__ flags) {
  using L_ = LrSmem<T, W, D>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L_::off_bar);
  Consts* s_k = reinterpret_cast<Consts*>(smem + L_::off_k);
  int* s_ok = reinterpret_cast<int*>(smem + L_::off_k + sizeof(Consts));
  uint32_t* s_win = reinterpret_cast<uint32_t*>(smem + L_::off_hist);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  HistSmem hs;
  hist_init(hs, s_win, s_win + LR_HW, a.R, LR_HW);
  if (threadIdx.x == 0) {
    for (int s = 0; s < W * D; s++) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbar_init();
  }
  if (!cta_consts(a, s_k, s_ok)) return;
  const Consts K = *s_k;
  const Geo& g = a.g;
  T* ring = reinterpret_cast<T*>(smem) + (size_t)warp * D * TILE_ELEMS;
  uint16_t* sR = reinterpret_cast<uint16_t*>(smem + L_::off_slab + (size_t)warp * L_::slab_bytes);
  uint64_t* bar = full + warp * D;
  TileWalk tw(warp, a.chunk, W), tl(warp, a.chunk, W);
  if (lane == 0) {
    ptx::prefetch_tensormap(&tm_x);
    for (int d = 0; d < D; d++, tl.next()) {
      const uint64_t t = tl.tile();
      if (t >= g.ntiles) break;
      const TileCoord tc = decode_tile(t, g);
      ptx::mbar_arrive_expect_tx(&bar[d], (uint32_t)L_::stage_bytes);
      ptx::tma_load_3d(ring + (size_t)d * TILE_ELEMS, &tm_x, &bar[d], (int)(tc.c * TK), (int)(tc.b * BS), (int)(tc.a * BS));
    }
  }
  for (uint32_t k = 0;; k++, tw.next()) {
    const uint64_t t = tw.tile();
    if (t >= g.ntiles) break;
    const uint32_t s = k % D, ph = (k / D) & 1u;
    const TileCoord tc = decode_tile(t, g);
    if (lane == 0) ptx::bulk_wait_read0();   // the previous tile's code store has read sR
    SZ3G_SYNCWARP();
    ptx::mbar_wait(&bar[s], ph);
    const T* xs = ring + (size_t)s * TILE_ELEMS;
    const LrSlabL sL{nullptr, reinterpret_cast<uint32_t*>(ring + (size_t)s * TILE_ELEMS), (int)(sizeof(T) / 4)};
    const T* xg = x + ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)tc.c * TK;
    if (tile_full(tc, g)) lr_compress_tile<T, true, true, true>(xs, BS * TK, TK, xg, sR, sL, tc, g, K, a.R, o, flags, hs, &tm_c);
    else lr_compress_tile<T, true, false, true>(xs, BS * TK, TK, xg, sR, sL, tc, g, K, a.R, o, flags, hs, &tm_c);
    SZ3G_SYNCWARP();
    if (lane == 0) {   // every lane's reads of the stage are done: refill it with tile k + D
      const uint64_t t2 = tl.tile();
      if (t2 < g.ntiles) {
        const TileCoord tc2 = decode_tile(t2, g);
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive_expect_tx(&bar[s], (uint32_t)L_::stage_bytes);
        ptx::tma_load_3d(ring + (size_t)s * TILE_ELEMS, &tm_x, &bar[s], (int)(tc2.c * TK), (int)(tc2.b * BS),
                         (int)(tc2.a * BS));
      }
      tl.next();
    }
  }
  if (lane == 0) ptx::bulk_wait0();
  SZ3G_SYNCTHREADS();
  if (o.hist) hist_flush(hs, o.hist);
  overflow_check(a, o.ocount, o.cap);
}

// Shapes without a TMA map: one warp per tile straight from the field (4 warps per CTA).
#ifndef SZ3G_LR_PW
#define SZ3G_LR_PW 4
#endif
constexpr int LR_PW = SZ3G_LR_PW;
template <typename T>
__global__ void __launch_bounds__(LR_PW * 32) k_lr_compress_plain(const T* __restrict__ x, KArgs a, CompressOut<T> o,
                                                                  uint8_t* __restrict__ flags) {
  extern __shared__ __align__(16) uint8_t psmem[];
  uint16_t* slabs = reinterpret_cast<uint16_t*>(psmem);
  uint32_t* s_win = reinterpret_cast<uint32_t*>(psmem + (size_t)LR_PW * 2 * TILE_ELEMS * sizeof(uint16_t));
  __shared__ Consts s_k;
  __shared__ int s_ok;
  HistSmem hs;
  hist_init(hs, s_win, s_win + LR_HW, a.R, LR_HW);
  if (!cta_consts(a, &s_k, &s_ok)) return;
  const Consts K = s_k;
  const Geo& g = a.g;
  const int warp = threadIdx.x >> 5;
  uint16_t* sR = slabs + (size_t)warp * 2 * TILE_ELEMS;
  const LrSlabL sL{sR + TILE_ELEMS, nullptr, 0};
  const uint64_t warps = (uint64_t)gridDim.x * LR_PW;
  for (uint64_t t = blockIdx.x * (uint64_t)LR_PW + warp; t < g.ntiles; t += warps) {
    const TileCoord tc = decode_tile(t, g);
    const uint64_t off = ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)tc.c * TK;
    lr_compress_tile<T, false, false, false>(x + off, g.n1 * g.n2, g.n2, x + off, sR, sL, tc, g, K, a.R, o, flags, hs,
                                             nullptr);
  }
  SZ3G_SYNCTHREADS();
  if (o.hist) hist_flush(hs, o.hist);
  overflow_check(a, o.ocount, o.cap);
}
size_t lr_plain_smem() { return (size_t)LR_PW * 2 * TILE_ELEMS * sizeof(uint16_t) + sizeof(uint32_t) * (LR_HW + 36); }

// ---------------------------------------------------------------------------------- LR decompress
// One warp per tile straight from global memory.  Regression blocks: x' = (T)(p + twoeb (c - R)).
// Lorenzo blocks: with r(i,j,k) = q(i,j,k) - q(i-1,j,k) - q(i,j-1,k) + q(i-1,j-1,k) (the (i,j)
// difference), delta = r(k) - r(k-1), so along each row r is a running sum of the residuals, restarted
// at an outlier (whose q is L1 of its stored value, already scattered into x_out), and
// q = r + q(i-1,j,k) + q(i,j-1,k) - q(i-1,j-1,k).  The block's right lane takes the left lane's last r
// by a shuffle: both lanes first run their columns from r = 0, then the right lane adds the left lane's
// final r to its columns before its first outlier.  Outliers are not written (the scatter did that).
// QT: the recurrence's integer type.  Without an outlier a Lorenzo block's q are prefix sums of residuals
// |delta| < R, so |q| <= 216 R < 2^23 and int32 is exact (a value with a large q is an outlier at the block
// origin); an outlier brings an arbitrary q (L1 of its stored value): with QT = int32 the routine then
// reports it and the caller redoes the tile in int64 (the writes are idempotent).
#ifndef SZ3G_LRD_JU
#define SZ3G_LRD_JU 1
#endif
constexpr int LRD_JU = SZ3G_LRD_JU;   // unroll of the regression phase's row loop (A/B tuning)
#ifndef SZ3G_LRD_COAL
#define SZ3G_LRD_COAL 1
#endif
#ifndef SZ3G_LRD_SPLIT
#define SZ3G_LRD_SPLIT 1
#endif
#ifndef SZ3G_LRD_COMPACT
#define SZ3G_LRD_COMPACT 0   // 1: Lorenzo blocks in their own pass over a warp-compacted block list (below;
                             // bit-exact, measured 8.8 vs 6.5 ms on c5: the tile pass without the recurrence
                             // still takes 6.4 ms, the separate pass 2.3 ms)
#endif
template <typename T, bool FULL, bool IN_SMEM, typename QT = int64_t>
__device__ __forceinline__ bool lr_decompress_tile(const uint16_t* __restrict__ cs, uint64_t ci, uint64_t cj,
                                                   const int32_t* __restrict__ coef,
                                                   const uint8_t* __restrict__ flags, T* __restrict__ xo,
                                                   const TileCoord tc, const Geo& g, const Consts& K, uint32_t R) {
  if (IN_SMEM) { ci = BS * TK; cj = TK; }
  const LaneGeom L = lane_geom<FULL>(tc, g);
  const int h = L.h;
  const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
  int4 cc = make_int4(0, 0, 0, 0);
  bool lor = false;
  if (L.m2 > 0) {
    cc = __ldg(reinterpret_cast<const int4*>(coef) + bid);
    lor = __ldg(flags + bid) != 0;
  }
  double bh[4];
  decode_coefs(cc, K, bh);
  const double cR = __dadd_rn(I2D_MAGIC, (double)R);
  const uint64_t gbase = ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)tc.c * TK + L.kcol;
#if SZ3G_LRD_SPLIT
  // Regression blocks first (O12), row by row with the six planes' chains independent; the Lorenzo
  // recurrence below then runs only in tiles that hold a Lorenzo block.  A full tile is walked with the
  // lanes across the row (columns lane, lane + 32, lane + 64, each with its own block's coefficients), so
  // every store instruction writes 128 contiguous bytes.
  if (FULL && IN_SMEM && SZ3G_LRD_COAL) {
    const int lane = threadIdx.x & 31;
    const uint64_t brow = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + (uint64_t)tc.c * 16u;
    double b1[3], b2[3], bk[3];
    bool reg[3];
#pragma unroll
    for (int m = 0; m < 3; m++) {
      const int k = lane + 32 * m;
      const int4 c4 = __ldg(reinterpret_cast<const int4*>(coef) + brow + k / BS);
      reg[m] = __ldg(flags + brow + k / BS) == 0;
      double bb[4];
      decode_coefs(c4, K, bb);
      b1[m] = bb[1];
      b2[m] = bb[2];
      bk[m] = __fma_rn(bb[3], (double)(k % BS), bb[0]);
    }
    const uint64_t rbase = ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)tc.c * TK + lane;
#pragma unroll LRD_JU
    for (int j = 0; j < BS; j++) {
#pragma unroll
      for (int m = 0; m < 3; m++) {
        const double base = __fma_rn(b2[m], (double)j, bk[m]);
        uint32_t c[BS];
#pragma unroll
        for (int i = 0; i < BS; i++) c[i] = cs[(i * BS + j) * TK + lane + 32 * m];
#pragma unroll
        for (int i = 0; i < BS; i++) {
          if (!reg[m] || c[i] == 0) continue;
          const double p = __fma_rn(b1[m], (double)i, base);
          const double qd = __dsub_rn(__hiloint2double(0x43300000, (int)c[i]), cR);
          xo[rbase + ((uint64_t)i * g.n1 + j) * g.n2 + 32 * m] = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, qd)));
        }
      }
    }
  } else if (!lor) {
#pragma unroll LRD_JU
    for (int j = 0; j < BS; j++) {
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        const bool cv = FULL || (j < L.m1 && L.kv(kk));
        const double base = __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * h + kk), bh[0]));
        const uint16_t* ccol = cs + (uint64_t)j * cj + L.kcol + kk;
        uint32_t c[BS];
#pragma unroll
        for (int i = 0; i < BS; i++) c[i] = (FULL || (cv && i < L.m0)) ? (uint32_t)ccol[(uint64_t)i * ci] : 0u;
#pragma unroll
        for (int i = 0; i < BS; i++) {
          if (c[i] == 0) continue;
          const double p = __fma_rn(bh[1], (double)i, base);
          const double qd = __dsub_rn(__hiloint2double(0x43300000, (int)c[i]), cR);
          xo[gbase + ((uint64_t)i * g.n1 + j) * g.n2 + kk] = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, qd)));
        }
      }
    }
  }
  if (SZ3G_LRD_COMPACT || !__any_sync(0xffffffffu, lor)) return false;   // COMPACT: k_lr_lorenzo_blocks
#endif
  // P[j] = q of row j of the previous plane; C = q of the previous row of this plane.  Row j needs
  // P[j] and P[j - 1]; once it is done P[j - 1] is free and takes this plane's row j - 1.
  QT P[BS][3];
  bool wide = false;
#pragma unroll
  for (int j = 0; j < BS; j++) P[j][0] = P[j][1] = P[j][2] = 0;
  for (int i = 0; i < BS; i++) {
    QT C[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < BS; j++) {
      uint32_t c[3];
      bool valid[3];
      const uint64_t e0 = gbase + ((uint64_t)i * g.n1 + j) * g.n2;
      const uint16_t* crow = cs + (uint64_t)i * ci + (uint64_t)j * cj + L.kcol;
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        valid[kk] = FULL || (i < L.m0 && j < L.m1 && L.kv(kk));
        c[kk] = valid[kk] ? (uint32_t)crow[kk] : R;
      }
      if (!SZ3G_LRD_SPLIT && !lor) {   // regression block (O12)
#pragma unroll
        for (int kk = 0; kk < 3; kk++) {
          if (!valid[kk] || c[kk] == 0) continue;
          const double p = __fma_rn(bh[1], (double)i, __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * h + kk), bh[0])));
          const double qd = __dsub_rn(__hiloint2double(0x43300000, (int)c[kk]), cR);
          xo[e0 + kk] = from_d<T>(__dadd_rn(p, __dmul_rn(K.twoeb, qd)));
        }
      }
      // Lorenzo recurrence, run by every lane (the shuffle needs the whole warp; regression lanes compute
      // throw-away values)
      QT r[3], base[3];
      bool nocarry[3];
      QT run = 0;
      bool cut = false;   // from an outlier on, r no longer depends on the left lane
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        base[kk] = P[j][kk] + C[kk] - (j > 0 ? P[j - 1][kk] : 0);
        if (lor && valid[kk] && c[kk] == 0) {
          if (sizeof(QT) < 8) {   // the int64 redo recomputes the tile: no need for this q here
            wide = true;
            run = 0;
          } else {
            bool ok;
            const double qd = lr_prequant(to_d<T>(xo[e0 + kk]), K, ok);
            run = (QT)__double2ll_rn(qd) - base[kk];
          }
          cut = true;
        } else {
          run += valid[kk] ? (QT)c[kk] - (QT)R : (QT)0;
        }
        r[kk] = run;
        nocarry[kk] = cut;
      }
      QT carry = __shfl_up_sync(0xffffffffu, r[2], 1);
      if (h == 0) carry = 0;
      QT q[3];
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        q[kk] = valid[kk] ? (nocarry[kk] ? r[kk] : r[kk] + carry) + base[kk] : 0;
        if (lor && valid[kk] && c[kk] != 0) xo[e0 + kk] = from_d<T>(__dmul_rn(K.twoeb, (double)q[kk]));
      }
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        if (j > 0) P[j - 1][kk] = C[kk];
        C[kk] = q[kk];
      }
    }
#pragma unroll
    for (int kk = 0; kk < 3; kk++) P[BS - 1][kk] = C[kk];
  }
  return wide;
}

// L7 for the Lorenzo blocks alone (SZ3G_LRD_COMPACT): the tile decompressor writes only the regression
// blocks, and this pass runs the recurrence for the Lorenzo blocks (5.4% of c5's blocks) instead of in
// every lane of every tile that holds one (58% of c5's tiles).  A warp scans the flags of 16 consecutive
// blocks, compacts the Lorenzo ones by ballot and gives each two lanes (columns 0-2 / 3-5, the tile
// decompressor's lane pairs, so the recurrence and its carry shuffle are the same), reading codes from
// global memory; int64 throughout.  Outliers: their stored values were scattered first (L7).
constexpr int LRL_WARPS = 8, LRL_GROUP = 512;
template <typename T>
__global__ void __launch_bounds__(LRL_WARPS * 32) k_lr_lorenzo_blocks(const uint16_t* __restrict__ codes,
                                                                     const uint8_t* __restrict__ flags,
                                                                     T* __restrict__ xo, KArgs a) {
  __shared__ Consts s_k;
  __shared__ int s_ok;
  __shared__ uint32_t s_list[LRL_WARPS][LRL_GROUP];   // a warp's compacted Lorenzo blocks (group offsets)
  if (!cta_consts(a, &s_k, &s_ok)) return;
  const Consts K = s_k;
  const Geo& g = a.g;
  const uint32_t R = a.R;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* list = s_list[wl];
  const uint64_t nb = (uint64_t)g.NB0 * g.NB1 * g.NB2;
  const uint64_t ngroups = (nb + LRL_GROUP - 1) / LRL_GROUP;
  const uint64_t warps = (uint64_t)gridDim.x * LRL_WARPS;
  for (uint64_t grp = blockIdx.x * (uint64_t)LRL_WARPS + wl; grp < ngroups; grp += warps) {
    const uint64_t b0 = grp * LRL_GROUP;
    // compact the group's Lorenzo blocks (ballot per 32 flags)
    uint32_t nl = 0;
    for (int q = 0; q < LRL_GROUP; q += 32) {
      const bool is = b0 + q + lane < nb && flags[b0 + q + lane] != 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, is);
      if (is) list[nl + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)(q + lane);
      nl += __popc(bal);
    }
    SZ3G_SYNCWARP();
    // batches of 16 blocks: lane pair (2 r, 2 r + 1) takes block r of the batch
    for (uint32_t s0 = 0; s0 < nl; s0 += 16) {
      const int rnk = lane >> 1, h = lane & 1;
      const bool act = s0 + rnk < nl;
      const uint64_t bid = b0 + (act ? list[s0 + rnk] : 0u);
      const uint64_t bc = bid % g.NB2, bab = bid / g.NB2, bb = bab % g.NB1, ba = bab / g.NB1;
      const int m0 = (int)umin64(BS, g.n0 - ba * BS), m1 = (int)umin64(BS, g.n1 - bb * BS);
      const int m2 = (int)umin64(BS, g.n2 - bc * BS);
      const uint64_t gbase = ((ba * BS) * g.n1 + bb * BS) * g.n2 + bc * BS + 3 * h;
      int64_t P[BS][3];
#pragma unroll
      for (int j = 0; j < BS; j++) P[j][0] = P[j][1] = P[j][2] = 0;
      for (int i = 0; i < BS; i++) {
        // the plane's 6 x 3 codes of this lane, loaded together (independent of the recurrence)
        uint32_t c[BS][3];
#pragma unroll
        for (int j = 0; j < BS; j++)
#pragma unroll
          for (int kk = 0; kk < 3; kk++) {
            const bool v = act && i < m0 && j < m1 && 3 * h + kk < m2;
            c[j][kk] = v ? (uint32_t)codes[gbase + ((uint64_t)i * g.n1 + j) * g.n2 + kk] : 0xffffffffu;
          }
        int64_t C[3] = {0, 0, 0};
#pragma unroll
        for (int j = 0; j < BS; j++) {
          const uint64_t e0 = gbase + ((uint64_t)i * g.n1 + j) * g.n2;
          int64_t r[3], base[3];
          bool nocarry[3];
          int64_t run = 0;
          bool cut = false;
#pragma unroll
          for (int kk = 0; kk < 3; kk++) {
            const bool valid = c[j][kk] != 0xffffffffu;
            base[kk] = P[j][kk] + C[kk] - (j > 0 ? P[j - 1][kk] : 0);
            if (valid && c[j][kk] == 0) {
              bool ok;
              const double qd = lr_prequant(to_d<T>(xo[e0 + kk]), K, ok);
              run = (int64_t)__double2ll_rn(qd) - base[kk];
              cut = true;
            } else {
              run += valid ? (int64_t)c[j][kk] - (int64_t)R : (int64_t)0;
            }
            r[kk] = run;
            nocarry[kk] = cut;
          }
          int64_t carry = __shfl_up_sync(0xffffffffu, r[2], 1);
          if (h == 0) carry = 0;
#pragma unroll
          for (int kk = 0; kk < 3; kk++) {
            const bool valid = c[j][kk] != 0xffffffffu;
            const int64_t q = valid ? (nocarry[kk] ? r[kk] : r[kk] + carry) + base[kk] : 0;
            if (valid && c[j][kk] != 0) xo[e0 + kk] = from_d<T>(__dmul_rn(K.twoeb, (double)q));
            if (j > 0) P[j - 1][kk] = C[kk];
            C[kk] = q;
          }
        }
#pragma unroll
        for (int kk = 0; kk < 3; kk++) P[BS - 1][kk] = C[kk];
      }
    }
    SZ3G_SYNCWARP();
  }
}

constexpr int LR_DW = 4;   // decompress: warps per CTA
template <typename T>
__global__ void __launch_bounds__(LR_DW * 32) k_lr_decompress(const uint16_t* __restrict__ codes,
                                                              const int32_t* __restrict__ coef,
                                                              const uint8_t* __restrict__ flags, T* __restrict__ xo,
                                                              KArgs a) {
  __shared__ Consts s_k;
  __shared__ int s_ok;
  if (!cta_consts(a, &s_k, &s_ok)) return;
  const Consts K = s_k;
  const Geo& g = a.g;
  const uint64_t warps = (uint64_t)gridDim.x * LR_DW;
  for (uint64_t t = blockIdx.x * (uint64_t)LR_DW + (threadIdx.x >> 5); t < g.ntiles; t += warps) {
    const TileCoord tc = decode_tile(t, g);
    const uint16_t* cs = codes + ((uint64_t)tc.a * BS * g.n1 + (uint64_t)tc.b * BS) * g.n2 + (uint64_t)tc.c * TK;
    if (tile_full(tc, g)) lr_decompress_tile<T, true, false>(cs, g.n1 * g.n2, g.n2, coef, flags, xo, tc, g, K, a.R);
    else lr_decompress_tile<T, false, false>(cs, g.n1 * g.n2, g.n2, coef, flags, xo, tc, g, K, a.R);
  }
}

// The code tiles through a private 2-stage TMA ring per warp (self-fed, as k_analyze_tma): the
// recurrence reads them from shared memory instead of waiting on a global load per row.
template <int W, int D>
struct LrDecSmem {
  static constexpr size_t stage_bytes = sizeof(uint16_t) * TILE_ELEMS;
  static constexpr size_t off_bar = (size_t)W * D * stage_bytes;
  static constexpr size_t off_k = off_bar + (size_t)W * D * sizeof(uint64_t);
  static constexpr size_t total = off_k + sizeof(Consts) + 16;
};

#ifndef SZ3G_LRD_MINB
#define SZ3G_LRD_MINB 4   // 128 registers: 4 CTAs (16 warps) per SM (A/B: 1 -> 7.57 ms, 4 -> 6.61 ms on c5)
#endif
template <typename T, int W, int D>
__global__ void __launch_bounds__(W * 32, SZ3G_LRD_MINB)
    k_lr_decompress_tma(const __grid_constant__ CUtensorMap tm_c, const int32_t* __restrict__ coef,
                        const uint8_t* __restrict__ flags, T* __restrict__ xo, KArgs a) {
  using L_ = LrDecSmem<W, D>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L_::off_bar);
  Consts* s_k = reinterpret_cast<Consts*>(smem + L_::off_k);
  int* s_ok = reinterpret_cast<int*>(smem + L_::off_k + sizeof(Consts));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < W * D; s++) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbar_init();
  }
  if (!cta_consts(a, s_k, s_ok)) return;
  const Consts K = *s_k;
  const Geo& g = a.g;
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem) + (size_t)warp * D * TILE_ELEMS;
  uint64_t* bar = full + warp * D;
  TileWalk tw(warp, a.chunk, W), tl(warp, a.chunk, W);
  if (lane == 0) {
    ptx::prefetch_tensormap(&tm_c);
    for (int d = 0; d < D; d++, tl.next()) {
      const uint64_t t = tl.tile();
      if (t >= g.ntiles) break;
      const TileCoord tc = decode_tile(t, g);
      ptx::mbar_arrive_expect_tx(&bar[d], (uint32_t)L_::stage_bytes);
      ptx::tma_load_3d(ring + (size_t)d * TILE_ELEMS, &tm_c, &bar[d], (int)(tc.c * TK), (int)(tc.b * BS), (int)(tc.a * BS));
    }
  }
  for (uint32_t k = 0;; k++, tw.next()) {
    const uint64_t t = tw.tile();
    if (t >= g.ntiles) break;
    const uint32_t s = k % D, ph = (k / D) & 1u;
    const TileCoord tc = decode_tile(t, g);
    ptx::mbar_wait(&bar[s], ph);
    const uint16_t* cs = ring + (size_t)s * TILE_ELEMS;
    if (tile_full(tc, g)) {
      if (__any_sync(0xffffffffu, lr_decompress_tile<T, true, true, int32_t>(cs, 0, 0, coef, flags, xo, tc, g, K, a.R)))
        lr_decompress_tile<T, true, true, int64_t>(cs, 0, 0, coef, flags, xo, tc, g, K, a.R);
    } else {
      lr_decompress_tile<T, false, true, int64_t>(cs, 0, 0, coef, flags, xo, tc, g, K, a.R);
    }
    SZ3G_SYNCWARP();
    if (lane == 0) {
      const uint64_t t2 = tl.tile();
      if (t2 < g.ntiles) {
        const TileCoord tc2 = decode_tile(t2, g);
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive_expect_tx(&bar[s], (uint32_t)L_::stage_bytes);
        ptx::tma_load_3d(ring + (size_t)s * TILE_ELEMS, &tm_c, &bar[s], (int)(tc2.c * TK), (int)(tc2.b * BS),
                         (int)(tc2.a * BS));
      }
      tl.next();
    }
  }
}

// ---------------------------------------------------------------------------------- LR compress, pairs
// Two warps per tile: warp half HW takes planes [3 HW, 3 HW + 3) and the second half also runs plane 2
// (q and its j,k-differences only) for its first i-difference, so each lane carries 3 (+1) x 3
// differences instead of 6 x 3 and the unrolled body holds 9 elements -- the single-warp kernel's
// 18-element body was ~48 KB of hot code, bound by instruction fetch.  Per tile three pair barriers:
// slabs free (the previous tile's TMA store has read them), block costs exchanged, codes complete.
template <typename T, bool FULL>
__device__ __forceinline__ void lr_half_compute(const T* __restrict__ xs, uint16_t* sR, uint16_t* sL, const LaneGeom& L,
                                                const double bh[4], const Fast32& F, const Fast32& F0, const Consts& K,
                                                uint32_t R, uint32_t& costR, uint32_t& costL, bool& big, int HW) {
  // one code path for both halves (one hot body in the instruction cache): planes P0 .. P0 + 3, codes for
  // i >= I0; the first half's helper plane is plane -1 (outside the block: q = 0)
  constexpr bool F32 = sizeof(T) == 4;
  constexpr int NP = 4;
  const int I0 = 3 * HW, P0 = 3 * HW - 1;
  const int h = L.h;
  const float inv2eb32 = K.inv2eb32;
  const float M32 = 12582912.0f;                 // 1.5 * 2^23
  const float Rf = (float)R;
  const int iR = (int)R;
  int32_t Dp[3][NP];
#pragma unroll
  for (int kk = 0; kk < 3; kk++)
#pragma unroll
    for (int ii = 0; ii < NP; ii++) Dp[kk][ii] = 0;
#pragma unroll 1
  for (int j = 0; j < BS; j++) {
    int32_t q[3][NP];
    uint32_t cr[3][NP];
    bool lv[3][NP];
    const float fj = (float)j;
#pragma unroll
    for (int kk = 0; kk < 3; kk++) {
      const bool cv = FULL || ((j < L.m1) && L.kv(kk));
      T xv[NP];
#pragma unroll
      for (int ii = 0; ii < NP; ii++) xv[ii] = (P0 + ii >= 0) ? xs[(P0 + ii) * (BS * TK) + j * TK + L.kcol + kk] : T(0);
      bool need = false;
      if (F32) {
        // packed fp32x2 over pairs of planes (FFMA2 / FADD2: each lane the IEEE result of the scalar op)
        const float base32 = __fmaf_rn(F.a2, fj, __fmaf_rn(F.a3, (float)(3 * h + kk), F.a0));
        const uint64_t inv2 = pack2(inv2eb32, inv2eb32), M2 = pack2(M32, M32);
#pragma unroll
        for (int ii = 0; ii < NP; ii += 2) {
          const int i = P0 + ii;
          const uint64_t x2 = pack2((float)xv[ii], (float)xv[ii + 1]);
          // regression: P = fma(a1, i, base) (exactly base at i = 0 for a finite a1), t = fma(x, inv, -P)
          const uint64_t nP = fma2(pack2(-F.a1, -F.a1), pack2((float)i, (float)(i + 1)), pack2(-base32, -base32));
          const uint64_t t2 = fma2(x2, inv2, nP);
          const uint64_t r2 = sub2(add2(t2, M2), M2);
          const uint64_t e2 = sub2(t2, r2);
          // Lorenzo prequantisation: t = x * inv (fma with a -0 addend rounds once, like the product)
          const uint64_t tL2 = fma2(x2, inv2, pack2(-0.0f, -0.0f));
          const uint64_t rL2 = sub2(add2(tL2, M2), M2);
          const uint64_t eL2 = sub2(tL2, rL2);
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            const int ip = i + hh;
            const bool valid = ip >= 0 && (FULL || (cv && ip < L.m0));
            if (ip >= I0) {
              const float t32 = lane_of(t2, hh), r = lane_of(r2, hh), e = lane_of(e2, hh);
              const bool ok = __fmaf_rn(F.k1, fabsf(t32), fabsf(e)) <= F.thr && fabsf(r) < Rf;
              cr[kk][ii + hh] = ok ? (uint32_t)((int)r + iR) : 0u;
              need |= valid && !ok;
            } else {
              cr[kk][ii + hh] = R;
            }
            const float tL = lane_of(tL2, hh), rL = lane_of(rL2, hh), eL = lane_of(eL2, hh);
            const bool okL = __fmaf_rn(F0.k1, fabsf(tL), fabsf(eL)) <= F0.thr && fabsf(tL) < 4194304.0f;
            q[kk][ii + hh] = okL ? (int32_t)rL : 0;
            lv[kk][ii + hh] = okL;
            need |= valid && !okL;
          }
        }
      } else {
        const double base = __fma_rn(bh[2], (double)j, __fma_rn(bh[3], (double)(3 * h + kk), bh[0]));
#pragma unroll
        for (int ii = 0; ii < NP; ii++) {
          const int i = P0 + ii;
          const bool valid = i >= 0 && (FULL || (cv && i < L.m0));
          const double xd = to_d<T>(xv[ii]);
          if (i >= I0) {
            const double p = __fma_rn(bh[1], (double)i, base);
            const double t = __dmul_rn(__dsub_rn(xd, p), K.inv2eb);
            const double rq = __dsub_rn(__dadd_rn(t, RINT_MAGIC), RINT_MAGIC);
            const bool ok = __fma_rn(K.vc, fabs(xd), fabs(__dsub_rn(t, rq))) <= K.vthr && fabs(rq) < (double)R;
            cr[kk][ii] = ok ? (uint32_t)((int)rq + iR) : 0u;
            need |= valid && !ok;
          } else {
            cr[kk][ii] = R;
          }
          const double tL = __dmul_rn(xd, K.inv2eb);
          const double rL = __dsub_rn(__dadd_rn(tL, RINT_MAGIC), RINT_MAGIC);
          const bool okL = __fma_rn(K.vc, fabs(xd), fabs(__dsub_rn(tL, rL))) <= K.vthr && fabs(tL) < 67108864.0;
          q[kk][ii] = okL ? (int32_t)rL : 0;
          lv[kk][ii] = okL;
          need |= valid && !okL;
        }
      }
      if (__any_sync(0xffffffffu, need)) {   // the exact definitions (rare)
#pragma unroll
        for (int ii = 0; ii < NP; ii++) {
          const int i = P0 + ii;
          const bool valid = i >= 0 && (FULL || (cv && i < L.m0));
          const bool wr = i >= I0 && cr[kk][ii] == 0u;
          if (valid && (wr || !lv[kk][ii])) {
            const LrExact ex = lr_exact_elem<T>(xv[ii], bh[0], bh[1], bh[2], bh[3], i, j, 3 * h + kk, K, R, wr,
                                                !lv[kk][ii]);
            if (wr) cr[kk][ii] = ex.cr;
            if (!lv[kk][ii]) {
              big |= ex.big;
              q[kk][ii] = ex.q;
              lv[kk][ii] = ex.lv;
            }
          }
        }
      }
#pragma unroll
      for (int ii = 0; ii < NP; ii++) {
        const bool valid = P0 + ii >= 0 && (FULL || (cv && P0 + ii < L.m0));
        if (!valid) { q[kk][ii] = 0; lv[kk][ii] = false; cr[kk][ii] = R; }
      }
    }
    int32_t left[NP];
#pragma unroll
    for (int ii = 0; ii < NP; ii++) {
      left[ii] = __shfl_up_sync(0xffffffffu, q[2][ii], 1);
      if (h == 0) left[ii] = 0;
    }
#pragma unroll
    for (int kk = 0; kk < 3; kk++) {
      const bool cv = FULL || ((j < L.m1) && L.kv(kk));
      int32_t Eprev = 0;
#pragma unroll
      for (int ii = 0; ii < NP; ii++) {
        const int i = P0 + ii;
        const int32_t D = q[kk][ii] - (kk == 0 ? left[ii] : q[kk - 1][ii]);
        const int32_t E = D - Dp[kk][ii];
        Dp[kk][ii] = D;
        const int32_t delta = E - Eprev;
        Eprev = E;
        if (i < I0) continue;   // the helper plane
        const bool valid = FULL || (cv && i < L.m0);
        // |delta| < R <=> delta + R - 1 in [0, 2R - 1) (|delta| < 2^25: no wrap)
        uint32_t cl = (lv[kk][ii] && (uint32_t)(delta + iR - 1) < 2u * R - 1u) ? (uint32_t)(delta + iR) : 0u;
        if (!valid) cl = R;
        const uint32_t c = cr[kk][ii];
        // an outlier (code 0) costs R = |0 - R|
        costR += (uint32_t)abs((int)c - iR);
        costL += (uint32_t)abs((int)cl - iR);
        const uint32_t sidx = (uint32_t)(i * (BS * TK) + j * TK + L.kcol + kk);
        sR[sidx] = (uint16_t)c;
        sL[sidx] = (uint16_t)cl;
      }
    }
  }
}

// outliers of planes [i0, i0 + 3) (rare_path over a plane range)
template <typename T, bool HIST>
__device__ __forceinline__ void lr_rare_planes(const T* __restrict__ xs, const uint16_t* cs, int i0, const LaneGeom& L,
                                               bool has_out, const TileCoord tc, const Geo& g, const CompressOut<T>& o,
                                               const HistSmem& hs) {
  const int lane = threadIdx.x & 31;
  if (!__any_sync(0xffffffffu, has_out)) return;
  const int i1 = min(i0 + 3, L.m0);
  uint32_t nout = 0;
  if (has_out) {
    for (int i = i0; i < i1; i++)
      for (int j = 0; j < L.m1; j++)
        for (int kk = 0; kk < 3; kk++)
          if (L.kv(kk)) nout += (cs[i * (BS * TK) + j * TK + L.kcol + kk] == 0u) ? 1u : 0u;
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
    for (int i = i0; i < i1; i++)
      for (int j = 0; j < L.m1; j++)
        for (int kk = 0; kk < 3; kk++) {
          if (!L.kv(kk) || cs[i * (BS * TK) + j * TK + L.kcol + kk] != 0) continue;
          if (pos < o.cap) {
            o.oidx[pos] = gbase + ((uint64_t)i * g.n1 + j) * g.n2 + kk;
            o.oval[pos] = xs[i * (BS * TK) + j * TK + L.kcol + kk];
          }
          pos++;
        }
  }
}

template <typename T, int NPAIR>
struct LrPairSmem {
  static constexpr size_t stage_bytes = sizeof(T) * TILE_ELEMS;
  static constexpr size_t slab_bytes = sizeof(uint16_t) * TILE_ELEMS;
  // + costs + flag, rounded to 128 bytes: every pair's stage is a TMA destination
  static constexpr size_t pair_bytes = (stage_bytes + 2 * slab_bytes + 2 * 16 * 8 + 16 + 127) / 128 * 128;
  static constexpr size_t off_hist = (size_t)NPAIR * pair_bytes;
  static constexpr size_t off_bar = off_hist + sizeof(uint32_t) * (LR_HW + 36);
  static constexpr size_t off_k = off_bar + (size_t)NPAIR * sizeof(uint64_t);
  static constexpr size_t total = off_k + sizeof(Consts) + 16;
};

__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// Histogram of a half's codes (planes [i0, i0 + 3)); returns whether the lane holds an outlier.  The window
// starts at lo >= 1, so code 0 is never in it; codes outside the window (and the outliers) are rare and
// handled in a second walk, keeping the hot loop free of branches.
template <bool HIST, bool FULL>
__device__ __forceinline__ bool lr_pair_hist(const uint16_t* sR, int i0, const LaneGeom& L, const HistSmem& hs,
                                             unsigned long long* ghist, uint32_t hb, uint32_t sink) {
  bool rare = false;
#pragma unroll 1
  for (int i = i0; i < i0 + 3; i++)
#pragma unroll
    for (int j = 0; j < BS; j++)
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        const bool valid = FULL || (i < L.m0 && j < L.m1 && L.kv(kk));
        const uint32_t code = sR[i * (BS * TK) + j * TK + L.kcol + kk];
        if (HIST) {
          const bool inwin = valid && code - hs.lo < hs.nwin;
          red_smem_add(inwin ? hb + 4u * code : sink, 1u);
          rare |= valid && !inwin;
        } else {
          rare |= valid && code == 0u;
        }
      }
  if (!HIST || !rare) return rare;
  bool has_out = false;
  for (int i = i0; i < i0 + 3; i++)
    for (int j = 0; j < BS; j++)
      for (int kk = 0; kk < 3; kk++) {
        const bool valid = FULL || (i < L.m0 && j < L.m1 && L.kv(kk));
        const uint32_t code = sR[i * (BS * TK) + j * TK + L.kcol + kk];
        if (!valid) continue;
        if (code == 0u) has_out = true;
        else if (code - hs.lo >= hs.nwin) atomicAdd(&ghist[code], 1ull);
      }
  return has_out;
}

template <typename T, bool FULL>
__device__ __forceinline__ void lr_pair_tile(const T* __restrict__ xs, uint16_t* sR, uint16_t* sL, uint2* s_cost,
                                             int* s_big, int hw, int bar_id, const TileCoord tc, const Geo& g,
                                             const Consts& K, uint32_t R, const CompressOut<T>& o,
                                             uint8_t* __restrict__ flags, const HistSmem& hs, const CUtensorMap* tm_c) {
  const LaneGeom L = lane_geom<FULL>(tc, g);
  const int h = L.h, lane = threadIdx.x & 31, bl = lane >> 1;
  double beta[4] = {0.0, 0.0, 0.0, 0.0}, bh[4];
  int32_t cc[4];
  const uint64_t bid = ((uint64_t)tc.a * g.NB1 + tc.b) * g.NB2 + L.kb;
  if (L.m2 > 0) {
    const double2 b01 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid);
    const double2 b23 = __ldg(reinterpret_cast<const double2*>(o.beta_in) + 2 * bid + 1);
    beta[0] = b01.x; beta[1] = b01.y; beta[2] = b23.x; beta[3] = b23.y;
  }
  block_codes(beta, K, cc, bh);
  const Fast32 F = fast32_consts(bh, K);
  const double zero[4] = {0.0, 0.0, 0.0, 0.0};
  const Fast32 F0 = fast32_consts(zero, K);
  uint32_t costR = 0, costL = 0;
  bool big = false;
  lr_half_compute<T, FULL>(xs, sR, sL, L, bh, F, F0, K, R, costR, costL, big, hw);
  costR += __shfl_xor_sync(0xffffffffu, costR, 1);
  costL += __shfl_xor_sync(0xffffffffu, costL, 1);
  if (h == 0) s_cost[hw * 16 + bl] = make_uint2(costR, costL);
  if (__any_sync(0xffffffffu, big) && lane == 0) *s_big = 1;
  pair_bar(bar_id);   // (2) both halves' costs and the big flag
  if (*s_big) {       // a q beyond the int32 residuals: the whole tile by the int64 routine (first warp)
    if (hw == 0)
      lr_compress_tile_exact<T, true, FULL, true>(xs, BS * TK, TK, sR, LrSlabL{sL, nullptr, 0}, tc, g, K, R, o, flags,
                                                  hs, tm_c);
    return;
  }
  const uint2 c0 = s_cost[bl], c1 = s_cost[16 + bl];
  const bool useL = c0.y + c1.y < c0.x + c1.x;
  if (hw == 0 && L.m2 > 0 && h == 0) {
    reinterpret_cast<int4*>(o.coef)[bid] = useL ? make_int4(0, 0, 0, 0) : make_int4(cc[0], cc[1], cc[2], cc[3]);
    flags[bid] = useL ? 1 : 0;
  }
  const int i0 = 3 * hw;
  const uint32_t hb = (uint32_t)__cvta_generic_to_shared(hs.win) - 4u * hs.lo;
  const uint32_t sink = (uint32_t)__cvta_generic_to_shared(hs.dummy) + 4u * lane;
  const bool hist = o.hist != nullptr;
  bool has_out = false;
  if (__any_sync(0xffffffffu, useL)) {   // the Lorenzo blocks' codes into the stored slab
    if (useL) {
#pragma unroll 1
      for (int i = i0; i < i0 + 3; i++)
#pragma unroll
        for (int j = 0; j < BS; j++)
#pragma unroll
          for (int kk = 0; kk < 3; kk++) {
            const uint32_t s = (uint32_t)(i * (BS * TK) + j * TK + L.kcol + kk);
            sR[s] = sL[s];
          }
    }
    SZ3G_SYNCWARP();
  }
  if (hist) has_out = lr_pair_hist<true, FULL>(sR, i0, L, hs, o.hist, hb, sink);
  else has_out = lr_pair_hist<false, FULL>(sR, i0, L, hs, o.hist, hb, sink);
  SZ3G_SYNCWARP();
  if (hist) lr_rare_planes<T, true>(xs, sR, i0, L, has_out, tc, g, o, hs);
  else lr_rare_planes<T, false>(xs, sR, i0, L, has_out, tc, g, o, hs);
  ptx::fence_proxy_async_smem();   // this warp's code writes, before the pair's TMA store
}

template <typename T, int NPAIR>
__global__ void __launch_bounds__(NPAIR * 64, 1)
    k_lr_compress_pair(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_c, KArgs a,
                       CompressOut<T> o, uint8_t* __restrict__ flags) {
  using L_ = LrPairSmem<T, NPAIR>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L_::off_bar);
  Consts* s_k = reinterpret_cast<Consts*>(smem + L_::off_k);
  int* s_ok = reinterpret_cast<int*>(smem + L_::off_k + sizeof(Consts));
  uint32_t* s_win = reinterpret_cast<uint32_t*>(smem + L_::off_hist);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = warp >> 1, hw = warp & 1, bar_id = 1 + p;
  HistSmem hs;
  hist_init(hs, s_win, s_win + LR_HW, a.R, LR_HW);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NPAIR; s++) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbar_init();
  }
  if (!cta_consts(a, s_k, s_ok)) return;
  const Consts K = *s_k;
  const Geo& g = a.g;
  uint8_t* pb = smem + (size_t)p * L_::pair_bytes;
  T* stage = reinterpret_cast<T*>(pb);
  uint16_t* sR = reinterpret_cast<uint16_t*>(pb + L_::stage_bytes);
  uint16_t* sL = sR + TILE_ELEMS;
  uint2* s_cost = reinterpret_cast<uint2*>(pb + L_::stage_bytes + 2 * L_::slab_bytes);
  int* s_big = reinterpret_cast<int*>(pb + L_::stage_bytes + 2 * L_::slab_bytes + 2 * 16 * 8);
  const bool loader = hw == 0 && lane == 0;
  TileWalk tw(p, a.chunk, NPAIR), tl(p, a.chunk, NPAIR);
  if (loader) {
    ptx::prefetch_tensormap(&tm_x);
    const uint64_t t = tl.tile();
    if (t < g.ntiles) {
      const TileCoord tc = decode_tile(t, g);
      ptx::mbar_arrive_expect_tx(&full[p], (uint32_t)L_::stage_bytes);
      ptx::tma_load_3d(stage, &tm_x, &full[p], (int)(tc.c * TK), (int)(tc.b * BS), (int)(tc.a * BS));
    }
    tl.next();
  }
  for (uint32_t k = 0;; k++, tw.next()) {
    const uint64_t t = tw.tile();
    if (t >= g.ntiles) break;
    const TileCoord tc = decode_tile(t, g);
    if (loader) {
      ptx::bulk_wait_read0();   // the previous tile's code store has read sR
      *s_big = 0;
    }
    pair_bar(bar_id);   // (1) slabs free, flag reset
    ptx::mbar_wait(&full[p], k & 1u);
    if (tile_full(tc, g)) lr_pair_tile<T, true>(stage, sR, sL, s_cost, s_big, hw, bar_id, tc, g, K, a.R, o, flags, hs, &tm_c);
    else lr_pair_tile<T, false>(stage, sR, sL, s_cost, s_big, hw, bar_id, tc, g, K, a.R, o, flags, hs, &tm_c);
    pair_bar(bar_id);   // (3) the tile's codes complete, the stage no longer read
    if (loader) {
      if (!*s_big) {
        ptx::tma_store_3d(&tm_c, sR, (int)(tc.c * TK), (int)(tc.b * BS), (int)(tc.a * BS));
        ptx::bulk_commit();
      }
      const uint64_t t2 = tl.tile();
      if (t2 < g.ntiles) {
        const TileCoord tc2 = decode_tile(t2, g);
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive_expect_tx(&full[p], (uint32_t)L_::stage_bytes);
        ptx::tma_load_3d(stage, &tm_x, &full[p], (int)(tc2.c * TK), (int)(tc2.b * BS), (int)(tc2.a * BS));
      }
      tl.next();
    }
  }
  if (loader) ptx::bulk_wait0();
  SZ3G_SYNCTHREADS();
  if (o.hist) hist_flush(hs, o.hist);
  overflow_check(a, o.ocount, o.cap);
}
