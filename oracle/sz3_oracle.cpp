// =====================================================================================
//  oracle/sz3_oracle.cpp -- TEST INFRASTRUCTURE ONLY (not part of the product path).
//
//  A plain, slow, single-threaded CPU definition of SZ3's block-wise linear-regression
//  predictor with linear-scaling quantisation, written from PAPER.md (arxiv 2111.02925):
//    * Lemma 1 / Eq. (thm1sol)  P:46-67   closed-form regression coefficients
//    * "Prediction"             P:156     f^(r)_ijk = b0 + i b1 + j b2 + k b3, residual,
//                                         linear-scaling quantisation
//    * Quantizer instances      P:406-409 equal bins of width 2*eb, out-of-range residuals
//                                         are "unpredictable" and stored separately
//    * quantize / recover       P:400-404, App. A
//    * block-then-element loop  App. A, Alg. 1
//    * value-range-relative eb
//    * SZ3-LR (NEXT-4)          P:845  Lorenzo / regression per block ("better result in between
//                                      based on blockwise error estimation"); DEFINITION.md L1-L7
//    * SZ3-Interp (NEXT-4)      P:852-853 "Both linear interpolation and cubic spline interpolation
//                                      are included", "constant coefficients"; DEFINITION.md I1-I6
//  Readings of silent / garbled passages (coefficient bins, tie rule, verify step, ...) are the
//  ones listed in DESIGN.md section "Readings" (G1..G18) and in oracle/DEFINITION.md.
//
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
//  load this library. It shares no code, header, table or constant with
//  paper_2111_02925_b200/ (the CUDA path), and neither side includes the other.
//
//  Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -shared -fPIC
//  (-ffp-contract=off: no multiply-add contraction except where std::fma is written out.)
// =====================================================================================
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>

extern "C" {

// Status codes (same meaning as include/sz3g.h, restated here on purpose: no shared header).
enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_EUNSUPPORTED = -2, ORC_ERANGE = -3, ORC_EBADRANGE = -5,
       ORC_EOVERFLOW = -6 };

// Counters reported next to the outputs (SURVEY 8(c) "Reported counters").
struct orc_counters {
  uint64_t elem_near_ties;      // (i)  frac((x-p)/(2eb)) within 1e-9 of 1/2 (true division)
  uint64_t elem_div_mismatch;   // (ii) rint((x-p)/(2eb)) != rint((x-p)*fl(1/(2eb)))
  uint64_t coef_near_ties;      // (iii) coefficients whose beta/w lies in the tie window
  uint64_t coef_tie_blocks;     //       blocks holding at least one such coefficient
  uint64_t radius_outliers;     // |t| >= R or |rint(t)| >= R (finite t)
  uint64_t verify_outliers;     // failed the O9 verify step
  uint64_t nonfinite_outliers;  // t not finite (NaN / Inf input)
  uint64_t zero_predictor_blocks; // O6 fallback: non-finite or int32-overflowing coefficient
};

}  // extern "C"

namespace {

// ---------------------------------------------------------------- element type helpers
template <typename T> struct dtype_of;
template <> struct dtype_of<float> { static constexpr int id = 0; };
template <> struct dtype_of<double> { static constexpr int id = 1; };

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- O1 / O2: error bound
// O1: ABS -> eb_abs = eb; REL (value range) -> eb_abs = eb * (hi - lo).
// O2: twoeb = 2 eb_abs, inv2eb = 1/twoeb, w0 = eb_abs/2, ws = eb_abs/(2B)  (DESIGN G1, G5).
struct Bounds {
  double eb_abs, twoeb, inv2eb, w0, ws;
};

inline bool make_bounds(int eb_mode, double eb, double lo, double hi, uint32_t B, Bounds* out) {
  double eb_abs;
  if (eb_mode == 0) {
    eb_abs = eb;
  } else {
    double range = hi - lo;
    eb_abs = eb * range;
  }
  if (!std::isfinite(eb_abs) || !(eb_abs > 0.0)) return false;
  out->eb_abs = eb_abs;
  out->twoeb = 2.0 * eb_abs;
  out->inv2eb = 1.0 / out->twoeb;
  out->w0 = eb_abs / 2.0;
  out->ws = eb_abs / (2.0 * (double)B);
  return true;
}

// ---------------------------------------------------------------- O4: block moments
// V0 = sum f, Vx = sum i f, Vy = sum j f, Vz = sum k f  (Lemma 1), sequential loops
// i -> j -> k with k fastest, f = (double) x.
template <typename T>
void block_moments(const T* x, uint64_t n1, uint64_t n2, uint64_t i0, uint64_t j0, uint64_t k0,
                   int m0, int m1, int m2, double V[4]) {
  double V0 = 0.0, Vx = 0.0, Vy = 0.0, Vz = 0.0;
  for (int i = 0; i < m0; i++)
    for (int j = 0; j < m1; j++)
      for (int k = 0; k < m2; k++) {
        double f = (double)x[((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k)];
        V0 += f;
        Vx += (double)i * f;
        Vy += (double)j * f;
        Vz += (double)k * f;
      }
  V[0] = V0; V[1] = Vx; V[2] = Vy; V[3] = Vz;
}

// ---------------------------------------------------------------- O5: Lemma 1
// beta_d = 6 / (n1 n2 n3 (n_d + 1)) * (2 V_d / (n_d - 1) - V0)
// beta_0 = V0 / (n1 n2 n3) - ((n1-1)/2 b1 + (n2-1)/2 b2 + (n3-1)/2 b3)
// Extent-1 axis: slope 0 (DESIGN G2; the Lemma divides by n_d - 1).
void lemma_beta(const double V[4], int m0, int m1, int m2, double beta[4]) {
  const int m[3] = {m0, m1, m2};
  const double Nb = (double)m0 * (double)m1 * (double)m2;
  for (int d = 0; d < 3; d++) {
    if (m[d] > 1) {
      double scale = 6.0 / (Nb * (double)(m[d] + 1));
      double inner = 2.0 * V[d + 1] / (double)(m[d] - 1) - V[0];
      beta[d + 1] = scale * inner;
    } else {
      beta[d + 1] = 0.0;
    }
  }
  beta[0] = V[0] / Nb - ((double)(m0 - 1) / 2.0 * beta[1] + (double)(m1 - 1) / 2.0 * beta[2] +
                         (double)(m2 - 1) / 2.0 * beta[3]);
}

// ---------------------------------------------------------------- O6: coefficient codes
// Independent per-block linear quantisation (DESIGN G1): c0 = rint(b0/w0), c_d = rint(b_d/ws),
// ties to even; non-finite or |c| > 2^31-1 -> all four codes 0 ("zero predictor").
// Returns true if the zero predictor was used.
bool coef_codes(const double beta[4], const Bounds& bd, int32_t c[4], double bhat[4]) {
  double r[4];
  bool bad = false;
  for (int d = 0; d < 4; d++) {
    double w = (d == 0) ? bd.w0 : bd.ws;
    r[d] = std::nearbyint(beta[d] / w);
    if (!std::isfinite(r[d]) || std::fabs(r[d]) > 2147483647.0) bad = true;
  }
  for (int d = 0; d < 4; d++) c[d] = bad ? 0 : (int32_t)r[d];
  bhat[0] = (double)c[0] * bd.w0;
  for (int d = 1; d < 4; d++) bhat[d] = (double)c[d] * bd.ws;
  return bad;
}

// ---------------------------------------------------------------- O7: prediction
// p = b0 + i b1 + j b2 + k b3 evaluated as fma(b1, i, fma(b2, j, fma(b3, k, b0)))
// (DESIGN G12: fixed order, explicit fused multiply-adds).
inline double predict(const double bh[4], int i, int j, int k) {
  return std::fma(bh[1], (double)i, std::fma(bh[2], (double)j, std::fma(bh[3], (double)k, bh[0])));
}

// ---------------------------------------------------------------- O8-O10: one element
// t = (x - p) * inv2eb; outlier if !(|t| < R); q = rint(t); outlier if |q| >= R;
// x' = (T)(p + twoeb*q) (mul then add, no FMA); outlier if |x' - x| > eb_abs; code = R + q.
// kind: 0 predictable, 1 radius, 2 verify, 3 non-finite.
template <typename T>
inline int quantize_element(T xv, double p, const Bounds& bd, uint32_t R, uint16_t* code,
                            T* xprime) {
  const double xd = (double)xv;
  const double t = (xd - p) * bd.inv2eb;
  if (!(std::fabs(t) < (double)R)) {
    *code = 0; *xprime = xv;
    return std::isfinite(t) ? 1 : 3;
  }
  const double q = std::nearbyint(t);
  if (std::fabs(q) >= (double)R) {
    *code = 0; *xprime = xv;
    return 1;
  }
  const double prod = bd.twoeb * q;
  const double y = p + prod;
  const T xp = (T)y;
  if (std::fabs((double)xp - xd) > bd.eb_abs) {
    *code = 0; *xprime = xv;
    return 2;
  }
  *code = (uint16_t)((int64_t)R + (int64_t)q);
  *xprime = xp;
  return 0;
}

inline bool near_half(double u, double window) {
  double fl = std::floor(u);
  return std::fabs(u - fl - 0.5) <= window;
}

// ---------------------------------------------------------------- whole-field compression
template <typename T>
int compress_impl(const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R,
                  int eb_mode, double eb, const double* range, const T* x, uint16_t* codes,
                  int32_t* coef, double* coef_raw, uint8_t* block_exempt, uint64_t* out_idx,
                  T* out_val, uint64_t cap, uint64_t* n_out, int64_t* hist, double* eb_abs_out,
                  orc_counters* cnt, T* xprime) {
  const uint64_t n0 = dims[0], n1 = dims[1], n2 = dims[2];
  const uint64_t N = n0 * n1 * n2;
  double lo = 0.0, hi = 0.0;
  if (eb_mode == 1) {
    if (range) {
      lo = range[0]; hi = range[1];
    } else {
      // a0 / O1: value range over the (local) field, as T widened to fp64.
      lo = hi = (double)x[0];
      for (uint64_t e = 0; e < N; e++) {
        double v = (double)x[e];
        if (std::isnan(v)) { lo = hi = v; break; }
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
    }
  }
  Bounds bd;
  if (!make_bounds(eb_mode, eb, lo, hi, B, &bd)) return ORC_EBADRANGE;
  if (eb_abs_out) *eb_abs_out = bd.eb_abs;

  orc_counters c{};
  uint64_t nout = 0;
  const uint64_t NB0 = ceil_div(n0, B), NB1 = ceil_div(n1, B), NB2 = ceil_div(n2, B);
  if (hist) std::memset(hist, 0, sizeof(int64_t) * 2 * (size_t)R);

  // O3: blocks in row-major block order; edge blocks clipped (DESIGN G3).
  for (uint64_t a = 0; a < NB0; a++)
    for (uint64_t b = 0; b < NB1; b++)
      for (uint64_t cc = 0; cc < NB2; cc++) {
        const uint64_t bid = (a * NB1 + b) * NB2 + cc;
        const uint64_t i0 = a * B, j0 = b * B, k0 = cc * B;
        const int m0 = (int)std::min<uint64_t>(B, n0 - i0);
        const int m1 = (int)std::min<uint64_t>(B, n1 - j0);
        const int m2 = (int)std::min<uint64_t>(B, n2 - k0);
        double V[4], beta[4], bhat[4];
        int32_t cd[4];
        block_moments(x, n1, n2, i0, j0, k0, m0, m1, m2, V);
        lemma_beta(V, m0, m1, m2, beta);
        if (coef_codes(beta, bd, cd, bhat)) c.zero_predictor_blocks++;
        for (int d = 0; d < 4; d++) {
          coef[4 * bid + d] = cd[d];
          if (coef_raw) coef_raw[4 * bid + d] = beta[d];
        }
        // (iii) coefficient tie window: the GPU may sum moments in another order, so its beta
        // can differ by the parity tolerance 1e-12 * max(|beta|, mean|f|); a code can then
        // differ only if beta/w lies within that distance (or 1e-9) of a half-integer.
        double absum = 0.0;
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++)
              absum += std::fabs((double)x[((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k)]);
        const double scale = absum / ((double)m0 * m1 * m2);
        bool tie_block = false;
        for (int d = 0; d < 4; d++) {
          const double w = (d == 0) ? bd.w0 : bd.ws;
          const double u = beta[d] / w;
          if (!std::isfinite(u)) continue;
          const double win = std::max(1e-9, 1e-12 * std::max(std::fabs(beta[d]), scale) / w);
          if (near_half(u, win)) { c.coef_near_ties++; tie_block = true; }
        }
        if (tie_block) c.coef_tie_blocks++;
        if (block_exempt) block_exempt[bid] = tie_block ? 1 : 0;

        // Alg. 1: for every element of the block, predict then quantize.
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) {
              const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
              const double p = predict(bhat, i, j, k);
              // counters (i), (ii): pre-rounding residual / (2 eb) by true division
              const double tdiv = ((double)x[e] - p) / bd.twoeb;
              const double tmul = ((double)x[e] - p) * bd.inv2eb;
              if (std::isfinite(tdiv) && std::fabs(tmul) < (double)R) {
                if (near_half(tdiv, 1e-9)) c.elem_near_ties++;
                if (std::nearbyint(tdiv) != std::nearbyint(tmul)) c.elem_div_mismatch++;
              }
              uint16_t code;
              T xp;
              const int kind = quantize_element<T>(x[e], p, bd, R, &code, &xp);
              codes[e] = code;
              if (xprime) xprime[e] = xp;
              if (kind != 0) {
                if (kind == 1) c.radius_outliers++;
                else if (kind == 2) c.verify_outliers++;
                else c.nonfinite_outliers++;
                if (nout < cap) {
                  out_idx[nout] = e + dim0_offset * n1 * n2;
                  out_val[nout] = x[e];
                }
                nout++;
              }
              if (hist) hist[code]++;  // O11 (bin 0 counts outliers)
            }
      }
  if (n_out) *n_out = nout;
  if (cnt) *cnt = c;
  return nout > cap ? ORC_EOVERFLOW : ORC_OK;
}

// ---------------------------------------------------------------- decompression
// recover: recompute O6-O7 from the codes, x' = (T)(p + twoeb*(c - R)) for c != 0
// (same ops as O9), x' = stored value for c == 0 ("stored separately").
template <typename T>
int decompress_impl(const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R,
                    double eb_abs, const uint16_t* codes, const int32_t* coef,
                    const uint64_t* out_idx, const T* out_val, uint64_t n_out, T* xo) {
  Bounds bd;
  if (!make_bounds(0, eb_abs, 0, 0, B, &bd)) return ORC_EINVAL;
  const uint64_t n0 = dims[0], n1 = dims[1], n2 = dims[2];
  const uint64_t NB0 = ceil_div(n0, B), NB1 = ceil_div(n1, B), NB2 = ceil_div(n2, B);
  for (uint64_t a = 0; a < NB0; a++)
    for (uint64_t b = 0; b < NB1; b++)
      for (uint64_t cc = 0; cc < NB2; cc++) {
        const uint64_t bid = (a * NB1 + b) * NB2 + cc;
        const uint64_t i0 = a * B, j0 = b * B, k0 = cc * B;
        const int m0 = (int)std::min<uint64_t>(B, n0 - i0);
        const int m1 = (int)std::min<uint64_t>(B, n1 - j0);
        const int m2 = (int)std::min<uint64_t>(B, n2 - k0);
        double bhat[4];
        bhat[0] = (double)coef[4 * bid] * bd.w0;
        for (int d = 1; d < 4; d++) bhat[d] = (double)coef[4 * bid + d] * bd.ws;
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) {
              const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
              const uint16_t code = codes[e];
              if (code == 0) { xo[e] = (T)0; continue; }
              const double p = predict(bhat, i, j, k);
              const double q = (double)((int64_t)code - (int64_t)R);
              const double prod = bd.twoeb * q;
              const double y = p + prod;
              xo[e] = (T)y;
            }
      }
  const uint64_t base = dim0_offset * n1 * n2;
  for (uint64_t m = 0; m < n_out; m++) {
    const uint64_t e = out_idx[m] - base;
    if (out_idx[m] < base || e >= n0 * n1 * n2) return ORC_EINVAL;
    xo[e] = out_val[m];
  }
  return ORC_OK;
}


// ---------------------------------------------------------------- SZ3-LR (NEXT-4; DEFINITION.md L1-L7)
// "a multialgorithm predictor ... a Lorenzo predictor and a regression-based predictor and predicts
// data using the better result in between based on blockwise error estimation".  The paper's
// Lorenzo section is empty (P:7); the readings are DESIGN G26-G29: the Lorenzo predictor works on the
// prequantised values q = rint(x / 2eb) (L1), first order, block-local (L2); a block's choice is the
// predictor with the smaller sum of |code - R| (outliers count R) over the block (L5).

// L1: q = rint(x * inv2eb) (the O8 product with p = 0); not usable (q = 0) if |x * inv2eb| >= 2^50 or
// x is not finite.
template <typename T>
inline int64_t lr_prequant(T xv, const Bounds& bd, bool* ok) {
  const double t = (double)xv * bd.inv2eb;
  if (!(std::fabs(t) < 1125899906842624.0)) { *ok = false; return 0; }
  *ok = true;
  return (int64_t)std::nearbyint(t);
}

// L2: delta(i,j,k) = sum over a,b,c in {0,1} of (-1)^(a+b+c) q(i-a, j-b, k-c), q = 0 outside the block
// (block extents m1, m2; q laid out [i][j][k] with strides m1*m2, m2).  Unsigned wrap-around keeps
// garbage streams defined; valid data never comes near 2^63.
inline int64_t lr_delta(const std::vector<int64_t>& q, int m1, int m2, int i, int j, int k) {
  uint64_t s = 0;
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++)
      for (int c = 0; c < 2; c++) {
        const int ii = i - a, jj = j - b, kk = k - c;
        if (ii < 0 || jj < 0 || kk < 0) continue;
        const uint64_t v = (uint64_t)q[((size_t)ii * m1 + jj) * m2 + kk];
        s = ((a + b + c) & 1) ? s - v : s + v;
      }
  return (int64_t)s;
}

template <typename T>
int lr_compress_impl(const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R, int eb_mode,
                     double eb, const double* range, const T* x, uint16_t* codes, int32_t* coef,
                     double* coef_raw, uint8_t* block_exempt, uint8_t* flags, uint64_t* out_idx, T* out_val,
                     uint64_t cap, uint64_t* n_out, int64_t* hist, double* eb_abs_out, T* xprime,
                     uint64_t* n_lorenzo) {
  const uint64_t n0 = dims[0], n1 = dims[1], n2 = dims[2];
  const uint64_t N = n0 * n1 * n2;
  double lo = 0.0, hi = 0.0;
  if (eb_mode == 1) {
    if (range) {
      lo = range[0]; hi = range[1];
    } else {
      lo = hi = (double)x[0];
      for (uint64_t e = 0; e < N; e++) {
        double v = (double)x[e];
        if (std::isnan(v)) { lo = hi = v; break; }
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
    }
  }
  Bounds bd;
  if (!make_bounds(eb_mode, eb, lo, hi, B, &bd)) return ORC_EBADRANGE;
  if (eb_abs_out) *eb_abs_out = bd.eb_abs;
  uint64_t nout = 0, nl = 0;
  const uint64_t NB0 = ceil_div(n0, B), NB1 = ceil_div(n1, B), NB2 = ceil_div(n2, B);
  if (hist) std::memset(hist, 0, sizeof(int64_t) * 2 * (size_t)R);
  const size_t BB = (size_t)B * B * B;
  std::vector<uint16_t> cR(BB), cL(BB);
  std::vector<T> xR(BB), xL(BB);
  std::vector<int64_t> q(BB);
  std::vector<uint8_t> qok(BB);
  for (uint64_t a = 0; a < NB0; a++)
    for (uint64_t b = 0; b < NB1; b++)
      for (uint64_t cc = 0; cc < NB2; cc++) {
        const uint64_t bid = (a * NB1 + b) * NB2 + cc;
        const uint64_t i0 = a * B, j0 = b * B, k0 = cc * B;
        const int m0 = (int)std::min<uint64_t>(B, n0 - i0);
        const int m1 = (int)std::min<uint64_t>(B, n1 - j0);
        const int m2 = (int)std::min<uint64_t>(B, n2 - k0);
        // L4: the regression side is O4-O10 unchanged
        double V[4], beta[4], bhat[4];
        int32_t cd[4];
        block_moments(x, n1, n2, i0, j0, k0, m0, m1, m2, V);
        lemma_beta(V, m0, m1, m2, beta);
        coef_codes(beta, bd, cd, bhat);
        double absum = 0.0;
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) absum += std::fabs((double)x[((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k)]);
        const double scale = absum / ((double)m0 * m1 * m2);
        bool tie_block = false;
        for (int d = 0; d < 4; d++) {
          const double w = (d == 0) ? bd.w0 : bd.ws;
          const double u = beta[d] / w;
          if (!std::isfinite(u)) continue;
          const double win = std::max(1e-9, 1e-12 * std::max(std::fabs(beta[d]), scale) / w);
          if (near_half(u, win)) tie_block = true;
        }
        uint64_t costR = 0, costL = 0;
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) {
              const size_t l = ((size_t)i * m1 + j) * m2 + k;
              const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
              quantize_element<T>(x[e], predict(bhat, i, j, k), bd, R, &cR[l], &xR[l]);
              costR += cR[l] == 0 ? R : (uint64_t)std::llabs((int64_t)cR[l] - (int64_t)R);
              bool ok;
              q[l] = lr_prequant<T>(x[e], bd, &ok);
              qok[l] = ok ? 1 : 0;
            }
        // L2 + L3: Lorenzo residual, code, verify
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) {
              const size_t l = ((size_t)i * m1 + j) * m2 + k;
              const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
              cL[l] = 0;
              xL[l] = x[e];
              if (qok[l]) {
                const int64_t d = lr_delta(q, m1, m2, i, j, k);
                if (d > -(int64_t)R && d < (int64_t)R) {
                  const T xp = (T)(bd.twoeb * (double)q[l]);
                  if (std::fabs((double)xp - (double)x[e]) <= bd.eb_abs) {
                    cL[l] = (uint16_t)((int64_t)R + d);
                    xL[l] = xp;
                  }
                }
              }
              costL += cL[l] == 0 ? R : (uint64_t)std::llabs((int64_t)cL[l] - (int64_t)R);
            }
        // L5 + L6: the cheaper predictor (ties -> regression)
        const bool useL = costL < costR;
        nl += useL ? 1 : 0;
        if (flags) flags[bid] = useL ? 1 : 0;
        for (int d = 0; d < 4; d++) {
          coef[4 * bid + d] = useL ? 0 : cd[d];
          if (coef_raw) coef_raw[4 * bid + d] = beta[d];
        }
        if (block_exempt) block_exempt[bid] = tie_block ? 1 : 0;
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) {
              const size_t l = ((size_t)i * m1 + j) * m2 + k;
              const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
              const uint16_t code = useL ? cL[l] : cR[l];
              codes[e] = code;
              if (xprime) xprime[e] = useL ? xL[l] : xR[l];
              if (code == 0) {
                if (nout < cap) {
                  out_idx[nout] = e + dim0_offset * n1 * n2;
                  out_val[nout] = x[e];
                }
                nout++;
              }
              if (hist) hist[code]++;
            }
      }
  if (n_out) *n_out = nout;
  if (n_lorenzo) *n_lorenzo = nl;
  return nout > cap ? ORC_EOVERFLOW : ORC_OK;
}

// L7: outliers first (their stored x is the decompressed value and gives q by L1), then per block in
// (i, j, k) order: regression blocks as O12, Lorenzo blocks q = (code - R) + (q - delta(q)) at (i,j,k)
// (the seven earlier neighbours), x' = (T)(twoeb * q).
template <typename T>
int lr_decompress_impl(const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R, double eb_abs,
                       const uint16_t* codes, const int32_t* coef, const uint8_t* flags, const uint64_t* out_idx,
                       const T* out_val, uint64_t n_out, T* xo) {
  Bounds bd;
  if (!make_bounds(0, eb_abs, 0, 0, B, &bd)) return ORC_EINVAL;
  const uint64_t n0 = dims[0], n1 = dims[1], n2 = dims[2];
  const uint64_t base = dim0_offset * n1 * n2;
  for (uint64_t m = 0; m < n_out; m++) {
    const uint64_t e = out_idx[m] - base;
    if (out_idx[m] < base || e >= n0 * n1 * n2) return ORC_EINVAL;
    xo[e] = out_val[m];
  }
  const uint64_t NB0 = ceil_div(n0, B), NB1 = ceil_div(n1, B), NB2 = ceil_div(n2, B);
  std::vector<int64_t> q((size_t)B * B * B);
  for (uint64_t a = 0; a < NB0; a++)
    for (uint64_t b = 0; b < NB1; b++)
      for (uint64_t cc = 0; cc < NB2; cc++) {
        const uint64_t bid = (a * NB1 + b) * NB2 + cc;
        const uint64_t i0 = a * B, j0 = b * B, k0 = cc * B;
        const int m0 = (int)std::min<uint64_t>(B, n0 - i0);
        const int m1 = (int)std::min<uint64_t>(B, n1 - j0);
        const int m2 = (int)std::min<uint64_t>(B, n2 - k0);
        if (!flags[bid]) {
          double bhat[4];
          bhat[0] = (double)coef[4 * bid] * bd.w0;
          for (int d = 1; d < 4; d++) bhat[d] = (double)coef[4 * bid + d] * bd.ws;
          for (int i = 0; i < m0; i++)
            for (int j = 0; j < m1; j++)
              for (int k = 0; k < m2; k++) {
                const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
                const uint16_t code = codes[e];
                if (code == 0) continue;   // the stored value, scattered above
                const double p = predict(bhat, i, j, k);
                const double qd = (double)((int64_t)code - (int64_t)R);
                const double prod = bd.twoeb * qd;
                xo[e] = (T)(p + prod);
              }
          continue;
        }
        for (int i = 0; i < m0; i++)
          for (int j = 0; j < m1; j++)
            for (int k = 0; k < m2; k++) {
              const size_t l = ((size_t)i * m1 + j) * m2 + k;
              const uint64_t e = ((i0 + i) * n1 + (j0 + j)) * n2 + (k0 + k);
              const uint16_t code = codes[e];
              if (code == 0) {
                bool ok;
                q[l] = lr_prequant<T>(xo[e], bd, &ok);
                continue;
              }
              q[l] = 0;   // delta over the earlier neighbours only
              const uint64_t pred = (uint64_t)0 - (uint64_t)lr_delta(q, m1, m2, i, j, k);
              q[l] = (int64_t)(pred + (uint64_t)((int64_t)code - (int64_t)R));
              xo[e] = (T)(bd.twoeb * (double)q[l]);
            }
      }
  return ORC_OK;
}

// ---------------------------------------------------------------- SZ3-Interp (NEXT-4; DEFINITION.md I1-I6)
// I2: the level plan.  S = the largest power of two below the largest extent; levels s = S, S/2, .., 1;
// in a level, one pass per axis d = 0, 1, 2.  Pass (s, d) predicts the indices whose coordinate along
// d is an odd multiple of s, whose coordinates along the earlier axes are multiples of s and along the
// later axes multiples of 2s.  Every index but the anchor (0, 0, 0) belongs to exactly one pass.
inline uint64_t interp_top_stride(const uint64_t dims[3]) {
  const uint64_t n = std::max(dims[0], std::max(dims[1], dims[2]));
  uint64_t S = 1;
  while (2 * S < n) S *= 2;
  return n > 1 ? S : 0;
}

// I3: prediction along axis d from the reconstructed donors at -3s, -s, +s, +3s (cubic spline weights
// (-1, 9, 9, -1)/16 when all four exist, the midpoint when only -s and +s do, else a copy of -s).
// All in fp64, no contraction: u = b + c, v = a + e, p = (9 u - v) * 0.0625.
inline double interp_predict(double a, double b, double c, double e, int method) {
  if (method == 2) {
    const double u = b + c;
    const double v = a + e;
    const double w = 9.0 * u;
    return (w - v) * 0.0625;
  }
  if (method == 1) return (b + c) * 0.5;
  return b;
}

// method of a target at coordinate i along an axis of extent n with stride s
inline int interp_method(uint64_t i, uint64_t n, uint64_t s) {
  if (i >= 3 * s && i + 3 * s < n) return 2;
  if (i + s < n) return 1;
  return 0;
}

template <typename T>
int interp_compress_impl(const uint64_t dims[3], uint64_t dim0_offset, uint32_t R, int eb_mode, double eb,
                         const double* range, const T* x, uint16_t* codes, uint64_t* out_idx, T* out_val,
                         uint64_t cap, uint64_t* n_out, int64_t* hist, double* eb_abs_out, T* xp, orc_counters* cnt) {
  const uint64_t n0 = dims[0], n1 = dims[1], n2 = dims[2], N = n0 * n1 * n2;
  double lo = 0.0, hi = 0.0;
  if (eb_mode == 1) {   // I1 = O1
    if (range) {
      lo = range[0]; hi = range[1];
    } else {
      lo = hi = (double)x[0];
      for (uint64_t e = 0; e < N; e++) {
        double v = (double)x[e];
        if (std::isnan(v)) { lo = hi = v; break; }
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
    }
  }
  Bounds bd;
  if (!make_bounds(eb_mode, eb, lo, hi, 6, &bd)) return ORC_EBADRANGE;
  if (eb_abs_out) *eb_abs_out = bd.eb_abs;
  orc_counters c{};
  uint64_t nout = 0;
  auto outlier = [&](uint64_t e) {
    if (nout < cap) { out_idx[nout] = e + dim0_offset * n1 * n2; out_val[nout] = x[e]; }
    nout++;
  };
  // I4: the anchor is stored as it is
  codes[0] = 0;
  xp[0] = x[0];
  outlier(0);
  const uint64_t S = interp_top_stride(dims);
  const uint64_t st[3] = {n1 * n2, n2, 1};
  for (uint64_t s = S; s >= 1; s /= 2) {
    for (int d = 0; d < 3; d++) {
      uint64_t first[3], step[3];
      for (int a = 0; a < 3; a++) {
        first[a] = a == d ? s : 0;
        step[a] = (a == d || a > d) ? 2 * s : s;
      }
      for (uint64_t i0 = first[0]; i0 < n0; i0 += step[0])
        for (uint64_t i1 = first[1]; i1 < n1; i1 += step[1])
          for (uint64_t i2 = first[2]; i2 < n2; i2 += step[2]) {
            const uint64_t e = i0 * st[0] + i1 * st[1] + i2 * st[2];
            const uint64_t id = d == 0 ? i0 : (d == 1 ? i1 : i2);
            const int m = interp_method(id, dims[d], s);
            const uint64_t sd = s * st[d];
            const double a = m == 2 ? (double)xp[e - 3 * sd] : 0.0;
            const double b = (double)xp[e - sd];
            const double cc = m >= 1 ? (double)xp[e + sd] : 0.0;
            const double ee = m == 2 ? (double)xp[e + 3 * sd] : 0.0;
            const double p = interp_predict(a, b, cc, ee, m);
            // I5 = O8-O10 with the interpolated prediction
            uint16_t code;
            T xv;
            const int kind = quantize_element<T>(x[e], p, bd, R, &code, &xv);
            codes[e] = code;
            xp[e] = xv;
            if (kind != 0) {
              if (kind == 1) c.radius_outliers++;
              else if (kind == 2) c.verify_outliers++;
              else c.nonfinite_outliers++;
              outlier(e);
            }
          }
    }
    if (s == 1) break;
  }
  if (hist) {   // O11
    std::memset(hist, 0, sizeof(int64_t) * 2 * (size_t)R);
    for (uint64_t e = 0; e < N; e++) hist[codes[e]]++;
  }
  *n_out = nout;
  if (cnt) *cnt = c;
  return nout > cap ? ORC_EOVERFLOW : ORC_OK;
}

// I6: decompression replays the plan on x' (outlier values first, then the passes in order)
template <typename T>
int interp_decompress_impl(const uint64_t dims[3], uint64_t dim0_offset, uint32_t R, double eb_abs,
                           const uint16_t* codes, const uint64_t* out_idx, const T* out_val, uint64_t n_out,
                           T* xo) {
  const uint64_t n0 = dims[0], n1 = dims[1], n2 = dims[2], N = n0 * n1 * n2;
  Bounds bd;
  if (!make_bounds(0, eb_abs, 0, 0, 6, &bd)) return ORC_EBADRANGE;
  for (uint64_t e = 0; e < N; e++) xo[e] = T(0);
  for (uint64_t o = 0; o < n_out; o++) {
    const uint64_t e = out_idx[o] - dim0_offset * n1 * n2;
    if (e < N) xo[e] = out_val[o];
  }
  const uint64_t S = interp_top_stride(dims);
  const uint64_t st[3] = {n1 * n2, n2, 1};
  for (uint64_t s = S; s >= 1; s /= 2) {
    for (int d = 0; d < 3; d++) {
      uint64_t first[3], step[3];
      for (int a = 0; a < 3; a++) {
        first[a] = a == d ? s : 0;
        step[a] = (a == d || a > d) ? 2 * s : s;
      }
      for (uint64_t i0 = first[0]; i0 < n0; i0 += step[0])
        for (uint64_t i1 = first[1]; i1 < n1; i1 += step[1])
          for (uint64_t i2 = first[2]; i2 < n2; i2 += step[2]) {
            const uint64_t e = i0 * st[0] + i1 * st[1] + i2 * st[2];
            if (codes[e] == 0) continue;   // outlier: its value is already in place
            const uint64_t id = d == 0 ? i0 : (d == 1 ? i1 : i2);
            const int m = interp_method(id, dims[d], s);
            const uint64_t sd = s * st[d];
            const double a = m == 2 ? (double)xo[e - 3 * sd] : 0.0;
            const double b = (double)xo[e - sd];
            const double cc = m >= 1 ? (double)xo[e + sd] : 0.0;
            const double ee = m == 2 ? (double)xo[e + 3 * sd] : 0.0;
            const double p = interp_predict(a, b, cc, ee, m);
            const double q = (double)((int64_t)codes[e] - (int64_t)R);
            const double prod = bd.twoeb * q;
            xo[e] = (T)(p + prod);
          }
    }
    if (s == 1) break;
  }
  return ORC_OK;
}

bool check_dims(const uint64_t* dims, uint32_t B, uint32_t R) {
  if (!dims || dims[0] == 0 || dims[1] == 0 || dims[2] == 0) return false;
  if (B < 1 || R < 1 || R > 32768) return false;
  return true;
}

}  // namespace

extern "C" {

// a0: value range [lo, hi] of an n-element T array (NaN anywhere -> both NaN).
int orc_value_range(int dtype, uint64_t n, const void* x, double out[2]) {
  if (!x || n == 0) return ORC_EINVAL;
  double lo, hi;
  if (dtype == 0) {
    const float* f = (const float*)x;
    lo = hi = f[0];
    for (uint64_t e = 0; e < n; e++) {
      double v = f[e];
      if (std::isnan(v)) { lo = hi = v; break; }
      lo = std::min(lo, v); hi = std::max(hi, v);
    }
  } else if (dtype == 1) {
    const double* f = (const double*)x;
    lo = hi = f[0];
    for (uint64_t e = 0; e < n; e++) {
      double v = f[e];
      if (std::isnan(v)) { lo = hi = v; break; }
      lo = std::min(lo, v); hi = std::max(hi, v);
    }
  } else {
    return ORC_EUNSUPPORTED;
  }
  out[0] = lo; out[1] = hi;
  return ORC_OK;
}

int orc_compress(int dtype, const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R,
                 int eb_mode, double eb, const double* range, const void* x, uint16_t* codes,
                 int32_t* coef, double* coef_raw, uint8_t* block_exempt, uint64_t* out_idx,
                 void* out_val, uint64_t cap, uint64_t* n_out, int64_t* hist, double* eb_abs_out,
                 orc_counters* cnt, void* xprime /* nullable: compress-time x' (T) */) {
  if (!check_dims(dims, B, R)) return (R < 1 || R > 32768) ? ORC_ERANGE : ORC_EINVAL;
  if (!x || !codes || !coef || (cap > 0 && (!out_idx || !out_val))) return ORC_EINVAL;
  if (!(eb > 0.0) || !std::isfinite(eb) || (eb_mode != 0 && eb_mode != 1)) return ORC_EINVAL;
  if (dtype == 0)
    return compress_impl<float>(dims, dim0_offset, B, R, eb_mode, eb, range, (const float*)x,
                                codes, coef, coef_raw, block_exempt, out_idx, (float*)out_val, cap,
                                n_out, hist, eb_abs_out, cnt, (float*)xprime);
  if (dtype == 1)
    return compress_impl<double>(dims, dim0_offset, B, R, eb_mode, eb, range, (const double*)x,
                                 codes, coef, coef_raw, block_exempt, out_idx, (double*)out_val,
                                 cap, n_out, hist, eb_abs_out, cnt, (double*)xprime);
  return ORC_EUNSUPPORTED;
}

int orc_decompress(int dtype, const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R,
                   double eb_abs, const uint16_t* codes, const int32_t* coef,
                   const uint64_t* out_idx, const void* out_val, uint64_t n_out, void* x_out) {
  if (!check_dims(dims, B, R)) return (R < 1 || R > 32768) ? ORC_ERANGE : ORC_EINVAL;
  if (!codes || !coef || !x_out || (n_out > 0 && (!out_idx || !out_val))) return ORC_EINVAL;
  if (dtype == 0)
    return decompress_impl<float>(dims, dim0_offset, B, R, eb_abs, codes, coef, out_idx,
                                  (const float*)out_val, n_out, (float*)x_out);
  if (dtype == 1)
    return decompress_impl<double>(dims, dim0_offset, B, R, eb_abs, codes, coef, out_idx,
                                   (const double*)out_val, n_out, (double*)x_out);
  return ORC_EUNSUPPORTED;
}

// ----- block / element level entry points (used by the pins in tests/test_oracle_pins.py)

// O4 + O5 on one dense m0 x m1 x m2 block of fp64 values (row-major, k fastest).
void orc_block_beta(const double* f, int m0, int m1, int m2, double V_out[4], double beta[4]) {
  double V[4];
  block_moments<double>(f, (uint64_t)m1, (uint64_t)m2, 0, 0, 0, m0, m1, m2, V);
  lemma_beta(V, m0, m1, m2, beta);
  if (V_out) for (int d = 0; d < 4; d++) V_out[d] = V[d];
}

// O6 on given raw coefficients; returns 1 if the zero predictor was chosen.
int orc_coef_codes(const double beta[4], double eb_abs, uint32_t B, int32_t c[4], double bhat[4]) {
  Bounds bd;
  if (!make_bounds(0, eb_abs, 0, 0, B, &bd)) return -1;
  return coef_codes(beta, bd, c, bhat) ? 1 : 0;
}

// O7.
double orc_predict(const double bhat[4], int i, int j, int k) { return predict(bhat, i, j, k); }

// O8-O10 for one element of dtype (value passed widened to fp64; for f32 it must be an f32
// value). Returns the outlier kind (0 predictable, 1 radius, 2 verify, 3 non-finite).
int orc_quantize_element(int dtype, double x, double p, double eb_abs, uint32_t R, uint16_t* code,
                         double* xprime) {
  Bounds bd;
  if (!make_bounds(0, eb_abs, 0, 0, 6, &bd)) return -1;
  if (dtype == 0) {
    float xp;
    int k = quantize_element<float>((float)x, p, bd, R, code, &xp);
    *xprime = xp;
    return k;
  }
  double xp;
  int k = quantize_element<double>(x, p, bd, R, code, &xp);
  *xprime = xp;
  return k;
}


// SZ3-LR (NEXT-4): compress -> codes, coefficient codes (0 for Lorenzo blocks), per-block predictor
// flags (1 = Lorenzo), outliers, histogram; decompress -> x'.
int orc_lr_compress(int dtype, const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R, int eb_mode,
                    double eb, const double* range, const void* x, uint16_t* codes, int32_t* coef, double* coef_raw,
                    uint8_t* block_exempt, uint8_t* flags, uint64_t* out_idx, void* out_val, uint64_t cap,
                    uint64_t* n_out, int64_t* hist, double* eb_abs_out, void* xprime, uint64_t* n_lorenzo) {
  if (!check_dims(dims, B, R)) return (R < 1 || R > 32768) ? ORC_ERANGE : ORC_EINVAL;
  if (!x || !codes || !coef || !flags || (cap > 0 && (!out_idx || !out_val))) return ORC_EINVAL;
  if (!(eb > 0.0) || !std::isfinite(eb) || (eb_mode != 0 && eb_mode != 1)) return ORC_EINVAL;
  if (dtype == 0)
    return lr_compress_impl<float>(dims, dim0_offset, B, R, eb_mode, eb, range, (const float*)x, codes, coef, coef_raw,
                                   block_exempt, flags, out_idx, (float*)out_val, cap, n_out, hist, eb_abs_out,
                                   (float*)xprime, n_lorenzo);
  if (dtype == 1)
    return lr_compress_impl<double>(dims, dim0_offset, B, R, eb_mode, eb, range, (const double*)x, codes, coef,
                                    coef_raw, block_exempt, flags, out_idx, (double*)out_val, cap, n_out, hist,
                                    eb_abs_out, (double*)xprime, n_lorenzo);
  return ORC_EUNSUPPORTED;
}

int orc_lr_decompress(int dtype, const uint64_t dims[3], uint64_t dim0_offset, uint32_t B, uint32_t R, double eb_abs,
                      const uint16_t* codes, const int32_t* coef, const uint8_t* flags, const uint64_t* out_idx,
                      const void* out_val, uint64_t n_out, void* x_out) {
  if (!check_dims(dims, B, R)) return (R < 1 || R > 32768) ? ORC_ERANGE : ORC_EINVAL;
  if (!codes || !coef || !flags || !x_out || (n_out > 0 && (!out_idx || !out_val))) return ORC_EINVAL;
  if (dtype == 0)
    return lr_decompress_impl<float>(dims, dim0_offset, B, R, eb_abs, codes, coef, flags, out_idx,
                                     (const float*)out_val, n_out, (float*)x_out);
  if (dtype == 1)
    return lr_decompress_impl<double>(dims, dim0_offset, B, R, eb_abs, codes, coef, flags, out_idx,
                                      (const double*)out_val, n_out, (double*)x_out);
  return ORC_EUNSUPPORTED;
}

// L2 on one dense block of integers (for the pins)
int64_t orc_lr_delta(const int64_t* q, int m0, int m1, int m2, int i, int j, int k) {
  std::vector<int64_t> v(q, q + (size_t)m0 * m1 * m2);
  return lr_delta(v, m1, m2, i, j, k);
}


// SZ3-Interp (NEXT-4): compress -> codes, outliers (the anchor first), histogram, x'; decompress -> x'.
int orc_interp_compress(int dtype, const uint64_t dims[3], uint64_t dim0_offset, uint32_t R, int eb_mode, double eb,
                        const double* range, const void* x, uint16_t* codes, uint64_t* out_idx, void* out_val,
                        uint64_t cap, uint64_t* n_out, int64_t* hist, double* eb_abs_out, void* xprime,
                        orc_counters* cnt) {
  if (!check_dims(dims, 6, R)) return (R < 1 || R > 32768) ? ORC_ERANGE : ORC_EINVAL;
  if (!x || !codes || !xprime || !n_out || cap < 1 || !out_idx || !out_val) return ORC_EINVAL;
  if (!(eb > 0.0) || !std::isfinite(eb) || (eb_mode != 0 && eb_mode != 1)) return ORC_EINVAL;
  if (dtype == 0)
    return interp_compress_impl<float>(dims, dim0_offset, R, eb_mode, eb, range, (const float*)x, codes, out_idx,
                                       (float*)out_val, cap, n_out, hist, eb_abs_out, (float*)xprime, cnt);
  if (dtype == 1)
    return interp_compress_impl<double>(dims, dim0_offset, R, eb_mode, eb, range, (const double*)x, codes, out_idx,
                                        (double*)out_val, cap, n_out, hist, eb_abs_out, (double*)xprime, cnt);
  return ORC_EUNSUPPORTED;
}

int orc_interp_decompress(int dtype, const uint64_t dims[3], uint64_t dim0_offset, uint32_t R, double eb_abs,
                          const uint16_t* codes, const uint64_t* out_idx, const void* out_val, uint64_t n_out,
                          void* x_out) {
  if (!check_dims(dims, 6, R)) return (R < 1 || R > 32768) ? ORC_ERANGE : ORC_EINVAL;
  if (!codes || !x_out || (n_out > 0 && (!out_idx || !out_val))) return ORC_EINVAL;
  if (dtype == 0)
    return interp_decompress_impl<float>(dims, dim0_offset, R, eb_abs, codes, out_idx, (const float*)out_val, n_out,
                                         (float*)x_out);
  if (dtype == 1)
    return interp_decompress_impl<double>(dims, dim0_offset, R, eb_abs, codes, out_idx, (const double*)out_val,
                                          n_out, (double*)x_out);
  return ORC_EUNSUPPORTED;
}

// I3 and the I2 pass of one index (for the pins): pass id = 3 * level + axis, level 0 = the top stride;
// -1 for the anchor
double orc_interp_predict(double a, double b, double c, double e, int method) {
  return interp_predict(a, b, c, e, method);
}

int64_t orc_interp_pass_of(const uint64_t dims[3], uint64_t i0, uint64_t i1, uint64_t i2) {
  const uint64_t S = interp_top_stride(dims);
  const uint64_t ii[3] = {i0, i1, i2};
  int64_t level = 0;
  for (uint64_t s = S; s >= 1; s /= 2, level++) {
    for (int d = 0; d < 3; d++) {
      bool in = ii[d] % (2 * s) == s;
      for (int a = 0; a < 3 && in; a++) {
        if (a < d) in = ii[a] % s == 0;
        if (a > d) in = ii[a] % (2 * s) == 0;
      }
      if (in) return 3 * level + d;
    }
    if (s == 1) break;
  }
  return -1;
}

uint64_t orc_num_blocks(const uint64_t dims[3], uint32_t B) {
  return ceil_div(dims[0], B) * ceil_div(dims[1], B) * ceil_div(dims[2], B);
}

}  // extern "C"
