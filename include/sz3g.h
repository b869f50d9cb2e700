/* =====================================================================================
 * sz3g.h -- C ABI of the B200 (sm_100a) block-regression compressor hot path.
 *
 * Implements, on device, SZ3's block-wise linear-regression predictor with linear-scaling
 * quantisation (arxiv 2111.02925, PAPER.md):
 *   - Lemma 1 / Eq. (thm1sol) closed-form coefficients ............ P:46-67
 *   - prediction f_ijk = b0 + i b1 + j b2 + k b3, residual,
 *     linear-scaling quantisation ................................. P:156
 *   - bins of width 2*eb, out-of-range residuals stored separately
 *   - quantize / recover ........................................... P:400-404, App. A
 *   - block-then-element iteration ................................. App. A
 *   - error bound normalised to the value range .................... P:833
 * The exact arithmetic (operation order, rounding, the readings of passages the paper leaves
 * silent) is oracle/DEFINITION.md O1-O11 + D; DESIGN.md lists the readings G1-G18.
 *
 * Conventions for every call:
 *   - Data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless a parameter
 *     says "host".  The caller owns every buffer; the library never allocates or frees device
 *     memory and keeps no state between calls (re-entrant on different streams).
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream) and returns
 *     before it completes.  Host-side argument errors are returned synchronously (SZ3G_E*);
 *     device-side conditions are written to a caller-provided device status word.
 *   - Grids are row-major, contiguous, slowest dimension first: element (i,j,k) lives at
 *     ((i*n1 + j)*n2 + k).  1D / 2D fields are passed as 3D with leading extents 1.
 *   - Blocks are B x B x B (B = block_size = 6), edge blocks clipped (never padded); block id
 *     (a*NB1 + b)*NB2 + c with NB_d = ceil(n_d / B).
 * ===================================================================================== */
#ifndef SZ3G_H
#define SZ3G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sz3g_stream_t; /* == cudaStream_t */

/* ---- return codes (host side, synchronous) */
#define SZ3G_OK            0
#define SZ3G_EINVAL       (-1) /* null pointer, a zero extent, eb <= 0 or not finite, bad enum   */
#define SZ3G_EUNSUPPORTED (-2) /* dtype / block_size / ndim not supported by the device path     */
#define SZ3G_ERANGE       (-3) /* radius outside [1, 32768] (codes must fit uint16)             */
#define SZ3G_ECUDA        (-4) /* a CUDA launch / driver call failed (see sz3g_last_cuda_error) */
#define SZ3G_ECORRUPT     (-5) /* a compressed stream failed validation (magic, version, length,
                                  section checksum)                                              */

/* ---- device status bits (written with atomicOr into *d_status; caller zeroes it first) */
#define SZ3G_STATUS_OUTLIER_OVERFLOW 0x1u /* *d_outlier_count > outlier_cap: retry, larger cap */
#define SZ3G_STATUS_BAD_RANGE        0x2u /* eb_abs not finite or <= 0 (REL: max-min <= 0/NaN) */
#define SZ3G_STATUS_BAD_HUFFMAN      0x4u /* codebook: no active symbol, a negative / >= 2^47 count,
                                             or 2^max_len < active symbols; encode: a code without
                                             a codeword; decode: a corrupt stream               */
#define SZ3G_STATUS_PAYLOAD_OVERFLOW 0x8u /* encode: the stream needs more than payload_cap words */

typedef enum { SZ3G_F32 = 0, SZ3G_F64 = 1 } sz3g_dtype;
/* ABS: eb is absolute.  REL: eb_abs = eb * (max - min) over the (global) field. */
typedef enum { SZ3G_EB_ABS = 0, SZ3G_EB_REL_RANGE = 1 } sz3g_eb_mode;

/* flags for sz3g_params.flags */
#define SZ3G_FLAG_FORCE_GENERIC 0x1u /* use the plain coalesced-load kernels even where the
                                        TMA/mbarrier pipeline applies (parity testing)        */

typedef struct {
  sz3g_dtype dtype;
  int        ndim;          /* 1..3 (informational; dims are always 3D, leading extents 1)    */
  uint64_t   dims[3];       /* local extents n0, n1, n2 (slowest first), all >= 1             */
  uint64_t   dim0_offset;   /* global index of this slab's first dim-0 plane (a multiple of B
                               when the field is sharded; 0 if not).  Only outlier indices
                               depend on it: they are global linear indices.                 */
} sz3g_grid;

typedef struct {
  uint32_t     block_size;  /* B; must be 6 (the tile shape of the device kernels)            */
  uint32_t     radius;      /* R in [1, 32768]: codes R+q for |q| < R, 0 = outlier; 2R bins  */
  sz3g_eb_mode eb_mode;
  double       eb;          /* > 0, finite; absolute or value-range relative                 */
  uint32_t     flags;       /* SZ3G_FLAG_*                                                    */
} sz3g_params;

/* a0 -- value range (needed for REL eb).
 * x: prod(dims) elements of grid->dtype.  d_minmax: device double[2] <- {min, max}, the
 * extrema widened to fp64.  If x holds a NaN, at least one of the two is NaN.  3 launches. */
int sz3g_value_range(const sz3g_grid* grid, const void* x, double* d_minmax, sz3g_stream_t stream);

/* a1-a7 -- compression (one fused kernel; 1 launch).
 *   x            in   prod(dims) T, row-major.
 *   d_minmax     in   device double[2] {min, max}; required iff eb_mode == REL (pass the GLOBAL
 *                     range when the field is sharded, so every slab uses the same eb).
 *   codes        out  prod(dims) uint16, same layout as x: R+q, or 0 for an outlier.
 *   coef_codes   out  4 x nblocks int32, [block][c0,c1,c2,c3]; b0 bin = eb/2, slopes eb/(2B).
 *   coef_raw     out  nullable; 4 x nblocks double, unquantised beta (parity checks only).
 *   outlier_idx  out  up to outlier_cap uint64 GLOBAL linear indices (dim0_offset applied),
 *   outlier_val  out  and their original values (T), in no particular order.
 *   d_outlier_count in/out device uint64 (caller zeroes it): incremented by the true number of
 *                     outliers; entries beyond outlier_cap are dropped and status bit 0 set.
 *   hist         in/out nullable; 2R int64 bins ACCUMULATED (+=): hist[code] counts codes,
 *                     hist[0] = outliers (P:418 frequency table).  Zero it for a fresh count.
 *   d_eb_abs     out  nullable; device double <- the absolute eb actually used.
 *   d_status     in/out device int32, SZ3G_STATUS_* bits or-ed in.
 * Host errors: EINVAL, EUNSUPPORTED (dtype, block_size != 6), ERANGE (radius), ECUDA.      */
int sz3g_regression_compress(const sz3g_grid* grid, const sz3g_params* params, const void* x,
                             const double* d_minmax, uint16_t* codes, int32_t* coef_codes,
                             double* coef_raw, uint64_t* outlier_idx, void* outlier_val,
                             uint64_t outlier_cap, unsigned long long* d_outlier_count,
                             int64_t* hist, double* d_eb_abs, int32_t* d_status,
                             sz3g_stream_t stream);

/* Two-pass compression (REL mode: the value range must be known before any coefficient or
 * element can be quantised).  Split so that each pass reads x once:
 *
 * a0 + a2 + a3 -- sz3g_regression_analyze: ONE read of x yields the value range and the
 * unquantised Lemma-1 coefficients of every block.
 *   x         in   prod(dims) T, row-major.
 *   d_minmax  out  device double[2] <- {min, max} as sz3g_value_range (NaN in max if a block of x
 *                  holds a NaN or infinities of both signs; either way REL compression then
 *                  reports SZ3G_STATUS_BAD_RANGE).  When sharded, all-reduce it (MIN, MAX)
 *                  before sz3g_regression_quantize.
 *   beta      out  4 x nblocks double, [block][b0,b1,b2,b3], 16-byte aligned: bit-identical to
 *                  the coef_raw output of sz3g_regression_compress on the same x.
 * Host errors: EINVAL (null / misaligned beta), EUNSUPPORTED, ECUDA.  3 launches (range init, the pass, range final;
 *           1 cooperative launch when built with -DSZ3G_ANA_COOP=1).
 *
 * a4-a7 -- sz3g_regression_quantize: compression from that beta.  Arguments and outputs are those
 * of sz3g_regression_compress (without coef_raw), plus
 *   beta      in   the analyze output for the same x (16-byte aligned).
 * Given the same x, params and d_minmax, codes / coef_codes / outliers / hist / d_eb_abs are
 * bit-identical to sz3g_regression_compress.  1 launch.                                        */
int sz3g_regression_analyze(const sz3g_grid* grid, const void* x, double* d_minmax, double* beta,
                            sz3g_stream_t stream);
int sz3g_regression_quantize(const sz3g_grid* grid, const sz3g_params* params, const void* x,
                             const double* d_minmax, const double* beta, uint16_t* codes,
                             int32_t* coef_codes, uint64_t* outlier_idx, void* outlier_val,
                             uint64_t outlier_cap, unsigned long long* d_outlier_count,
                             int64_t* hist, double* d_eb_abs, int32_t* d_status,
                             sz3g_stream_t stream);

/* a8 -- decompression (recover): x_out = (T)(p + 2 eb (c - R)) for c != 0, then the
 * stored outlier values are scattered to their indices (2 launches, stream-ordered).
 *   params           the compression parameters: ABS with eb = eb_abs, or REL with the same
 *                    relative eb and the same d_minmax (eb_abs is recomputed on the device with
 *                    the same operations, so it is bit-identical to the compress-time value).
 *   d_minmax         device double[2]; required iff params->eb_mode == REL.
 *   outlier_idx      global indices (grid->dim0_offset is subtracted), outlier_val their values.
 *   n_outliers       HOST count of stored outliers, or, when d_outlier_count is non-NULL, the
 *                    capacity of outlier_idx / outlier_val (an upper bound).
 *   d_outlier_count  nullable DEVICE uint64: the count written by sz3g_regression_compress;
 *                    min(*d_outlier_count, n_outliers) entries are scattered.
 * With d_minmax and d_outlier_count a compress -> decompress sequence needs no host
 * synchronisation.  The result is bit-identical to the compress-time x'.                     */
int sz3g_regression_decompress(const sz3g_grid* grid, const sz3g_params* params,
                               const double* d_minmax, const uint16_t* codes,
                               const int32_t* coef_codes, const uint64_t* outlier_idx,
                               const void* outlier_val, uint64_t n_outliers,
                               const unsigned long long* d_outlier_count, void* x_out,
                               sz3g_stream_t stream);

/* NEXT-4 -- SZ3-LR, the composite predictor: "a Lorenzo predictor and a regression-based predictor
 * and predicts data using the better result in between based on blockwise error estimation".
 * Definition oracle/DEFINITION.md L1-L7 (readings DESIGN G26-G29): per 6^3 block, the regression
 * codes (O7-O10, coefficients from sz3g_regression_analyze's beta) and block-local first-order 3D
 * Lorenzo codes of the prequantised values q = rint(x / 2eb) (code R + delta, decompressed value
 * (T)(2eb q)); the block keeps the predictor with the smaller sum of |code - R| (outliers count R).
 *
 * sz3g_lr_quantize -- compress from the analyze pass (run sz3g_regression_analyze first; it also
 * gives the REL range).  Arguments as sz3g_regression_quantize, plus
 *   flags       out  nblocks uint8: 1 = Lorenzo block, 0 = regression block.
 *   coef_codes  out  as sz3g_regression_quantize for regression blocks; {0,0,0,0} for Lorenzo blocks.
 *   codes / outliers / hist / d_outlier_count / d_eb_abs / d_status: of the chosen predictor, with
 *   the same semantics (outlier values are the original x).
 * Host errors: EINVAL (null or misaligned pointers), EUNSUPPORTED, ERANGE, ECUDA.  1 launch.
 *
 * sz3g_lr_decompress -- x' from the codes, coefficient codes, flags and outliers (arguments as
 * sz3g_regression_decompress plus flags).  The outlier values are scattered into x_out first:
 * Lorenzo blocks take their q from them (L7).  2 launches (1 without outliers).                 */
int sz3g_lr_quantize(const sz3g_grid* grid, const sz3g_params* params, const void* x, const double* d_minmax,
                     const double* beta, uint16_t* codes, int32_t* coef_codes, uint8_t* flags,
                     uint64_t* outlier_idx, void* outlier_val, uint64_t outlier_cap,
                     unsigned long long* d_outlier_count, int64_t* hist, double* d_eb_abs, int32_t* d_status,
                     sz3g_stream_t stream);
int sz3g_lr_decompress(const sz3g_grid* grid, const sz3g_params* params, const double* d_minmax,
                       const uint16_t* codes, const int32_t* coef_codes, const uint8_t* flags,
                       const uint64_t* outlier_idx, const void* outlier_val, uint64_t n_outliers,
                       const unsigned long long* d_outlier_count, void* x_out, sz3g_stream_t stream);

/* NEXT-4 -- SZ3-Interp, the multilevel interpolation predictor: "Both linear interpolation and cubic
 * spline interpolation are included ... SZ3-Interp has constant coefficients and therefore does not have
 * storage overhead".  Definition oracle/DEFINITION.md I1-I6 (readings DESIGN G30-G33): levels of
 * stride s = S .. 1 (S the largest power of two below the largest extent), one pass per axis; each
 * target is predicted from RECONSTRUCTED donors at -3s, -s, +s, +3s along the pass axis (cubic weights
 * (-1, 9, 9, -1)/16, the midpoint near the far edge, a copy of -s at it) and quantised as O8-O10; the
 * anchor (0,0,0) is stored as an outlier.  Level-serial: one launch per non-empty pass (<= 3 log2 S).
 * Not sharded (donors cross any slab boundary): one GPU per field.
 *
 * sz3g_interp_compress -- arguments as sz3g_regression_compress (no coefficients), plus
 *   xprime  out  prod(dims) T: the reconstruction x' (the method's working buffer; equal to what
 *                sz3g_interp_decompress returns).
 *   hist    nullable, 2R int64 bins ACCUMULATED (sz3g_histogram over the finished codes).
 *   outlier_cap >= 1 (the anchor is always stored).
 * Host errors: EINVAL, EUNSUPPORTED, ERANGE, ECUDA; device status bits as regression.
 *
 * sz3g_interp_decompress -- arguments as sz3g_regression_decompress (no coefficients): outlier
 * values scattered into x_out first, then the passes in plan order.                              */
int sz3g_interp_compress(const sz3g_grid* grid, const sz3g_params* params, const void* x, const double* d_minmax,
                         uint16_t* codes, void* xprime, uint64_t* outlier_idx, void* outlier_val,
                         uint64_t outlier_cap, unsigned long long* d_outlier_count, int64_t* hist,
                         double* d_eb_abs, int32_t* d_status, sz3g_stream_t stream);
int sz3g_interp_decompress(const sz3g_grid* grid, const sz3g_params* params, const double* d_minmax,
                           const uint16_t* codes, const uint64_t* outlier_idx, const void* outlier_val,
                           uint64_t n_outliers, const unsigned long long* d_outlier_count, void* x_out,
                           sz3g_stream_t stream);

/* a7 standalone -- histogram of n uint16 codes into 2R int64 bins, ACCUMULATED (+=).  Codes
 * >= 2R are ignored.  1 launch. */
int sz3g_histogram(const uint16_t* codes, uint64_t n, uint32_t radius, int64_t* hist,
                   sz3g_stream_t stream);

/* histogram of n uint16 symbols into nbins (<= 65536) int64 bins, ACCUMULATED; the shared-memory
 * window is [window_lo, window_lo + 8192) -- place it where the symbols' mass is (e.g. 0 for the
 * zigzag coefficient deltas); symbols >= nbins are ignored.  1 launch.                           */
int sz3g_histogram_bins(const uint16_t* codes, uint64_t n, uint32_t nbins, uint32_t window_lo,
                        int64_t* hist, sz3g_stream_t stream);

/* Reported counters (north_star parity rule: near-ties "are counted, and the count is reported";
 * SURVEY 8(c) "Reported counters"), a diagnostic pass over x after compression, ACCUMULATED (+=)
 * into device uint64 d_counts[4]:
 *   [0] (i)   elements whose pre-rounding residual / (2 eb) -- by TRUE division, t = (x - p) / 2eb --
 *             lies within 1e-9 of a half-integer;
 *   [1] (ii)  elements where rint(t by division) != rint((x - p) * fl(1 / 2eb)) (the definition's t,
 *             DESIGN G5); [0] and [1] count elements with a finite quotient and |t| < R only;
 *   [2] (iii) coefficients whose beta / w lies within max(1e-9, 1e-12 max(|beta|, mean |f|) / w)
 *             of a half-integer (w = eb/2 intercept, eb/12 slopes), the parity tie window;
 *   [3]       blocks holding at least one such coefficient.
 * p is the O7 prediction from coef_codes (the stored coefficients), eb_abs from params / d_minmax as
 * in compression.  beta (4 x nblocks double, the analyze pass's or coef_raw) is nullable: then [2]
 * and [3] are not touched.  Sums and counts follow the definition's loop order, so for the same
 * codes and beta they equal the oracle's counters exactly.  Not on the timed path.  1 launch. */
int sz3g_tie_counts(const sz3g_grid* grid, const sz3g_params* params, const double* d_minmax, const void* x,
                    const int32_t* coef_codes, const double* beta, unsigned long long* d_counts,
                    sz3g_stream_t stream);

/* number of regression blocks of a grid: prod ceil(n_d / block_size) (0 on bad input) */
uint64_t sz3g_num_blocks(const sz3g_grid* grid, uint32_t block_size);

/* 1 if the TMA/mbarrier pipelined kernels apply to this grid (alignment permitting), else 0 */
int sz3g_uses_tma(const sz3g_grid* grid, int decompress);

/* total device kernels this process has launched through the library (for launch counting) */
uint64_t sz3g_launch_count(void);

/* ---- Encoder stage (NEXT-1): Huffman coding of the quantisation codes.  P:156 "The data size will be
 * significantly reduced after conducting Huffman encoding on the quantization codes"; P:418 the
 * Huffman encoder "constructs a Huffman tree based on the frequency of input data using a greedy
 * algorithm, generates codebook according to the tree, and then compress the data using the
 * codebook"; encode / decode / save / load, App. A P:948-957.  Definition:
 * oracle/DEFINITION.md H1-H5 (readings G19-G23 in DESIGN.md).
 *
 * sz3g_huffman_codebook -- from the (merged) histogram of sz3g_regression_compress / _quantize:
 *   hist       in   nsym int64 counts (nsym = 2R, <= 65536; counts in [0, 2^47)).
 *   max_len    in   maximum code length, 1..16 (the stream format uses 16).
 *   lengths    out  nsym uint8: optimal code lengths under max_len (package-merge, tie rule H2);
 *                   0 for symbols with count 0; one active symbol gets length 1.
 *   codewords  out  nsym uint32: (length << 24) | canonical codeword (H3, right-aligned in the low
 *                   16 bits); 0 for absent symbols.  This packed table is what the encoder reads.
 *   dtable     out  sz3g_huffman_dtable_bytes(nsym) bytes, 16-byte aligned: the decoder's tables.
 *   scratch    in   sz3g_huffman_scratch_bytes(nsym, max_len) bytes of device memory.
 *   d_status   in/out SZ3G_STATUS_BAD_HUFFMAN on an empty histogram, a bad count or 2^max_len < n.
 *   One launch (a single CTA).  Bit-identical to the oracle's lengths and codewords.
 *
 * sz3g_huffman_encode -- n codes in chunks of `chunk` (1..2048; the format uses 2048), with the
 *   packed codewords of sz3g_huffman_codebook (nsym entries; a code >= nsym or with length 0 sets
 *   BAD_HUFFMAN):
 *   chunk_offsets out nchunks + 1 uint64: word offset of each chunk, then the total word count.
 *   payload       out the chunks, each packed MSB-first into whole 32-bit words (H4); at most
 *                     payload_cap_words words are written (SZ3G_STATUS_PAYLOAD_OVERFLOW beyond).
 *   scratch       in  sz3g_huffman_encode_scratch_bytes(n, chunk) bytes of device memory.
 *   5 launches (chunk sizes, 3-phase scan, pack).  Codes without a codeword set BAD_HUFFMAN.
 *
 * sz3g_huffman_decode -- the inverse: n codes from payload / chunk_offsets with the dtable of the
 *   same codebook (codes and payload 16-byte aligned); a corrupt stream sets BAD_HUFFMAN.
 *   1 launch.                                                                                  */
/* sz3g_huffman_codebook_from_lengths -- the same codewords and dtable from stored lengths alone (a
 *   canonical code is defined by its lengths, H3): lengths must be <= max_len with Kraft sum <= 1 and
 *   at least one symbol, else BAD_HUFFMAN.  lengths is read, not written.  1 launch.            */
uint64_t sz3g_huffman_scratch_bytes(uint32_t nsym, uint32_t max_len);
int sz3g_huffman_codebook_from_lengths(const uint8_t* lengths, uint32_t nsym, uint32_t max_len,
                                       uint32_t* codewords, void* dtable, int32_t* d_status,
                                       sz3g_stream_t stream);
uint64_t sz3g_huffman_dtable_bytes(uint32_t nsym);
uint64_t sz3g_huffman_encode_scratch_bytes(uint64_t n, uint32_t chunk);
int sz3g_huffman_codebook(const int64_t* hist, uint32_t nsym, uint32_t max_len, uint8_t* lengths,
                          uint32_t* codewords, void* dtable, void* scratch, int32_t* d_status,
                          sz3g_stream_t stream);
int sz3g_huffman_encode(const uint16_t* codes, uint64_t n, uint32_t chunk, const uint32_t* codewords,
                        uint32_t nsym, uint64_t* chunk_offsets, uint32_t* payload,
                        uint64_t payload_cap_words, void* scratch, int32_t* d_status,
                        sz3g_stream_t stream);
int sz3g_huffman_decode(const uint32_t* payload, const uint64_t* chunk_offsets, uint64_t n,
                        uint32_t chunk, const void* dtable, uint32_t max_len, uint16_t* codes,
                        int32_t* d_status, sz3g_stream_t stream);

/* ---- SZ3-Truncation (NEXT-2): "Given the target bytes k as input parameter, it
 * keeps k most-significant bytes of each floating-point data while discarding the rest of the bytes";
 * "it bypasses the other stages".  Definition: oracle/DEFINITION.md T1-T2 (reading G24).
 *   grid   dtype and extents (n = prod(dims) elements; dim0_offset unused).
 *   x      prod(dims) T; out / in: n * k bytes, element after element, each element's k
 *          most-significant bytes of its IEEE-754 pattern, most significant first.
 *   k      1..4 (f32) or 1..8 (f64), else ERANGE.  Buffers 16-byte aligned, else EINVAL.
 * Decompression writes the stored bytes as the most significant ones and zeros below.  1 launch
 * each; k = sizeof(T) is bitwise lossless.                                                      */
int sz3g_truncation_compress(const sz3g_grid* grid, const void* x, uint32_t k, uint8_t* out,
                             sz3g_stream_t stream);
int sz3g_truncation_decompress(const sz3g_grid* grid, const uint8_t* in, uint32_t k, void* x_out,
                               sz3g_stream_t stream);

/* ---- Distortion metrics of a reconstruction (NEXT-3): "The bit rate equals bits/cr
 * ... PSNR is inversely proportional to the mean square error of decompress data and original data
 * in logarithmic scale"; SPEC S:545 PSNR = 20 log10(range) - 10 log10(MSE).
 * sz3g_error_stats: one read of x and y (same grid) ->
 *   d_out  device double[3] <- {max |x - y|, sum (x - y)^2, #elements with |x - y| > eb}, fp64;
 *          elements whose x and y are bitwise identical contribute 0 (preserved NaN / Inf), a NaN
 *          difference makes the max NaN and counts as above eb.  Deterministic (fixed reduction order).
 *   scratch sz3g_error_stats_scratch_bytes(n) bytes of device memory.  2 launches.
 * MSE = sum / n; PSNR and the bit rate (bits / ratio) are formed by the caller.                */
uint64_t sz3g_error_stats_scratch_bytes(uint64_t n);
int sz3g_error_stats(const sz3g_grid* grid, const void* x, const void* y, double eb, double* d_out,
                     void* scratch, sz3g_stream_t stream);

/* ---- Coefficient-code delta coding (NEXT-3), reading G25 of the empty "Coefficient Compression"
 * heading; definition oracle/DEFINITION.md C1-C2.
 * sz3g_coef_delta_encode: coef [nb][4] int32 (sz3g_regression_compress output) ->
 *   sym      out  4 * nb uint16, channel-major [c][block]: zigzag(coef[b][c] - coef[b-1][c]) clipped
 *                 to 65535 (escape); Huffman-code them with their own histogram (R = 32768 bins).
 *   escapes  out  the full zigzag values of the escaped positions, in position order (up to esc_cap).
 *   d_nesc   out  device uint64: the number of escapes.
 *   scratch  in   sz3g_coef_delta_scratch_bytes(nb) bytes.  3 launches.
 * sz3g_coef_delta_decode: the inverse (running sums per channel); too few escapes set
 *   SZ3G_STATUS_BAD_HUFFMAN in *d_status.  5 launches.                                          */
uint64_t sz3g_coef_delta_scratch_bytes(uint64_t nb);
int sz3g_coef_delta_encode(const int32_t* coef, uint64_t nb, uint16_t* sym, uint64_t* escapes,
                           uint64_t esc_cap, uint64_t* d_nesc, void* scratch, sz3g_stream_t stream);
int sz3g_coef_delta_decode(const uint16_t* sym, uint64_t nb, const uint64_t* escapes, uint64_t nesc,
                           int32_t* coef, void* scratch, int32_t* d_status, sz3g_stream_t stream);

/* ---- Self-describing compressed stream (NEXT-3): "magic ..., version u16, ... each inner
 * section: tag u8, length u64, payload".  HOST code and HOST buffers only.  Layout (little-endian):
 * "SZ3G" | version u16 (1) | 96-byte header | nsec u32 | nsec x {tag u8 | length u64 | FNV-1a-64 of
 * the payload u64 | payload}.  Reading checks magic, version, every length and checksum and returns
 * SZ3G_ECORRUPT (with the failing section's tag in *bad_tag) on any mismatch; the returned sections
 * point into the input buffer.  Section tags used by the Python layer: SZ3G_SEC_*.             */
typedef struct {
  sz3g_dtype   dtype;
  uint32_t     ndim;
  uint64_t     dims[3];
  sz3g_eb_mode eb_mode;
  double       eb;          /* as given (absolute, or relative to the value range)            */
  double       eb_abs;      /* the absolute bound used                                         */
  uint32_t     radius, block_size, chunk, max_len, flags;
  uint64_t     n_outliers, nblocks;
  uint64_t     dim0_offset; /* global plane offset of the slab (outlier indices are global); 0 unsharded */
} sz3g_stream_header;
typedef struct {
  uint32_t    tag;
  const void* data;         /* host */
  uint64_t    bytes;
} sz3g_section;
enum {
  SZ3G_SEC_CODE_BOOK = 1,   /* canonical codebook of the element codes: u32 n, n x (u16 sym, u8 len) */
  SZ3G_SEC_CODE_OFFS = 2,   /* chunk word offsets, u64 x (nchunks + 1)                                */
  SZ3G_SEC_CODE_DATA = 3,   /* Huffman payload words of the element codes                             */
  SZ3G_SEC_COEF_BOOK = 4,   /* codebook of the coefficient delta symbols                              */
  SZ3G_SEC_COEF_OFFS = 5,
  SZ3G_SEC_COEF_DATA = 6,
  SZ3G_SEC_COEF_ESC = 7,    /* coefficient escapes, u64 zigzag values in position order               */
  SZ3G_SEC_OUT_IDX = 8,     /* outlier global indices, u64                                            */
  SZ3G_SEC_OUT_VAL = 9,     /* outlier values, T                                                      */
  SZ3G_SEC_LR_FLAGS = 10    /* SZ3-LR predictor flags, one bit per block (LSB first; 1 = Lorenzo);
                               present iff header.flags has SZ3G_STREAM_LR                            */
};
#define SZ3G_STREAM_LR 0x1u   /* sz3g_stream_header.flags: an SZ3-LR stream (decompress with sz3g_lr_decompress) */
#define SZ3G_STREAM_INTERP 0x2u   /* an SZ3-Interp stream: nblocks 0, no COEF_* sections (sz3g_interp_decompress) */
uint64_t sz3g_stream_size(const sz3g_section* sections, uint32_t nsec);
int sz3g_stream_write(const sz3g_stream_header* hdr, const sz3g_section* sections, uint32_t nsec,
                      void* out, uint64_t cap, uint64_t* written);
int sz3g_stream_read(const void* in, uint64_t len, sz3g_stream_header* hdr, sz3g_section* sections,
                     uint32_t sec_cap, uint32_t* nsec, uint32_t* bad_tag);
/* Consistency of a parsed compressed-field stream (sections as returned by sz3g_stream_read) BEFORE
 * anything is launched on it: the checksums only catch accidental damage, this catches a stream that is
 * internally inconsistent (and would make a decoder read past a buffer).  Checks: dtype, 1 <= ndim <= 3
 * with leading extents 1, block_size 6, radius in [1, 32768], 1 <= max_len <= 16, chunk >= 1, eb_abs
 * finite and > 0, nblocks == sz3g_num_blocks(dims); every required section present once (LR_FLAGS iff
 * the LR flag; no coefficient sections and nblocks 0 with the INTERP flag); OUT_IDX = 8 n_outliers and OUT_VAL = sizeof(T) n_outliers bytes, every outlier index in
 * the slab [dim0_offset n1 n2, (dim0_offset + n0) n1 n2); CODE_OFFS / COEF_OFFS hold exactly
 * ceil(n / chunk) + 1 u64 offsets (n = N codes, 4 nblocks coefficient symbols), starting at 0,
 * non-decreasing, each chunk at most ceil(chunk max_len / 32) words, ending at the payload's word count
 * (CODE_DATA / COEF_DATA a whole number of u32 words); codebooks u32 m then m (u16 symbol < 2R (65536
 * for the coefficients), u8 length in 1..max_len) records, symbols strictly increasing; COEF_ESC a
 * whole number of u64; LR_FLAGS ceil(nblocks / 8) bytes.  Returns SZ3G_OK, SZ3G_EINVAL (null
 * arguments) or SZ3G_ECORRUPT with the offending section's tag (0 = the header) in *bad_tag. */
int sz3g_stream_validate(const sz3g_stream_header* hdr, const sz3g_section* sections, uint32_t nsec,
                         uint32_t* bad_tag);

/* Performance tuning only (no call changes a result): set knob `key` ("CHUNK_C", "CHUNK_D", "CCFG",
 * "PF"; defaults are the measured best, environment SZ3G_<KEY> overrides them) for
 * launches issued after the call.  Process-global, not thread-safe against concurrent launches.
 * Returns SZ3G_EINVAL for an unknown key. */
int sz3g_set_tuning(const char* key, int64_t value);

const char* sz3g_strerror(int code);
const char* sz3g_last_cuda_error(void);
const char* sz3g_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SZ3G_H */
