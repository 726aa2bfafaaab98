/*
 * enks_b200.h — C-ABI of the B200-native matrix-variate EnKS hot path.
 *
 * The reference (arXiv 2410.09663, package `enksmpc`) is pure Python/NumPy;
 * its hot path is enks.smooth_horizon (pkg/src/enksmpc/enks.py:256-284).  This
 * library replaces the NumPy/BLAS/LAPACK call sites of that path with sm_100a
 * kernels.  The Python host package `paper_2410_09663_b200` (a drop-in mirror
 * of the reference API) binds these entry points with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes only; no allocation inside the library.  All
 *     device pointers are caller-owned; `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).  Every call is stream-ordered and
 *     asynchronous unless stated otherwise.
 *   - Ensemble layout ("member-column"): a block of R rows for N members with
 *     m columns each is a row-major R x (N*m) fp32 matrix; member i's (r, j)
 *     entry is at [r * ld + i * m + j].  This is exactly the matrix the
 *     reference builds by copy in _pair_covariance (enks.py:151-152).
 *   - Return value: 0 on success, otherwise an ENKS_E_* code; the message is
 *     available from enks_last_error() (thread-local).
 */
#ifndef ENKS_B200_H
#define ENKS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENKS_OK 0
#define ENKS_E_ARG 1       /* bad argument (shape, null pointer, unsupported size) */
#define ENKS_E_CUDA 2      /* CUDA launch / runtime error */
#define ENKS_E_UNSUPPORTED 3

/* Library identity / diagnostics. */
int enks_version(void);
const char* enks_last_error(void);
/* 1 if the current device is sm_100 (B200) and the library's cubin loads. */
int enks_device_check(void);

/*
 * Noise substreams (K1+K2).  Replaces the per-member loop of
 *   enks.py:131-145 _member_noise  ->  matvar.py:149-151 NoiseStreams.substream(i, t, ch)
 *   .standard_normal((rows, cols))  ->  matvar.py:183-188 transform_standard_normal.
 * Bit-identical to numpy SeedSequence -> Philox4x64-10 -> ziggurat.
 *   head/n_head : SeedSequence entropy words common to all streams — the seed's
 *                 uint32 words zero-padded to 4, followed by NoiseStreams.prefix
 *                 words (n_head <= 32).  The stream ids (member0+i, t, channel)
 *                 are appended on device (each < 2^32, one word).
 *   diag        : optional row scaling (rows doubles) = diagonal of the row
 *                 Cholesky factor; NULL -> raw standard normals.  A dense
 *                 factor is applied afterwards with enks_gemm.
 *   out         : rows x (n_members*cols) block, leading dimension ld_out.
 *   base/out_plus (optional, both or neither): out_plus = base + value
 *                 (the "u + w" slot of enks.py:168 and the "x + v" / "u + v"
 *                 observations of enks.py:200).
 *   out may be NULL when out_plus is given.
 */
int enks_noise_fill(const uint32_t* head, int n_head, uint32_t t, uint32_t channel,
                    int64_t member0, int64_t n_members, int rows, int cols,
                    const double* diag, float* out, int64_t ld_out,
                    const float* base, int64_t ld_base, float* out_plus, int64_t ld_plus,
                    void* stream);

/*
 * Several noise channels of one step in a single launch (one warp per
 * (member, job) substream), e.g. W, V_X, V_U of step t: job q draws channel
 * channel[q] at time t[q] into rows[q] rows with the same out/base/out_plus
 * semantics as enks_noise_fill (arrays of n_jobs <= 4 entries; host memory).
 */
int enks_noise_fill_multi(const uint32_t* head, int n_head, int64_t member0, int64_t n_members,
                          int cols, int n_jobs, const uint32_t* t, const uint32_t* channel,
                          const int* rows, const double* const* diag, float* const* out,
                          const int64_t* ld_out, const float* const* base, const int64_t* ld_base,
                          float* const* out_plus, const int64_t* ld_plus, void* ws,
                          int64_t ws_bytes, void* stream);
/* Workspace for the segmented launch (few substreams: each substream cut into chunks drawn by
 * separate warps, chained in order); 0 = one warp per substream.  ws may be NULL (then never
 * segmented). */
int64_t enks_noise_ws_bytes(int64_t n_members, int n_jobs, int max_rows, int cols);
/* Same, with the head words in DEVICE memory (n_head of them), so a captured CUDA graph can
 * be replayed for another (seed, prefix) by rewriting the words (closed-loop MPC steps use
 * NoiseStreams.child(k), matvar.py:153-154). */
int enks_noise_fill_multi_dev(const uint32_t* head_dev, int n_head, int64_t member0,
                              int64_t n_members, int cols, int n_jobs, const uint32_t* t,
                              const uint32_t* channel, const int* rows, const double* const* diag,
                              float* const* out, const int64_t* ld_out, const float* const* base,
                              const int64_t* ld_base, float* const* out_plus,
                              const int64_t* ld_plus, void* ws, int64_t ws_bytes, void* stream);

/* Both member sums of a predict in one pass (enks.py:171 slice mean, enks.py:194-200 + 231
 * observation mean): acc/amax = sums of src's rows relative to the first member (z0 = NULL
 * semantics of enks_member_sum), acc2/amax2 = the same for src + src2 over the first rows2 rows
 * (rows2 <= rows); src's first rows2 rows are read once.  cols % 4 == 0, 16-byte aligned rows.
 * ws: enks_member_sum2_ws_bytes(rows, rows2, n_members, cols) bytes of device memory. */
int64_t enks_member_sum2_ws_bytes(int rows, int rows2, int64_t n_members, int cols);
int enks_member_sum2(const float* src, int64_t ld_src, int rows, const float* src2,
                     int64_t ld_src2, int rows2, int64_t n_members, int cols, double* acc,
                     float* amax, double* acc2, float* amax2, void* ws, void* stream);
/*
 * Member statistics (K4/K5).  Replaces members.mean(axis=0) (enks.py:171, 248),
 * obs.mean(axis=0) (enks.py:231) and the anomaly formation (enks.py:232-233).
 * Anomalies are formed relative to a per-(row, col) shift z0 (global member
 * 0), so identical members give exactly zero anomalies at any N.
 *   enks_member_sum    : acc[r*cols+j] (double) = sum over local members of (src - z0);
 *                        amax (optional) = max over local members of |src - z0|.
 *                        z0 == NULL -> z0 is local member 0 (single-rank case).
 *   enks_member_center : mean = z0 + acc/n_total; anom = (src - z0) - acc/n_total.
 *                        anom may be NULL (mean only) and may alias src.
 * `ws` for enks_member_sum: enks_member_sum_ws_bytes() bytes of device scratch.
 */
int64_t enks_member_sum_ws_bytes(int rows, int64_t n_members, int cols);
int enks_member_sum(const float* src, int64_t ld_src, const float* src2, int64_t ld_src2, int rows,
                    int64_t n_members, int cols, const float* z0, double* acc, float* amax, void* ws,
                    void* stream);
/* Multi-rank member sums without a broadcast of global member 0: each rank sums relative to its
 * OWN first member s (z0 = NULL), converts to absolute sums with coef = +n_local
 * (acc += coef * s), the ranks allreduce, and each converts back with coef = -n_total, so the
 * centring kernels again see sums relative to their local s.  Identical members still give
 * exactly zero anomalies (n * s is exact in fp64).  src2 as in enks_member_sum (s = src + src2
 * in fp32).  Replaces the member-0 broadcast of the enks.py:171 / 231 means under sharding. */
int enks_member_sum_rebase(const float* src, int64_t ld_src, const float* src2, int64_t ld_src2,
                           int rows, int cols, double* acc, double coef, void* stream);
int enks_member_center(const float* src, int64_t ld_src, int rows, int64_t n_members, int cols,
                       const float* z0, const double* acc, int64_t n_total, float* mean,
                       float* anom, int64_t ld_anom, void* stream);

/*
 * Centring straight into the fp16-pair basis (see enks_f16pair_split): per-row scale
 * from the bound max|src - z0| + |mean shift| (amax from enks_member_sum), then
 * h/l planes (ld ldh) + inv_scale, the member mean, and optionally an fp32 copy of
 * the first rows_f32 rows (f32, ld_f32).  scale_ws: `rows` floats of scratch.
 * Rows [skip0, skip1) are not stored in the basis (later rows move up); skip1 <= skip0: none.
 */
int enks_member_center_f16pair(const float* src, int64_t ld_src, int rows, int64_t n_members,
                               int cols, const float* z0, const double* acc, const float* amax,
                               int64_t n_total, float* mean, void* h, void* l, int64_t ldh,
                               float* inv_scale, float* scale_ws, float* f32, int64_t ld_f32,
                               int rows_f32, int skip0, int skip1, void* stream);

/*
 * Forecast + noise in one launch (enks.py:165-168 and 194-200 at step t): the fused 2-32-32-1
 * CNN forecast (as enks_cnn_forward) whose otherwise idle warps draw the noise jobs of
 * enks_noise_fill_multi (head words on the host, or head_dev in device memory for graph
 * replays).  enks_cnn_noise_fusable tells whether the model/shape takes this path (else
 * ENKS_E_UNSUPPORTED: use enks_noise_fill_multi + enks_cnn_forward).
 */
int enks_cnn_noise_fusable(int n_layers, const int* widths, int rows, int cols);
int enks_cnn_forward_noise(int n_layers, const int* widths, const float* weights,
                           const float* biases, float alpha, const float* x, int64_t ldx,
                           const float* u, int64_t ldu, float* out, int64_t ldo, int rows, int cols,
                           int64_t n_members, const uint32_t* head, const uint32_t* head_dev,
                           int n_head, int64_t member0, int n_jobs, const uint32_t* t,
                           const uint32_t* channel, const int* job_rows, const double* const* diag,
                           float* const* nout, const int64_t* ld_nout, const float* const* base,
                           const int64_t* ld_base, float* const* out_plus,
                           const int64_t* ld_plus, void* stream);

/*
 * Derived-U chain (replaces the U rows of enks.py:233-248 for slices 1..n_slices): the slice
 * rows [X; U; dU] obey U_s = U_{s-1} + dU_s member-wise (enks.py:168), so the basis holds only
 * [X; dU] (n + l rows per slice).  mean (full (n + 2l)-row slices from slice 1, ld_mean) +=
 * delta (compact increments G (y_ref - y_bar), ld_delta) with U rows getting the prefix sum of
 * the dU increments; gtt (n + l x p) = [X rows of the newest slice's compact gain;
 * sum over slices of its dU rows].  Either pair of pointers may be NULL to skip that part.
 */
/*
 * Observation centring (enks.py:194-200, 231-233) with the perturbed observation formed on the
 * fly as src + src2 ([x; u] + [v_x; v_u]; enks_member_sum takes the same src2): writes the
 * fp16-pair basis rows (h, l, inv_scale, as enks_member_center_f16pair), the member mean, and
 * the transposed pair planes th / tl (K x rows, ld ldt) with one scale per K row (t_inv) --
 * the K-major B operand of the newest-slice shift (enks.py:247).  rows <= 256.  th, tl and
 * t_inv may all be NULL: no transposed planes (the shift then reads the basis rows MN-major,
 * enks_gemm_f16pair_ex_mn).
 */
int enks_member_center_f16pair_t(const float* src, int64_t ld_src, const float* src2,
                                 int64_t ld_src2, int rows, int64_t n_members, int cols,
                                 const float* z0, const double* acc, const float* amax,
                                 int64_t n_total, float* mean, void* h, void* l, int64_t ldh,
                                 float* inv_scale, float* scale_ws, void* th, void* tl, int64_t ldt,
                                 float* t_inv, void* stream);

int enks_uchain_apply(const float* delta, int64_t ld_delta, float* mean, int64_t ld_mean,
                      const float* gcol, int64_t ld_g, float* gtt, int64_t ld_gtt, int n_slices,
                      int n, int l, int m, int p, void* stream);

/*
 * Dense fp32 GEMM used by every contraction of the path (K2 dense colouring,
 * linear forecast, K6/K7 covariances, correction and gain products, K9
 * member shift, mean update):
 *   C[M x N] = alpha * op(A) op(B) + beta * C0 + bias[i, n % bias_cols]
 *   op(A) = A (M x K, lda) or A^T when trans_a (A stored K x M)
 *   op(B) = B (K x N, ldb) or B^T when trans_b (B stored N x K)
 * C0/bias optional (NULL); C0 may alias C.  tri_rows/tri_k > 0 skip the
 * structurally-zero leading K range of block upper-triangular A: rows in
 * block r0/tri_rows start at k = (r0/tri_rows)*tri_k.
 * split_k > 1 requires ws of enks_gemm_ws_bytes(M, N, split_k) bytes and is
 * reduced deterministically (fixed order).  Replaces numpy `@` / OpenBLAS
 * dgemm at enks.py:153, 247 and matvar.py:188.
 * `engine`: 0/1 = SIMT fp32 FFMA; 2 = tcgen05 3xTF32 (trans_a=0, trans_b=1, N <= 256,
 * no bias/tri; `ws` must then hold enks_tc_gemm_ws_bytes(M, N, K, split_k) bytes).
 */
int64_t enks_gemm_ws_bytes(int64_t M, int64_t N, int split_k);
int enks_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, float alpha,
              const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
              const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias, int bias_cols,
              float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k, int split_k, void* ws,
              int engine, void* stream);

/*
 * tcgen05 3xTF32 contraction with a pre-split B operand (the cross moments
 * P = [A; Yc] Yc^T of the append-only basis; enks.py:234-236):
 *   C[M x N] = alpha * A B^T,  B = Bh + Bl with Bh = rna_tf32(B) (enks_tf32_split).
 * Splitting B once per step lets both basis segments reuse it.  `ws` holds
 * split_k * M * N floats of deterministic split-K partials (split_k <= 0: auto).
 */
int64_t enks_tc_gemm_ws_bytes(int64_t M, int64_t N, int64_t K, int split_k);
int enks_tf32_split(const float* src, int64_t ld, int64_t rows, int64_t cols, float* hi, float* lo,
                    int transpose, void* stream);
int enks_gemm_nt_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                    const float* Bh, const float* Bl, int64_t ldb, float* C, int64_t ldc,
                    int split_k, void* ws, void* stream);

/*
 * General tcgen05 3xTF32 GEMM with a pre-split B (B = Bh + Bl):
 *   C = alpha * A op(B) + beta * C0 + bias[r, c % bias_cols]
 * b_mn_major = 0: Bh/Bl are N x K (K-major; op(B) = B^T, any N, N-tiles of 256);
 * b_mn_major = 1: K x N MN-major operands (experimental, not used by the engine).
 * enks_tf32_split(..., transpose=1) produces the K-major planes of a K x N matrix.
 * tri_rows/tri_k as in enks_gemm.  Used for the newest-slice member shift
 * (enks.py:247 restated), the gain correction and the gain itself.
 * `ws`: split_k * M * N floats when split_k != 1 (split_k <= 0: auto).
 */
int enks_gemm_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                 const float* Bh, const float* Bl, int64_t ldb, int b_mn_major, float beta,
                 const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias, int bias_cols,
                 float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k, int split_k, void* ws,
                 void* stream);

/*
 * fp16-pair storage and contraction of the append-only basis (the dominant
 * cross moments P = [A; Yc] Yc^T, enks.py:148-153, 234-236):
 *   enks_f16pair_split : per row r, s_r = 2^e with max|x_r| s_r in [2^13, 2^14);
 *                        h = fp16(x s), l = fp16(x s - h) (fp16 planes, ld ldo),
 *                        inv_scale[r] = 1 / s_r.  x = (h + l) / s to ~2^-22.
 *   enks_f16pair_recon : fp32 reconstruction (members read-back).
 *   enks_gemm_f16pair  : C[M x N] = alpha * diag(inv_sa) (Ah+Al)(Bh+Bl)^T diag(inv_sb)
 *                        on tcgen05 kind::f16 (three MMAs per K=16 step, dropped l*l
 *                        term ~2^-22), N <= 256; `ws` of enks_gemm_f16pair_ws_bytes bytes.
 */
int enks_f16pair_split(const float* src, int64_t ld, int64_t rows, int64_t K, void* h, void* l,
                       int64_t ldo, float* inv_scale, void* stream);
/* enks_f16pair_split of src[r][k] * col_scale[k] (a per-column power of two folded in first:
 * the per-row scale of the other operand of a reduction over k, e.g. Yc_tau's for G_tt). */
int enks_f16pair_split_cs(const float* src, int64_t ld, int64_t rows, int64_t K,
                          const float* col_scale, void* h, void* l, int64_t ldo, float* inv_scale,
                          void* stream);
int enks_f16pair_recon(const void* h, const void* l, int64_t ldi, const float* inv_scale,
                       int64_t rows, int64_t K, float* out, int64_t ldo, void* stream);
int64_t enks_gemm_f16pair_ws_bytes(int64_t M, int64_t N, int64_t K);

/* Leave `sms` SMs (0..16) free in the grids of the following enks_gemm_f16pair launches (split-K
 * and persistent-pair sizing), so a concurrent one-CTA kernel -- the side-stream gain solve of
 * enks.py:234-246, which overlaps the cross moments of enks.py:148-153 -- gets an SM at once
 * instead of after the first cross-moment CTA drains.  Host-side state, read at launch (and so
 * baked into captured graphs); 0 restores full grids.  Returns ENKS_OK. */
int enks_set_sm_reserve(int sms);
int enks_gemm_f16pair(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah, const void* Al,
                      int64_t lda, const float* inv_sa, const void* Bh, const void* Bl, int64_t ldb,
                      const float* inv_sb, float* C, int64_t ldc, void* ws, void* stream);

/*
 * Gain solve (K8).  Replaces enks.py:234-235 (symmetrize) and 238-246
 * (cho_factor with the jitter fallback, cho_solve):
 *   Sy = scale * 0.5 * (S + S^T); try Cholesky; on failure (pivot <= 0 or NaN)
 *   retry once with Sy + (1e-9 * tr(Sy)/p + 1e-30) I and increment *jitter_events;
 *   if that fails too set *status = 1 (the reference raises LinAlgError).
 *   Writes Sy^{-1} (p x p, ld p) to `inv` (consumed by enks_gemm).
 * Runs on one CTA in shared memory; p <= enks_spd_max_p().  `ws`: p*p floats.
 * status / jitter_events are device ints (no host sync).
 */
/*
 * Fused-epilogue variant (no split-K), any N (256-column tiles):
 * C = alpha diag(inv_sa) (Ah + Al)(Bh + Bl)^T diag(inv_sb) + beta C0 + bias[:, c % bias_cols].
 * Used for the newest-slice shift last = mean + A_tau - G_tt Yc_tau (enks.py:247 restricted to
 * the newest slice) with B = Yc_tau^T planes from enks_f16pair_transpose (rows <= 256 source
 * rows re-split into K-major transposed planes with per-output-row scales).
 */
int enks_gemm_f16pair_ex(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah,
                         const void* Al, int64_t lda, const float* inv_sa, const void* Bh,
                         const void* Bl, int64_t ldb, const float* inv_sb, float beta,
                         const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias,
                         int bias_cols, float* C, int64_t ldc, void* stream);
/* As enks_gemm_f16pair_ex, but B is given MN-major: Bh / Bl are K x N row-major (ldb), i.e. the
 * fp16-pair rows of the centred observations Yc_tau themselves (enks.py:247, newest-slice shift
 * last = C0 + bias - G_tt Yc_tau), so no transposed copy is needed.  B carries no per-reduction-row
 * scale here: fold it into A first (enks_f16pair_split_cs); inv_sn scales output columns (N > 128,
 * K % 32 == 0, N % 8 == 0; CTA-pair kernel). */
int enks_gemm_f16pair_ex_mn(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah,
                            const void* Al, int64_t lda, const float* inv_sa, const void* Bh,
                            const void* Bl, int64_t ldb, const float* inv_sn, float beta,
                            const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias,
                            int bias_cols, float* C, int64_t ldc, void* stream);
int enks_f16pair_transpose(const void* h, const void* l, int64_t ldi, const float* inv_src,
                           int rows, int64_t cols, void* oh, void* ol, int64_t ldo, float* inv_out,
                           void* stream);

int enks_spd_max_p(void);
/* workspace bytes for enks_spd_inverse at this p (p x p floats up to 288; for 288 < p <= 576 the
 * solve runs as a 2 x 2 Schur complement of two one-CTA factorisations, both with and without
 * the reference jitter, and selects on device -- no host synchronisation). */
int64_t enks_spd_ws_bytes(int p);
int enks_spd_inverse(const float* S, int64_t lds, int p, float scale, float* inv, float* ws,
                     int* status, int* jitter_events, void* stream);

/*
 * CNN forecast (K3): X' = X + alpha * conv_L(...tanh(conv_1([X, U]))...), 3x3
 * kernels, zero 'same' padding, tanh between layers, torch conv2d weight
 * layout.  The reference's model seam is MatrixDynamics.step
 * (dynamics.py:40-50) called at enks.py:168; the CNN itself is not in the
 * reference.  x/u/out use the member-column layout (image rows =
 * block rows, image cols = m).  widths[0..n_layers] with widths[0] == 2 and
 * widths[n_layers] == 1; weights/biases concatenated per layer (device).
 */
int enks_cnn_max_width(void);
/* Deep surrogates (widths 2-32-...-32-1, fields a multiple of 128 pixels wide, e.g. BASELINE C4):
 * one tcgen05 kernel per 32 -> 32 layer with fp16-pair activations through HBM (csrc/cnn_deep.cu);
 * needs the workspace enks_cnn_ws_bytes reports (0 = none needed), processed in member chunks. */
int64_t enks_cnn_ws_bytes(int n_layers, const int* widths, int rows, int cols, int64_t n_members);
int enks_cnn_forward_ws(int n_layers, const int* widths, const float* weights,
                        const float* biases, float alpha, const float* x, int64_t ldx,
                        const float* u, int64_t ldu, float* out, int64_t ldo, int rows, int cols,
                        int64_t n_members, void* ws, int64_t ws_bytes, void* stream);
int enks_cnn_forward(int n_layers, const int* widths, const float* weights, const float* biases,
                     float alpha, const float* x, int64_t ldx, const float* u, int64_t ldu,
                     float* out, int64_t ldo, int rows, int cols, int64_t n_members,
                     void* stream);

/*
 * Burgers forecast: cfg.substeps forward-Euler steps of the
 * 2-D viscous Burgers solver for every member, force held constant
 * (replaces BurgersDynamics.step, dynamics.py:264-270 -> _step_packed 183-216,
 * called at enks.py:168).  x/out: (2*grid_n x n_members*grid_n) member-column
 * layout, phi_x rows above phi_y rows; u: u_rows x K with u_rows = 2 (boundary
 * force on rows grid_n-1 / 2*grid_n-1) or 2*grid_n (pointwise source), 0 = none.
 * CFL (dynamics.py:168-180): max|phi| over every substep input is folded into
 * *vmax (device float, caller zeroes it) and a non-finite entry sets bit 0 of
 * *flags; the caller raises CflError from them.  ws: enks_burgers_ws_bytes bytes
 * (0 when the member field fits in shared memory).
 */
int64_t enks_burgers_ws_bytes(int grid_n, int n_members, int substeps);
int enks_burgers_forward(const float* x, int64_t ldx, const float* u, int64_t ldu, int u_rows,
                         float* out, int64_t ldo, int grid_n, int n_members, int substeps,
                         double nu, double dt, double dx, float* vmax, int* flags, void* ws,
                         void* stream);

/*
 * Constraint barrier observation row (enks.py:201-208,
 * virtualsys.py:289-302).  S: predicted slices (d x n_members*m, member-column layout).
 * g_i = <coef, S_i> + c0 (kind 0, coef d x m) or max_{r0<=r<r1}|S_i[r,:]| + c0 (kind 1);
 * out[i*m + j] = softplus_{alpha,beta}(g_i) + sqrt_var * eps[i] for all j (fp64 math).
 * eps: the first draw of substream (i, t, CH_EPS) per member (enks_noise_fill, 1 x 1).
 */
int enks_barrier_row(const float* S, int64_t lds, int d, int m, int64_t n_members, int kind,
                     const float* coef, int64_t ldc, double c0, int r0, int r1, double alpha,
                     double beta, double sqrt_var, const float* eps, float* out, void* stream);

/*
 * Quadratic trace for the closed-loop metrics:
 * out[0] = (accumulate ? out[0] : 0) + scale * sum_ij E[i,j] X[i,j] in fp64, one CTA,
 * fixed reduction order.  stage_cost (virtualsys.py:279-286) is tr[e^T W^-1 e] summed over
 * the x / u / dU blocks = sum(e * (W^-1 e)); the SPEC controller's rmse is
 * ||phi - phi_ref||_F^2 / points (SPEC.md controller.rmse).
 */
int enks_quad_form(const float* E, int64_t lde, const float* X, int64_t ldx, int64_t rows,
                   int64_t cols, double scale, double* out, int accumulate, void* stream);

/* Small elementwise helpers. */
/* out[r, j] = a[r, j] + b[r, j] (the "u + w + v" observation of enks.py:168, 200). */
int enks_add(const float* a, int64_t lda, const float* b, int64_t ldb, float* out, int64_t ldo,
             int64_t rows, int64_t cols, void* stream);
/* out[r, j] = a[r, j] - b[r, j] for an R x C block (innovation y_ref - obs_mean, enks.py:247). */
int enks_sub(const float* a, int64_t lda, const float* b, int64_t ldb, float* out, int64_t ldo,
             int64_t rows, int64_t cols, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ENKS_B200_H */
