/*
 * jigsaw_sm100.h — C ABI of libjigsaw_sm100.so, the sm_100a (B200) kernels behind
 * the WeatherMixer training step and its Jigsaw-sharded layers.
 *
 * The reference (`jigsaw` 0.1.0, /root/reference/pkg/src/jigsaw) is pure numpy and has
 * no FFI; its operator boundary is the Python functions in tensor.py / parallel.py /
 * model.py. Every entry point below replaces one of those operators (cited per entry),
 * and the Python host package `paper_2507_05753_b200` binds them with ctypes
 * (INTEGRATION.md shows the binding a maintainer would add to the reference).
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless stated otherwise; sizes are element counts.
 *   - Every call is asynchronous on the given cudaStream_t (passed as void*), allocates
 *     nothing and never synchronises the host.
 *   - Return value: 0 = OK, JG_ERR_SHAPE = shape/dtype/alignment error (Python maps it to
 *     ShapeError, the reference's tensor.py:23), JG_ERR_CUDA = launch/driver error
 *     (RuntimeError). jg_last_error() returns a thread-local message naming the problem.
 */
#ifndef JIGSAW_SM100_H
#define JIGSAW_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#pragma GCC visibility push(default)

#define JG_OK 0
#define JG_ERR_SHAPE 1
#define JG_ERR_CUDA 2

/* element types */
#define JG_F32 0
#define JG_BF16 1

/* operand storage order for jg_gemm (tensor.py:27-33 MatmulMode is expressed through these) */
#define JG_KMAJOR 0  /* operand stored [rows(M or N)][K], K contiguous              */
#define JG_MNMAJOR 1 /* operand stored [K][rows(M or N)], the M (or N) axis contiguous */

/* arithmetic of jg_gemm */
#define JG_MATH_BF16 0   /* bf16 operands, fp32 accumulate in TMEM (tcgen05 kind::f16) */
#define JG_MATH_TF32X3 1 /* fp32 operands split hi/lo, 3 tcgen05 kind::tf32 passes   */

/* epilogue flags for jg_gemm */
#define JG_EPI_ACCUM 1u     /* D += result (fp32 D): weight-grad accumulation, parallel.py:490-493 */
#define JG_EPI_BIAS_COL 2u  /* result += bias[col]  (parallel.py:524-525)                          */
#define JG_EPI_BIAS_ROW 4u  /* result += bias[row]  (weight-first tok2, parallel.py:522-523)       */
#define JG_EPI_RESID 8u     /* result += resid[row,col] (residual add, model.py:274,280)           */
#define JG_EPI_GELU_FWD 16u /* D = result (pre-activation), D2 = gelu(result)  (tensor.py:75-77)   */
#define JG_EPI_GELU_BWD 32u /* result *= gelu'(pre[row,col])                   (tensor.py:80-84)   */
#define JG_EPI_COPY_D2 64u  /* D2 = result as well (e.g. bf16 operand copy of an fp32 output)     */
#define JG_EPI_STATS 128u   /* stats[row] += (sum_col result, sum_col result^2)  (model.py:234)     */
#define JG_EPI_ADAM 256u    /* result is a complete weight gradient: apply Adam to D = fp32 master
                               in place (m, v, bf16 copy alongside) instead of storing the gradient
                               (fused into the producer; no gradient round trip) */
#define JG_EPI_LNB 512u     /* the result is the upstream gradient g of a layer norm: accumulate its
                               backward row moments stats[row] += (sum_col g*gamma, sum_col
                               g*gamma*xhat), xhat = (x - mean) * rstd  (model.py:242-250) */

/* Extra destinations of an output (the same element offsets relative to each base): used to
 * push a Jigsaw all-gather operand straight from its producer into the peers' NVLink-mapped
 * gather slots, so the gather overlaps the producing kernel. NULL / n = 0: none. */
typedef struct jg_bcast {
  void* ptr[4];
  int32_t n;
} jg_bcast;

/* Learning-rate schedule of one lr class: linear warm-up from warm_start to
 * base_lr over warmup_steps (epoch 1), then cosine annealing to final_lr at step total_steps-1.
 * total_steps <= 0: constant base_lr. */
#define JG_MAX_LR_CLASSES 4
typedef struct jg_lr_schedule {
  float base_lr, warm_start, final_lr;
  int64_t warmup_steps, total_steps;
} jg_lr_schedule;

/*
 * jg_gemm — one (batched) GEMM with a fused epilogue.
 * Replaces tensor.matmul (tensor.py:59-72) as called by MpContext._mm (parallel.py:65-69),
 * plus the bias add / GELU / residual / layer-norm-moment elementwise work that follows
 * each call in ShardedLinear.forward (parallel.py:515-526) and MixerBlock (model.py:268-297).
 *
 * Logical problem, per batch index b:   R[b] = sum_k A[b](m,k) * B[b](n,k)    (m < M, n < N)
 *   A element (m,k) lives at a[b*a_bstride + m*lda + k]   when a_major == JG_KMAJOR
 *                            a[b*a_bstride + k*lda + m]   when a_major == JG_MNMAJOR
 *   (same for B with n in place of m). NT = (K,K), NN = (K,MN) for B, TN = (MN,MN).
 * reduce_batch != 0: R = sum_b R[b] (weight gradients summed over the batch, parallel.py:552-556),
 *   written to batch slot 0 of D.
 * a_bstride == 0 (or b_bstride == 0) broadcasts that operand over the batch.
 * For JG_MATH_TF32X3 the caller passes the fp32 hi/lo split of each operand (jg_split_tf32_2d),
 *   both K-major: a/b = hi parts, a_lo/b_lo = lo parts;  R = Ahi*Bhi + Ahi*Blo + Alo*Bhi.
 * The epilogue then applies, in order: alpha*R, +bias, +resid, (+D if ACCUM), GELU fwd/bwd,
 * stores D (d_type) and D2 (d2_type), and accumulates row moments.
 */
typedef struct jg_gemm_desc {
  int64_t m, n, k, batch;
  int32_t math;          /* JG_MATH_* */
  int32_t reduce_batch;  /* 0/1 */
  const void* a; const void* a_lo; int64_t lda, a_bstride; int32_t a_major;
  const void* b; const void* b_lo; int64_t ldb, b_bstride; int32_t b_major;
  uint32_t epi;          /* JG_EPI_* */
  float alpha;
  void* d;  int64_t ldd,  d_bstride;  int32_t d_type;
  void* d2; int64_t ldd2, d2_bstride; int32_t d2_type;
  const float* bias; int64_t bias_bstride;
  const float* resid; int64_t ldr, r_bstride;
  const void* pre; int64_t ldp, p_bstride; int32_t pre_type;
  float* stats; int64_t stats_bstride;   /* [rows][2] fp32, must be zeroed by the caller */
  /* JG_EPI_ADAM: moments with D's indexing (ld = ldd, batch stride = d_bstride), optional bf16
   * copy of the updated weight (same indexing), step counter t >= 1 on the device. */
  float* adam_m; float* adam_v; void* adam_pbf16; const int32_t* adam_step;
  float adam_lr, adam_beta1, adam_beta2, adam_eps;
  /* Per-output-batch destination override (Jigsaw fused reduce-scatter): when d_planes[b] is
   * non-NULL, batch b of D is written at d_planes[b] (row stride ldd) — typically a peer GPU's
   * symmetric buffer reached over NVLink — and the epilogue ends with a system-scope fence. */
  void* d_planes[8];
  /* extra destinations of D and D2 (TMA-store epilogue only; same ld / batch stride) */
  jg_bcast d_bcast, d2_bcast;
  /* Fused Jigsaw reduce-scatter over peer memory (replaces the partial-sum exchange of
   * pnt/pnn/ptn, parallel.py:118-132, 200-215, 287-300, and the sum + ShardedLinear tail that
   * follows it, parallel.py:521-525). Batch b of the GEMM is the partial product owned by group
   * member b; the d_planes[b] != NULL batches are stored raw (dtype rs_part_type, row stride ldd)
   * into their owners' buffers, and after a tile's stores have landed the epilogue adds 1
   * (system-scope release) to rs_flag_peers[b][flag(tile)]. With rs_flags != NULL, rs_own names
   * this rank's own batch (rs_flags == NULL: no own batch, rs_own ignored; a zeroed descriptor
   * disables the whole mode): its tiles run after every remote tile, each waits until rs_flags[flag(tile)] reaches
   * rs_need (one arrival per peer), then the epilogue forms sum_{j < rs_nsrc} plane_j in order —
   * plane rs_src_idx being this rank's accumulator rounded to rs_part_type, the others read from
   * rs_src + j * rs_src_stride (row stride ldd) — and applies the regular epilogue to it exactly
   * as jg_epilogue would (alpha, bias, residual, GELU, moments, D / D2 / broadcast stores; the
   * batch strides are ignored: batch 0 addressing). Flag counters are returned to zero by the
   * consumer. flag(tile) = (tile_in_batch * cta_group + cta_rank) * 8 + epilogue_warp, below
   * rs_flag_cap. */
  uint32_t* rs_flags;
  uint32_t* rs_flag_peers[8];
  const void* rs_src; int64_t rs_src_stride;
  int32_t rs_part_type, rs_nsrc, rs_src_idx, rs_own, rs_need, rs_flag_cap;
  /* JG_EPI_LNB operands: the layer norm's input x (fp32, row stride lnb_ldx, batch stride
   * lnb_x_bstride), gamma [n], (mean, rstd) per row with the stats layout (batch stride
   * stats_bstride); the moments go to `stats` (zeroed by the caller). */
  const float* lnb_x; int64_t lnb_ldx, lnb_x_bstride;
  const float* lnb_gamma; const float* lnb_mr;
  /* persistent grid limit: at most max_sms SMs (0 = all), leaving the rest to a concurrent
   * kernel (the optimiser overlapped with the backward, jg_adam_sms) */
  int32_t max_sms;
  /* d_planes with several samples per plane: with plane_div > 0, output batch b goes to plane
   * b / plane_div (d_planes[b / plane_div], at most 8 planes), at sample offset
   * (b % plane_div) * d_planes_bstride elements — one launch for the partial planes of every
   * sample of a Jigsaw token layer (parallel.py:118-132 per sample). TMA-store epilogue only. */
  int32_t plane_div;
  int64_t d_planes_bstride;
  /* output tile width: 0 = chosen per shape (wave-quantisation model), else 64 / 128 / 256
   * (64 only for problems of at most 128 rows: CTA pairs need 128 or 256) */
  int32_t tile_n;
} jg_gemm_desc;

int jg_gemm(const jg_gemm_desc* desc, void* stream);

/*
 * jg_epilogue — the jg_gemm epilogue (same descriptor fields: m, n, batch, epi, alpha, d, d2,
 * bias, resid, pre, stats; A/B fields ignored) applied to an accumulator that arrived by
 * another route: the sum of `nplanes` partial-product planes acc[p][m][lda] (plane stride
 * acc_bstride, fp32 or bf16) pushed by the Jigsaw peers into this rank's buffer
 * (parallel.py:118-132 sums partials; the bias/GELU/residual follow, parallel.py:521-525).
 * With nplanes == 1 and desc->batch > 1, acc_bstride is the batch stride instead.
 */
int jg_epilogue(const jg_gemm_desc* desc, const void* acc, int32_t acc_type, int64_t lda, int64_t acc_bstride,
                int32_t nplanes, void* stream);   /* honours desc->d_bcast / d2_bcast */

/* y += alpha * x (fp32): accumulate a reduce-scattered weight gradient (parallel.py:490-493). */
int jg_axpy(float* y, const float* x, float alpha, int64_t n, void* stream);

/* y = sum of nplanes planes x[p*plane_stride + i] (x_type JG_F32 or JG_BF16; fp32 sum, + y if
 * accumulate): reduce pushed Jigsaw partials that need no epilogue (weight gradients, gu). */
int jg_sum_planes(float* y, const void* x, int32_t x_type, int64_t n, int32_t nplanes, int64_t plane_stride,
                  int32_t accumulate, void* stream);

/* Asynchronous device copy (copy engine; either side may be a peer GPU's buffer over NVLink).
 * Used to push Jigsaw activation tiles into peers' symmetric gather buffers. */
/* SM-driven copy of `bytes` (multiple of 8; src / dst 8-byte aligned) from src to every dst->ptr[i] (own or NVLink peer
 * memory), ending with a system-scope fence: the small Jigsaw gathers (layer-norm row moments,
 * model.py:220-231 stats_peer) that must not wait behind host->device copies on the copy
 * engines. */
int jg_push(const void* src, int64_t bytes, const jg_bcast* dst, void* stream);
int jg_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* zero `bytes` of device memory (gradient / statistics accumulators at the start of a step;
 * model.py:447-449 zero_grads) */
int jg_memset(void* dst, int64_t bytes, void* stream);

/* Device-side barrier of a Jigsaw group over peer memory (graph-capturable; publishes the
 * producer-push gathers and reduce-scatter partials of the exchanges in parallel.py:118-353).
 * peer_slots[j] = member j's arrival counters (G uint32, NVLink-mapped), own_slots = this
 * member's; *epoch (this device) counts the barriers passed. One 32-thread block: epoch += 1,
 * system-scope release add of 1 into peer_slots[j][idx] for every j != idx, then acquire-spin
 * until own_slots[j] >= epoch for every j != idx (traps after ~4 s instead of hanging). */
int jg_group_barrier(uint32_t* const* peer_slots, uint32_t* own_slots, uint32_t* epoch, int32_t G, int32_t idx,
                     void* stream);   /* G <= 8 */

/* Split fp32 x into tf32-exact hi (low 13 mantissa bits cleared) and lo = x - hi. */
int jg_split_tf32(const float* x, float* hi, float* lo, int64_t n, void* stream);

/* 2-D split into K-major 3xTF32 operands: x[b][rows][cols] (row stride ldx, batch stride
 * x_bstride) -> hi/lo [b][transpose ? cols : rows][ldo], zero-padded up to ldo, so that
 * MN-major fp32 operands become K-major and any K becomes a 16-byte multiple. */
int jg_split_tf32_2d(const float* x, int64_t rows, int64_t cols, int64_t ldx, int64_t batch, int64_t x_bstride,
                     int32_t transpose, float* hi, float* lo, int64_t ldo, void* stream);

/* Elementwise cast fp32 -> bf16 (round to nearest even). */
int jg_cast_bf16(const float* x, void* y_bf16, int64_t n, void* stream);

/* GELU forward / backward as standalone ops (tensor.py:75-84). dtype = JG_F32 or JG_BF16 for
 * x/y/g; the math is fp32. y = gelu(x);  dx = g * (Phi(x) + x*phi(x)). */
int jg_gelu_fwd(const void* x, void* y, int32_t dtype, int64_t n, void* stream);
int jg_gelu_bwd(const void* x, const void* g, void* dx, int32_t dtype, int64_t n, void* stream);

/*
 * Layer norm over the last axis, possibly split across ranks (ShardedLayerNorm,
 * model.py:200-250; serial twin tensor.py:87-123).  Rows = R, local width = C,
 * normalised width = c_total (C * column-split ways).  Row moments are exchanged between
 * the two phases by the caller (an NCCL all-reduce over the row group) when C < c_total.
 */
/* phase 0 (forward): stats[r] += (sum x, sum x^2) over the local columns. */
int jg_ln_moments(const float* x, float* stats, int64_t rows, int64_t cols, int64_t ldx, void* stream);
/* phase 1 (forward): y = gamma * (x - mean) * inv_std + beta ; saves (mean, inv_std) per row. */
int jg_ln_apply(const float* x, const float* stats, const float* gamma, const float* beta,
                void* y, int32_t y_type, float* mean_rstd, int64_t rows, int64_t cols,
                int64_t c_total, float eps, const jg_bcast* y_bcast, void* stream);
/* backward phase 0: bstats[r] += (sum h, sum h*xhat) with h = g*gamma, xhat from x & mean_rstd. */
int jg_ln_bwd_moments(const float* x, const float* g, const float* gamma, const float* mean_rstd,
                      float* bstats, int64_t rows, int64_t cols, void* stream);
/* backward phase 1: dx = inv_std*(h - sum_h/c_total - xhat*sum_hx/c_total);
 * out = (resid ? resid : 0) + dx  (fp32), out_bf16 optional copy;
 * dgamma[c] += sum_r g*xhat ; dbeta[c] += sum_r g ;
 * optional, in the same pass over out (the bias gradients of the layers it feeds,
 * parallel.py:536, 548): rowsum_out[r % rowsum_period] += sum_c out  (tok2's row bias; the
 * period folds a batch of samples onto one bias), colsum_out[c] += sum_r out (a column bias). */
int jg_ln_bwd_apply(const float* x, const float* g, const float* gamma, const float* mean_rstd,
                    const float* bstats, const float* resid, float* out, void* out_bf16,
                    float* dgamma, float* dbeta, float* rowsum_out, int64_t rowsum_period, float* colsum_out,
                    int64_t rows, int64_t cols, int64_t c_total, const jg_bcast* op_bcast, void* stream);

/* Column sums (bias gradients, parallel.py:548,559-561): out[c] += sum_r x[r*ld + c];
 * Row sums (row-bias gradient of weight-first tok2, parallel.py:536): out[r] += sum_c x[r*ld+c]. */
int jg_colsum(const void* x, int32_t x_type, float* out, int64_t rows, int64_t cols, int64_t ldx, void* stream);
int jg_rowsum(const void* x, int32_t x_type, float* out, int64_t rows, int64_t cols, int64_t ldx, void* stream);

/* patchify / unpatchify (tensor.py:126-151): x [B, lat, lon, C] <-> tokens [B, T, C*p_lat*p_lon],
 * channel-major features, row-major tokens. x_type/t_type = JG_F32 or JG_BF16. */
int jg_patchify(const float* x, void* tokens, int32_t t_type, int64_t batch, int64_t lat, int64_t lon,
                int64_t chans, int64_t p_lat, int64_t p_lon, void* stream);
int jg_unpatchify(const float* tokens, float* x, int64_t batch, int64_t lat, int64_t lon,
                  int64_t chans, int64_t p_lat, int64_t p_lon, void* stream);

/*
 * Fused decoder tail + loss (model.py:420-438 blend forward/backward; SPEC.md:396-413
 * lat-weighted MSE).  dec_tok = decoder output in token layout [B, T, F] (fp32).
 *   decoded = unpatchify(dec_tok); out = w*decoded + (1-w)*x                      (model.py:424)
 *   loss_partial += sum lat_w[lat] * var_w[c] * (out - target)^2 * inv_count
 *   g_out = 2 * lat_w * var_w * (out - target) * inv_count * loss_scale
 *   g_blend[c] += sum g_out * (decoded - x)                                      (model.py:437)
 *   g_dec_tok = patchify(g_out * w)  written as fp32 and/or bf16                  (model.py:438-439)
 * out / g_dec_f32 / g_dec_bf16 may be NULL. loss_sum is one fp32 scalar (pre-zeroed).
 * g_out_ext (optional, [B,lat,lon,C] fp32): when non-NULL it REPLACES the MSE gradient
 * (the reference's model.backward(g_out) entry point, model.py:428). With neither target nor
 * g_out_ext only the forward blend (out) is computed (model.forward, model.py:420-426).
 */
int jg_blend_loss(const float* dec_tok, const float* x, const float* target, const float* blend_w,
                  const float* lat_w, const float* var_w, const float* g_out_ext,
                  float* out, float* loss_sum, float* g_blend, float* g_dec_f32, void* g_dec_bf16,
                  int64_t batch, int64_t lat, int64_t lon, int64_t chans, int64_t p_lat, int64_t p_lon,
                  float inv_count, float loss_scale, const jg_bcast* gdec_bcast, void* stream);

/*
 * Fused Adam over one flat fp32 parameter range (bias-corrected,
 * p -= lr * mhat / (sqrt(vhat) + eps)); writes the bf16 operand copy when p_bf16 != NULL.
 * The step counter t (>= 1) is read from device memory so a captured CUDA graph replays
 * correctly; *grad_scale_dev (NULL = 1.0) multiplies g first (global-norm clipping,
 * SPEC.md:473-481).
 */
int jg_adam(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n,
            float lr, float beta1, float beta2, float eps, const int32_t* step_dev,
            const float* grad_scale_dev, const float* lr_dev, void* stream);   /* lr_dev != NULL overrides lr */
/* jg_adam pinned to `sms` SMs (one 1024-thread block per SM, holding enough shared memory that
 * no GEMM CTA fits beside it): runs beside a persistent jg_gemm limited to the other SMs
 * (jg_gemm_desc.max_sms), so a block's optimiser update overlaps the rest of the backward. */
int jg_adam_sms(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n,
                float lr, float beta1, float beta2, float eps, const int32_t* step_dev,
                const float* grad_scale_dev, const float* lr_dev, int32_t sms, void* stream);
/* jg_adam + Jigsaw weight-panel push: segment k of this call's range ([start, start+len),
 * 64-element aligned, len % 4 == 0) is additionally stored as bf16 at every dst[k][0..ndst)
 * (8-byte aligned) — the column-group members' gather slots of a channel-mixing weight, so the
 * next step's weight-panel all-gather is done by the optimiser (replaces the per-panel copies
 * of jigsaw_grid.gather_panels). */
#define JG_MAX_PUSH_SEGS 16
typedef struct jg_push_seg {
  int64_t start, len;
  void* dst[4];
  int32_t ndst;
} jg_push_seg;
typedef struct jg_push_table {
  jg_push_seg seg[JG_MAX_PUSH_SEGS];
  int32_t nseg;
} jg_push_table;
int jg_adam_push(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n,
                 float lr, float beta1, float beta2, float eps, const int32_t* step_dev,
                 const float* grad_scale_dev, const float* lr_dev, const jg_push_table* push, void* stream);
/* *counter += 1 on the device (advances the Adam step inside a graph). */
int jg_step_increment(int32_t* counter, void* stream);

/* weight * (sum of squares of x) added into out[0] (global grad norm; weight
 * 1/k counts a vector duplicated on k ranks once, parallel.py:483-485). */
int jg_sqnorm(const float* x, int64_t n, float weight, float* out, void* stream);

/* Device-side optimiser schedule for a captured step: lr_out[i] = lr_at(*step_dev - 1, sched[i])
 * and, when clip_norm > 0, *grad_scale_out = min(1, clip_norm / sqrt(*sqsum_dev))
 * (global-norm clipping). Feeds jg_adam's lr_dev / grad_scale_dev. */
int jg_opt_schedule(const int32_t* step_dev, const jg_lr_schedule* sched, int32_t nsched, const float* sqsum_dev,
                    float clip_norm, float* lr_out, float* grad_scale_out, void* stream);

/* Introspection. */
const char* jg_version(void);
const char* jg_last_error(void);
/* number of kernels launched by this library since load (evidence counter for bench.py). */
int64_t jg_launch_count(void);
/* sizeof(jg_gemm_desc): bindings check their struct mirror against it at load time. */
size_t jg_gemm_desc_size(void);

#pragma GCC visibility pop
#ifdef __cplusplus
}
#endif
#endif /* JIGSAW_SM100_H */
