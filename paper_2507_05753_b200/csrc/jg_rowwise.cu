// jg_rowwise.cu — HBM-bound kernels of the WeatherMixer step: layer-norm phases, bias-grad
// reductions, patch permutes, the fused blend + lat-weighted-MSE tail, Adam, casts.
// All are coalesced along the contiguous (last) axis, vectorised to 16-byte accesses where
// the row length allows, warp-reduced, and grid-sized in multiples of the SM count.
#include "jg_common.cuh"
#include <mutex>
#include <cstring>

namespace {

using jgd::warp_sum;

struct Bcast {
  void* p[4];
  int n;
};
Bcast to_bcast(const jg_bcast* b) {
  Bcast o{};
  if (b) {
    o.n = b->n < 4 ? b->n : 4;
    for (int i = 0; i < o.n; ++i) o.p[i] = b->ptr[i];
  }
  return o;
}
__device__ __forceinline__ void store8_bc(void* base, const Bcast& bc, int64_t off, bool bf16, const float* v) {
  jgd::store8(base, off, bf16, v);
  for (int i = 0; i < bc.n; ++i) jgd::store8(bc.p[i], off, bf16, v);
}
__device__ __forceinline__ void store1_bc(void* base, const Bcast& bc, int64_t off, bool bf16, float v) {
  jgd::store1(base, off, bf16, v);
  for (int i = 0; i < bc.n; ++i) jgd::store1(bc.p[i], off, bf16, v);
}

// Grid of at most (resident blocks per SM) x (SM count) for a grid-stride kernel: every block
// is resident from the start, so there is no second partial wave.
template <typename Kern>
int resident_grid(Kern kernel, int block, int64_t work_blocks) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  const int64_t cap = static_cast<int64_t>(per_sm) * jg::num_sms();
  return static_cast<int>(work_blocks < 1 ? 1 : (work_blocks < cap ? work_blocks : cap));
}

// Column chunk per warp unit of the row-wise kernels: whole rows when the rows alone give every
// SM 64 warps; otherwise 256 columns (one 16-byte vector per lane) so short row counts (Jigsaw
// tiles) still fill the GPU.
int64_t row_chunk(int64_t rows, int64_t cols) {
  return rows >= static_cast<int64_t>(jg::num_sms()) * 64 ? (cols > 0 ? cols : 1) : 256;
}

int grid_for(int64_t work_items, int per_block) {
  int64_t b = (work_items + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(jg::num_sms()) * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

// ---------------------------------------------------------------- casts / splits / gelu
__global__ void split_tf32_kernel(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = v - h;
  }
}

// 2-D split (optionally transposing) into K-major hi / lo operands for the 3xTF32 GEMM.
// in : x[b][r][c] (row stride ldx, batch stride xbs); out: [b][transpose ? c : r][ldo] zero-padded.
__global__ void split_tf32_2d_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                     int64_t xbs, bool transpose, float* __restrict__ hi, float* __restrict__ lo,
                                     int64_t ldo) {
  __shared__ float tile[32][33];
  const int64_t b = blockIdx.z;
  const int64_t out_rows = transpose ? cols : rows;
  const int64_t out_cols = transpose ? rows : cols;
  const int64_t obs = out_rows * ldo;
  const float* xb = x + b * xbs;
  if (!transpose) {
    const int64_t r = blockIdx.y * 32 + threadIdx.y;
    for (int64_t rr = r; rr < blockIdx.y * 32 + 32 && rr < rows; rr += 8) {
      const int64_t c = blockIdx.x * 32 + threadIdx.x;
      if (c < ldo) {
        const float v = c < cols ? xb[rr * ldx + c] : 0.f;
        const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        hi[b * obs + rr * ldo + c] = h;
        lo[b * obs + rr * ldo + c] = v - h;
      }
    }
    return;
  }
  // transpose: read a 32x32 tile of x (rows r0.., cols c0..), write it to out rows c0.., cols r0..
  const int64_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? xb[r * ldx + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t orow = c0 + i, ocol = r0 + threadIdx.x;
    if (orow < out_rows && ocol < ldo) {
      const float v = tile[threadIdx.x][i];
      const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
      hi[b * obs + orow * ldo + ocol] = h;
      lo[b * obs + orow * ldo + ocol] = v - h;
    }
  }
  (void)out_cols;
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

__global__ void gelu_fwd_kernel(const void* __restrict__ x, void* __restrict__ y, bool bf16, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    jgd::store1(y, i, bf16, jgd::gelu_f(jgd::load1(x, i, bf16)));
}

__global__ void gelu_bwd_kernel(const void* __restrict__ x, const void* __restrict__ g, void* __restrict__ dx,
                                bool bf16, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    jgd::store1(dx, i, bf16, jgd::load1(g, i, bf16) * jgd::gelu_grad_f(jgd::load1(x, i, bf16)));
}

// ---------------------------------------------------------------- layer norm
// Warp per row. The moment formula is the reference's one-pass E[x^2] - mean^2
// (tensor.py:87-94, model.py:234-237) so sharded partial moments compose exactly.
__global__ void ln_moments_kernel(const float* __restrict__ x, float* __restrict__ stats, int64_t rows,
                                  int64_t cols, int64_t ldx) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool vec = (cols % 4 == 0) && (ldx % 4 == 0);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const float* xr = x + r * ldx;
    float s = 0.f, ss = 0.f;
    if (vec) {
      for (int64_t c = lane * 4; c < cols; c += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + c);
        s += v.x + v.y + v.z + v.w;
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32) {
        const float v = xr[c];
        s += v;
        ss += v * v;
      }
    }
    s = warp_sum(s);
    ss = warp_sum(ss);
    if (lane == 0) {
      atomicAdd(stats + 2 * r, s);
      atomicAdd(stats + 2 * r + 1, ss);
    }
  }
}

__global__ void ln_apply_kernel(const float* __restrict__ x, const float* __restrict__ stats,
                                const float* __restrict__ gamma, const float* __restrict__ beta, void* __restrict__ y,
                                bool y_bf16, float* __restrict__ mean_rstd, int64_t rows, int64_t cols,
                                float inv_ctotal, float eps, const Bcast bc, int64_t cw_arg) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool vec = (cols % 8 == 0);
  // vector path: warp unit = (row, column chunk of cw = k*256 columns; nch chunks per row);
  // scalar path: warp per row
  const int64_t cw = vec ? cw_arg : cols, nch = (cols + cw - 1) / cw;
  for (int64_t u = wid; u < rows * nch; u += warps) {
    const int64_t r = u / nch, ch = u - r * nch;
    const float mean = stats[2 * r] * inv_ctotal;
    const float var = stats[2 * r + 1] * inv_ctotal - mean * mean;
    const float rstd = 1.0f / sqrtf(var + eps);
    if (ch == 0 && lane == 0 && mean_rstd) {
      mean_rstd[2 * r] = mean;
      mean_rstd[2 * r + 1] = rstd;
    }
    const float* xr = x + r * cols;
    const int64_t yo = r * cols;
    if (vec) {
      const int64_t ce = (ch + 1) * cw < cols ? (ch + 1) * cw : cols;
      for (int64_t c = ch * cw + lane * 8; c < ce; c += 256) {
        float v[8], gm[8], bt[8];
        jgd::load8(xr, c, false, v);
        jgd::load8(gamma, c, false, gm);
        jgd::load8(beta, c, false, bt);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = gm[j] * ((v[j] - mean) * rstd) + bt[j];
        store8_bc(y, bc, yo + c, y_bf16, v);
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32)
        store1_bc(y, bc, yo + c, y_bf16, gamma[c] * ((xr[c] - mean) * rstd) + beta[c]);
    }
  }
  if (bc.n) __threadfence_system();  // peer copies complete before the group barrier
}

__global__ void ln_bwd_moments_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                      const float* __restrict__ gamma, const float* __restrict__ mean_rstd,
                                      float* __restrict__ bstats, int64_t rows, int64_t cols, int64_t cw_arg) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool vec = (cols % 8 == 0);
  const int64_t cw = vec ? cw_arg : cols, nch = (cols + cw - 1) / cw;  // vector path: (row, chunk) units
  for (int64_t u = wid; u < rows * nch; u += warps) {
    const int64_t r = u / nch, ch = u - r * nch;
    const float mean = mean_rstd[2 * r], rstd = mean_rstd[2 * r + 1];
    const float* xr = x + r * cols;
    const float* gr = g + r * cols;
    float sh = 0.f, shx = 0.f;
    if (vec) {
      const int64_t ce = (ch + 1) * cw < cols ? (ch + 1) * cw : cols;
      for (int64_t c = ch * cw + lane * 8; c < ce; c += 256) {
        float xv[8], gv[8], gm[8];
        jgd::load8(xr, c, false, xv);
        jgd::load8(gr, c, false, gv);
        jgd::load8(gamma, c, false, gm);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float h = gv[j] * gm[j];
          sh += h;
          shx += h * ((xv[j] - mean) * rstd);
        }
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32) {
        const float h = gr[c] * gamma[c];
        sh += h;
        shx += h * ((xr[c] - mean) * rstd);
      }
    }
    sh = warp_sum(sh);
    shx = warp_sum(shx);
    if (lane == 0) {
      atomicAdd(bstats + 2 * r, sh);
      atomicAdd(bstats + 2 * r + 1, shx);
    }
  }
}

// 2-D tiled: block = 256 threads over 4*256 = 1024 columns, LNB_ROWS rows, processed LNB_U rows
// at a time (all their loads issued before any math or store: LNB_U x 3 16-byte loads in flight
// per thread). Column partials of dgamma / dbeta stay in registers; one atomic per column per block.
constexpr int LNB_ROWS = 64, LNB_U = 4;
__global__ void ln_bwd_apply_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                    const float* __restrict__ gamma, const float* __restrict__ mean_rstd,
                                    const float* __restrict__ bstats, const float* __restrict__ resid,
                                    float* __restrict__ out, __nv_bfloat16* __restrict__ out_bf16,
                                    float* __restrict__ dgamma, float* __restrict__ dbeta,
                                    float* __restrict__ rowsum_out, int64_t rowsum_period,
                                    float* __restrict__ colsum_out, int64_t rows, int64_t cols,
                                    float inv_ctotal, const Bcast bc) {
  const int64_t c0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
  const int64_t r0 = blockIdx.y * (int64_t)LNB_ROWS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // row-sum partials of the 8 warps meet in shared memory: one atomic per row per block
  __shared__ float srow[LNB_ROWS][8];
  // threads past the last column stay (nc = 0) so whole warps reduce the row sums
  const int nc = c0 >= cols ? 0 : (cols - c0 >= 4 ? 4 : static_cast<int>(cols - c0));
  if (nc == 0 && !rowsum_out) return;
  const int64_t r1 = r0 + LNB_ROWS < rows ? r0 + LNB_ROWS : rows;
  const bool v4 = nc == 4 && (cols % 4 == 0);
  float gm[4], dg[4] = {0, 0, 0, 0}, db[4] = {0, 0, 0, 0}, cs[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < 4; ++j) gm[j] = j < nc ? gamma[c0 + j] : 0.f;
  for (int64_t rb = r0; rb < r1; rb += LNB_U) {
    float xv[LNB_U][4], gv[LNB_U][4], rv[LNB_U][4];
#pragma unroll
    for (int u = 0; u < LNB_U; ++u) {
      const int64_t r = rb + u;
      const int64_t o = r * cols + c0;
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[u][j] = gv[u][j] = rv[u][j] = 0.f;
      if (r >= r1) continue;
      if (v4) {
        const float4 a = *reinterpret_cast<const float4*>(x + o);
        const float4 b = *reinterpret_cast<const float4*>(g + o);
        xv[u][0] = a.x; xv[u][1] = a.y; xv[u][2] = a.z; xv[u][3] = a.w;
        gv[u][0] = b.x; gv[u][1] = b.y; gv[u][2] = b.z; gv[u][3] = b.w;
        if (resid) {
          const float4 c = *reinterpret_cast<const float4*>(resid + o);
          rv[u][0] = c.x; rv[u][1] = c.y; rv[u][2] = c.z; rv[u][3] = c.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < nc) {
            xv[u][j] = x[o + j];
            gv[u][j] = g[o + j];
            rv[u][j] = resid ? resid[o + j] : 0.f;
          }
      }
    }
#pragma unroll
    for (int u = 0; u < LNB_U; ++u) {
      const int64_t r = rb + u;
      if (r >= r1) continue;
      const float mean = mean_rstd[2 * r], rstd = mean_rstd[2 * r + 1];
      const float msh = bstats[2 * r] * inv_ctotal, mshx = bstats[2 * r + 1] * inv_ctotal;
      const int64_t o = r * cols + c0;
      float ov[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float xh = (xv[u][j] - mean) * rstd;
        const float h = gv[u][j] * gm[j];
        ov[j] = rv[u][j] + rstd * (h - msh - xh * mshx);
        if (j < nc) {
          dg[j] += gv[u][j] * xh;
          db[j] += gv[u][j];
          cs[j] += ov[j];
        }
      }
      if (rowsum_out) {
        float rs = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) rs += j < nc ? ov[j] : 0.f;
        rs = warp_sum(rs);
        if (lane == 0) srow[r - r0][warp] = rs;
      }
      if (nc == 0) continue;
      if (v4) {
        *reinterpret_cast<float4*>(out + o) = make_float4(ov[0], ov[1], ov[2], ov[3]);
        if (out_bf16) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(ov[0], ov[1]), hi = __floats2bfloat162_rn(ov[2], ov[3]);
          uint2 raw;
          raw.x = *reinterpret_cast<uint32_t*>(&lo);
          raw.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(out_bf16 + o) = raw;
          for (int i = 0; i < bc.n; ++i) *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(bc.p[i]) + o) = raw;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < nc) {
            out[o + j] = ov[j];
            if (out_bf16) {
              out_bf16[o + j] = __float2bfloat16_rn(ov[j]);
              for (int i = 0; i < bc.n; ++i) reinterpret_cast<__nv_bfloat16*>(bc.p[i])[o + j] = __float2bfloat16_rn(ov[j]);
            }
          }
      }
    }
  }
  if (rowsum_out) {  // uniform over the block: no thread returned early
    __syncthreads();
    if (threadIdx.x < r1 - r0) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += srow[threadIdx.x][w];
      atomicAdd(rowsum_out + (r0 + threadIdx.x) % rowsum_period, s);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (j < nc) {
      if (dgamma) atomicAdd(dgamma + c0 + j, dg[j]);
      if (dbeta) atomicAdd(dbeta + c0 + j, db[j]);
      if (colsum_out) atomicAdd(colsum_out + c0 + j, cs[j]);
    }
  if (bc.n) __threadfence_system();
}

// ---------------------------------------------------------------- bias-grad reductions
// colsum: block = 8 warps over 256 columns (8 per lane, 16-byte loads) x CS_ROWS rows; warp w
// takes rows w, w+8, ... (CS_ROWS/8 independent loads in flight per thread); the 8 warp
// partials meet in shared memory and one atomic per column per block goes to global.
constexpr int CS_ROWS = 256;
__global__ void colsum_kernel(const void* __restrict__ x, bool bf16, float* __restrict__ out, int64_t rows,
                              int64_t cols, int64_t ldx, bool vec) {
  __shared__ float part[8][8 * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = blockIdx.x * (int64_t)256 + lane * 8;
  const int64_t r0 = blockIdx.y * (int64_t)CS_ROWS;
  const int64_t r1 = r0 + CS_ROWS < rows ? r0 + CS_ROWS : rows;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (c0 < cols) {
    if (vec) {
#pragma unroll 4
      for (int64_t r = r0 + w; r < r1; r += 8) {
        float t[8];
        jgd::load8(x, r * ldx + c0, bf16, t);
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] += t[j];
      }
    } else {
      for (int64_t r = r0 + w; r < r1; r += 8)
        for (int j = 0; j < 8; ++j)
          if (c0 + j < cols) s[j] += jgd::load1(x, r * ldx + c0 + j, bf16);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[w][j * 32 + lane] = s[j];
  __syncthreads();
  if (w == 0 && c0 < cols) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float t = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += part[k][j * 32 + lane];
      if (c0 + j < cols) atomicAdd(out + c0 + j, t);
    }
  }
}
__global__ void rowsum_kernel(const void* __restrict__ x, bool bf16, float* __restrict__ out, int64_t rows,
                              int64_t cols, int64_t ldx) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    float s = 0.f;
    for (int64_t c = lane; c < cols; c += 32) s += jgd::load1(x, r * ldx + c, bf16);
    s = warp_sum(s);
    if (lane == 0) out[r] += s;
  }
}

// ---------------------------------------------------------------- patch permutes
// token t = gi*gw + gj ; feature f = c*pl*pw + i*pw + j ; grid (gi*pl+i, gj*pw+j, c)
// Work unit = (b, gi, i, gj, c), c fastest: the pw grid values of channel c along one patch
// row (lanes = consecutive channels, so each of the pw loads is a coalesced warp-wide run) map
// to pw CONTIGUOUS token features c*pl*pw + i*pw + [0, pw) — one 8/16/32-byte vector per
// thread (whole 32-byte sectors; the neighbouring rows' halves merge in L2). Every unit is
// independent: no shared-memory transpose, no barriers, pw loads in flight per thread.
struct PatchIdx {
  int64_t b, y, gj, tk;
  int c, i;
};
__device__ __forceinline__ PatchIdx patch_unit(uint32_t u, int chans, uint32_t gw, int pl, uint32_t gh) {
  PatchIdx q;
  q.c = static_cast<int>(u % chans);
  u /= chans;
  q.gj = u % gw;
  u /= gw;
  q.i = static_cast<int>(u % pl);
  u /= pl;
  const int64_t gi = u % gh;
  q.b = u / gh;
  q.y = gi * pl + q.i;
  q.tk = (q.b * gh + gi) * gw + q.gj;
  return q;
}

template <int PW>
__device__ __forceinline__ void store_run(void* base, int64_t off, bool bf16, const float* v) {
  if constexpr (PW == 8) {
    jgd::store8(base, off, bf16, v);
  } else if constexpr (PW == 4) {
    if (bf16) {
      uint2 raw;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
      h[0] = __floats2bfloat162_rn(v[0], v[1]);
      h[1] = __floats2bfloat162_rn(v[2], v[3]);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + off) = raw;
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + off) = make_float4(v[0], v[1], v[2], v[3]);
    }
  } else if constexpr (PW == 2) {
    if (bf16)
      *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(base) + off) = __floats2bfloat162_rn(v[0], v[1]);
    else
      *reinterpret_cast<float2*>(reinterpret_cast<float*>(base) + off) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int j = 0; j < PW; ++j) jgd::store1(base, off + j, bf16, v[j]);
  }
}
template <int PW>
__device__ __forceinline__ void load_run(const float* base, int64_t off, float* v) {
  if constexpr (PW == 8) {
    jgd::load8(base, off, false, v);
  } else if constexpr (PW == 4) {
    const float4 a = *reinterpret_cast<const float4*>(base + off);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else if constexpr (PW == 2) {
    const float2 a = *reinterpret_cast<const float2*>(base + off);
    v[0] = a.x; v[1] = a.y;
  } else {
#pragma unroll
    for (int j = 0; j < PW; ++j) v[j] = base[off + j];
  }
}

// PW > 0: compile-time patch width (vector path); PW == 0: runtime width, scalar token side.
template <int PW>
__global__ void patchify_kernel(const float* __restrict__ x, void* __restrict__ tok, bool bf16, int64_t batch,
                                int64_t lat, int64_t lon, int chans, int pl, int pw_rt) {
  const int pw = PW > 0 ? PW : pw_rt;
  const uint32_t gw = static_cast<uint32_t>(lon / pw), gh = static_cast<uint32_t>(lat / pl);
  const uint32_t units = static_cast<uint32_t>(batch) * gh * pl * gw * chans;
  const int64_t PP = static_cast<int64_t>(pl) * pw, F = PP * chans;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < units; u += gridDim.x * blockDim.x) {
    const PatchIdx q = patch_unit(u, chans, gw, pl, gh);
    const float* src = x + ((q.b * lat + q.y) * lon + q.gj * pw) * chans + q.c;
    const int64_t dst = q.tk * F + q.c * PP + q.i * pw;
    if constexpr (PW > 0) {
      float v[PW];
#pragma unroll
      for (int j = 0; j < PW; ++j) v[j] = src[static_cast<int64_t>(j) * chans];
      store_run<PW>(tok, dst, bf16, v);
    } else {
      for (int j = 0; j < pw; ++j) jgd::store1(tok, dst + j, bf16, src[static_cast<int64_t>(j) * chans]);
    }
  }
}

__global__ void unpatchify_kernel(const float* __restrict__ tok, float* __restrict__ x, int64_t batch, int64_t lat,
                                  int64_t lon, int64_t chans, int64_t pl, int64_t pw) {
  const int64_t gw = lon / pw, T = (lat / pl) * gw, F = chans * pl * pw;
  const int64_t n = batch * lat * lon * chans;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx % chans;
    const int64_t xo = (idx / chans) % lon;
    const int64_t ya = (idx / (chans * lon)) % lat;
    const int64_t b = idx / (chans * lon * lat);
    const int64_t t = (ya / pl) * gw + xo / pw;
    const int64_t f = c * pl * pw + (ya % pl) * pw + (xo % pw);
    x[idx] = tok[(b * T + t) * F + f];
  }
}

// ---------------------------------------------------------------- blend + loss
// Same work units as patchify (b, gi, i, gj, c): one vector of pw decoder features per thread,
// pw coalesced x / target (/ out / g_ext) values, one vector of pw gradient features stored.
// The grid-stride step is a multiple of C (only the first C*floor(blockDim/C) threads of a
// block work), so each thread keeps ONE channel for the whole kernel and its blend-gradient
// and loss partials stay in registers; one shared atomic per thread and one global atomic per
// channel per block at the end.
constexpr int MAX_CH = 256;
template <int PW>
__global__ void blend_loss_kernel(const float* __restrict__ dec_tok, const float* __restrict__ x,
                                  const float* __restrict__ target, const float* __restrict__ blend_w,
                                  const float* __restrict__ lat_w, const float* __restrict__ var_w,
                                  const float* __restrict__ g_ext, float* __restrict__ out, float* __restrict__ loss_sum,
                                  float* __restrict__ g_blend, float* __restrict__ g_dec_f32,
                                  __nv_bfloat16* __restrict__ g_dec_bf16, int64_t batch, int64_t lat, int64_t lon,
                                  int chans, int pl, int pw_rt, float inv_count, float loss_scale, const Bcast bc) {
  __shared__ float s_part[1024];  // per-thread blend-gradient partials (blockDim <= 1024)
  __shared__ float s_loss[32];
  const int pw = PW > 0 ? PW : pw_rt;
  const int C = chans;
  const uint32_t gw = static_cast<uint32_t>(lon / pw), gh = static_cast<uint32_t>(lat / pl);
  const uint32_t units = static_cast<uint32_t>(batch) * gh * pl * gw * C;
  const int64_t PP = static_cast<int64_t>(pl) * pw, F = PP * C;
  const bool want_grad = (g_ext != nullptr) || (target != nullptr);
  const int act = (static_cast<int>(blockDim.x) / C) * C;  // > 0: host guarantees C <= blockDim
  const int t0 = static_cast<int>(threadIdx.x);
  float lsum = 0.f, gb = 0.f;
  if (t0 < act) {
    const int my_c = t0 % C;
    const float w = blend_w[my_c], vw = var_w ? var_w[my_c] : 0.f;
    constexpr int VMAX = PW > 0 ? PW : 16;
    for (uint32_t u = blockIdx.x * act + t0; u < units; u += gridDim.x * act) {
      const PatchIdx q = patch_unit(u, C, gw, pl, gh);
      const int64_t ga0 = ((q.b * lat + q.y) * lon + q.gj * pw) * C + my_c;
      const int64_t to = q.tk * F + my_c * PP + q.i * pw;
      float dec[VMAX], xv[VMAX], tv[VMAX];
      if constexpr (PW > 0) {
        load_run<PW>(dec_tok, to, dec);
      } else {
#pragma unroll
        for (int j = 0; j < VMAX; ++j)
          if (j < pw) dec[j] = dec_tok[to + j];
      }
#pragma unroll
      for (int j = 0; j < VMAX; ++j)
        if (PW > 0 || j < pw) {
          xv[j] = x[ga0 + static_cast<int64_t>(j) * C];
          tv[j] = want_grad ? (g_ext ? g_ext[ga0 + static_cast<int64_t>(j) * C] : target[ga0 + static_cast<int64_t>(j) * C])
                            : 0.f;
        }
      const float wt = (target && !g_ext) ? lat_w[q.y] * vw : 0.f;
      float gd[VMAX];
#pragma unroll
      for (int j = 0; j < VMAX; ++j)
        if (PW > 0 || j < pw) {
          const float o = w * dec[j] + (1.0f - w) * xv[j];
          if (out) out[ga0 + static_cast<int64_t>(j) * C] = o;
          float g;
          if (g_ext) {
            g = tv[j];
          } else {
            const float er = o - tv[j];
            lsum += wt * er * er;
            g = 2.0f * wt * er * inv_count * loss_scale;
          }
          gb += g * (dec[j] - xv[j]);
          gd[j] = g * w;
        }
      if (!want_grad) continue;
      if constexpr (PW > 0) {
        if (g_dec_f32) {
          store_run<PW>(g_dec_f32, to, false, gd);
          for (int k = 0; k < bc.n; ++k) store_run<PW>(bc.p[k], to, false, gd);
        }
        if (g_dec_bf16) {
          store_run<PW>(g_dec_bf16, to, true, gd);
          for (int k = 0; k < bc.n; ++k) store_run<PW>(bc.p[k], to, true, gd);
        }
      } else {
#pragma unroll
        for (int j = 0; j < VMAX; ++j)
          if (j < pw) {
            if (g_dec_f32) store1_bc(g_dec_f32, bc, to + j, false, gd[j]);
            if (g_dec_bf16) store1_bc(g_dec_bf16, bc, to + j, true, gd[j]);
          }
      }
    }
  }
  s_part[t0] = gb;
  lsum = warp_sum(lsum);
  if ((threadIdx.x & 31) == 0) s_loss[threadIdx.x >> 5] = lsum;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? s_loss[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0 && loss_sum && target && !g_ext) atomicAdd(loss_sum, v * inv_count);
  }
  if (g_blend && want_grad)  // fixed-order sum of the act / C threads that own channel c
    for (int c = t0; c < C; c += blockDim.x) {
      float t = 0.f;
      for (int k = c; k < act; k += C) t += s_part[k];
      atomicAdd(g_blend + c, t);
    }
  if (bc.n) __threadfence_system();
}

// ---------------------------------------------------------------- Adam
// Segments of the range whose bf16 copy is also pushed to peer gather slots (jg_adam_push).
__device__ __forceinline__ void push_bf16x4(const jg_push_table& t, int64_t e, uint2 raw) {
  for (int k = 0; k < t.nseg; ++k) {
    const jg_push_seg& sg = t.seg[k];
    if (e >= sg.start && e < sg.start + sg.len) {
      for (int d = 0; d < sg.ndst; ++d)
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(sg.dst[d]) + (e - sg.start)) = raw;
      return;
    }
  }
}
__device__ __forceinline__ void push_bf16x1(const jg_push_table& t, int64_t e, __nv_bfloat16 h) {
  for (int k = 0; k < t.nseg; ++k) {
    const jg_push_seg& sg = t.seg[k];
    if (e >= sg.start && e < sg.start + sg.len) {
      for (int d = 0; d < sg.ndst; ++d) reinterpret_cast<__nv_bfloat16*>(sg.dst[d])[e - sg.start] = h;
      return;
    }
  }
}

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, __nv_bfloat16* __restrict__ pb, int64_t n, float lr, float b1,
                            float b2, float eps, const int32_t* __restrict__ step, const float* __restrict__ gscale,
                            const float* __restrict__ lr_dev, const jg_push_table push) {
  const int t = *step;
  if (lr_dev) lr = *lr_dev;
  const float bc1 = 1.0f / (1.0f - powf(b1, (float)t));
  const float bc2 = 1.0f / (1.0f - powf(b2, (float)t));
  const float s = gscale ? *gscale : 1.0f;
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* pa = &pp.x; const float* ga = &gg.x; float* ma = &mm.x; float* va = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gj = ga[j] * s;
      ma[j] = b1 * ma[j] + (1.0f - b1) * gj;
      va[j] = b2 * va[j] + (1.0f - b2) * gj * gj;
      pa[j] -= lr * (ma[j] * bc1) / (sqrtf(va[j] * bc2) + eps);
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (pb) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y), hi = __floats2bfloat162_rn(pp.z, pp.w);
      uint2 raw;
      raw.x = *reinterpret_cast<uint32_t*>(&lo);
      raw.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(pb)[i] = raw;
      if (push.nseg) push_bf16x4(push, 4 * i, raw);
    }
  }
  // scalar tail
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gj = g[i] * s;
    m[i] = b1 * m[i] + (1.0f - b1) * gj;
    v[i] = b2 * v[i] + (1.0f - b2) * gj * gj;
    p[i] -= lr * (m[i] * bc1) / (sqrtf(v[i] * bc2) + eps);
    if (pb) pb[i] = __float2bfloat16_rn(p[i]);
    if (pb && push.nseg) push_bf16x1(push, i, __float2bfloat16_rn(p[i]));
  }
  if (push.nseg) __threadfence_system();  // peer copies complete before the next group barrier
}

__global__ void step_inc_kernel(int32_t* counter) { *counter += 1; }

__global__ void sqnorm_kernel(const float* __restrict__ x, int64_t n, float weight, float* __restrict__ out,
                              bool vec) {
  __shared__ float part[32];
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 4; i += stride) {
      const float4 v = reinterpret_cast<const float4*>(x)[i];
      s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const float v = x[i];
      s += v * v;
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) atomicAdd(out, v * weight);
  }
}

// lr_at for each lr class, evaluated at optimiser step *step - 1, and the
// global-norm clip factor from the summed squares.
struct SchedArgs { jg_lr_schedule s[JG_MAX_LR_CLASSES]; int n; };

__device__ float lr_at_dev(const jg_lr_schedule& c, int64_t step) {
  if (c.total_steps <= 0) return c.base_lr;  // no schedule: constant lr
  if (step < 0) step = 0;
  if (step > c.total_steps - 1) step = c.total_steps - 1;
  if (step < c.warmup_steps)
    return c.warm_start + (c.base_lr - c.warm_start) * (float)((double)step / (double)c.warmup_steps);
  const int64_t span = c.total_steps - 1 - c.warmup_steps;
  const double u = span > 0 ? (double)(step - c.warmup_steps) / (double)span : 1.0;
  return (float)(c.final_lr + 0.5 * ((double)c.base_lr - c.final_lr) * (1.0 + cos(3.14159265358979323846 * u)));
}

__global__ void opt_schedule_kernel(const int32_t* __restrict__ step, const SchedArgs a, const float* __restrict__ sq,
                                    float clip, float* __restrict__ lr_out, float* __restrict__ gscale) {
  if (threadIdx.x != 0) return;
  const int64_t t = (int64_t)(*step) - 1;
  for (int i = 0; i < a.n; ++i) lr_out[i] = lr_at_dev(a.s[i], t);
  if (gscale) {
    float f = 1.0f;
    if (clip > 0.f && sq) {
      const float norm = sqrtf(*sq);
      if (norm > clip) f = clip / norm;
    }
    *gscale = f;
  }
}

// ---------------------------------------------------------------- standalone epilogue
// The jg_gemm epilogue applied to an fp32 accumulator that arrived by another route (an NCCL
// reduce-scatter of Jigsaw partial products). Warp per row, lanes over columns.
struct EpiArgs {
  int64_t m, n;
  uint32_t epi;
  float alpha;
  const void* acc; int64_t lda, a_bs; int nplanes; bool acc_bf16;
  void* d; int64_t ldd, d_bs; bool d_bf16;
  void* d2; int64_t ldd2, d2_bs; bool d2_bf16;
  const float* bias; int64_t bias_bs;
  const float* resid; int64_t ldr, r_bs;
  const void* pre; int64_t ldp, p_bs; bool pre_bf16;
  float* stats; int64_t stats_bs;
  Bcast dbc, d2bc;
};

// F: the epilogue flags when known at compile time (EPI_DYN: read a.epi). With constant flags the
// operand loads are unconditional, so the compiler issues them together (one memory round trip
// per unit) and allocates registers only for the operands in use.
constexpr uint32_t EPI_DYN = 0xFFFFFFFFu;
template <uint32_t F = EPI_DYN>
__device__ __forceinline__ void epi_apply8(const EpiArgs& a, int64_t b, int64_t r, int64_t c, float rb, float* v,
                                           float& s1, float& s2) {
  const uint32_t epi = F == EPI_DYN ? a.epi : F;
  if (a.nplanes > 1) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.f;
    for (int pl = 0; pl < a.nplanes; ++pl) {
      float t[8];
      jgd::load8(a.acc, pl * a.a_bs + r * a.lda + c, a.acc_bf16, t);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] += t[k];
    }
  } else {
    jgd::load8(a.acc, b * a.a_bs + r * a.lda + c, a.acc_bf16, v);
  }
  float t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = v[k] * a.alpha + rb;
  if (epi & JG_EPI_BIAS_COL) {
    jgd::load8(a.bias, b * a.bias_bs + c, false, t);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += t[k];
  }
  if (epi & JG_EPI_RESID) {
    jgd::load8(a.resid, b * a.r_bs + r * a.ldr + c, false, t);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += t[k];
  }
  if (epi & JG_EPI_GELU_BWD) {
    jgd::load8(a.pre, b * a.p_bs + r * a.ldp + c, a.pre_bf16, t);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] *= jgd::gelu_grad_f(t[k]);
  }
  const int64_t od = b * a.d_bs + r * a.ldd + c;
  if (epi & JG_EPI_ACCUM) {
    jgd::load8(a.d, od, false, t);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += t[k];
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    s1 += v[k];
    s2 += v[k] * v[k];
  }
  if (a.d) store8_bc(a.d, a.dbc, od, a.d_bf16, v);
  if (epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) {
    if (epi & JG_EPI_GELU_FWD) {
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = jgd::gelu_f(v[k]);
      store8_bc(a.d2, a.d2bc, b * a.d2_bs + r * a.ldd2 + c, a.d2_bf16, t);
    } else {
      store8_bc(a.d2, a.d2bc, b * a.d2_bs + r * a.ldd2 + c, a.d2_bf16, v);
    }
  }
}

// Vector path: warp unit = (row, 256-column chunk), so even a few thousand rows give tens of
// thousands of independent units (enough loads in flight without long per-warp row loops);
// LN-moment partials are warp-reduced per unit and added with one atomic pair per unit.
// Minimum resident blocks per SM (register cap) per flag set, from A/Bs of 1 / 6 / 8 on 2x2 tiles
// (tools/membench.py; profiles/r2/r3x_epilogue_minblocks.log, r3y_epilogue_bounds_vs_none.log):
// against no launch bounds, the residual + moments forms gain 6-8 %, GELU' 9 %, GELU 5-15 %.
template <uint32_t F>
constexpr int epi_min_blocks() {
  return F == (JG_EPI_BIAS_ROW | JG_EPI_RESID | JG_EPI_STATS)   ? 8
         : F == (JG_EPI_BIAS_COL | JG_EPI_RESID | JG_EPI_STATS) ? 6
         : F == JG_EPI_GELU_BWD                                  ? 6
                                                                 : 1;
}
template <uint32_t F = EPI_DYN>
__global__ void __launch_bounds__(256, epi_min_blocks<F>()) epilogue_kernel(const EpiArgs a, bool vec) {
  const uint32_t epi = F == EPI_DYN ? a.epi : F;
  const int64_t b = blockIdx.y;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (vec) {
    const int64_t nch = (a.n + 255) / 256;
    const int64_t units = a.m * nch;
    for (int64_t u = wid; u < units; u += warps) {
      const int64_t r = u / nch, c = (u - r * nch) * 256 + lane * 8;
      const float rb = (epi & JG_EPI_BIAS_ROW) ? a.bias[b * a.bias_bs + r] : 0.f;
      float s1 = 0.f, s2 = 0.f;
      if (c < a.n) {
        float v[8];
        epi_apply8<F>(a, b, r, c, rb, v, s1, s2);
      }
      if (epi & JG_EPI_STATS) {
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if (lane == 0) {
          atomicAdd(a.stats + b * a.stats_bs + 2 * r, s1);
          atomicAdd(a.stats + b * a.stats_bs + 2 * r + 1, s2);
        }
      }
    }
    if (a.dbc.n || a.d2bc.n) __threadfence_system();
    return;
  }
  for (int64_t r = wid; r < a.m; r += warps) {
    const float rb = (epi & JG_EPI_BIAS_ROW) ? a.bias[b * a.bias_bs + r] : 0.f;
    float s1 = 0.f, s2 = 0.f;
    for (int64_t c = lane; c < a.n; c += 32) {
      float v = 0.f;
      if (a.nplanes > 1) {
        for (int pl = 0; pl < a.nplanes; ++pl) v += jgd::load1(a.acc, pl * a.a_bs + r * a.lda + c, a.acc_bf16);
      } else {
        v = jgd::load1(a.acc, b * a.a_bs + r * a.lda + c, a.acc_bf16);
      }
      v = v * a.alpha + rb;
      if (epi & JG_EPI_BIAS_COL) v += a.bias[b * a.bias_bs + c];
      if (epi & JG_EPI_RESID) v += a.resid[b * a.r_bs + r * a.ldr + c];
      if (epi & JG_EPI_GELU_BWD) v *= jgd::gelu_grad_f(jgd::load1(a.pre, b * a.p_bs + r * a.ldp + c, a.pre_bf16));
      const int64_t od = b * a.d_bs + r * a.ldd + c;
      if (epi & JG_EPI_ACCUM) v += reinterpret_cast<const float*>(a.d)[od];
      s1 += v;
      s2 += v * v;
      if (a.d) store1_bc(a.d, a.dbc, od, a.d_bf16, v);
      if (epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2))
        store1_bc(a.d2, a.d2bc, b * a.d2_bs + r * a.ldd2 + c, a.d2_bf16, (epi & JG_EPI_GELU_FWD) ? jgd::gelu_f(v) : v);
    }
    if (epi & JG_EPI_STATS) {
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        atomicAdd(a.stats + b * a.stats_bs + 2 * r, s1);
        atomicAdd(a.stats + b * a.stats_bs + 2 * r + 1, s2);
      }
    }
  }
  if (a.dbc.n || a.d2bc.n) __threadfence_system();
}

template <bool BF>
__global__ void sum_planes_kernel(float* __restrict__ y, const void* __restrict__ x, int64_t n, int nplanes,
                                  int64_t ps, bool accumulate, bool vec) {
  // vec: 8 consecutive elements per thread (16-byte loads / two 16-byte stores)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; i < n; i += stride * 8) {
      float s[8], t[8];
      if (accumulate) jgd::load8(y, i, false, s);
      else {
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] = 0.f;
      }
      for (int p = 0; p < nplanes; ++p) {
        jgd::load8(x, p * ps + i, BF, t);
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] += t[e];
      }
      jgd::store8(y, i, false, s);
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float s = accumulate ? y[i] : 0.f;
    for (int p = 0; p < nplanes; ++p) s += jgd::load1(x, p * ps + i, BF);
    y[i] = s;
  }
}

__global__ void axpy_kernel(float* __restrict__ y, const float* __restrict__ x, float alpha, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += alpha * x[i];
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// SM-driven copy of one buffer to up to 4 destinations (own or NVLink-mapped peer memory):
// 16-byte vector loads / stores when everything is 16-byte aligned, else 8-byte. For the small
// Jigsaw gathers (layer-norm row moments) that must not queue behind bulk host->device copies on
// the copy engines.
template <typename V>
__global__ void push_kernel(const uint8_t* __restrict__ src, int64_t bytes, Bcast dst) {
  const int64_t n = bytes / (int64_t)sizeof(V);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const V v = reinterpret_cast<const V*>(src)[i];
    for (int d = 0; d < dst.n; ++d) reinterpret_cast<V*>(dst.p[d])[i] = v;
  }
  const int64_t t0 = n * (int64_t)sizeof(V);
  if (blockIdx.x == 0 && (int64_t)threadIdx.x < (bytes - t0) / 8) {
    const int64_t o = t0 + threadIdx.x * 8;
    const uint2 v = *reinterpret_cast<const uint2*>(src + o);
    for (int d = 0; d < dst.n; ++d) *reinterpret_cast<uint2*>(static_cast<uint8_t*>(dst.p[d]) + o) = v;
  }
  __threadfence_system();  // peers read after the group barrier that follows
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int jg_split_tf32(const float* x, float* hi, float* lo, int64_t n, void* stream) {
  JG_SHAPE_CHECK(n >= 0, "jg_split_tf32: negative size");
  if (n == 0) return JG_OK;
  split_tf32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, hi, lo, n);
  JG_LAUNCH_CHECK("split_tf32");
  return JG_OK;
}

int jg_split_tf32_2d(const float* x, int64_t rows, int64_t cols, int64_t ldx, int64_t batch, int64_t x_bstride,
                     int32_t transpose, float* hi, float* lo, int64_t ldo, void* stream) {
  JG_SHAPE_CHECK(rows > 0 && cols > 0 && batch > 0 && ldx >= cols, "jg_split_tf32_2d: bad shape");
  JG_SHAPE_CHECK(ldo >= (transpose ? rows : cols), "jg_split_tf32_2d: ldo too small");
  dim3 block(32, 8);
  dim3 grid;
  if (transpose)
    grid = dim3((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32), (unsigned)batch);
  else
    grid = dim3((unsigned)((ldo + 31) / 32), (unsigned)((rows + 31) / 32), (unsigned)batch);
  split_tf32_2d_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(x, rows, cols, ldx, x_bstride, transpose != 0, hi,
                                                                 lo, ldo);
  JG_LAUNCH_CHECK("split_tf32_2d");
  return JG_OK;
}

int jg_cast_bf16(const float* x, void* y, int64_t n, void* stream) {
  if (n == 0) return JG_OK;
  cast_bf16_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, (__nv_bfloat16*)y, n);
  JG_LAUNCH_CHECK("cast_bf16");
  return JG_OK;
}

int jg_gelu_fwd(const void* x, void* y, int32_t dtype, int64_t n, void* stream) {
  JG_SHAPE_CHECK(dtype == JG_F32 || dtype == JG_BF16, "jg_gelu_fwd: bad dtype %d", dtype);
  if (n == 0) return JG_OK;
  gelu_fwd_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, y, dtype == JG_BF16, n);
  JG_LAUNCH_CHECK("gelu_fwd");
  return JG_OK;
}

int jg_gelu_bwd(const void* x, const void* g, void* dx, int32_t dtype, int64_t n, void* stream) {
  JG_SHAPE_CHECK(dtype == JG_F32 || dtype == JG_BF16, "jg_gelu_bwd: bad dtype %d", dtype);
  if (n == 0) return JG_OK;
  gelu_bwd_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, g, dx, dtype == JG_BF16, n);
  JG_LAUNCH_CHECK("gelu_bwd");
  return JG_OK;
}

int jg_ln_moments(const float* x, float* stats, int64_t rows, int64_t cols, int64_t ldx, void* stream) {
  JG_SHAPE_CHECK(rows >= 0 && cols > 0 && ldx >= cols, "jg_ln_moments: bad shape");
  if (rows == 0) return JG_OK;
  ln_moments_kernel<<<grid_for(rows, 8), 256, 0, (cudaStream_t)stream>>>(x, stats, rows, cols, ldx);
  JG_LAUNCH_CHECK("ln_moments");
  return JG_OK;
}

int jg_ln_apply(const float* x, const float* stats, const float* gamma, const float* beta, void* y, int32_t y_type,
                float* mean_rstd, int64_t rows, int64_t cols, int64_t c_total, float eps, const jg_bcast* y_bcast,
                void* stream) {
  JG_SHAPE_CHECK(eps > 0.f, "layer_norm eps must be > 0, got %g", (double)eps);
  JG_SHAPE_CHECK(rows >= 0 && cols > 0 && c_total >= cols, "jg_ln_apply: bad shape");
  JG_SHAPE_CHECK(al16(x) && al16(y) && al16(gamma) && al16(beta), "jg_ln_apply: pointers must be 16B aligned");
  if (rows == 0) return JG_OK;
  const int64_t cw = row_chunk(rows, cols);
  const int64_t lnu = rows * ((cols + cw - 1) / cw);
  ln_apply_kernel<<<resident_grid(ln_apply_kernel, 256, (lnu + 7) / 8), 256, 0, (cudaStream_t)stream>>>(x, stats, gamma, beta, y, y_type == JG_BF16,
                                                                      mean_rstd, rows, cols, 1.0f / (float)c_total, eps,
                                                                      to_bcast(y_bcast), cw);
  JG_LAUNCH_CHECK("ln_apply");
  return JG_OK;
}

int jg_ln_bwd_moments(const float* x, const float* g, const float* gamma, const float* mean_rstd, float* bstats,
                      int64_t rows, int64_t cols, void* stream) {
  JG_SHAPE_CHECK(rows >= 0 && cols > 0, "jg_ln_bwd_moments: bad shape");
  JG_SHAPE_CHECK(al16(x) && al16(g) && al16(gamma), "jg_ln_bwd_moments: pointers must be 16B aligned");
  if (rows == 0) return JG_OK;
  const int64_t cw = row_chunk(rows, cols);
  const int64_t lnu = rows * ((cols + cw - 1) / cw);
  ln_bwd_moments_kernel<<<resident_grid(ln_bwd_moments_kernel, 256, (lnu + 7) / 8), 256, 0, (cudaStream_t)stream>>>(x, g, gamma, mean_rstd, bstats, rows, cols, cw);
  JG_LAUNCH_CHECK("ln_bwd_moments");
  return JG_OK;
}

int jg_ln_bwd_apply(const float* x, const float* g, const float* gamma, const float* mean_rstd, const float* bstats,
                    const float* resid, float* out, void* out_bf16, float* dgamma, float* dbeta, float* rowsum_out,
                    int64_t rowsum_period, float* colsum_out, int64_t rows, int64_t cols, int64_t c_total,
                    const jg_bcast* op_bcast, void* stream) {
  JG_SHAPE_CHECK(rows >= 0 && cols > 0 && c_total >= cols, "jg_ln_bwd_apply: bad shape");
  JG_SHAPE_CHECK(al16(x) && al16(g) && al16(out) && (!resid || al16(resid)), "jg_ln_bwd_apply: pointers must be 16B aligned");
  if (rows == 0) return JG_OK;
  dim3 grid((unsigned)((cols + 1023) / 1024), (unsigned)((rows + LNB_ROWS - 1) / LNB_ROWS));
  JG_SHAPE_CHECK(!rowsum_out || rowsum_period > 0, "jg_ln_bwd_apply: rowsum_period must be > 0");
  ln_bwd_apply_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, g, gamma, mean_rstd, bstats, resid, out,
                                                               (__nv_bfloat16*)out_bf16, dgamma, dbeta, rowsum_out,
                                                               rowsum_out ? rowsum_period : 1, colsum_out, rows, cols,
                                                               1.0f / (float)c_total, to_bcast(op_bcast));
  JG_LAUNCH_CHECK("ln_bwd_apply");
  return JG_OK;
}

int jg_colsum(const void* x, int32_t x_type, float* out, int64_t rows, int64_t cols, int64_t ldx, void* stream) {
  JG_SHAPE_CHECK(rows >= 0 && cols > 0 && ldx >= cols, "jg_colsum: bad shape");
  if (rows == 0) return JG_OK;
  const bool vec = cols % 8 == 0 && ldx % 8 == 0 && al16(x);
  dim3 grid((unsigned)((cols + 255) / 256), (unsigned)((rows + CS_ROWS - 1) / CS_ROWS));
  colsum_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, x_type == JG_BF16, out, rows, cols, ldx, vec);
  JG_LAUNCH_CHECK("colsum");
  return JG_OK;
}

int jg_rowsum(const void* x, int32_t x_type, float* out, int64_t rows, int64_t cols, int64_t ldx, void* stream) {
  JG_SHAPE_CHECK(rows >= 0 && cols > 0 && ldx >= cols, "jg_rowsum: bad shape");
  if (rows == 0) return JG_OK;
  rowsum_kernel<<<grid_for(rows, 8), 256, 0, (cudaStream_t)stream>>>(x, x_type == JG_BF16, out, rows, cols, ldx);
  JG_LAUNCH_CHECK("rowsum");
  return JG_OK;
}

int jg_patchify(const float* x, void* tokens, int32_t t_type, int64_t batch, int64_t lat, int64_t lon, int64_t chans,
                int64_t p_lat, int64_t p_lon, void* stream) {
  JG_SHAPE_CHECK(p_lat > 0 && p_lon > 0 && lat % p_lat == 0 && lon % p_lon == 0,
                 "grid %lldx%lld not divisible by patch %lldx%lld", (long long)lat, (long long)lon, (long long)p_lat,
                 (long long)p_lon);
  const int64_t units = batch * lat * (lon / p_lon) * chans;
  if (units == 0) return JG_OK;
  JG_SHAPE_CHECK(units < (int64_t(1) << 31), "jg_patchify: %lld patch rows exceed 2^31", (long long)units);
  const bool bf = t_type == JG_BF16;
  const int vb = static_cast<int>(p_lon) * (bf ? 2 : 4);  // vector bytes per thread on the token side
  const bool al = (reinterpret_cast<uintptr_t>(tokens) % (vb >= 16 ? 16 : vb)) == 0;
  auto* st = (cudaStream_t)stream;
  const int C = static_cast<int>(chans), PL = static_cast<int>(p_lat), PW = static_cast<int>(p_lon);
  const int64_t nb = (units + 255) / 256;
#define JG_PATCH(PWV)                                                                       \
  patchify_kernel<PWV><<<resident_grid(patchify_kernel<PWV>, 256, nb), 256, 0, st>>>(x, tokens, bf, batch, lat, \
                                                                                      lon, C, PL, PW)
  if (al && p_lon == 8)
    JG_PATCH(8);
  else if (al && p_lon == 4)
    JG_PATCH(4);
  else if (al && p_lon == 2)
    JG_PATCH(2);
  else
    JG_PATCH(0);
#undef JG_PATCH
  JG_LAUNCH_CHECK("patchify");
  return JG_OK;
}

int jg_unpatchify(const float* tokens, float* x, int64_t batch, int64_t lat, int64_t lon, int64_t chans, int64_t p_lat,
                  int64_t p_lon, void* stream) {
  JG_SHAPE_CHECK(p_lat > 0 && p_lon > 0 && lat % p_lat == 0 && lon % p_lon == 0,
                 "token tensor does not fit grid %lldx%lld", (long long)lat, (long long)lon);
  const int64_t n = batch * lat * lon * chans;
  if (n == 0) return JG_OK;
  unpatchify_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(tokens, x, batch, lat, lon, chans, p_lat, p_lon);
  JG_LAUNCH_CHECK("unpatchify");
  return JG_OK;
}

int jg_blend_loss(const float* dec_tok, const float* x, const float* target, const float* blend_w, const float* lat_w,
                  const float* var_w, const float* g_out_ext, float* out, float* loss_sum, float* g_blend,
                  float* g_dec_f32, void* g_dec_bf16, int64_t batch, int64_t lat, int64_t lon, int64_t chans,
                  int64_t p_lat, int64_t p_lon, float inv_count, float loss_scale, const jg_bcast* gdec_bcast,
                  void* stream) {
  JG_SHAPE_CHECK(chans > 0 && chans <= MAX_CH, "jg_blend_loss: 1..%d channels", MAX_CH);
  JG_SHAPE_CHECK(lat % p_lat == 0 && lon % p_lon == 0, "jg_blend_loss: grid not divisible by patch");
  JG_SHAPE_CHECK(!target || (lat_w && var_w), "jg_blend_loss: a target needs lat/var weights");
  JG_SHAPE_CHECK(p_lon <= 16, "jg_blend_loss: patch width %lld > 16", (long long)p_lon);
  const int64_t units = batch * lat * (lon / p_lon) * chans;
  if (units == 0) return JG_OK;
  JG_SHAPE_CHECK(units < (int64_t(1) << 31), "jg_blend_loss: %lld patch rows exceed 2^31", (long long)units);
  const Bcast bc = to_bcast(gdec_bcast);
  // vector path: every token-side base (the decoder tokens, gradient outputs, peer copies) aligned
  // to the per-thread run (pw floats / bf16)
  const int vf = static_cast<int>(p_lon) * 4, vh = static_cast<int>(p_lon) * 2;
  auto al = [](const void* p, int bytes) {
    return p == nullptr || (reinterpret_cast<uintptr_t>(p) % (bytes >= 16 ? 16 : bytes)) == 0;
  };
  bool vec = al(dec_tok, vf) && al(g_dec_f32, vf) && al(g_dec_bf16, vh);
  for (int k = 0; k < bc.n; ++k) vec = vec && al(bc.p[k], g_dec_f32 ? vf : vh);
  const int block = 256;
  const int act = (block / static_cast<int>(chans)) * static_cast<int>(chans);
  const int64_t nb = (units + act - 1) / act;
  auto* st = (cudaStream_t)stream;
  const int C = static_cast<int>(chans), PL = static_cast<int>(p_lat), PW = static_cast<int>(p_lon);
#define JG_BLEND(PWV)                                                                                           \
  blend_loss_kernel<PWV><<<resident_grid(blend_loss_kernel<PWV>, block, nb), block, 0, st>>>(dec_tok, x, target, blend_w, lat_w, var_w, g_out_ext, out,      \
                                                 loss_sum, g_blend, g_dec_f32, (__nv_bfloat16*)g_dec_bf16, batch, \
                                                 lat, lon, C, PL, PW, inv_count, loss_scale, bc)
  if (vec && p_lon == 8)
    JG_BLEND(8);
  else if (vec && p_lon == 4)
    JG_BLEND(4);
  else if (vec && p_lon == 2)
    JG_BLEND(2);
  else
    JG_BLEND(0);
#undef JG_BLEND
  JG_LAUNCH_CHECK("blend_loss");
  return JG_OK;
}

int jg_adam_push(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n, float lr, float beta1,
                 float beta2, float eps, const int32_t* step_dev, const float* grad_scale_dev, const float* lr_dev,
                 const jg_push_table* push, void* stream) {
  JG_SHAPE_CHECK(n >= 0 && step_dev, "jg_adam: bad arguments");
  JG_SHAPE_CHECK(al16(p) && al16(g) && al16(m) && al16(v) && (!p_bf16 || (reinterpret_cast<uintptr_t>(p_bf16) & 7u) == 0),
                 "jg_adam: buffers must be 16B aligned");
  jg_push_table t{};
  if (push && push->nseg > 0) {
    JG_SHAPE_CHECK(p_bf16 && push->nseg <= JG_MAX_PUSH_SEGS, "jg_adam_push: needs the bf16 copy, <= %d segments",
                   JG_MAX_PUSH_SEGS);
    for (int k = 0; k < push->nseg; ++k) {
      const jg_push_seg& sg = push->seg[k];
      JG_SHAPE_CHECK(sg.start >= 0 && sg.len >= 0 && sg.start + sg.len <= n && sg.start % 4 == 0 && sg.len % 4 == 0 &&
                         sg.ndst >= 0 && sg.ndst <= 4,
                     "jg_adam_push: bad segment %d", k);
      for (int d = 0; d < sg.ndst; ++d)
        JG_SHAPE_CHECK((reinterpret_cast<uintptr_t>(sg.dst[d]) & 7u) == 0, "jg_adam_push: dst must be 8B aligned");
    }
    t = *push;
  }
  if (n == 0) return JG_OK;
  adam_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, (cudaStream_t)stream>>>(
      p, g, m, v, (__nv_bfloat16*)p_bf16, n, lr, beta1, beta2, eps, step_dev, grad_scale_dev, lr_dev, t);
  JG_LAUNCH_CHECK("adam");
  return JG_OK;
}

int jg_adam_sms(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n, float lr, float beta1,
                float beta2, float eps, const int32_t* step_dev, const float* grad_scale_dev, const float* lr_dev,
                int32_t sms, void* stream) {
  JG_SHAPE_CHECK(n >= 0 && step_dev && sms > 0, "jg_adam_sms: bad arguments");
  JG_SHAPE_CHECK(al16(p) && al16(g) && al16(m) && al16(v) && (!p_bf16 || (reinterpret_cast<uintptr_t>(p_bf16) & 7u) == 0),
                 "jg_adam: buffers must be 16B aligned");
  if (n == 0) return JG_OK;
  // one 1024-thread block per SM (48 registers per thread) holding 100 KB of (unused) dynamic
  // shared memory, so none fits beside a GEMM CTA: the blocks land on the SMs the GEMM grid
  // leaves free
  constexpr int kSmem = 100 * 1024;
  static std::once_flag once;
  std::call_once(once, [] { cudaFuncSetAttribute(adam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem); });
  jg_push_table t{};
  adam_kernel<<<sms, 1024, kSmem, (cudaStream_t)stream>>>(p, g, m, v, (__nv_bfloat16*)p_bf16, n, lr, beta1, beta2,
                                                              eps, step_dev, grad_scale_dev, lr_dev, t);
  JG_LAUNCH_CHECK("adam_sms");
  return JG_OK;
}

int jg_adam(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n, float lr, float beta1, float beta2,
            float eps, const int32_t* step_dev, const float* grad_scale_dev, const float* lr_dev, void* stream) {
  return jg_adam_push(p, g, m, v, p_bf16, n, lr, beta1, beta2, eps, step_dev, grad_scale_dev, lr_dev, nullptr, stream);
}

int jg_opt_schedule(const int32_t* step_dev, const jg_lr_schedule* sched, int32_t nsched, const float* sqsum_dev,
                    float clip_norm, float* lr_out, float* grad_scale_out, void* stream) {
  JG_SHAPE_CHECK(step_dev && nsched >= 0 && nsched <= JG_MAX_LR_CLASSES && (nsched == 0 || (sched && lr_out)),
                 "jg_opt_schedule: bad arguments");
  JG_SHAPE_CHECK(clip_norm <= 0.f || (sqsum_dev && grad_scale_out), "jg_opt_schedule: clipping needs sqsum and scale");
  SchedArgs a{};
  a.n = nsched;
  for (int i = 0; i < nsched; ++i) {
    JG_SHAPE_CHECK(sched[i].total_steps <= 0 || (sched[i].warmup_steps >= 0 && sched[i].warmup_steps < sched[i].total_steps),
                   "jg_opt_schedule: warm-up must end before the last step");
    a.s[i] = sched[i];
  }
  opt_schedule_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(step_dev, a, sqsum_dev, clip_norm, lr_out, grad_scale_out);
  JG_LAUNCH_CHECK("opt_schedule");
  return JG_OK;
}

int jg_step_increment(int32_t* counter, void* stream) {
  step_inc_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(counter);
  JG_LAUNCH_CHECK("step_inc");
  return JG_OK;
}

int jg_sqnorm(const float* x, int64_t n, float weight, float* out, void* stream) {
  if (n == 0) return JG_OK;
  const bool vec = n % 4 == 0 && al16(x);
  sqnorm_kernel<<<grid_for(vec ? n / 4 : n, 256), 256, 0, (cudaStream_t)stream>>>(x, n, weight, out, vec);
  JG_LAUNCH_CHECK("sqnorm");
  return JG_OK;
}

int jg_epilogue(const jg_gemm_desc* g, const void* acc, int32_t acc_type, int64_t lda, int64_t acc_bstride,
                int32_t nplanes, void* stream) {
  JG_SHAPE_CHECK(g && acc && g->m > 0 && g->n > 0 && g->batch > 0, "jg_epilogue: bad shape");
  JG_SHAPE_CHECK(nplanes >= 1 && (nplanes == 1 || g->batch == 1), "jg_epilogue: planes need batch 1");
  JG_SHAPE_CHECK(!(g->epi & JG_EPI_ACCUM) || (g->d && g->d_type == JG_F32), "jg_epilogue: ACCUM needs an fp32 D");
  JG_SHAPE_CHECK(!(g->epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) || g->d2, "jg_epilogue: missing D2");
  JG_SHAPE_CHECK(!(g->epi & (JG_EPI_BIAS_COL | JG_EPI_BIAS_ROW)) || g->bias, "jg_epilogue: missing bias");
  JG_SHAPE_CHECK(!(g->epi & JG_EPI_RESID) || g->resid, "jg_epilogue: missing resid");
  JG_SHAPE_CHECK(!(g->epi & JG_EPI_GELU_BWD) || g->pre, "jg_epilogue: missing pre");
  JG_SHAPE_CHECK(!(g->epi & JG_EPI_STATS) || g->stats, "jg_epilogue: missing stats");
  EpiArgs a;
  a.m = g->m; a.n = g->n; a.epi = g->epi; a.alpha = g->alpha;
  a.acc = acc; a.lda = lda; a.a_bs = acc_bstride; a.nplanes = nplanes; a.acc_bf16 = acc_type == JG_BF16;
  a.d = g->d; a.ldd = g->ldd; a.d_bs = g->d_bstride; a.d_bf16 = g->d_type == JG_BF16;
  a.d2 = g->d2; a.ldd2 = g->ldd2; a.d2_bs = g->d2_bstride; a.d2_bf16 = g->d2_type == JG_BF16;
  a.bias = g->bias; a.bias_bs = g->bias_bstride;
  a.resid = g->resid; a.ldr = g->ldr; a.r_bs = g->r_bstride;
  a.pre = g->pre; a.ldp = g->ldp; a.p_bs = g->p_bstride; a.pre_bf16 = g->pre_type == JG_BF16;
  a.stats = g->stats; a.stats_bs = g->stats_bstride;
  a.dbc = to_bcast(&g->d_bcast);
  a.d2bc = to_bcast(&g->d2_bcast);
  auto a16 = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool vec = g->n % 8 == 0 && lda % 8 == 0 && acc_bstride % 8 == 0 && g->ldd % 8 == 0 && g->ldd2 % 8 == 0 &&
                   g->ldr % 8 == 0 && g->ldp % 8 == 0 && g->bias_bstride % 8 == 0 && a16(acc) && a16(g->d) &&
                   a16(g->d2) && a16(g->bias) && a16(g->resid) && a16(g->pre) && g->d_bstride % 8 == 0 &&
                   g->r_bstride % 8 == 0 && g->p_bstride % 8 == 0 && g->d2_bstride % 8 == 0;
  const int64_t units = vec ? g->m * ((g->n + 255) / 256) : g->m;  // warp units per batch entry
  // the flag sets of the Jigsaw step get their own instantiation (loads issued together)
  auto launch = [&](auto kern) {
    dim3 grid((unsigned)resident_grid(kern, 256, (units + 7) / 8), (unsigned)g->batch);
    kern<<<grid, 256, 0, (cudaStream_t)stream>>>(a, vec);
  };
  switch (g->epi) {
    case JG_EPI_BIAS_ROW | JG_EPI_RESID | JG_EPI_STATS: launch(epilogue_kernel<JG_EPI_BIAS_ROW | JG_EPI_RESID | JG_EPI_STATS>); break;
    case JG_EPI_BIAS_COL | JG_EPI_GELU_FWD: launch(epilogue_kernel<JG_EPI_BIAS_COL | JG_EPI_GELU_FWD>); break;
    case JG_EPI_BIAS_COL | JG_EPI_RESID | JG_EPI_STATS: launch(epilogue_kernel<JG_EPI_BIAS_COL | JG_EPI_RESID | JG_EPI_STATS>); break;
    case JG_EPI_BIAS_COL | JG_EPI_RESID: launch(epilogue_kernel<JG_EPI_BIAS_COL | JG_EPI_RESID>); break;
    case JG_EPI_BIAS_COL | JG_EPI_RESID | JG_EPI_COPY_D2: launch(epilogue_kernel<JG_EPI_BIAS_COL | JG_EPI_RESID | JG_EPI_COPY_D2>); break;
    case JG_EPI_BIAS_COL | JG_EPI_STATS: launch(epilogue_kernel<JG_EPI_BIAS_COL | JG_EPI_STATS>); break;
    case JG_EPI_BIAS_COL: launch(epilogue_kernel<JG_EPI_BIAS_COL>); break;
    case JG_EPI_GELU_BWD: launch(epilogue_kernel<JG_EPI_GELU_BWD>); break;
    case 0: launch(epilogue_kernel<0u>); break;
    default: launch(epilogue_kernel<EPI_DYN>); break;
  }
  JG_LAUNCH_CHECK("epilogue");
  return JG_OK;
}

int jg_sum_planes(float* y, const void* x, int32_t x_type, int64_t n, int32_t nplanes, int64_t plane_stride,
                  int32_t accumulate, void* stream) {
  if (n == 0) return JG_OK;
  const bool bf = x_type == JG_BF16;
  const bool vec = n % 8 == 0 && plane_stride % 8 == 0 && al16(y) && al16(x);
  const int64_t work = vec ? n / 8 : n;
  if (bf) sum_planes_kernel<true><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(y, x, n, nplanes, plane_stride, accumulate != 0, vec);
  else sum_planes_kernel<false><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(y, x, n, nplanes, plane_stride, accumulate != 0, vec);
  JG_LAUNCH_CHECK("sum_planes");
  return JG_OK;
}

struct BarrierArgs { uint32_t* peer[8]; uint32_t* own; uint32_t* epoch; int G, idx; };

__global__ void group_barrier_kernel(const BarrierArgs a) {
  __shared__ uint32_t e;
  const int lane = threadIdx.x;
  if (lane == 0) {
    e = *a.epoch + 1;
    *a.epoch = e;
  }
  __syncthreads();
  __threadfence_system();  // this GPU's earlier (peer) stores are visible before it signals
  if (lane < a.G && lane != a.idx) {
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.peer[lane] + a.idx) : "memory");
    const long long t0 = clock64();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.own + lane) : "memory");
      if (static_cast<int32_t>(v - e) >= 0) break;
      if (clock64() - t0 > (1ll << 33)) __trap();  // a member never arrived: fail loudly
    }
  }
  __syncthreads();
}

int jg_group_barrier(uint32_t* const* peer_slots, uint32_t* own_slots, uint32_t* epoch, int32_t G, int32_t idx,
                     void* stream) {
  JG_SHAPE_CHECK(G >= 1 && G <= 8 && idx >= 0 && idx < G && own_slots && epoch, "jg_group_barrier: bad group");
  BarrierArgs a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < G; ++j) a.peer[j] = peer_slots[j];
  a.own = own_slots;
  a.epoch = epoch;
  a.G = G;
  a.idx = idx;
  group_barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(a);
  JG_LAUNCH_CHECK("group_barrier");
  return JG_OK;
}

int jg_push(const void* src, int64_t bytes, const jg_bcast* dst, void* stream) {
  auto al8 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; };
  JG_SHAPE_CHECK(bytes >= 0 && bytes % 8 == 0 && al8(src), "jg_push: bytes and src must be 8-byte multiples");
  Bcast b = to_bcast(dst);
  bool a16 = al16(src);
  for (int d = 0; d < b.n; ++d) {
    JG_SHAPE_CHECK(al8(b.p[d]), "jg_push: destinations must be 8-byte aligned");
    a16 = a16 && al16(b.p[d]);
  }
  if (bytes == 0 || b.n == 0) return JG_OK;
  const uint8_t* s = static_cast<const uint8_t*>(src);
  if (a16)
    push_kernel<uint4><<<grid_for((bytes + 15) / 16, 256), 256, 0, (cudaStream_t)stream>>>(s, bytes, b);
  else
    push_kernel<uint2><<<grid_for((bytes + 7) / 8, 256), 256, 0, (cudaStream_t)stream>>>(s, bytes, b);
  JG_LAUNCH_CHECK("push");
  return JG_OK;
}

int jg_memset(void* dst, int64_t bytes, void* stream) {
  if (bytes == 0) return JG_OK;
  return jg::cuda_check(cudaMemsetAsync(dst, 0, (size_t)bytes, (cudaStream_t)stream), "cudaMemsetAsync");
}

int jg_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes == 0) return JG_OK;
  return jg::cuda_check(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
                        "cudaMemcpyAsync");
}

int jg_axpy(float* y, const float* x, float alpha, int64_t n, void* stream) {
  if (n == 0) return JG_OK;
  axpy_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(y, x, alpha, n);
  JG_LAUNCH_CHECK("axpy");
  return JG_OK;
}

}  // extern "C"
