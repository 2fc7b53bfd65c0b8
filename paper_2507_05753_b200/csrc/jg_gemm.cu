// jg_gemm.cu — persistent, warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
// Replaces tensor.matmul (reference tensor.py:59-72) as used by every Jigsaw primitive
// (parallel.py:107-353) and fuses the elementwise tails of ShardedLinear / MixerBlock
// (bias parallel.py:521-525, GELU tensor.py:75-84, residual model.py:274/280, layer-norm
// row moments model.py:234) into the accumulator read-out.
//
// Structure (one CTA per SM, persistent over output tiles of 128 x BN):
//   warp 0 lane 0 : TMA producer — fills a STAGES-deep ring of (A,B) K-slices in smem,
//                   128B-swizzled, completion counted on full[] mbarriers.
//   warp 1 lane 0 : MMA issuer — 4 x tcgen05.mma per K-slice into a TMEM accumulator
//                   (double-buffered: 2 x BN fp32 columns), frees smem via tcgen05.commit.
//   warp 2        : TMEM allocator.
//   warps 4..11   : epilogue — two warps per TMEM lane quarter, each draining alternate
//                   32-column chunks: tcgen05.ld 32 lanes x 32 columns per step (thread ==
//                   row), applies bias / residual / GELU / GELU' / accumulate / row moments,
//                   stores fp32 and/or bf16; releases the TMEM buffer to the MMA warp.
// Operands may be K-major or MN-major (the NN / NT / TN modes of tensor.py:27-33), are
// loaded with 3-D TMA (batch as the 3rd dimension) and may be summed over the batch
// (weight gradients, parallel.py:552-556) or over up to three K segments (3xTF32 split).
#include "jg_common.cuh"
#include <cudaTypedefs.h>
#include <mutex>

namespace {

constexpr int BM = 128;
#ifndef JG_EPI_WARPS
#define JG_EPI_WARPS 8
#endif
#ifndef JG_REG_LO
#define JG_REG_LO 88
#define JG_REG_HI 208
#endif
constexpr int NUM_EPI_WARPS = JG_EPI_WARPS;  // 8: two per TMEM lane quarter, splitting a tile's column chunks
static_assert(NUM_EPI_WARPS == 4 || NUM_EPI_WARPS == 8,
              "epilogue warps: 4 or 8 (12 deadlocks the pipeline and overflows shared memory)");
constexpr int NUM_THREADS = 128 + 32 * NUM_EPI_WARPS;
constexpr int SMEM_BUDGET = 196 * 1024;

struct GemmParams {
  CUtensorMap tma_a[3];
  CUtensorMap tma_b[3];
  CUtensorMap tma_d[8];   // D store maps: [0] = batched D, or one per remote output plane
  CUtensorMap tma_d2;
  CUtensorMap tma_dx[4];  // extra destinations (peer gather slots) of D and of D2
  CUtensorMap tma_d2x[4];
  int nb_d, nb_d2;
  int tma_store;          // 1: epilogue writes D / D2 through TMA bulk tensor stores
  int nseg;
  int m, n, k;
  int batch;
  int reduce_batch;
  int a_mn, b_mn;          // operand majors (1 = MN-major)
  int a_batched, b_batched;
  int num_kb;              // K blocks per (segment, batch)
  int m_tiles, n_tiles;
  int num_tiles;
  // epilogue
  uint32_t epi;
  float alpha;
  void* d; int64_t ldd, d_bs; int d_bf16;
  void* d2; int64_t ldd2, d2_bs; int d2_bf16;
  const float* bias; int64_t bias_bs;
  const float* resid; int64_t ldr, r_bs;
  const void* pre; int64_t ldp, p_bs; int pre_bf16;
  float* stats; int64_t stats_bs;
  float* adam_m; float* adam_v; __nv_bfloat16* adam_pbf16; const int32_t* adam_step;
  float adam_lr, adam_b1, adam_b2, adam_eps;
  void* d_planes[8];
  int remote;              // some output goes to a peer: system-scope fence at the end
  int planes;              // d_planes in use: per-batch D store maps
  int plane_div;           // > 0: batch b -> store map b / plane_div, sample coordinate b % plane_div
  int plane_minor;         // tile order with the output plane fastest (JG_PLANE_MAJOR=1 disables)
  // fused reduce-scatter (jg_gemm_desc rs_*): raw partial tiles to the owners + arrival flags,
  // own-plane tiles last, summed with the peers' partials in this rank's buffer
  int rs_mode;
  int dmap_bf16[8];        // dtype of tma_d[b]
  uint32_t* rs_flags;
  uint32_t* rs_flag_peers[8];
  const void* rs_src; int64_t rs_src_stride;
  int rs_part_bf16, rs_nsrc, rs_src_idx, rs_own, rs_need;
  // wave schedule of a fused reduce-scatter with an own plane: the persistent loop's positions
  // come in waves of `units` tiles (one per CTA unit); wave k holds own-plane tiles
  // wave_idx[k]*units.. (wave_kind 1) or remote-partial tiles (0). Own waves alternate with
  // remote waves (after a head of remote waves), so each CTA alternates the heavy own epilogue
  // (peer partial loads, residual, two outputs) with light raw partial stores, and an own tile
  // always follows its peers' partials by at least one wave. nwaves == 0: linear order.
  int num_pos, units, nwaves;
  uint8_t wave_kind[64], wave_idx[64];
  const float* lnb_x; int64_t lnb_ldx, lnb_x_bs; const float* lnb_gamma; const float* lnb_mr;
  int rs_dbg;              // JG_RS_DBG ablations (timing only, results wrong): 1 no fences, 2 no own wait, 4 no peer loads
};

// Fused reduce-scatter: the own plane's tiles run after every remote tile (logical batch order
// own+1, own+2, ..., own), so each rank first feeds its peers, then consumes what they fed it.
template <bool RS>
__device__ __forceinline__ int rs_batch(const GemmParams& p, int lb) {
  return (RS && p.rs_own >= 0) ? (p.rs_own + 1 + lb) % p.batch : lb;
}

// position of the persistent tile loop -> (output batch, tile within the batch); false: a hole
template <bool RS>
__device__ __forceinline__ bool tile_at(const GemmParams& p, int pos, int tiles_per_batch, int& tb, int& rem) {
  if (!RS && p.planes && p.plane_minor) {
    // partial planes for several owners: plane-minor order, so every wave mixes local tiles
    // with tiles stored into peers over NVLink (plane-major order bunches each peer's whole
    // plane into one stretch that NVLink cannot absorb; measured -22..28 % at K ~ 2160)
    rem = pos / p.batch;
    tb = pos - rem * p.batch;
    return true;
  }
  if (!RS || p.nwaves == 0) {
    const int lb = p.reduce_batch ? 0 : pos / tiles_per_batch;
    rem = pos - lb * tiles_per_batch;
    tb = p.reduce_batch ? 0 : rs_batch<RS>(p, lb);
    return true;
  }
  const int k = pos / p.units;
  const int t = p.wave_idx[k] * p.units + (pos - k * p.units);
  if (p.wave_kind[k]) {
    tb = p.rs_own;
    rem = t;
    return t < tiles_per_batch;
  }
  const int nr = p.batch - 1;
  if (t >= nr * tiles_per_batch) return false;
  rem = t / nr;
  const int b = t - rem * nr;
  tb = b < p.rs_own ? b : b + 1;
  return true;
}

__device__ __forceinline__ void rs_wait_flag(const uint32_t* f, uint32_t need) {
  const long long t0 = clock64();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v >= need) break;
    __nanosleep(64);
    if (clock64() - t0 > (1ll << 33)) __trap();  // a peer never arrived (~4 s): fail loudly, never hang
  }
}

__device__ __forceinline__ void rs_add_flag(uint32_t* f, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

// wait until at most n of this thread's most recent bulk async-groups are still pending
__device__ __forceinline__ void bulk_wait_le(int n) {
  switch (n) {
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
  }
}

// Arrival of a partial tile at its owner, signalled lazily: the tile's stores are left in flight
// while the warp drains the next tile, whose own store groups (`newer`) may stay pending.
__device__ __forceinline__ void rs_signal(uint32_t*& pend, int newer, int lane, int dbg) {
  if (pend == nullptr) return;
  if (lane == 0) {
    if (!(dbg & 1)) {
      bulk_wait_le(newer);  // the tile's stores are complete ...
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }                       // ... and ordered before the release below
    rs_add_flag(pend, 1u);
  }
  __syncwarp();
  pend = nullptr;
}

// 8 contiguous partial-product elements written by a peer during this kernel (L2, not L1)
__device__ __forceinline__ void load8_cg(const void* base, int64_t off, bool bf16, float* v) {
  if (bf16) {
    const uint4 raw = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + off));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  } else {
    const float4* q = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off);
    const float4 a = __ldcg(q), b = __ldcg(q + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <int BN, bool TF32, int CG = 1>
struct Cfg {
  static constexpr int ESIZE = TF32 ? 4 : 2;
  static constexpr int BK = 128 / ESIZE;           // one 128-byte swizzle atom of K
  static constexpr int UMMA_K = TF32 ? 8 : 16;     // 32 bytes of K per instruction
  static constexpr int ATOM = 128 / ESIZE;         // elements per 128B row of an MN-major box
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = (BN / CG) * 128;  // 2-CTA: each CTA holds half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (SMEM_BUDGET / STAGE_BYTES) > 8 ? 8 : (SMEM_BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS = 2 * BN;          // double-buffered fp32 accumulator
  static constexpr int EPI_STAGE_BYTES = NUM_EPI_WARPS * 4096;  // one 32x32 fp32 staging tile per epilogue warp
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t IDESC_BASE =
      (1u << 4)                                    // D format: f32
      | ((TF32 ? 2u : 1u) << 7)                    // A format: tf32 / bf16
      | ((TF32 ? 2u : 1u) << 10)                   // B format
      | (static_cast<uint32_t>(BN >> 3) << 17)     // N
      | (static_cast<uint32_t>((BM * CG) >> 4) << 24);  // M (256 for a CTA pair)
};

// Stage one warp's 32 x 32 accumulator chunk (thread = row) in 128B / 64B-swizzled smem and
// TMA-store it: rows become contiguous bulk writes (HBM or an NVLink peer), conflict-free smem.
__device__ __forceinline__ void stage_store(uint8_t* stg, const float* v, bool bf16, int lane,
                                            const CUtensorMap* map, int c0, int c1, int c2,
                                            const CUtensorMap* extra = nullptr, int n_extra = 0) {
  if (lane == 0) jgd::bulk_wait_read0();
  __syncwarp();
  if (bf16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 raw;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[8 * i + 2 * k], v[8 * i + 2 * k + 1]);
      *reinterpret_cast<uint4*>(stg + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4)) = raw;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      *reinterpret_cast<float4*>(stg + lane * 128 + ((i ^ (lane & 7)) << 4)) =
          make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
  jgd::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    jgd::tma_store_3d(map, stg, c0, c1, c2);
    for (int i = 0; i < n_extra; ++i) jgd::tma_store_3d(extra + i, stg, c0, c1, c2);  // same tile, peers
    jgd::bulk_commit();
  }
}

// L2-aware tile order: tiles run m-fastest inside groups of TILE_GROUP_M row tiles, so one wave of
// ~148 CTAs covers a ~8 x (units/8) block of the output and reads ~8 + units/8 operand panels per
// k-step from DRAM instead of (units / n_tiles) + n_tiles (long-K token GEMMs: B re-read per wave).
#ifndef JG_TILE_GROUP_M
#define JG_TILE_GROUP_M 8
#endif
constexpr int TILE_GROUP_M = JG_TILE_GROUP_M;
__device__ __forceinline__ void tile_coords(int rem, int m_tiles, int n_tiles, int& mi, int& ni) {
  const int per_group = TILE_GROUP_M * n_tiles;
  const int g = rem / per_group;
  const int first = g * TILE_GROUP_M;
  const int gm = min(TILE_GROUP_M, m_tiles - first);
  const int r = rem - g * per_group;
  mi = first + r % gm;
  ni = r / gm;
}

template <int BN, bool TF32, int CG, bool RS>
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_kernel(const __grid_constant__ GemmParams p) {
  using C = Cfg<BN, TF32, CG>;
  static_assert(CG == 1 || !TF32, "2-CTA path is bf16 only");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::STAGES * C::A_BYTES;
  constexpr int A_STRIDE = C::A_BYTES, B_STRIDE = C::B_BYTES;
  uint8_t* smem_epi = smem + C::STAGES * C::STAGE_BYTES;  // 1024-aligned: 4 x 4 KB staging tiles
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + C::EPI_STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.nseg; ++s) {
      jgd::tma_prefetch_desc(&p.tma_a[s]);
      jgd::tma_prefetch_desc(&p.tma_b[s]);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      jgd::mbar_init(&full[s], 1);
      jgd::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      jgd::mbar_init(&tfull[s], 1);
      jgd::mbar_init(&tempty[s], NUM_EPI_WARPS * CG);  // every epilogue warp of the pair drains the leader's slot
    }
    jgd::mbar_fence_init();
  }
  const uint32_t cta_rank = CG == 2 ? jgd::cluster_ctarank() : 0;
  const bool leader = cta_rank == 0;
  if (warp == 2) {
    if constexpr (CG == 2)
      jgd::tmem_alloc_2sm(tmem_slot, C::TMEM_COLS);
    else
      jgd::tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  jgd::tc_fence_before();
  if constexpr (CG == 2)
    jgd::cluster_sync();
  else
    __syncthreads();
  jgd::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int tile0 = blockIdx.x / CG, tstep = gridDim.x / CG;

  const int kb_batches = p.reduce_batch ? p.batch : 1;
  const int kb_per_tile = p.nseg * kb_batches * p.num_kb;
  const int tiles_per_batch = p.m_tiles * p.n_tiles;

  // register split: warpgroup 0 (TMA producer, MMA issuer, TMEM allocator) needs few; the two
  // epilogue warpgroups get the rest (128 x 88 + 256 x 208 <= 64K; 40 / 232 and no split measured slower at locked clocks)
#define JG_STR2(x) #x
#define JG_STR(x) JG_STR2(x)
  if (warp < 4) {
#if JG_REG_LO > 0
  asm volatile("setmaxnreg.dec.sync.aligned.u32 " JG_STR(JG_REG_LO) ";\n" ::: "memory");
#endif
  if (warp == 0 && lane == 0) {
    // ===================== TMA producer =====================
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = tile0; tile < p.num_pos; tile += tstep) {
      int tb, rem;
      if (!tile_at<RS>(p, tile, tiles_per_batch, tb, rem)) continue;
      int mi, ni;
      tile_coords(rem, p.m_tiles, p.n_tiles, mi, ni);
      const int m0 = mi * (BM * CG) + BM * static_cast<int>(cta_rank);
      const int n0 = ni * BN + (BN / CG) * static_cast<int>(cta_rank);
      for (int seg = 0; seg < p.nseg; ++seg) {
        for (int bb = 0; bb < kb_batches; ++bb) {
          const int b = p.reduce_batch ? bb : tb;
          const int ba = p.a_batched ? b : 0;
          const int bbz = p.b_batched ? b : 0;
          for (int kb = 0; kb < p.num_kb; ++kb) {
            jgd::mbar_wait(&empty[stage], phase ^ 1);
            if (leader) jgd::mbar_arrive_expect_tx(&full[stage], CG * C::STAGE_BYTES);
            const int k0 = kb * C::BK;
            uint8_t* sa = smem_a + stage * A_STRIDE;
            uint8_t* sb = smem_b + stage * B_STRIDE;
            auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, int c2) {
              if constexpr (CG == 2)
                jgd::tma_load_3d_2sm(dst, map, &full[stage], c0, c1, c2);
              else
                jgd::tma_load_3d(dst, map, &full[stage], c0, c1, c2);
            };
            if (p.a_mn) {
#pragma unroll
              for (int j = 0; j < BM / C::ATOM; ++j) load(sa + j * (C::BK * 128), &p.tma_a[seg], m0 + j * C::ATOM, k0, ba);
            } else {
              load(sa, &p.tma_a[seg], k0, m0, ba);
            }
            if (p.b_mn) {
#pragma unroll
              for (int j = 0; j < BN / CG / C::ATOM; ++j)
                load(sb + j * (C::BK * 128), &p.tma_b[seg], n0 + j * C::ATOM, k0, bbz);
            } else {
              load(sb, &p.tma_b[seg], k0, n0, bbz);
            }
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ===================== MMA issuer (leader CTA of a pair issues for both) =====================
    const uint32_t idesc = C::IDESC_BASE | (static_cast<uint32_t>(p.a_mn) << 15) | (static_cast<uint32_t>(p.b_mn) << 16);
    // K-major: SBO = 8 rows * 128B, per-instruction K step = 32 bytes inside the swizzle atom.
    // MN-major: LBO = one (ATOM x BK) box, SBO = 8 K-rows * 128B, K step = UMMA_K rows * 128B.
    const uint32_t a_lbo = p.a_mn ? C::BK * 128 : 16, b_lbo = p.b_mn ? C::BK * 128 : 16;
    const uint32_t a_kstep = p.a_mn ? C::UMMA_K * 128 : 32, b_kstep = p.b_mn ? C::UMMA_K * 128 : 32;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = tile0; tile < p.num_pos; tile += tstep) {
      int tb_, rem_;
      if (!tile_at<RS>(p, tile, tiles_per_batch, tb_, rem_)) continue;
      jgd::mbar_wait(&tempty[acc], acc_phase ^ 1);
      jgd::tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
      for (int i = 0; i < kb_per_tile; ++i) {
        jgd::mbar_wait(&full[stage], phase);
        jgd::tc_fence_after();
        const uint32_t sa = jgd::smem_u32(smem_a + stage * A_STRIDE);
        const uint32_t sb = jgd::smem_u32(smem_b + stage * B_STRIDE);
#pragma unroll
        for (int kk = 0; kk < C::BK / C::UMMA_K; ++kk) {
          const uint64_t ad = jgd::make_sdesc(sa + kk * a_kstep, a_lbo, 1024);
          const uint64_t bd = jgd::make_sdesc(sb + kk * b_kstep, b_lbo, 1024);
          if constexpr (TF32)
            jgd::umma_tf32(d_tmem, ad, bd, idesc, (i | kk) != 0);
          else if constexpr (CG == 2)
            jgd::umma_bf16_2sm(d_tmem, ad, bd, idesc, (i | kk) != 0);
          else
            jgd::umma_bf16(d_tmem, ad, bd, idesc, (i | kk) != 0);
        }
        if constexpr (CG == 2)
          jgd::umma_commit_2sm(&empty[stage], 0x3);
        else
          jgd::umma_commit(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if constexpr (CG == 2)
        jgd::umma_commit_2sm(&tfull[acc], 0x3);
      else
        jgd::umma_commit(&tfull[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  } else {
#if JG_REG_LO > 0
    asm volatile("setmaxnreg.inc.sync.aligned.u32 " JG_STR(JG_REG_HI) ";\n" ::: "memory");
#endif
    // ===================== epilogue =====================
    const int q = warp & 3;             // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;   // which alternate 32-column chunks of the tile it drains
    constexpr int CSTEP = NUM_EPI_WARPS / 4;
    uint8_t* stg = smem_epi + (warp - 4) * 4096;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t epi = p.epi;
    float bc1 = 1.f, bc2 = 1.f;
    const float ab1 = p.adam_b1, ab2 = p.adam_b2, alr = p.adam_lr, aeps = p.adam_eps;
    if (epi & JG_EPI_ADAM) {
      const int t = *p.adam_step;
      bc1 = 1.0f / (1.0f - powf(ab1, (float)t));
      bc2 = 1.0f / (1.0f - powf(ab2, (float)t));
    }
    uint32_t* pend = nullptr;  // flag of the last partial tile whose arrival is not yet signalled
    for (int tile = tile0; tile < p.num_pos; tile += tstep) {
      int tb, rem;
      if (!tile_at<RS>(p, tile, tiles_per_batch, tb, rem)) continue;
      int mi, ni;
      tile_coords(rem, p.m_tiles, p.n_tiles, mi, ni);
      const int m0 = mi * (BM * CG) + BM * static_cast<int>(cta_rank);
      const int n0 = ni * BN;
      int ngroups = 0;  // bulk store groups this warp commits for this tile
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < p.m;
      // fused reduce-scatter roles of this tile: own plane (sum + full epilogue) or a raw
      // partial for its owner (no epilogue); eb = batch index of the epilogue operands
      const bool own = RS && p.rs_mode && tb == p.rs_own;
      const bool part = RS && p.rs_mode && !own;
      const uint32_t tepi = part ? 0u : epi;
      const int eb = (RS && p.rs_mode) ? 0 : tb;
      const int fidx = (rem * CG + static_cast<int>(cta_rank)) * NUM_EPI_WARPS + (warp - 4);
      jgd::mbar_wait(&tfull[acc], acc_phase);
      jgd::tc_fence_after();
      if (RS && own) {
        rs_signal(pend, 0, lane, p.rs_dbg);  // peers may be waiting for it: never hold it across a wait
        if (!(p.rs_dbg & 2)) rs_wait_flag(p.rs_flags + fidx, static_cast<uint32_t>(p.rs_need));
        __syncwarp();
        if (lane == 0) rs_add_flag(p.rs_flags + fidx, static_cast<uint32_t>(-p.rs_need));  // re-arm for reuse
      }

      // per-batch destination (fused reduce-scatter into a peer's buffer) or the regular strided D
      void* dbase = p.d;
      int64_t drow = tb * p.d_bs + static_cast<int64_t>(row) * p.ldd;
      if (p.remote && tb < 8 && p.d_planes[tb] != nullptr) {
        dbase = p.d_planes[tb];
        drow = static_cast<int64_t>(row) * p.ldd;
      }
      const int64_t d2row = eb * p.d2_bs + static_cast<int64_t>(row) * p.ldd2;
      const int64_t rrow = eb * p.r_bs + static_cast<int64_t>(row) * p.ldr;
      const int64_t prow = eb * p.p_bs + static_cast<int64_t>(row) * p.ldp;
      float rbias = 0.f;
      if ((tepi & JG_EPI_BIAS_ROW) && row_ok) rbias = p.bias[eb * p.bias_bs + row];
      float s1 = 0.f, s2 = 0.f;
      float lnb_mean = 0.f, lnb_rstd = 0.f;
      if ((tepi & JG_EPI_LNB) && row_ok) {
        lnb_mean = p.lnb_mr[eb * p.stats_bs + static_cast<int64_t>(row) * 2];
        lnb_rstd = p.lnb_mr[eb * p.stats_bs + static_cast<int64_t>(row) * 2 + 1];
      }

#pragma unroll 1
      for (int c = half; c < BN / 32; c += CSTEP) {
        const int col0 = n0 + c * 32;
        if (col0 >= p.n) break;  // warp-uniform
        float v[32];
        jgd::tmem_ld32(tmem_base + static_cast<uint32_t>(acc * BN + c * 32) + (static_cast<uint32_t>(q * 32) << 16), v);
        const bool full_chunk = col0 + 32 <= p.n;
        const int ncol = full_chunk ? 32 : p.n - col0;
        if (own && row_ok) {
          // sum of the group's partial planes in member order (exactly jg_epilogue's sum of the
          // reduce-scattered planes: this rank's own plane rounded to the partial dtype), then
          // the epilogue in jg_epilogue's order: alpha, row bias, column bias, residual, GELU'
          float s[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) s[j] = 0.f;
          const int64_t srow = static_cast<int64_t>(row) * p.ldd + col0;
          for (int src = 0; src < p.rs_nsrc; ++src) {
            if (src == p.rs_src_idx || (p.rs_dbg & 4)) {
#pragma unroll
              for (int j = 0; j < 32; ++j) s[j] += p.rs_part_bf16 ? __bfloat162float(__float2bfloat16_rn(v[j])) : v[j];
            } else if (full_chunk) {
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                float t[8];
                load8_cg(p.rs_src, src * p.rs_src_stride + srow + g * 8, p.rs_part_bf16, t);
#pragma unroll
                for (int j = 0; j < 8; ++j) s[g * 8 + j] += t[j];
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < ncol) s[j] += jgd::load1(p.rs_src, src * p.rs_src_stride + srow + j, p.rs_part_bf16);
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = s[j] * p.alpha + rbias;
          if (epi & JG_EPI_BIAS_COL) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += (j < ncol) ? __ldg(p.bias + col0 + j) : 0.f;
          }
        }
        if (row_ok && !own && !part) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
        if (epi & JG_EPI_BIAS_COL) {
          const float* bp = p.bias + tb * p.bias_bs + col0;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += (j < ncol) ? __ldg(bp + j) : 0.f;
        }
        if (epi & JG_EPI_BIAS_ROW) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += rbias;
        }
        }  // regular (non-reduce-scatter) alpha / bias
        if (row_ok && !part) {
        if (epi & JG_EPI_RESID) {
          if (full_chunk) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float t[8];
              jgd::load8(p.resid, rrow + col0 + g * 8, false, t);
#pragma unroll
              for (int j = 0; j < 8; ++j) v[g * 8 + j] += t[j];
            }
          } else {
            #pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncol) v[j] += p.resid[rrow + col0 + j];
          }
        }
        if (epi & JG_EPI_GELU_BWD) {
          if (full_chunk) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float t[8];
              jgd::load8(p.pre, prow + col0 + g * 8, p.pre_bf16, t);
#pragma unroll
              for (int j = 0; j < 8; ++j) v[g * 8 + j] *= jgd::gelu_grad_f(t[j]);
            }
          } else {
            #pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncol) v[j] *= jgd::gelu_grad_f(jgd::load1(p.pre, prow + col0 + j, p.pre_bf16));
          }
        }
        if (epi & JG_EPI_ACCUM) {
          if (full_chunk) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float t[8];
              jgd::load8(dbase, drow + col0 + g * 8, false, t);
#pragma unroll
              for (int j = 0; j < 8; ++j) v[g * 8 + j] += t[j];
            }
          } else {
            #pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncol) v[j] += reinterpret_cast<const float*>(dbase)[drow + col0 + j];
          }
        }
        if (epi & JG_EPI_STATS) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = (j < ncol) ? v[j] : 0.f;
            s1 += x;
            s2 += x * x;
          }
        }
        if (epi & JG_EPI_LNB) {
          // layer-norm backward moments of this gradient: (sum g*gamma, sum g*gamma*xhat)
          const float* xr = p.lnb_x + eb * p.lnb_x_bs + static_cast<int64_t>(row) * p.lnb_ldx + col0;
          if (full_chunk) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float t[8];
              jgd::load8(xr, g * 8, false, t);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float h = v[g * 8 + j] * __ldg(p.lnb_gamma + col0 + g * 8 + j);
                s1 += h;
                s2 += h * ((t[j] - lnb_mean) * lnb_rstd);
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) {
                const float h = v[j] * __ldg(p.lnb_gamma + col0 + j);
                s1 += h;
                s2 += h * ((xr[j] - lnb_mean) * lnb_rstd);
              }
          }
        }
        }  // row_ok: math done
        if (epi & JG_EPI_ADAM) {
          // v[] is the complete gradient of this weight tile. Transpose the warp's 32 x 32 chunk
          // through its staging buffer (XOR swizzle) and update 4 rows x 32 columns per warp
          // instruction: lane = (row-in-4, float4 column), every master / m / v access a full
          // 128B row segment, all 24 vector loads of the chunk in flight before any math
          // (the epilogue is HBM-bound: 26 B per parameter).
          float* sf = reinterpret_cast<float*>(stg);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) sf[lane * 32 + (j ^ lane)] = v[j];
          __syncwarp();
          float* dp = reinterpret_cast<float*>(p.d);
          const int sr = lane >> 3, c4 = (lane & 7) * 4;
          const int col = col0 + c4;
          const int rbase = m0 + q * 32;
          float4 w4[8], m4[8], v4[8];
          int64_t off[8];
          bool ok[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = rbase + i * 4 + sr;
            off[i] = tb * p.d_bs + static_cast<int64_t>(rr) * p.ldd + col;
            ok[i] = rr < p.m && col + 3 < p.n;
            if (ok[i]) {
              w4[i] = *reinterpret_cast<const float4*>(dp + off[i]);
              m4[i] = *reinterpret_cast<const float4*>(p.adam_m + off[i]);
              v4[i] = *reinterpret_cast<const float4*>(p.adam_v + off[i]);
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + sr;
            if (ok[i]) {
              float* w = &w4[i].x;
              float* mm = &m4[i].x;
              float* vv = &v4[i].x;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float gj = sf[r * 32 + ((c4 + k) ^ r)];
                mm[k] = ab1 * mm[k] + (1.0f - ab1) * gj;
                vv[k] = ab2 * vv[k] + (1.0f - ab2) * gj * gj;
                w[k] -= alr * (mm[k] * bc1) / (sqrtf(vv[k] * bc2) + aeps);
              }
              *reinterpret_cast<float4*>(dp + off[i]) = w4[i];
              *reinterpret_cast<float4*>(p.adam_m + off[i]) = m4[i];
              *reinterpret_cast<float4*>(p.adam_v + off[i]) = v4[i];
              if (p.adam_pbf16) {
                __nv_bfloat162 lo = __floats2bfloat162_rn(w[0], w[1]), hi = __floats2bfloat162_rn(w[2], w[3]);
                uint2 raw;
                raw.x = *reinterpret_cast<uint32_t*>(&lo);
                raw.y = *reinterpret_cast<uint32_t*>(&hi);
                *reinterpret_cast<uint2*>(p.adam_pbf16 + off[i]) = raw;
              }
            } else if (rbase + r < p.m) {  // ragged column tail: scalar
              for (int k = 0; k < 4; ++k) {
                if (col + k >= p.n) break;
                const int64_t o = off[i] + k;
                const float gj = sf[r * 32 + ((c4 + k) ^ r)];
                const float mm = ab1 * p.adam_m[o] + (1.0f - ab1) * gj;
                const float vv = ab2 * p.adam_v[o] + (1.0f - ab2) * gj * gj;
                const float w = dp[o] - alr * (mm * bc1) / (sqrtf(vv * bc2) + aeps);
                dp[o] = w;
                p.adam_m[o] = mm;
                p.adam_v[o] = vv;
                if (p.adam_pbf16) p.adam_pbf16[o] = __float2bfloat16_rn(w);
              }
            }
          }
          continue;
        }
        if (p.tma_store) {
          // stage the warp's 32 x 32 chunk in swizzled smem, one TMA bulk tensor store per output
          const int rbase = m0 + q * 32;
          if (part) {
            stage_store(stg, v, p.dmap_bf16[tb], lane, &p.tma_d[tb], col0, rbase, 0);
            ++ngroups;
            continue;
          }
          const bool per_batch_map = p.planes || (RS && p.rs_mode);
          const int mi = per_batch_map ? (p.plane_div ? tb / p.plane_div : tb) : 0;
          const int c2 = per_batch_map ? (p.plane_div ? tb % p.plane_div : 0) : tb;
          if (per_batch_map || p.d != nullptr)
            stage_store(stg, v, p.dmap_bf16[mi], lane, &p.tma_d[mi], col0, rbase, c2, p.tma_dx, p.nb_d);
          if (epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) {
            if (epi & JG_EPI_GELU_FWD) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = jgd::gelu_f(v[j]);
            }
            stage_store(stg, v, p.d2_bf16, lane, &p.tma_d2, col0, rbase, eb, p.tma_d2x, p.nb_d2);
          }
          continue;
        }
        if (!row_ok) continue;
        // primary output
        if (dbase != nullptr) {
          if (full_chunk) {
#pragma unroll
            for (int g = 0; g < 4; ++g) jgd::store8(dbase, drow + col0 + g * 8, p.d_bf16, v + g * 8);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncol) jgd::store1(dbase, drow + col0 + j, p.d_bf16, v[j]);
          }
        }
        // secondary output: gelu(result) or a plain copy
        if (epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) {
          if (epi & JG_EPI_GELU_FWD) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = jgd::gelu_f(v[j]);
          }
          if (full_chunk) {
#pragma unroll
            for (int g = 0; g < 4; ++g) jgd::store8(p.d2, d2row + col0 + g * 8, p.d2_bf16, v + g * 8);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) if (j < ncol) jgd::store1(p.d2, d2row + col0 + j, p.d2_bf16, v[j]);
          }
        }
      }
      if ((tepi & (JG_EPI_STATS | JG_EPI_LNB)) && row_ok) {
        float* sp = p.stats + eb * p.stats_bs + static_cast<int64_t>(row) * 2;
        atomicAdd(sp, s1);
        atomicAdd(sp + 1, s2);
      }
      if (RS && part && p.rs_flag_peers[tb] != nullptr) {
        // the previous partial tile's stores are older than this tile's ngroups: signal it now,
        // this one after the next tile (or before any own-tile wait / at the end)
        rs_signal(pend, ngroups, lane, p.rs_dbg);
        pend = p.rs_flag_peers[tb] + fidx;
      }
      jgd::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          jgd::mbar_arrive_leader(&tempty[acc]);
        else
          jgd::mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if constexpr (RS) rs_signal(pend, 0, lane, p.rs_dbg);
    if (lane == 0) jgd::bulk_wait0();  // every TMA store of this warp has landed
    __syncwarp();
    if (p.remote) __threadfence_system();  // peer stores visible before the group barrier
  }

  jgd::tc_fence_before();
  if constexpr (CG == 2)
    jgd::cluster_sync();  // the leader's MMAs read the peer's smem: nobody leaves early
  else
    __syncthreads();
  if (warp == 2) {
    jgd::tc_fence_after();
    if constexpr (CG == 2)
      jgd::tmem_dealloc_2sm(tmem_base, C::TMEM_COLS);
    else
      jgd::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// Operand map. K-major: dims (K, rows, batch), box (BK, rows_box). MN-major: dims (rows, K, batch),
// box (ATOM, BK). rows = M or N extent.
int make_operand_map(CUtensorMap* map, const void* ptr, bool tf32, bool mn_major, int64_t rows, int64_t k,
                     int64_t ld, int64_t bstride, int64_t batch, int box_rows) {
  const int esize = tf32 ? 4 : 2;
  const int atom = 128 / esize;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  if (mn_major) {
    dims[0] = rows; dims[1] = k;
    box[0] = atom; box[1] = atom;  // BK == ATOM
  } else {
    dims[0] = k; dims[1] = rows;
    box[0] = atom; box[1] = box_rows;
  }
  dims[2] = batch;
  box[2] = 1;
  strides[0] = static_cast<cuuint64_t>(ld) * esize;
  strides[1] = static_cast<cuuint64_t>(batch > 1 ? bstride : ld * (mn_major ? k : rows)) * esize;
  if (strides[1] == 0 || strides[1] % 16) strides[1] = ((strides[0] * dims[1] + 15) / 16) * 16;
  auto fn = encode_fn();
  if (!fn) {
    jg::set_error("cuTensorMapEncodeTiled unavailable (driver entry point lookup failed)");
    return JG_ERR_CUDA;
  }
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = fn(map, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): rows=%lld k=%lld ld=%lld", (int)r,
             (long long)rows, (long long)k, (long long)ld);
    return jg::shape_error(buf);
  }
  return JG_OK;
}

// Store map for an epilogue output: dims (cols, rows, batches), 32 x 32 boxes, swizzled to match
// stage_store (128B rows for fp32, 64B rows for bf16).
int make_store_map(CUtensorMap* map, void* ptr, bool bf16, int64_t rows, int64_t cols, int64_t ld, int64_t bstride,
                   int64_t batches) {
  const int es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(batches)};
  cuuint64_t strides[2];
  strides[0] = static_cast<cuuint64_t>(ld) * es;
  strides[1] = batches > 1 ? static_cast<cuuint64_t>(bstride) * es : strides[0] * dims[1];
  if (strides[1] == 0 || strides[1] % 16) strides[1] = ((strides[0] * dims[1] + 15) / 16) * 16;
  cuuint32_t box[3] = {32, 32, 1}, estr[3] = {1, 1, 1};
  auto fn = encode_fn();
  if (!fn) {
    jg::set_error("cuTensorMapEncodeTiled unavailable");
    return JG_ERR_CUDA;
  }
  CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[200];
    snprintf(buf, sizeof(buf), "store tensor map failed (%d): rows=%lld cols=%lld ld=%lld", (int)r, (long long)rows,
             (long long)cols, (long long)ld);
    return jg::shape_error(buf);
  }
  return JG_OK;
}

template <int BN, bool TF32, int CG, bool RS = false>
int launch(GemmParams& p, cudaStream_t stream) {
  using C = Cfg<BN, TF32, CG>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_kernel<BN, TF32, CG, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return jg::cuda_check(attr_err, "cudaFuncSetAttribute(gemm)");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.units * CG);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_kernel<BN, TF32, CG, RS>, p);
  if (e != cudaSuccess) return jg::cuda_check(e, "gemm_kernel launch");
  JG_LAUNCH_CHECK("gemm_kernel");
  return JG_OK;
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

extern "C" int jg_gemm(const jg_gemm_desc* g, void* stream_v) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  JG_SHAPE_CHECK(g != nullptr, "jg_gemm: null descriptor");
  JG_SHAPE_CHECK(g->m > 0 && g->n > 0 && g->k > 0 && g->batch > 0, "jg_gemm: empty problem m=%lld n=%lld k=%lld batch=%lld",
                 (long long)g->m, (long long)g->n, (long long)g->k, (long long)g->batch);
  JG_SHAPE_CHECK(g->m < (1ll << 31) && g->n < (1ll << 31) && g->k < (1ll << 31), "jg_gemm: dimension too large");
  const bool tf32 = g->math == JG_MATH_TF32X3;
  JG_SHAPE_CHECK(g->math == JG_MATH_BF16 || tf32, "jg_gemm: unknown math %d", g->math);
  const int esize = tf32 ? 4 : 2;
  JG_SHAPE_CHECK(g->a && g->b && aligned16(g->a) && aligned16(g->b), "jg_gemm: operands must be 16-byte aligned");
  JG_SHAPE_CHECK((g->lda * esize) % 16 == 0 && (g->ldb * esize) % 16 == 0,
                 "jg_gemm: operand leading dims (%lld, %lld) must be multiples of %d elements", (long long)g->lda,
                 (long long)g->ldb, 16 / esize);
  JG_SHAPE_CHECK((g->a_bstride * esize) % 16 == 0 && (g->b_bstride * esize) % 16 == 0,
                 "jg_gemm: operand batch strides must be multiples of 16 bytes");
  JG_SHAPE_CHECK(g->lda >= (g->a_major == JG_MNMAJOR ? g->m : g->k), "jg_gemm: lda too small");
  JG_SHAPE_CHECK(g->ldb >= (g->b_major == JG_MNMAJOR ? g->n : g->k), "jg_gemm: ldb too small");
  if (tf32) {
    JG_SHAPE_CHECK(g->a_lo && g->b_lo && aligned16(g->a_lo) && aligned16(g->b_lo), "jg_gemm: tf32x3 needs lo parts");
    JG_SHAPE_CHECK(g->a_major == JG_KMAJOR && g->b_major == JG_KMAJOR,
                   "jg_gemm: tf32x3 operands must be K-major (jg_split_tf32_2d transposes)");
  }

  const uint32_t epi = g->epi;
  auto out_ok = [](const void* ptr, int64_t ld, int type) {
    const int es = type == JG_BF16 ? 2 : 4;
    return aligned16(ptr) && (ld * es) % 16 == 0;
  };
  JG_SHAPE_CHECK(g->d == nullptr || out_ok(g->d, g->ldd, g->d_type), "jg_gemm: D must be 16B aligned with ld %% 16B == 0");
  for (int i = 0; i < 8; ++i)
    JG_SHAPE_CHECK(g->d_planes[i] == nullptr || out_ok(g->d_planes[i], g->ldd, g->d_type), "jg_gemm: misaligned d_planes");
  JG_SHAPE_CHECK(!(epi & JG_EPI_ACCUM) || (g->d && g->d_type == JG_F32), "jg_gemm: ACCUM needs an fp32 D");
  JG_SHAPE_CHECK(!(epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) || (g->d2 && out_ok(g->d2, g->ldd2, g->d2_type)),
                 "jg_gemm: GELU_FWD/COPY_D2 need an aligned D2");
  JG_SHAPE_CHECK(!(epi & (JG_EPI_BIAS_COL | JG_EPI_BIAS_ROW)) || g->bias, "jg_gemm: bias flag without bias");
  JG_SHAPE_CHECK(!(epi & JG_EPI_RESID) || (g->resid && out_ok(g->resid, g->ldr, JG_F32)), "jg_gemm: bad resid");
  JG_SHAPE_CHECK(!(epi & JG_EPI_GELU_BWD) || (g->pre && out_ok(g->pre, g->ldp, g->pre_type)), "jg_gemm: bad pre");
  JG_SHAPE_CHECK(!(epi & JG_EPI_STATS) || g->stats, "jg_gemm: STATS without stats buffer");
  JG_SHAPE_CHECK(!(epi & JG_EPI_LNB) || (g->stats && g->lnb_x && g->lnb_gamma && g->lnb_mr && aligned16(g->lnb_x) &&
                                         g->lnb_ldx % 4 == 0 && g->lnb_x_bstride % 4 == 0 && !(epi & JG_EPI_STATS) &&
                                         !(epi & JG_EPI_ADAM)),
                 "jg_gemm: LNB needs stats, an aligned fp32 x (ld %% 4 == 0), gamma and mean/rstd, and no STATS/ADAM");
  JG_SHAPE_CHECK(!(epi & JG_EPI_ADAM) || (g->d && g->d_type == JG_F32 && g->adam_m && g->adam_v && g->adam_step &&
                                          aligned16(g->adam_m) && aligned16(g->adam_v) &&
                                          !(epi & (JG_EPI_ACCUM | JG_EPI_GELU_FWD | JG_EPI_COPY_D2 | JG_EPI_STATS))),
                 "jg_gemm: ADAM needs fp32 D (the master weights), aligned m/v, a step counter, and no other outputs");

  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.m = static_cast<int>(g->m);
  p.n = static_cast<int>(g->n);
  p.k = static_cast<int>(g->k);
  p.batch = static_cast<int>(g->batch);
  p.reduce_batch = g->reduce_batch ? 1 : 0;
  p.a_mn = g->a_major == JG_MNMAJOR;
  p.b_mn = g->b_major == JG_MNMAJOR;
  p.a_batched = g->batch > 1 && g->a_bstride != 0;
  p.b_batched = g->batch > 1 && g->b_bstride != 0;
  const int bk = 128 / esize;
  p.num_kb = static_cast<int>((g->k + bk - 1) / bk);

  // tile width: the widest N tile that still gives at least one full wave of tiles; bf16 problems
  // taller than one 128-row tile run on CTA pairs (cta_group::2, 256-row tiles, B split in two).
  const int64_t out_batches = p.reduce_batch ? 1 : g->batch;
  static const bool no_2sm = getenv("JG_NO_2SM") != nullptr;
  const int cg = (!tf32 && g->m > BM && g->n > 64 && !no_2sm) ? 2 : 1;
  const int64_t mt = (g->m + BM * cg - 1) / (BM * cg);
  int bn = 256;
  if (g->n <= 64) bn = 64;
  else if (g->n <= 128) bn = 128;
  else {
    const int64_t t256 = mt * ((g->n + 255) / 256) * out_batches;
    if (t256 < jg::num_sms() / cg) bn = 128;
  }
  if (g->tile_n != 0) {
    JG_SHAPE_CHECK(g->tile_n == 256 || g->tile_n == 128 || (g->tile_n == 64 && cg == 1),
                   "jg_gemm: tile_n must be 0, 64 (at most 128 rows), 128 or 256");
    bn = g->tile_n;
  }
  p.m_tiles = static_cast<int>(mt);
  p.n_tiles = static_cast<int>((g->n + bn - 1) / bn);
  const int64_t nt = static_cast<int64_t>(p.m_tiles) * p.n_tiles * out_batches;
  JG_SHAPE_CHECK(nt < (1ll << 31), "jg_gemm: too many tiles");
  p.num_tiles = static_cast<int>(nt);
  p.num_pos = p.num_tiles;
  {
    static const int env_cap = getenv("JG_GEMM_SMS") ? atoi(getenv("JG_GEMM_SMS")) : 0;  // experiment only
    const int sm_cap = g->max_sms > 0 ? g->max_sms : env_cap;
    const int sms = (sm_cap >= 2 * cg && sm_cap < jg::num_sms()) ? sm_cap : jg::num_sms();
    const int max_units = sms / cg;
    p.units = p.num_tiles < max_units ? p.num_tiles : max_units;
  }
  p.nwaves = 0;

  p.nseg = tf32 ? 3 : 1;
  const void* as[3] = {g->a, g->a, g->a_lo};
  const void* bs[3] = {g->b, g->b_lo, g->b};
  for (int s = 0; s < p.nseg; ++s) {
    int rc = make_operand_map(&p.tma_a[s], as[s], tf32, p.a_mn, g->m, g->k, g->lda, g->a_bstride,
                              p.a_batched ? g->batch : 1, BM);
    if (rc) return rc;
    rc = make_operand_map(&p.tma_b[s], bs[s], tf32, p.b_mn, g->n, g->k, g->ldb, g->b_bstride,
                          p.b_batched ? g->batch : 1, bn / cg);
    if (rc) return rc;
  }

  p.epi = epi;
  p.alpha = g->alpha;
  p.d = g->d; p.ldd = g->ldd; p.d_bs = g->d_bstride; p.d_bf16 = g->d_type == JG_BF16;
  p.d2 = g->d2; p.ldd2 = g->ldd2; p.d2_bs = g->d2_bstride; p.d2_bf16 = g->d2_type == JG_BF16;
  p.bias = g->bias; p.bias_bs = g->bias_bstride;
  p.resid = g->resid; p.ldr = g->ldr; p.r_bs = g->r_bstride;
  p.pre = g->pre; p.ldp = g->ldp; p.p_bs = g->p_bstride; p.pre_bf16 = g->pre_type == JG_BF16;
  p.stats = g->stats; p.stats_bs = g->stats_bstride;
  p.lnb_x = g->lnb_x; p.lnb_ldx = g->lnb_ldx; p.lnb_x_bs = g->lnb_x_bstride;
  p.lnb_gamma = g->lnb_gamma; p.lnb_mr = g->lnb_mr;
  p.adam_m = g->adam_m; p.adam_v = g->adam_v; p.adam_pbf16 = static_cast<__nv_bfloat16*>(g->adam_pbf16);
  p.adam_step = g->adam_step; p.adam_lr = g->adam_lr; p.adam_b1 = g->adam_beta1; p.adam_b2 = g->adam_beta2;
  p.adam_eps = g->adam_eps;
  p.remote = 0;
  for (int i = 0; i < 8; ++i) {
    p.d_planes[i] = g->d_planes[i];
    if (g->d_planes[i] != nullptr) p.remote = 1;
    p.rs_flag_peers[i] = g->rs_flag_peers[i];
  }
  p.planes = p.remote;
  static const bool plane_major = getenv("JG_PLANE_MAJOR") != nullptr;
  p.plane_minor = plane_major ? 0 : 1;
  const bool rs_has_own = g->rs_flags != nullptr;  // rs_own is meaningful only with a flag array
  p.rs_own = rs_has_own ? g->rs_own : -1;
  p.rs_mode = rs_has_own ? 1 : 0;
  for (int i = 0; i < 8; ++i)
    if (g->rs_flag_peers[i] != nullptr) p.rs_mode = 1;
  p.plane_div = (p.remote && g->plane_div > 0) ? g->plane_div : 0;
  const int64_t nplanes_out = p.plane_div ? g->batch / p.plane_div : g->batch;
  JG_SHAPE_CHECK(!p.plane_div || (g->batch % p.plane_div == 0 && !p.rs_mode && g->d_planes_bstride > 0),
                 "jg_gemm: plane_div needs batch = planes x plane_div, a sample stride, no fused reduce-scatter");
  JG_SHAPE_CHECK(!p.remote || (!g->reduce_batch && nplanes_out <= 8 && !(epi & (JG_EPI_ACCUM | JG_EPI_ADAM))),
                 "jg_gemm: d_planes needs <= 8 independent output planes and no ACCUM/ADAM");
  if (p.rs_mode) {
    JG_SHAPE_CHECK(!g->reduce_batch && g->batch <= 8 && p.rs_own >= -1 && p.rs_own < g->batch && !(epi & (JG_EPI_ACCUM | JG_EPI_ADAM)),
                   "jg_gemm: fused reduce-scatter needs <= 8 independent output batches and no ACCUM/ADAM");
    JG_SHAPE_CHECK(NUM_EPI_WARPS == 8 && static_cast<int64_t>(p.m_tiles) * p.n_tiles * cg * NUM_EPI_WARPS <= g->rs_flag_cap,
                   "jg_gemm: fused reduce-scatter flag array too small (%lld tiles, cap %d)",
                   (long long)p.m_tiles * p.n_tiles, g->rs_flag_cap);
    JG_SHAPE_CHECK(g->rs_part_type == JG_BF16 || g->rs_part_type == JG_F32, "jg_gemm: rs_part_type must be f32 or bf16");
    for (int b = 0; b < static_cast<int>(g->batch); ++b) {
      const bool own = b == p.rs_own;
      JG_SHAPE_CHECK(own ? g->d_planes[b] == nullptr : (g->d_planes[b] != nullptr && g->rs_flag_peers[b] != nullptr),
                     "jg_gemm: fused reduce-scatter batch %d needs %s", b,
                     own ? "no d_planes entry (own plane)" : "a d_planes entry and a peer flag array");
    }
    if (p.rs_own >= 0)
      JG_SHAPE_CHECK(g->d != nullptr && g->rs_src != nullptr && g->rs_nsrc >= 1 &&
                         g->rs_nsrc <= 8 && g->rs_src_idx >= 0 && g->rs_src_idx < g->rs_nsrc && g->rs_need >= 0 &&
                         aligned16(g->rs_src) && (g->rs_src_stride * (g->rs_part_type == JG_BF16 ? 2 : 4)) % 16 == 0,
                     "jg_gemm: fused reduce-scatter own plane needs D, flags and an aligned partial-plane source");
  }
  p.rs_flags = g->rs_flags;
  p.rs_src = g->rs_src;
  p.rs_src_stride = g->rs_src_stride;
  p.rs_part_bf16 = g->rs_part_type == JG_BF16;
  p.rs_nsrc = g->rs_nsrc;
  p.rs_src_idx = g->rs_src_idx;
  p.rs_need = g->rs_need;
  static const int rs_dbg = getenv("JG_RS_DBG") ? atoi(getenv("JG_RS_DBG")) : 0;
  p.rs_dbg = rs_dbg;
  static const bool rs_linear = getenv("JG_RS_LINEAR") != nullptr;
  if (p.rs_own >= 0 && p.batch >= 2 && !rs_linear) {
    // head of nr + 1 remote waves, then (own wave, nr remote waves) cycles; leftovers at the end
    const int64_t T = static_cast<int64_t>(p.m_tiles) * p.n_tiles, U = p.units, nr = p.batch - 1;
    const int64_t wo = (T + U - 1) / U, wr = (nr * T + U - 1) / U;
    if (wo + wr <= 64) {
      int64_t io = 0, ir = 0, w = 0;
      auto push = [&](int kind, int64_t idx) {
        p.wave_kind[w] = static_cast<uint8_t>(kind);
        p.wave_idx[w] = static_cast<uint8_t>(idx);
        ++w;
      };
      for (; ir < wr && ir < nr + 1; ++ir) push(0, ir);
      while (io < wo || ir < wr) {
        if (io < wo) push(1, io++);
        for (int64_t j = 0; j < nr && ir < wr; ++j) push(0, ir++);
      }
      p.nwaves = static_cast<int>(w);
      p.num_pos = static_cast<int>(w * U);
    }
  }
  // TMA-store epilogue whenever D is write-only (no read-modify-write of D)
  p.tma_store = !(epi & (JG_EPI_ACCUM | JG_EPI_ADAM)) && (g->d != nullptr || p.remote);
  JG_SHAPE_CHECK(!p.rs_mode || p.tma_store, "jg_gemm: fused reduce-scatter needs the TMA-store epilogue");
  JG_SHAPE_CHECK(!p.rs_mode || !(epi & JG_EPI_LNB), "jg_gemm: LNB is not supported with a fused reduce-scatter");
  if (p.tma_store) {
    const bool dbf = g->d_type == JG_BF16;
    // per-output-batch maps (d_planes / fused reduce-scatter) address one plane each (batch 0)
    const int64_t eb_batches = p.rs_mode ? 1 : out_batches;
    if (p.rs_mode) {
      for (int b = 0; b < static_cast<int>(out_batches); ++b) {
        const bool own = b == p.rs_own;
        p.dmap_bf16[b] = own ? dbf : p.rs_part_bf16;
        int rc = make_store_map(&p.tma_d[b], own ? g->d : g->d_planes[b], p.dmap_bf16[b], g->m, g->n, g->ldd, 0, 1);
        if (rc) return rc;
      }
    } else if (p.remote && p.plane_div) {
      for (int b = 0; b < static_cast<int>(nplanes_out); ++b) {
        JG_SHAPE_CHECK(g->d_planes[b] != nullptr, "jg_gemm: plane_div needs every d_planes entry");
        p.dmap_bf16[b] = dbf;
        int rc = make_store_map(&p.tma_d[b], g->d_planes[b], dbf, g->m, g->n, g->ldd, g->d_planes_bstride, p.plane_div);
        if (rc) return rc;
      }
    } else if (p.remote) {
      for (int b = 0; b < static_cast<int>(out_batches); ++b) {
        p.dmap_bf16[b] = dbf;
        int rc = make_store_map(&p.tma_d[b], g->d_planes[b] ? g->d_planes[b] : g->d, dbf, g->m, g->n, g->ldd, 0, 1);
        if (rc) return rc;
      }
    } else {
      p.dmap_bf16[0] = dbf;
      int rc = make_store_map(&p.tma_d[0], g->d, dbf, g->m, g->n, g->ldd, g->d_bstride, out_batches);
      if (rc) return rc;
    }
    if (epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) {
      int rc = make_store_map(&p.tma_d2, g->d2, g->d2_type == JG_BF16, g->m, g->n, g->ldd2, g->d2_bstride, eb_batches);
      if (rc) return rc;
    }
    p.nb_d = (p.remote && !p.rs_mode) ? 0 : g->d_bcast.n;
    p.nb_d2 = (epi & (JG_EPI_GELU_FWD | JG_EPI_COPY_D2)) ? g->d2_bcast.n : 0;
    JG_SHAPE_CHECK(p.nb_d >= 0 && p.nb_d <= 4 && p.nb_d2 >= 0 && p.nb_d2 <= 4, "jg_gemm: at most 4 broadcast targets");
    for (int i = 0; i < p.nb_d; ++i) {
      int rc = make_store_map(&p.tma_dx[i], g->d_bcast.ptr[i], dbf, g->m, g->n, g->ldd, g->d_bstride, eb_batches);
      if (rc) return rc;
    }
    for (int i = 0; i < p.nb_d2; ++i) {
      int rc = make_store_map(&p.tma_d2x[i], g->d2_bcast.ptr[i], g->d2_type == JG_BF16, g->m, g->n, g->ldd2,
                              g->d2_bstride, eb_batches);
      if (rc) return rc;
    }
  } else {
    JG_SHAPE_CHECK(g->d_bcast.n == 0 && g->d2_bcast.n == 0, "jg_gemm: broadcast outputs need a write-only D");
  }
  if (p.nb_d || p.nb_d2) p.remote = 1;  // system fence at the end: peers read after the barrier

  JG_SHAPE_CHECK(!(tf32 && p.rs_mode), "jg_gemm: fused reduce-scatter is bf16 only");
  if (tf32) {
    if (bn == 256) return launch<256, true, 1>(p, stream);
    if (bn == 128) return launch<128, true, 1>(p, stream);
    return launch<64, true, 1>(p, stream);
  }
  if (p.rs_mode) {  // fused reduce-scatter variant (bf16 only; rs code compiled out of the others)
    if (cg == 2) {
      if (bn == 256) return launch<256, false, 2, true>(p, stream);
      return launch<128, false, 2, true>(p, stream);
    }
    if (bn == 256) return launch<256, false, 1, true>(p, stream);
    if (bn == 128) return launch<128, false, 1, true>(p, stream);
    return launch<64, false, 1, true>(p, stream);
  }
  if (cg == 2) {
    if (bn == 256) return launch<256, false, 2>(p, stream);
    return launch<128, false, 2>(p, stream);
  }
  if (bn == 256) return launch<256, false, 1>(p, stream);
  if (bn == 128) return launch<128, false, 1>(p, stream);
  return launch<64, false, 1>(p, stream);
}
