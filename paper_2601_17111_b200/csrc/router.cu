// Router of Eq. 2 on the 5th-generation tensor cores, sm_100a (row f4).
//
//   z = uᵀ W_r (u ∈ R^D, W_r ∈ R^{D×N}),  s = softmax(z) over all N experts,
//   ids = the K largest s (descending, ties -> lower id; R31/R32),  gates = s[ids].
//
// One persistent kernel per call on CTA pairs (cta_group::2, clusters of 2); per 256-token tile:
//   warp 0      TMA producer (both CTAs): its 128 token rows [128 x 64] (evict-first: streamed once)
//               + HALF of the router weight box [Npad/2 x 64] (evict-last: every tile re-reads it
//               from L2), 128-byte swizzle; both CTAs' loads complete on the leader's barrier
//   warp 1      TMEM allocator; in the leader CTA the warp-converged tcgen05.mma issue (M=256 over
//               the pair, N=box, K=16 steps) -- the pair halves the weight bytes each SM stages and
//               reads per token, the shared-memory traffic that bounded the 1-CTA version
//   warps 2-5   epilogue, one token row per thread, one pass over the fp32 logits in TMEM (64
//               columns per wait): online softmax (running max, Σ exp rescaled per chunk) and a
//               branch-free register top-K insertion; gates = exp(z - max) / Σ.
// The logits never touch HBM (optional debug copy).  The whole call is bound by reading the tokens
// once (2·D bytes per token): the contraction is 2·N·D FLOP per token, i.e. N FLOP/byte — below
// the tensor/HBM ridge for every N this supports (≤ 512).
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

namespace llep {

namespace {

constexpr int RBM = 128;                 // token rows per tile (= TMEM lanes)
constexpr int RBK = 64;                  // K per stage (one 128-byte swizzle row)
constexpr int kRouterThreads = 320;     // producer, MMA, 8 epilogue warps (2 per TMEM lane quarter)
constexpr int kRouterSmemBudget = 227 * 1024;

struct RouterParams {
  CUtensorMap tmX;     // tokens [B, D] bf16
  CUtensorMap tmW;     // router weight [N, D] bf16 (row i = column i of W_r)
  int32_t n_tiles, d_model, n_experts, top_k;
  int32_t box_rows, n_box, stages, nacc, acc_cols;
  int64_t n_tokens;
  int32_t *ids;
  float *gates;
  float *logits;       // [B, N] or null
};

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 32 consecutive fp32 TMEM columns of this thread's lane (no wait)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// KMAX = K exactly when EXACT (K <= 8), else an upper bound with runtime K (K in 9..16)
// NB = weight boxes (MMAs) per K step: 1 for N <= 256, 2 above
template <int KMAX, bool EXACT, int NB>
__global__ void __launch_bounds__(kRouterThreads, 1) router_kernel(const __grid_constant__ RouterParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  constexpr int A_BYTES = RBM * RBK * 2;
  const int HB = p.box_rows / 2;                 // weight rows per box staged by each CTA of the pair
  const int B_BYTES = NB * HB * 128;
  const int STAGE = A_BYTES + B_BYTES;
  const int S = p.stages;
  uint8_t *sA = smem;
  uint8_t *sB = smem + S * A_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * STAGE);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(tfull + i), 1);
      mbar_init(smem_u32(tempty + i), 16);       // 8 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmW)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nk = (p.d_model + RBK - 1) / RBK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      const uint64_t pol_x = policy_evict_first(), pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < p.n_tiles; t += n_pairs) {
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fl = smem_u32(full + stage);
          if (leader) mbar_expect_tx(fl, 2 * STAGE);   // both CTAs' loads complete on the leader
          const uint32_t fb = mapa_shared(fl, 0);
          tma_load_2d_pair(smem_u32(sA + stage * A_BYTES), &p.tmX, fb, kb * RBK, t * 2 * RBM + (int)crank * RBM,
                           pol_x);
#pragma unroll
          for (int c = 0; c < NB; ++c)
            tma_load_2d_pair(smem_u32(sB + stage * B_BYTES + c * HB * 128), &p.tmW, fb, kb * RBK,
                             c * p.box_rows + (int)crank * HB, pol_w);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------------ MMA issue (leader warp)
      // M=256 over the pair (128 token rows per CTA), N=box (each CTA stages half of each box)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.box_rows >> 3) << 17) |
                             ((uint32_t)((2 * RBM) >> 4) << 24);
      const uint64_t adesc0 = smem_desc(smem_u32(sA)), bdesc0 = smem_desc(smem_u32(sB));
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < p.n_tiles; t += n_pairs, ++it) {
        const int acc = p.nacc == 2 ? (it & 1) : 0;
        const uint32_t aphase = p.nacc == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(smem_u32(tempty + acc), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * p.acc_cols;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          __syncwarp();
          const uint64_t ad = adesc0 + (uint32_t)((stage * A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + (uint32_t)((stage * B_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < RBK / 16; ++kk)
#pragma unroll
            for (int c = 0; c < NB; ++c)
              tc_mma_pair_w(d_tmem + c * p.box_rows, ad + (uint32_t)(kk * 2),
                            bd + (uint32_t)((c * HB * 128 + kk * 32) >> 4), idesc, (kb | kk) != 0);
          tc_commit_pair_w(smem_u32(empty + stage));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair_w(smem_u32(tfull + acc));
      }
    }
  } else {
    // -------------------------------------------------------------------- epilogue: softmax top-K
    // 8 warps: warp w reads TMEM lanes 32*(w % 4) .. +31 (its rows) and column half h = (w-2) / 4:
    // h = 0 -> experts [0, C0), h = 1 -> [C0, N).  Each computes its half's max, Σ exp and top-K;
    // h = 1 hands its partial to h = 0 through shared memory, which merges and writes the row.
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int N = p.n_experts, K = p.top_k;
    const int C0 = ((N + 1) / 2 + 31) / 32 * 32;
    const int j0 = h == 0 ? 0 : C0, j1 = h == 0 ? (C0 < N ? C0 : N) : N;
    constexpr int STR = 2 + 2 * KMAX + 1;         // partial record stride (odd: no bank conflicts)
    float *xp = reinterpret_cast<float *>(smem + S * STAGE + 256) + (q * 32 + lane) * STR;
    int it = 0;
    for (int t = pair; t < p.n_tiles; t += n_pairs, ++it) {
      const int acc = p.nacc == 2 ? (it & 1) : 0;
      const uint32_t aphase = p.nacc == 2 ? ((it >> 1) & 1) : (it & 1);
      mbar_wait(smem_u32(tfull + acc), aphase);
      tc_fence_after();
      const int64_t row = (int64_t)t * 2 * RBM + (int64_t)crank * RBM + q * 32 + lane;
      const bool row_ok = row < p.n_tokens;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * p.acc_cols;
      float tv[KMAX];
      int ti[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        tv[i] = -INFINITY;
        ti[i] = 0;
      }
      float mx = -INFINITY, last = -INFINITY, sum = 0.f;
      // one pass over this half's logits in 64-column chunks (two x32 TMEM loads, one wait):
      // running max with the sum rescaled once per chunk (online softmax), and the top-K by
      // logit (softmax is monotone in z)
      for (int j = j0; j < j1; j += 64) {
        float v[64];
        tmem_ld32(taddr + j, v);
        tmem_ld32(taddr + j + 32, v + 32);
        tmem_ld_wait();
        float cm = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (j + i < j1) cm = fmaxf(cm, v[i]);
        const float nm = fmaxf(mx, cm);
        sum *= expf(mx - nm);          // 0 on the first chunk (exp(-inf) = 0)
        mx = nm;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int e = j + i;
          if (e < j1) {
            const float z = v[i];
            if (p.logits && row_ok) p.logits[row * N + e] = z;
            sum += expf(z - mx);
            if (z > last) {            // strictly greater: an equal later id never displaces
              // branch-free insertion into the descending list (positions are compile-time, so
              // tv / ti stay in registers): entry r takes entry r-1 if z beats that one, else z
              // if z beats entry r
#pragma unroll
              for (int r = KMAX - 1; r >= 1; --r) {
                if (EXACT || r < K) {
                  const bool up = z > tv[r - 1], here = z > tv[r];
                  tv[r] = up ? tv[r - 1] : (here ? z : tv[r]);
                  ti[r] = up ? ti[r - 1] : (here ? e : ti[r]);
                }
              }
              if (z > tv[0]) {
                tv[0] = z;
                ti[0] = e;
              }
              if (EXACT) {
                last = tv[KMAX - 1];
              } else {
#pragma unroll
                for (int r = 0; r < KMAX; ++r)
                  if (r == K - 1) last = tv[r];
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty + acc), 0));
      __syncwarp();   // reconverge: named barriers (bar.sync) that follow require converged warps
      if (h == 1) {
        if (it > 0) asm volatile("barrier.sync 2, 256;" ::: "memory");   // h = 0 has read the last one
        xp[0] = mx;
        xp[1] = sum;
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
          xp[2 + r] = tv[r];
          xp[2 + KMAX + r] = __int_as_float(ti[r]);
        }
        asm volatile("barrier.sync 1, 256;" ::: "memory");
      } else {
        // the two column halves meet at named barriers from different code locations: the
        // non-.aligned barrier forms (bar.sync / bar.arrive are .aligned: one instruction per barrier)
        asm volatile("barrier.sync 1, 256;" ::: "memory");
        const float m1 = xp[0], s1 = xp[1];
        float bv[KMAX];
        int bi[KMAX];
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
          bv[r] = xp[2 + r];
          bi[r] = __float_as_int(xp[2 + KMAX + r]);
        }
        asm volatile("barrier.arrive 2, 256;" ::: "memory");
        // merge: softmax sums at the common max; top-K of two descending lists (on equal values
        // the first half -- lower expert ids -- goes first)
        const float m = fmaxf(mx, m1);
        const float tot = (mx == -INFINITY ? 0.f : sum * expf(mx - m)) + (m1 == -INFINITY ? 0.f : s1 * expf(m1 - m));
        if (row_ok) {
          int a = 0, b = 0;
#pragma unroll
          for (int r = 0; r < KMAX; ++r) {
            if (r < K) {
              float va = -INFINITY, vb = -INFINITY;
              int ia = 0, ib = 0;
#pragma unroll
              for (int k = 0; k < KMAX; ++k) {
                if (k == a) { va = tv[k]; ia = ti[k]; }
                if (k == b) { vb = bv[k]; ib = bi[k]; }
              }
              const bool takeb = vb > va;
              const float z = takeb ? vb : va;
              const int e = takeb ? ib : ia;
              a += takeb ? 0 : 1;
              b += takeb ? 1 : 0;
              p.ids[row * K + r] = e;
              p.gates[row * K + r] = __fdiv_rn(expf(z - m), tot);
            }
          }
        }
      }
    }
    if (h == 1 && it > 0) asm volatile("barrier.sync 2, 256;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                 : "memory");
}

template <int KMAX, bool EXACT>
llep_status launch_router(RouterParams &prm, int grid, int smem, cudaStream_t s) {
  auto kern = prm.n_box == 1 ? router_kernel<KMAX, EXACT, 1> : router_kernel<KMAX, EXACT, 2>;
  static int smem_set[2] = {0, 0};
  if (smem > smem_set[prm.n_box - 1]) {
    LLEP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    smem_set[prm.n_box - 1] = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kRouterThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LLEP_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  return LLEP_OK;
}

}  // namespace

llep_status run_router(const RouterArgs &a, cudaStream_t s) {
  if (a.n_tokens == 0) return LLEP_OK;
  RouterParams prm;
  memset(&prm, 0, sizeof(prm));
  // MMA N per weight box: <= 256, a multiple of 16; the rows past N read as zeros (TMA OOB fill)
  const int n16 = (a.n_experts + 15) / 16 * 16;
  prm.n_box = (n16 + 255) / 256;
  prm.box_rows = ((n16 + prm.n_box - 1) / prm.n_box + 15) / 16 * 16;
  const int npad = prm.n_box * prm.box_rows;
  prm.nacc = npad <= 256 ? 2 : 1;
  prm.acc_cols = npad <= 256 ? 256 : 512;
  const int stage = RBM * RBK * 2 + prm.n_box * (prm.box_rows / 2) * 128;   // per CTA of a pair
  const int kmax = a.top_k <= 8 ? a.top_k : 16;
  const int extra = 1024 + 256 + 128 * (2 + 2 * kmax + 1) * 4;   // + the column-half partials
  prm.stages = (kRouterSmemBudget - extra) / stage;
  if (prm.stages > 8) prm.stages = 8;
  const int smem = prm.stages * stage + extra;
  if (!tma_map_kmajor(&prm.tmX, a.x, a.n_tokens, a.d_model, RBM) ||
      !tma_map_kmajor(&prm.tmW, a.w_router, a.n_experts, a.d_model, prm.box_rows / 2)) {
    set_error("cuTensorMapEncodeTiled failed for the router (d_model %% 8 == 0, 16-byte aligned bases)");
    return LLEP_ERR_CUDA;
  }
  const int64_t tiles = (a.n_tokens + 2 * RBM - 1) / (2 * RBM);   // 256-token pair tiles
  prm.n_tiles = (int32_t)tiles;
  prm.n_tokens = a.n_tokens;
  prm.d_model = a.d_model;
  prm.n_experts = a.n_experts;
  prm.top_k = a.top_k;
  prm.ids = a.ids;
  prm.gates = a.gates;
  prm.logits = a.logits;
  // as few CTA pairs as give every pair the same number of tiles (128 tiles at G120: 64 pairs x 2
  // instead of 74 pairs with 54 doing a second tile): -2 % at G120, -3.4 % at Q3 (router_bench A/B)
  int pairs = (int)(tiles < a.num_sms / 2 ? tiles : a.num_sms / 2);
  if (pairs > 0) {
    const int64_t waves = (tiles + pairs - 1) / pairs;
    pairs = (int)((tiles + waves - 1) / waves);
  }
  const int grid = 2 * pairs;
  switch (a.top_k) {
    case 1: return launch_router<1, true>(prm, grid, smem, s);
    case 2: return launch_router<2, true>(prm, grid, smem, s);
    case 3: return launch_router<3, true>(prm, grid, smem, s);
    case 4: return launch_router<4, true>(prm, grid, smem, s);
    case 5: return launch_router<5, true>(prm, grid, smem, s);
    case 6: return launch_router<6, true>(prm, grid, smem, s);
    case 7: return launch_router<7, true>(prm, grid, smem, s);
    case 8: return launch_router<8, true>(prm, grid, smem, s);
    default: return launch_router<16, false>(prm, grid, smem, s);
  }
}

}  // namespace llep
