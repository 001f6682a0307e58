// Router of Eq. 2 on the 5th-generation tensor cores, sm_100a (row f4).
//
//   z = uᵀ W_r (u ∈ R^D, W_r ∈ R^{D×N}),  s = softmax(z) over all N experts,
//   ids = the K largest s (descending, ties -> lower id; R31/R32),  gates = s[ids].
//
// One persistent kernel per call; per 128-token tile:
//   warp 0      TMA producer: token tile [128 x 64] (evict-first: streamed once) + the router weight
//               [Npad x 64] (evict-last: every tile re-reads it from L2), 128-byte swizzle
//   warp 1      TMEM allocator + warp-converged tcgen05.mma issue (M=128, N=box, K=16 steps)
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

#include "common.cuh"
#include "tc.cuh"

namespace llep {

namespace {

constexpr int RBM = 128;                 // token rows per tile (= TMEM lanes)
constexpr int RBK = 64;                  // K per stage (one 128-byte swizzle row)
constexpr int kRouterThreads = 192;
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

__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap *map, uint32_t bar,
                                                 int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
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

// warp-converged issue: the whole warp runs the loop, one elected lane issues
__device__ __forceinline__ void mma_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

// KMAX = K exactly when EXACT (K <= 8), else an upper bound with runtime K (K in 9..16)
// NB = weight boxes (MMAs) per K step: 1 for N <= 256, 2 above
template <int KMAX, bool EXACT, int NB>
__global__ void __launch_bounds__(kRouterThreads, 1) router_kernel(const __grid_constant__ RouterParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  constexpr int A_BYTES = RBM * RBK * 2;
  const int B_BYTES = NB * p.box_rows * 128;
  const int STAGE = A_BYTES + B_BYTES;
  const int S = p.stages;
  uint8_t *sA = smem;
  uint8_t *sB = smem + S * A_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * STAGE);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(tfull + i), 1);
      mbar_init(smem_u32(tempty + i), 4);        // 4 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmW)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nk = (p.d_model + RBK - 1) / RBK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      const uint64_t pol_x = policy_evict_first(), pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fb = smem_u32(full + stage);
          mbar_expect_tx(fb, STAGE);
          tma_load_2d_hint(smem_u32(sA + stage * A_BYTES), &p.tmX, fb, kb * RBK, t * RBM, pol_x);
#pragma unroll
          for (int c = 0; c < NB; ++c)
            tma_load_2d_hint(smem_u32(sB + stage * B_BYTES + c * p.box_rows * 128), &p.tmW, fb, kb * RBK,
                             c * p.box_rows, pol_w);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------------- MMA issue (whole warp)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.box_rows >> 3) << 17) |
                           ((uint32_t)(RBM >> 4) << 24);
    const uint64_t adesc0 = smem_desc(smem_u32(sA)), bdesc0 = smem_desc(smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
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
            mma_w(d_tmem + c * p.box_rows, ad + (uint32_t)(kk * 2),
                  bd + (uint32_t)((c * p.box_rows * 128 + kk * 32) >> 4), idesc, (kb | kk) != 0);
        commit_w(smem_u32(empty + stage));
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      commit_w(smem_u32(tfull + acc));
    }
  } else {
    // -------------------------------------------------------------------- epilogue: softmax top-K
    const int q = warp & 3;                      // TMEM lanes q*32 .. q*32+31
    const int N = p.n_experts, K = p.top_k;
    int it = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
      const int acc = p.nacc == 2 ? (it & 1) : 0;
      const uint32_t aphase = p.nacc == 2 ? ((it >> 1) & 1) : (it & 1);
      mbar_wait(smem_u32(tfull + acc), aphase);
      tc_fence_after();
      const int64_t row = (int64_t)t * RBM + q * 32 + lane;
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
      // one pass over the logits in 64-column chunks (two x32 TMEM loads, one wait): running max
      // with the sum rescaled once per chunk (online softmax), and the top-K by logit (softmax is
      // monotone in z)
      for (int j = 0; j < N; j += 64) {
        float v[64];
        tmem_ld32(taddr + j, v);
        tmem_ld32(taddr + j + 32, v + 32);
        tmem_ld_wait();
        float cm = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (j + i < N) cm = fmaxf(cm, v[i]);
        const float nm = fmaxf(mx, cm);
        sum *= expf(mx - nm);          // 0 on the first chunk (exp(-inf) = 0)
        mx = nm;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int e = j + i;
          if (e < N) {
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
      if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      if (row_ok) {
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
          if (r < K) {
            p.ids[row * K + r] = ti[r];
            p.gates[row * K + r] = __fdiv_rn(expf(tv[r] - mx), sum);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
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
  kern<<<grid, kRouterThreads, smem, s>>>(prm);
  LLEP_CUDA(cudaGetLastError());
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
  const int stage = RBM * RBK * 2 + prm.n_box * prm.box_rows * 128;
  const int extra = 1024 + 256;
  prm.stages = (kRouterSmemBudget - extra) / stage;
  if (prm.stages > 8) prm.stages = 8;
  const int smem = prm.stages * stage + extra;
  if (!tma_map_kmajor(&prm.tmX, a.x, a.n_tokens, a.d_model, RBM) ||
      !tma_map_kmajor(&prm.tmW, a.w_router, a.n_experts, a.d_model, prm.box_rows)) {
    set_error("cuTensorMapEncodeTiled failed for the router (d_model %% 8 == 0, 16-byte aligned bases)");
    return LLEP_ERR_CUDA;
  }
  const int64_t tiles = (a.n_tokens + RBM - 1) / RBM;
  prm.n_tiles = (int32_t)tiles;
  prm.n_tokens = a.n_tokens;
  prm.d_model = a.d_model;
  prm.n_experts = a.n_experts;
  prm.top_k = a.top_k;
  prm.ids = a.ids;
  prm.gates = a.gates;
  prm.logits = a.logits;
  const int grid = (int)(tiles < a.num_sms ? tiles : a.num_sms);
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
