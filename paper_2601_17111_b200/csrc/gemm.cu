// Grouped expert GEMMs on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// The expert FFN is the dense part of the layer (a8/a9; T_local of §3.2).  The paper
// ran it as a cuBLAS loop or a Triton grouped GEMM (F-gemm P:1127); here ONE persistent
// kernel per projection walks every (group, 128-row block, N tile) of this device:
//   warp 0      TMA producer: A tile [128 x 64] + B tile [BN x 64] per stage, 128-byte swizzle
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16 steps)
//   warps 2-5   epilogue: tcgen05.ld of the fp32 accumulator, fused activation, bf16 stores
// Accumulators are double-buffered in TMEM (2 x 256 columns) so the epilogue of tile i overlaps
// the MMAs of tile i+1.  Epilogues:
//   mode 0 (GEMM1 + SwiGLU): the B tile stacks BN/2 rows of W_gate over the matching BN/2 rows
//     of W_up (two TMA boxes), so one accumulator tile holds both halves of each output column:
//     A[r, n] = silu(acc[r, n]) * acc[r, BN/2 + n]   (no [n, 2H] intermediate in HBM)
//   mode 1 (GEMM2 + gate): Y[r, n] = gate[r] * acc[r, n]   (Ĥ = Ĝ ⊙ B̂W)
//   mode 2 (backward recompute): raw [g | u] rows;  mode 3 (training forward): mode 0 + mode 2 stores
// Groups start at 128-aligned rows, so an M tile never straddles two experts; rows past a
// group's end are computed on padding and masked at the store.
// The default kernels are the CTA-pair versions (grouped_gemm_2cta_kernel, cta_group::2, groups
// 256-row aligned): M=256 tiles, M=128 pair MMAs for blocks with <= 128 rows left, and SWAPPED tiles
// for groups of <= 64 rows (D = W·Xᵀ: M=256 over weight rows, N=64 over the group's tokens, three
// K sub-tiles per stage) -- at P=1 those are the cold experts, whose cost is streaming their weights
// (bounded by the ~60-70 GB/s of HBM ingest one SM sustains, profiles/r02_cold_stream_limit.txt).
// Producers wait per foreign group for its weight flag and per m-block for the dispatch arrival flags
// of the sources of its rows (row f2), so GEMM1 starts before the slowest peer has finished sending.
// A/B-only variants of the pair kernel: MC = 2 (LLEP_GEMM_MC=2: two pairs per cluster sharing the
// activation tile by TMA multicast) and the TMA gather4 of this rank's own rows (LLEP_GATHER=1); both
// are bit-identical and measured slower.
// Backward GEMMs (gemm_bwd_*_kernel, row f1) follow at the end of the file.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "tc.cuh"

#ifndef LLEP_SWAP_K
#define LLEP_SWAP_K 3   // K sub-tiles per stage of a swapped tile (A/B: -DLLEP_SWAP_K=2)
#endif

namespace llep {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;                 // 64 bf16 = 128 bytes = one swizzle row
constexpr int kGemmThreads = 192;
constexpr int kAccCols = 256;          // TMEM columns per accumulator buffer
constexpr int kSmemBudget = 227 * 1024;

struct GemmParams {
  CUtensorMap tmA;     // activations [rows, kdim]
  CUtensorMap tmW0;    // native weights [n_native * wrows, kdim]
  CUtensorMap tmW1;    // foreign weights [n_foreign * wrows, kdim]
  CUtensorMap tmAs;    // pair kernel, swapped tiles: activations, 32-row boxes (the N operand)
  CUtensorMap tmW0s;   //   native weights, 64-row boxes (the M operand)
  CUtensorMap tmW1s;   //   foreign weights, 64-row boxes
  int32_t swap;        // pair kernel: groups of <= 64 rows run as swapped tiles (weights x tokens)
  const Group *groups;
  const int32_t *sched;
  const int32_t *n_groups_dev;
  int32_t n_groups_host;
  int32_t kdim, nout, wrows, n_ntiles, wup_off;
  const float *gate;
  __nv_bfloat16 *out;
  const uint32_t *wflags;
  const uint32_t *ep;    // device epochs (common.cuh): weights landed at ep[kEpWeight], rows at ep[kEpArrive]
  int32_t *err;
  const uint32_t *arrive;
  const uint32_t *mblk_src;
  uint32_t src_all;      // every source rank (0: unknown)
  const int32_t *row_src;
  uint16_t *const *peer_slot;
  __nv_bfloat16 *out2;   // mode 3: raw [g | u] pre-activations, rows of 2 * nout (training forward)
  CUtensorMap tmXg;      // pair kernel, modes 0/3: the caller's tokens [xg_rows, kdim], {64 x 1} boxes
  const int32_t *rtok;   //   token row of each receive row of a gathered m-block (nullptr: no gather)
  int32_t xg_rows;
  uint32_t self_mask;    //   m-blocks with mblk_src == self_mask (all rows from this rank) are gathered
};

// Row f2: wait until foreign slot f's weights have landed (flag published by the native device
// with release semantics after its copy-engine push), then order the TMA reads after it.
// Bounded like the device barriers: after ~20 s (or once another wait / barrier of this rank has
// failed, err[1] != 0) it gives up and flags err[1] |= 16 (LLEP_ERR_COMM at the next check), so a peer
// that returned early cannot hang this GPU.
__device__ __forceinline__ void wait_weights(const GemmParams &p, int wslot, uint32_t wepoch) {
  if (wslot >= 0 || !p.wflags) return;
  const uint32_t *f = p.wflags + (-1 - wslot);
  uint32_t v;
  const long long t0 = clock64();
  long long spins = 0;
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if ((int32_t)(v - wepoch) >= 0) break;
    if (((++spins) & 255) == 0) {
      if (p.err && *reinterpret_cast<volatile int32_t *>(p.err + 1) != 0) break;
      if (clock64() - t0 > 40000000000LL) {
        if (p.err) atomicOr(p.err + 1, 16);
        break;
      }
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Row f2: the dispatch is overlapped with the GEMMs.  Before the first TMA load of an m-block's
// activation rows, wait until every source rank that dispatched rows into that block has published
// its arrival flag (release after all its rows were stored, route.cu dispatch_kernel), then order the
// async-proxy (TMA) reads after the acquire.  Bounded like wait_weights.
__device__ __forceinline__ void wait_sources(const GemmParams &p, int mblk, uint32_t &seen, uint32_t aepoch) {
  if (!p.arrive || (p.src_all && (seen & p.src_all) == p.src_all)) return;   // no per-tile lookup then
  uint32_t need = p.mblk_src[mblk] & ~seen;
  if (!need) return;
  const long long t0 = clock64();
  long long spins = 0;
  while (need) {
    const int q = __ffs(need) - 1;
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.arrive + q) : "memory");
    if ((int32_t)(v - aepoch) >= 0) {
      need &= need - 1;
      seen |= 1u << q;
      continue;
    }
    if (((++spins) & 255) == 0) {
      if (p.err && *reinterpret_cast<volatile int32_t *>(p.err + 1) != 0) break;
      if (clock64() - t0 > 40000000000LL) {
        if (p.err) atomicOr(p.err + 1, 32);
        break;
      }
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EXTRA = 1024 + 256 + (kMaxGroups + 1) * 4;
  static constexpr int STAGES_RAW = (kSmemBudget - EXTRA) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE + EXTRA;
  static_assert(B_BYTES % 1024 == 0, "B tile must keep 1024-byte swizzle alignment");
  static_assert(STAGES >= 2, "pipeline too shallow");
};

// ------------------------------------------------------------------------ PTX wrappers
// instruction descriptor: bf16 A/B, fp32 D, both K-major, M=128, N=BN
template <int BN>
__device__ __forceinline__ uint32_t instr_desc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

struct TileInfo {
  int row0, row_end, nb, wslot, small;
  int mblk;   // m-block index in group order (Group.mblk_start + m)
  int half;   // pair kernel: <= 128 rows left in this block -> M=128 pair MMA (64 rows per CTA)
  int swap;   // pair kernel: <= 64 rows -> swapped tile, D[weight rows x tokens] (M=256, N=64)
};

template <int TM = BM>
__device__ __forceinline__ TileInfo decode_tile(int t, int n_ntiles, const int *s_mblk,
                                                int n_groups, const Group *groups,
                                                const int32_t *sched) {
  TileInfo ti;
  const int mb = t / n_ntiles;
  ti.nb = t - mb * n_ntiles;
  int lo, m;
  if (sched) {                    // interleaved m-block order from the layout step
    const int32_t e = __ldg(sched + mb);
    lo = e >> 20;
    m = e & 0xFFFFF;
  } else {                        // group order: last g with s_mblk[g] <= mb
    lo = 0;
    int hi = n_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_mblk[mid] <= mb) lo = mid;
      else hi = mid - 1;
    }
    m = mb - s_mblk[lo];
  }
  const Group g = groups[lo];
  ti.mblk = g.mblk_start + m;
  ti.row0 = g.row_base + m * TM;
  ti.row_end = g.row_base + g.n_rows;
  ti.wslot = g.wslot;
  ti.small = g.n_rows <= kSmallGroupRows;  // its weights are streamed once: evict first from L2
  ti.half = ti.row_end - ti.row0 <= TM / 2;
  ti.swap = 0;
  return ti;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1) grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  using C = Cfg<BN>;
  constexpr int S = C::STAGES;
  constexpr int BNO = MODE != 1 ? BN / 2 : BN;   // output columns per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + S * C::A_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * C::STAGE);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
  int *s_mblk = reinterpret_cast<int *>(smem + S * C::STAGE + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_groups = p.n_groups_dev ? *p.n_groups_dev : p.n_groups_host;
  for (int g = threadIdx.x; g < n_groups; g += kGemmThreads) s_mblk[g] = p.groups[g].mblk_start;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(tfull + i), 1);
      mbar_init(smem_u32(tempty + i), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmW0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmW1)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kAccCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  int total_tiles = 0;
  if (n_groups > 0) {
    const Group last = p.groups[n_groups - 1];
    total_tiles = (last.mblk_start + (last.n_rows + BM - 1) / BM) * p.n_ntiles;
  }
  const int nk = (p.kdim + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      uint32_t seen = 0;   // sources whose arrival this thread already acquired
      const uint32_t wep = p.ep ? p.ep[kEpWeight] : 0u, aep = p.ep ? p.ep[kEpArrive] : 0u;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const TileInfo ti = decode_tile(t, p.n_ntiles, s_mblk, n_groups, p.groups, p.sched);
        const CUtensorMap *wm = ti.wslot >= 0 ? &p.tmW0 : &p.tmW1;
        const int wbase = (ti.wslot >= 0 ? ti.wslot : (-1 - ti.wslot)) * p.wrows + ti.nb * BNO;
        wait_weights(p, ti.wslot, wep);
        wait_sources(p, ti.mblk, seen, aep);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fb = smem_u32(full + stage);
          mbar_expect_tx(fb, C::STAGE);
          tma_load_2d(smem_u32(sA + stage * C::A_BYTES), &p.tmA, fb, kb * BK, ti.row0);
          if (MODE != 1) {
            tma_load_2d(smem_u32(sB + stage * C::B_BYTES), wm, fb, kb * BK, wbase);
            tma_load_2d(smem_u32(sB + stage * C::B_BYTES + (BN / 2) * BK * 2), wm, fb, kb * BK,
                        wbase + p.wup_off);
          } else {
            tma_load_2d(smem_u32(sB + stage * C::B_BYTES), wm, fb, kb * BK, wbase);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc = instr_desc<BN>();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(smem_u32(tempty + acc), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc_mma(d_tmem, smem_desc(a0 + kk * 32), smem_desc(b0 + kk * 32), idesc,
                   (kb | kk) != 0);
          tc_commit(smem_u32(empty + stage));  // frees the smem stage when these MMAs finish
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(smem_u32(tfull + acc));      // accumulator ready for the epilogue
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-5)
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const TileInfo ti = decode_tile(t, p.n_ntiles, s_mblk, n_groups, p.groups, p.sched);
      mbar_wait(smem_u32(tfull + acc), aphase);
      tc_fence_after();
      const int row = ti.row0 + q * 32 + lane;
      const bool row_ok = row < ti.row_end;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kAccCols;
      const int col0 = ti.nb * BNO;
      if (MODE == 2) {
        // raw gate / up pre-activations for the backward recompute: GU[r] = [g (nout) | u (nout)]
        __nv_bfloat16 *grow = p.out + (size_t)row * 2 * p.nout + col0;
#pragma unroll 1
        for (int j = 0; j < BNO; j += 8) {
          float g[8], u[8];
          tmem_ld8(taddr + j, g);
          tmem_ld8(taddr + BNO + j, u);
          tmem_ld_wait();
          if (row_ok && col0 + j < p.nout) {
            uint4 og, ou;
            __nv_bfloat162 *hg = reinterpret_cast<__nv_bfloat162 *>(&og);
            __nv_bfloat162 *hu = reinterpret_cast<__nv_bfloat162 *>(&ou);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              hg[i] = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
              hu[i] = __floats2bfloat162_rn(u[2 * i], u[2 * i + 1]);
            }
            *reinterpret_cast<uint4 *>(grow + j) = og;
            *reinterpret_cast<uint4 *>(grow + p.nout + j) = ou;
          }
        }
      } else if (MODE == 0) {
        __nv_bfloat16 *orow = p.out + (size_t)row * p.nout + col0;
#pragma unroll 1
        for (int j = 0; j < BNO; j += 8) {
          float g[8], u[8];
          tmem_ld8(taddr + j, g);
          tmem_ld8(taddr + BNO + j, u);
          tmem_ld_wait();
          if (row_ok && col0 + j < p.nout) {
            uint4 o;
            __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float a0 = __fdividef(g[2 * i], 1.f + __expf(-g[2 * i])) * u[2 * i];
              const float a1 = __fdividef(g[2 * i + 1], 1.f + __expf(-g[2 * i + 1])) * u[2 * i + 1];
              h[i] = __floats2bfloat162_rn(a0, a1);
            }
            *reinterpret_cast<uint4 *>(orow + j) = o;
          }
        }
      } else {
        const float gs = row_ok ? p.gate[row] : 0.f;
        __nv_bfloat16 *orow = p.out + (size_t)row * p.nout + col0;
        if (p.peer_slot && row_ok) {  // fused combine push: this row's output -> its home slot
          const int32_t src = p.row_src[row];
          orow = reinterpret_cast<__nv_bfloat16 *>(p.peer_slot[src & 31]) + (size_t)(src >> 5) * p.nout + col0;
        }
#pragma unroll 1
        for (int j = 0; j < BNO; j += 8) {
          float v[8];
          tmem_ld8(taddr + j, v);
          tmem_ld_wait();
          if (row_ok && col0 + j < p.nout) {
            uint4 o;
            __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(gs * v[2 * i], gs * v[2 * i + 1]);
            *reinterpret_cast<uint4 *>(orow + j) = o;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      __syncwarp();
    }
  }
  // fused combine push (mode 1): order this thread's peer stores before the kernel's completion and
  // the device barrier that follows (release at system scope there; per-thread fence here)
  if (MODE == 1 && p.peer_slot) asm volatile("fence.acq_rel.sys;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * kAccCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------------ 2-CTA variant
// A CTA pair (cluster of 2, one TPC) computes a 256-row tile with tcgen05.mma.cta_group::2.
// Each CTA stages its own 128 rows of A and HALF of the B tile (mode 0: CTA0 the W_gate rows,
// CTA1 the matching W_up rows; mode 1: the two halves of the N tile), so the per-SM shared-memory
// operand traffic per MMA drops by a third.  The leader (cluster rank 0) issues the MMAs; both
// CTAs' TMA loads complete on the leader's full barrier; the MMA commits are multicast to both
// CTAs' empty / accumulator-full barriers; each CTA's epilogue drains its own TMEM lanes (its 128
// rows of the 256-row accumulator) and arrives on the leader's TMEM-empty barrier.
// SwiGLU exchange buffer of a half tile (mode 0): [64 rows][S0+1] + [64 rows][S1+1] fp32 (odd strides)
constexpr int kXchgBytes = 64 * (65 + 65) * 4;   // S0, S1 <= 64 for BN <= 256
// coalesced epilogue stores: per epilogue warp a [32 rows][128 B] staging block (16-byte units
// XOR-swizzled by row) -- mode 0 places it inside its exchange buffer
constexpr int kStoreStageBytes = 4 * 32 * 128;

// The warp's 32 lanes each hold up to 8 16-byte units of their own row (o[0..nv)); write them so
// that one instruction stores 4 rows x 128 contiguous bytes (rows may be scattered in memory):
// stage in shared memory, then lane l writes unit (l & 7) of row (4 i + l / 8).
__device__ __forceinline__ void warp_store_rows(uint8_t *wst, int lane, const uint4 (&o)[8], int nv,
                                                unsigned long long dst, int ok) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < nv) *reinterpret_cast<uint4 *>(wst + lane * 128 + ((c ^ (lane & 7)) * 16)) = o[c];
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int rr = it * 4 + (lane >> 3), c = lane & 7;
    const unsigned long long d = __shfl_sync(0xffffffffu, dst, rr);
    const int k = __shfl_sync(0xffffffffu, ok, rr);
    if (k && c < nv)
      *reinterpret_cast<uint4 *>(d + c * 16) = *reinterpret_cast<const uint4 *>(wst + rr * 128 + ((c ^ (rr & 7)) * 16));
  }
  __syncwarp();
}

#ifndef LLEP_FWD_RING_CAP
#define LLEP_FWD_RING_CAP (227 * 1024)   // A/B builds: cap on the forward pair GEMMs' operand ring bytes
#endif
template <int BN, int KSUB = 1, int XB = 0>   // KSUB: 64-deep K sub-tiles per stage; XB: exchange bytes
struct Cfg2 {
  static constexpr int A_BYTES = BM * BK * 2 * KSUB;
  static constexpr int B_BYTES = (BN / 2) * BK * 2 * KSUB;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EXTRA = 1024 + 256 + XB;
  static constexpr int RING = kSmemBudget - EXTRA < LLEP_FWD_RING_CAP ? kSmemBudget - EXTRA : LLEP_FWD_RING_CAP;
  static constexpr int STAGES_RAW = RING / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE + EXTRA;
  static_assert(B_BYTES % 1024 == 0, "B half tile must keep 1024-byte swizzle alignment");
};


// MC = 1: clusters of one CTA pair.  MC = 2: clusters of two CTA pairs that compute the two adjacent N
// tiles (nb = 2j, 2j+1) of the same m-block in lockstep: the activation (A) tile they share is loaded ONCE
// from L2 and multicast to both pairs (each of the four CTAs issues one of the two 64-deep K sub-tiles of
// its row half, for itself and its counterpart in the other pair), halving the A operand's L2 reads; a
// stage is refilled only when both pairs' MMAs released it (empty barriers count one commit per pair).
template <int BN, int MODE, int KSUB, int MC>
__global__ void __launch_bounds__(kGemmThreads, 1) grouped_gemm_2cta_kernel(const __grid_constant__ GemmParams p) {
  static_assert(MC == 1 || (MC == 2 && KSUB == 2), "A multicast splits a stage's two K sub-tiles over the pairs");
  using C = Cfg2<BN, KSUB, (MODE == 0 || MODE == 3) ? kXchgBytes : kStoreStageBytes>;
  constexpr int KST = BK * KSUB;                 // K per pipeline stage
  constexpr int S = C::STAGES;
  constexpr int TM = 2 * BM;                     // rows per pair tile
  constexpr int BNO = MODE != 1 ? BN / 2 : BN;   // output columns per tile
  // swapped tiles carry 3 K sub-tiles per stage when the stage has room (A 16 KB + B 4 KB each; the
  // third A sub-tile goes into the B region): 50 % more weight bytes in flight for these HBM-fed tiles
  constexpr int SWK = C::B_BYTES >= BM * 128 + 3 * 32 * 128 ? LLEP_SWAP_K : 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + S * C::A_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * C::STAGE);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
  float *xchg = reinterpret_cast<float *>(smem + S * C::STAGE + 256);   // mode 0 half tiles

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ccr = cluster_ctarank();           // rank in the cluster (2 * MC CTAs)
  const uint32_t crank = ccr & 1u;                  // rank in the CTA pair
  const uint32_t lead = ccr & ~1u;                  // the pair's leader: issues the MMAs, owns the barriers
  const int cpair = (int)(ccr >> 1);                // which pair of the cluster (MC = 2: N tile 2j + cpair)
  const bool leader = crank == 0;
  const int n_groups = p.n_groups_dev ? *p.n_groups_dev : p.n_groups_host;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), MC);        // one MMA-completion commit per pair sharing the stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(tfull + i), 1);
      mbar_init(smem_u32(tempty + i), 8);        // 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmW0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmW1)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kAccCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  int total_tiles = 0;
  if (n_groups > 0) {
    const Group last = p.groups[n_groups - 1];
    total_tiles = (last.mblk_start + (last.n_rows + TM - 1) / TM) * p.n_ntiles;
  }
  const int nk = (p.kdim + KST - 1) / KST;
  // work units: one tile per pair (MC = 1) or the tile pair (2j, 2j+1) of an m-block per cluster (MC = 2)
  const int unit0 = blockIdx.x / (2 * MC), n_units = gridDim.x / (2 * MC);
  const int total_units = total_tiles / MC;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs)
    // Lane 0 waits for foreign weights / dispatched rows and issues the box loads; for a gathered
    // m-block (modes 0/3: every row of it was routed from this rank to itself) all 32 lanes issue
    // TMA gather4 loads of their 4 token rows of x (the dispatch did not copy them, a6 local rows).
    // L2 policy: a small group's weights are read by one m-block only (evict first) so they do
    // not push the large groups' re-used weights and activation tiles out of L2
    const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_normal();
    const uint64_t pol_act = l2_policy_evict_normal();
    const bool gather_on = (MODE == 0 || MODE == 3) && p.rtok != nullptr;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t seen = 0;   // sources whose arrival lane 0 already acquired
    const uint32_t wep = p.ep ? p.ep[kEpWeight] : 0u, aep = p.ep ? p.ep[kEpArrive] : 0u;
    // Without the gather (the default) lane 0 runs the loop alone, as in round 1: the warp-wide loop
    // (32 lanes polling each stage's empty barrier, a __syncwarp per stage) made GEMM1 / GEMM2 4-6 %
    // slower at base clocks (profiles/r02_gemm_regression_bisect.txt)
    const unsigned pmask = gather_on ? 0xffffffffu : 1u;
    if (gather_on || lane == 0)
    for (int u = unit0; u < total_units; u += n_units) {
      const int t = u * MC + cpair;
      TileInfo ti = decode_tile<TM>(t, p.n_ntiles, nullptr, n_groups, p.groups, p.sched);
      ti.swap = p.swap && ti.row_end - ti.row0 <= 64;
      const CUtensorMap *wm = ti.wslot >= 0 ? &p.tmW0 : &p.tmW1;
      const int wbase = (ti.wslot >= 0 ? ti.wslot : (-1 - ti.wslot)) * p.wrows + ti.nb * BNO;
      const int brow = MODE != 1 ? wbase + (int)crank * p.wup_off : wbase + (int)crank * (BN / 2);
      if (lane == 0) {
        wait_weights(p, ti.wslot, wep);
        wait_sources(p, ti.mblk, seen, aep);
      }
      // gathered block: lane l holds the token rows of this CTA's rows base + 4l .. base + 4l + 3
      // (rows past the group's end read token 0; they are computed on and masked at the store)
      const bool gat = gather_on && __ldg(p.mblk_src + ti.mblk) == p.self_mask;
      const int gbase = ti.swap ? ti.row0 + (int)crank * 32 : ti.row0 + (int)crank * (ti.half ? BM / 2 : BM);
      const int gn = ti.swap ? 8 : 32;   // lanes with rows: 32 rows (swapped B operand) or 128
      int gi[4] = {0, 0, 0, 0};
      if (gat && lane < gn) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = gbase + 4 * lane + i;
          const int tk = r < ti.row_end ? __ldg(p.rtok + r) : 0;
          gi[i] = (unsigned)tk < (unsigned)p.xg_rows ? tk : 0;
        }
      }
      __syncwarp(pmask);
      // swapped tile: this CTA's 128 weight rows as the A operand (mode 0/2/3: 64 gate + the
      // matching 64 up rows of features nb*BNO + crank*64 ...; mode 1: rows nb*BN + crank*BN/2
      // ...) and its 32 of the group's <= 64 token rows as the B operand
      const CUtensorMap *wms = ti.wslot >= 0 ? &p.tmW0s : &p.tmW1s;
      const int srow = MODE != 1 ? wbase + (int)crank * 64 : wbase + (int)crank * (BN / 2);
      const int srow2 = MODE != 1 ? srow + p.wup_off : srow + 64;
      if (ti.swap) {
        for (int kb = 0; kb * SWK * BK < p.kdim; ++kb) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const int nsub = min(SWK, (p.kdim - kb * SWK * BK + BK - 1) / BK);
          const uint32_t fl = smem_u32(full + stage);
          const uint32_t fb = mapa_shared(fl, lead);
          if (lane == 0) {
            if (leader) mbar_expect_tx(fl, 2 * nsub * (BM * 128 + 32 * 128));
            // per sub-tile: the weight rows, then (unless gathered) the token rows -- round 1's issue
            // order; all weights first and the tokens last measured ~3 % slower in GEMM1 (tokens
            // first: same as this order), profiles/r02_gemm_regression_bisect.txt
            for (int s2 = 0; s2 < nsub; ++s2) {
              const uint32_t ad = s2 < 2 ? smem_u32(sA + stage * C::A_BYTES + s2 * (BM * 128))
                                         : smem_u32(sB + stage * C::B_BYTES);
              tma_load_2d_pair(ad, wms, fb, (kb * SWK + s2) * BK, srow, ti.small ? pol_first : pol_last);
              tma_load_2d_pair(ad + 64 * 128, wms, fb, (kb * SWK + s2) * BK, srow2, ti.small ? pol_first : pol_last);
              if (!gat)
                tma_load_2d_pair(smem_u32(sB + stage * C::B_BYTES + (SWK == 3 ? BM * 128 : 0) + s2 * (32 * 128)),
                                 &p.tmAs, fb, (kb * SWK + s2) * BK, ti.row0 + (int)crank * 32, pol_act);
            }
          }
          if (gat && lane < gn) {
            for (int s2 = 0; s2 < nsub; ++s2) {
              const uint32_t bd = smem_u32(sB + stage * C::B_BYTES + (SWK == 3 ? BM * 128 : 0) + s2 * (32 * 128));
              tma_gather4_pair(bd + lane * 512, &p.tmXg, fb, (kb * SWK + s2) * BK, gi[0], gi[1], gi[2], gi[3], pol_act);
            }
          }
          __syncwarp(pmask);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        continue;
      }
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(smem_u32(empty + stage), phase ^ 1);
        const int nsub = min(KSUB, (p.kdim - kb * KST + BK - 1) / BK);   // skip all-OOB sub-tiles
        const uint32_t fl = smem_u32(full + stage);
        const uint32_t fb = mapa_shared(fl, lead);
        if (lane == 0) {
          if (leader) mbar_expect_tx(fl, 2 * nsub * (C::STAGE / KSUB));
          for (int s2 = 0; s2 < nsub; ++s2) {
            const uint32_t adst = smem_u32(sA + stage * C::A_BYTES + s2 * (BM * 128));
            const int arow = ti.row0 + (int)crank * (ti.half ? BM / 2 : BM);
            if (MC == 2) {   // sub-tile s2 of this row half, issued by pair s2, into both pairs' CTAs
              if (s2 == cpair)
                tma_load_2d_pair_mc(adst, &p.tmA, fb, (kb * KSUB + s2) * BK, arow,
                                    (uint16_t)((1u << crank) | (1u << (2 + crank))), pol_act);
            } else if (!gat) {
              tma_load_2d_pair(adst, &p.tmA, fb, (kb * KSUB + s2) * BK, arow, pol_act);
            }
            tma_load_2d_pair(smem_u32(sB + stage * C::B_BYTES + s2 * ((BN / 2) * 128)), wm, fb,
                             (kb * KSUB + s2) * BK, brow, ti.small ? pol_first : pol_last);
          }
        }
        if (gat) {
          for (int s2 = 0; s2 < nsub; ++s2)
            tma_gather4_pair(smem_u32(sA + stage * C::A_BYTES + s2 * (BM * 128)) + lane * 512, &p.tmXg, fb,
                             (kb * KSUB + s2) * BK, gi[0], gi[1], gi[2], gi[3], pol_act);
        }
        __syncwarp(pmask);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------------------------------------------------------- MMA issuer (leader warp)
      // M=256 for a full pair tile, M=128 (64 rows per CTA) when <= 128 rows of the block remain
      const uint32_t idesc_full = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                  ((uint32_t)(TM >> 4) << 24);
      const uint32_t idesc_half = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                  ((uint32_t)((TM / 2) >> 4) << 24);
      const uint32_t idesc_swap = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) |
                                  ((uint32_t)(TM >> 4) << 24);
      const uint64_t adesc0 = smem_desc(smem_u32(sA)), bdesc0 = smem_desc(smem_u32(sB));
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint16_t m_empty = MC == 2 ? 0xF : 0x3, m_full = (uint16_t)(0x3u << lead);
      for (int u = unit0; u < total_units; u += n_units, ++it) {
        const int t = u * MC + cpair;
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        TileInfo ti = decode_tile<TM>(t, p.n_ntiles, nullptr, n_groups, p.groups, p.sched);
        ti.swap = p.swap && ti.row_end - ti.row0 <= 64;
        const uint32_t idesc = ti.swap ? idesc_swap : ti.half ? idesc_half : idesc_full;
        mbar_wait(smem_u32(tempty + acc), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        if (ti.swap) {
          for (int kb = 0; kb * SWK * BK < p.kdim; ++kb) {
            mbar_wait(smem_u32(full + stage), phase);
            tc_fence_after();
            __syncwarp();
            const int nsub = min(SWK, (p.kdim - kb * SWK * BK + BK - 1) / BK);
#pragma unroll
            for (int s2 = 0; s2 < SWK; ++s2) {
              if (s2 < nsub) {
                const uint64_t ad = smem_desc(s2 < 2 ? smem_u32(sA + stage * C::A_BYTES + s2 * (BM * 128))
                                                     : smem_u32(sB + stage * C::B_BYTES));
                const uint64_t bd = smem_desc(smem_u32(sB + stage * C::B_BYTES + (SWK == 3 ? BM * 128 : 0) +
                                                       s2 * (32 * 128)));
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  tc_mma_pair_w(d_tmem, ad + (uint32_t)((kk * 32) >> 4), bd + (uint32_t)((kk * 32) >> 4), idesc,
                                (kb | s2 | kk) != 0);
              }
            }
            tc_commit_pair_mask(smem_u32(empty + stage), m_empty);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc_commit_pair_mask(smem_u32(tfull + acc), m_full);
          continue;
        }
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          __syncwarp();
          // descriptor start-address field is addr >> 4: advance it by the byte offset >> 4
          const uint64_t ad = adesc0 + (uint32_t)((stage * C::A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + (uint32_t)((stage * C::B_BYTES) >> 4);
          const int nsub = min(KSUB, (p.kdim - kb * KST + BK - 1) / BK);
#pragma unroll
          for (int s2 = 0; s2 < KSUB; ++s2) {
            if (s2 < nsub) {
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                tc_mma_pair_w(d_tmem, ad + (uint32_t)((s2 * (BM * 128) + kk * 32) >> 4),
                              bd + (uint32_t)((s2 * ((BN / 2) * 128) + kk * 32) >> 4), idesc,
                              (kb | s2 | kk) != 0);
            }
          }
          tc_commit_pair_mask(smem_u32(empty + stage), m_empty);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair_mask(smem_u32(tfull + acc), m_full);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    int it = 0;
    for (int u = unit0; u < total_units; u += n_units, ++it) {
      const int t = u * MC + cpair;
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      TileInfo ti = decode_tile<TM>(t, p.n_ntiles, nullptr, n_groups, p.groups, p.sched);
        ti.swap = p.swap && ti.row_end - ti.row0 <= 64;
      mbar_wait(smem_u32(tfull + acc), aphase);
      tc_fence_after();
      const int row = ti.row0 + (int)crank * BM + q * 32 + lane;
      const bool row_ok = row < ti.row_end;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kAccCols;
      const int col0 = ti.nb * BNO;
      constexpr int bno = BNO;
      if (ti.swap) {
        // swapped tile: TMEM lane L = weight row (feature) of this CTA, column j = token row0 + j
        const int L = q * 32 + lane;
        if (MODE == 1) {
          const int fl = L;                                   // this CTA's rows nb*BN + crank*BN/2 + L
          const int d = ti.nb * BN + (int)crank * (BN / 2) + fl;
          const bool fok = fl < BN / 2 && d < p.nout;
#pragma unroll 1
          for (int j = 0; j < 64; j += 8) {
            float v[8];
            tmem_ld8(taddr + j, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int row = ti.row0 + j + i;
              if (fok && row < ti.row_end) {
                __nv_bfloat16 *orow = p.out + (size_t)row * p.nout;
                if (p.peer_slot) {
                  const int32_t src = p.row_src[row];
                  orow = reinterpret_cast<__nv_bfloat16 *>(p.peer_slot[src & 31]) + (size_t)(src >> 5) * p.nout;
                }
                orow[d] = __float2bfloat16_rn(p.gate[row] * v[i]);
              }
            }
          }
        } else {
          // lanes 0-63: gate rows of features f0 + L, lanes 64-127: the matching up rows
          const int hi = L >> 6, fl = L & 63;
          const int fr = (int)crank * 64 + fl;               // feature within the tile's BNO
          const int f = ti.nb * BNO + fr;
          const bool fok = fr < BNO && f < p.nout;
          if (MODE == 2 || MODE == 3) {   // raw [g | u] rows
            __nv_bfloat16 *gdst = (MODE == 2 ? p.out : p.out2) + (size_t)hi * p.nout + f;
#pragma unroll 1
            for (int j = 0; j < 64; j += 8) {
              float v[8];
              tmem_ld8(taddr + j, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (fok && ti.row0 + j + i < ti.row_end)
                  gdst[(size_t)(ti.row0 + j + i) * 2 * p.nout] = __float2bfloat16_rn(v[i]);
            }
          }
          if (MODE == 0 || MODE == 3) {
            // SwiGLU: gate lanes finish tokens [0, 32), up lanes tokens [32, 64); each sends the
            // other half of its 64 columns through shared memory ([2][64 features][33])
            float *xs = xchg;
            asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll 1
            for (int jj = 0; jj < 32; jj += 8) {
              float v[8];
              tmem_ld8(taddr + (hi == 0 ? 32 : 0) + jj, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i) xs[(hi * 64 + fl) * 33 + jj + i] = v[i];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int jb = hi == 0 ? 0 : 32;
#pragma unroll 1
            for (int jj = 0; jj < 32; jj += 8) {
              float v[8];
              tmem_ld8(taddr + jb + jj, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float o = xs[((1 - hi) * 64 + fl) * 33 + jj + i];
                const float g = hi == 0 ? v[i] : o, u = hi == 0 ? o : v[i];
                const int row = ti.row0 + jb + jj + i;
                if (fok && row < ti.row_end)
                  p.out[(size_t)row * p.nout + f] = __float2bfloat16_rn(__fdividef(g, 1.f + __expf(-g)) * u);
              }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
          }
        }
      } else if (ti.half) {
        // M=128 pair tile: this CTA's 64 rows.  TMEM lanes 0-63 hold accumulator columns [0, BN/2)
        // (the B rows staged by CTA 0) and lanes 64-127 columns [BN/2, BN) (CTA 1's) of the SAME
        // 64 rows, both at TMEM columns 0 .. BN/2-1.
        constexpr int BH = BN / 2;
        const int L = q * 32 + lane, hi = L >> 6, r = L & 63;
        const int hrow = ti.row0 + (int)crank * (BM / 2) + r;
        const bool hok = hrow < ti.row_end;
        if (MODE == 1) {
          const float gs = hok ? p.gate[hrow] : 0.f;
          __nv_bfloat16 *orow = p.out + (size_t)hrow * p.nout + col0 + hi * BH;
          if (p.peer_slot && hok) {
            const int32_t src = p.row_src[hrow];
            orow = reinterpret_cast<__nv_bfloat16 *>(p.peer_slot[src & 31]) + (size_t)(src >> 5) * p.nout +
                   col0 + hi * BH;
          }
#pragma unroll 1
          for (int j = 0; j < BH; j += 8) {
            float v[8];
            tmem_ld8(taddr + j, v);
            tmem_ld_wait();
            if (hok && col0 + hi * BH + j < p.nout) {
              uint4 o;
              __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
              for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(gs * v[2 * i], gs * v[2 * i + 1]);
              *reinterpret_cast<uint4 *>(orow + j) = o;
            }
          }
        } else if (MODE == 2) {
          // lanes 0-63 hold gate pre-activations, lanes 64-127 up: GU[r] = [g (nout) | u (nout)]
          __nv_bfloat16 *dst = p.out + (size_t)hrow * 2 * p.nout + hi * p.nout + col0;
#pragma unroll 1
          for (int j = 0; j < BH; j += 8) {
            float v[8];
            tmem_ld8(taddr + j, v);
            tmem_ld_wait();
            if (hok && col0 + j < p.nout) {
              uint4 o;
              __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
              for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
              *reinterpret_cast<uint4 *>(dst + j) = o;
            }
          }
        } else {
          // SwiGLU needs g (lanes 0-63) and u (lanes 64-127) of the same row: exchange through
          // shared memory.  Gate lanes finish columns [0, S0), up lanes [S0, BH).
          constexpr int S0 = (BH / 2 + 7) / 8 * 8, S1 = BH - S0;
          if (MODE == 3) {   // saved pre-activations: gate lanes write g, up lanes u (as mode 2)
            __nv_bfloat16 *dst = p.out2 + (size_t)hrow * 2 * p.nout + hi * p.nout + col0;
#pragma unroll 1
            for (int j = 0; j < BH; j += 8) {
              float v[8];
              tmem_ld8(taddr + j, v);
              tmem_ld_wait();
              if (hok && col0 + j < p.nout) {
                uint4 o;
                __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
                for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                *reinterpret_cast<uint4 *>(dst + j) = o;
              }
            }
          }
          float *xu = xchg;                          // [64][S0+1] up values of columns [0, S0)
          float *xg = xchg + 64 * (S0 + 1);          // [64][S1+1] gate values of columns [S0, BH)
          asm volatile("bar.sync 1, 128;" ::: "memory");   // the previous half tile's reads are done
          if (hi == 0) {
#pragma unroll 1
            for (int j = S0; j < BH; j += 8) {
              float v[8];
              tmem_ld8(taddr + j, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i) xg[r * (S1 + 1) + (j - S0) + i] = v[i];
            }
          } else {
#pragma unroll 1
            for (int j = 0; j < S0; j += 8) {
              float v[8];
              tmem_ld8(taddr + j, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i) xu[r * (S0 + 1) + j + i] = v[i];
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          __nv_bfloat16 *orow = p.out + (size_t)hrow * p.nout + col0;
          const int j0 = hi == 0 ? 0 : S0, j1 = hi == 0 ? S0 : BH;
#pragma unroll 1
          for (int j = j0; j < j1; j += 8) {
            float v[8], g[8], u[8];
            tmem_ld8(taddr + j, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              g[i] = hi == 0 ? v[i] : xg[r * (S1 + 1) + (j - S0) + i];
              u[i] = hi == 0 ? xu[r * (S0 + 1) + j + i] : v[i];
            }
            if (hok && col0 + j < p.nout) {
              uint4 o;
              __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float a0 = __fdividef(g[2 * i], 1.f + __expf(-g[2 * i])) * u[2 * i];
                const float a1 = __fdividef(g[2 * i + 1], 1.f + __expf(-g[2 * i + 1])) * u[2 * i + 1];
                h[i] = __floats2bfloat162_rn(a0, a1);
              }
              *reinterpret_cast<uint4 *>(orow + j) = o;
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");   // exchange reads done before any reuse
        }
      } else {
        // full tile: lane = row; 64-column chunks converted in registers, stored coalesced
        uint8_t *wst = reinterpret_cast<uint8_t *>(xchg) + q * (32 * 128);
        const int okr = row_ok ? 1 : 0;
        float gs = 1.f;
        __nv_bfloat16 *orow;
        if (MODE == 1) {
          gs = row_ok ? p.gate[row] : 0.f;
          orow = p.out + (size_t)row * p.nout + col0;
          if (p.peer_slot && row_ok) {  // fused combine push: this row's output -> its home slot
            const int32_t src = p.row_src[row];
            orow = reinterpret_cast<__nv_bfloat16 *>(p.peer_slot[src & 31]) + (size_t)(src >> 5) * p.nout + col0;
          }
        } else if (MODE == 0 || MODE == 3) {
          orow = p.out + (size_t)row * p.nout + col0;
        } else {
          orow = p.out + (size_t)row * 2 * p.nout + col0;   // GU[r] = [g (nout) | u (nout)]
        }
#pragma unroll 1
        for (int j = 0; j < bno; j += 64) {
          const int nch = (bno - j) >= 64 ? 8 : (bno - j) / 8;
          const int left = (p.nout - col0 - j) / 8;          // masked tail of the output width
          const int nv = nch < left ? nch : (left > 0 ? left : 0);
          float v[64];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < nch) tmem_ld8(taddr + j + 8 * c, v + 8 * c);
          if (MODE != 1) {
            float u[64];
#pragma unroll
            for (int c = 0; c < 8; ++c)
              if (c < nch) tmem_ld8(taddr + bno + j + 8 * c, u + 8 * c);
            tmem_ld_wait();
            uint4 o[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o[c]);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float g0 = v[8 * c + 2 * i], g1 = v[8 * c + 2 * i + 1];
                const float u0 = u[8 * c + 2 * i], u1 = u[8 * c + 2 * i + 1];
                if (MODE != 2)
                  h[i] = __floats2bfloat162_rn(__fdividef(g0, 1.f + __expf(-g0)) * u0,
                                               __fdividef(g1, 1.f + __expf(-g1)) * u1);
                else
                  h[i] = __floats2bfloat162_rn(g0, g1);
              }
            }
            warp_store_rows(wst, lane, o, nv, reinterpret_cast<unsigned long long>(orow + j), okr);
            if (MODE == 3) {   // saved pre-activations [g | u] of this row (bit-identical to mode 2)
              __nv_bfloat16 *grow = p.out2 + (size_t)row * 2 * p.nout + col0;
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o[c]);
#pragma unroll
                for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[8 * c + 2 * i], v[8 * c + 2 * i + 1]);
              }
              warp_store_rows(wst, lane, o, nv, reinterpret_cast<unsigned long long>(grow + j), okr);
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o[c]);
#pragma unroll
                for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(u[8 * c + 2 * i], u[8 * c + 2 * i + 1]);
              }
              warp_store_rows(wst, lane, o, nv, reinterpret_cast<unsigned long long>(grow + p.nout + j), okr);
            }
            if (MODE == 2) {
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o[c]);
#pragma unroll
                for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(u[8 * c + 2 * i], u[8 * c + 2 * i + 1]);
              }
              warp_store_rows(wst, lane, o, nv, reinterpret_cast<unsigned long long>(orow + p.nout + j), okr);
            }
          } else {
            tmem_ld_wait();
            uint4 o[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o[c]);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                h[i] = __floats2bfloat162_rn(gs * v[8 * c + 2 * i], gs * v[8 * c + 2 * i + 1]);
            }
            warp_store_rows(wst, lane, o, nv, reinterpret_cast<unsigned long long>(orow + j), okr);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty + acc), lead));
      __syncwarp();   // reconverge: named barriers (bar.sync) that follow require converged warps
    }
  }
  // fused combine push (mode 1): order this thread's peer stores before the kernel's completion and
  // the device barrier that follows (release at system scope there; per-thread fence here)
  if (MODE == 1 && p.peer_slot) asm volatile("fence.acq_rel.sys;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * kAccCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

bool make_map(CUtensorMap *m, const void *ptr, int64_t rows, int32_t kdim, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kdim * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int MODE>
llep_status launch(const GemmArgs &g, GemmParams &prm, cudaStream_t s) {
  using C = Cfg<BN>;
  auto kern = grouped_gemm_kernel<BN, MODE>;
  static bool attr_set = false;
  if (!attr_set) {
    LLEP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const int box_w = MODE != 1 ? BN / 2 : BN;
  const int wrows = MODE != 1 ? 2 * g.nout : g.nout;
  if (!make_map(&prm.tmA, g.a, g.a_rows, g.kdim, BM) ||
      !make_map(&prm.tmW0, g.w_native, (int64_t)g.n_native * wrows, g.kdim, box_w) ||
      !make_map(&prm.tmW1, g.w_foreign ? g.w_foreign : g.w_native,
                (int64_t)(g.w_foreign ? g.n_foreign : g.n_native) * wrows, g.kdim, box_w)) {
    set_error("cuTensorMapEncodeTiled failed (alignment: kdim %% 8 == 0, 16-byte aligned bases)");
    return LLEP_ERR_CUDA;
  }
  prm.wrows = wrows;
  prm.wup_off = MODE != 1 ? g.nout : 0;
  prm.n_ntiles = (g.nout + box_w - 1) / box_w;
  grouped_gemm_kernel<BN, MODE><<<g.num_sms, kGemmThreads, C::SMEM, s>>>(prm);
  LLEP_CUDA(cudaGetLastError());
  return LLEP_OK;
}

#ifndef LLEP_FWD_KSUB
#define LLEP_FWD_KSUB 2   // forward pair GEMMs: 64-deep K sub-tiles per pipeline stage (A/B: 3)
#endif
template <int BN, int MODE, int KSUB = LLEP_FWD_KSUB>
llep_status launch_pair(const GemmArgs &g, GemmParams &prm, cudaStream_t s) {
  using C = Cfg2<BN, KSUB, (MODE == 0 || MODE == 3) ? kXchgBytes : kStoreStageBytes>;
  // opt-in (LLEP_GEMM_MC=2): two-pair clusters with the A tile multicast when the N tiles pair up.
  // Correct (bit-identical) and 25 % fewer L2 bytes, but clusters of 4 fit only 132 of the 148 SMs
  // (GPCs' SM counts are not multiples of 4), which costs more than the multicast saves: G120 layer
  // step +12 %, Q3 +7 % (profiles/r02_ab_multicast.txt).  Default: single pairs on all 148 SMs.
  const int n_nt = (g.nout + (MODE != 1 ? BN / 2 : BN) - 1) / (MODE != 1 ? BN / 2 : BN);
  const char *mce = getenv("LLEP_GEMM_MC");
  const int mc = (KSUB == 2 && n_nt % 2 == 0 && !g.rtok && mce && atoi(mce) == 2) ? 2 : 1;
  auto kern = mc == 2 ? grouped_gemm_2cta_kernel<BN, MODE, KSUB, (KSUB == 2 ? 2 : 1)>
                      : grouped_gemm_2cta_kernel<BN, MODE, KSUB, 1>;
  if (!g.sched) {   // the pair kernels walk the layout's interleaved m-block schedule
    set_error("pair GEMM needs the m-block schedule (LLEP_GEMM_GROUP_ORDER applies to the 1-CTA kernels)");
    return LLEP_ERR_INVALID;
  }
  static bool attr_set[2] = {false, false};
  if (!attr_set[mc - 1]) {
    LLEP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set[mc - 1] = true;
  }
  const int box_w = BN / 2;
  const int wrows = MODE != 1 ? 2 * g.nout : g.nout;
  if (!make_map(&prm.tmA, g.a, g.a_rows, g.kdim, BM) ||
      !make_map(&prm.tmW0, g.w_native, (int64_t)g.n_native * wrows, g.kdim, box_w) ||
      !make_map(&prm.tmW1, g.w_foreign ? g.w_foreign : g.w_native,
                (int64_t)(g.w_foreign ? g.n_foreign : g.n_native) * wrows, g.kdim, box_w)) {
    set_error("cuTensorMapEncodeTiled failed (alignment: kdim %% 8 == 0, 16-byte aligned bases)");
    return LLEP_ERR_CUDA;
  }
  if (!make_map(&prm.tmAs, g.a, g.a_rows, g.kdim, 32) ||
      !make_map(&prm.tmW0s, g.w_native, (int64_t)g.n_native * wrows, g.kdim, 64) ||
      !make_map(&prm.tmW1s, g.w_foreign ? g.w_foreign : g.w_native,
                (int64_t)(g.w_foreign ? g.n_foreign : g.n_native) * wrows, g.kdim, 64)) {
    set_error("cuTensorMapEncodeTiled failed (swapped-tile maps)");
    return LLEP_ERR_CUDA;
  }
  if ((MODE == 0 || MODE == 3) && g.rtok && g.xg && g.xg_rows > 0 && g.mblk_src) {
    if (!make_map(&prm.tmXg, g.xg, g.xg_rows, g.kdim, 1)) {
      set_error("cuTensorMapEncodeTiled failed (token gather map)");
      return LLEP_ERR_CUDA;
    }
    prm.rtok = g.rtok;
    prm.xg_rows = (int32_t)g.xg_rows;
    prm.self_mask = g.self_mask;
  }
  prm.wrows = wrows;
  prm.wup_off = MODE != 1 ? g.nout : 0;
  prm.n_ntiles = (g.nout + (MODE != 1 ? BN / 2 : BN) - 1) / (MODE != 1 ? BN / 2 : BN);
  cudaLaunchConfig_t cfg = {};
  int grid = g.num_sms & ~(2 * mc - 1);
  if (const char *gp = getenv("LLEP_GEMM_PAIRS"))   // measurement only: fewer CTA pairs (per-pair rates)
    grid = 2 * mc * std::max(1, std::min(grid / (2 * mc), atoi(gp) / mc));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * mc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (mc == 2) {
    // a persistent grid must be co-resident: clusters of 4 need 4 free SMs in one GPC, so size the grid
    // by the occupancy API (GPCs whose SM count is not a multiple of 4 lose their remainder SMs)
    static int max_clusters = 0;
    if (!max_clusters) {
      cudaLaunchConfig_t q = cfg;
      q.gridDim = dim3((unsigned)(g.num_sms & ~3));
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &q) != cudaSuccess || max_clusters < 1)
        max_clusters = (g.num_sms & ~3) / 4;
      (void)cudaGetLastError();
    }
    cfg.gridDim = dim3((unsigned)std::min(grid, 4 * max_clusters));
  }
  LLEP_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  return LLEP_OK;
}


// ------------------------------------------------------------------------ backward GEMMs (f1)
// The backward pass contracts the expert weights along the other dimension and the
// activations along the token dimension, so its operands are MN-major in shared memory: TMA boxes
// of 64 MN-elements (128 B, swizzled) x 64 K-rows, one 8 KB block per 64-wide MN chunk.  UMMA
// descriptor for such a tile: LBO = distance between MN chunks (8 KB), SBO = distance between
// 8-row K groups (1 KB); a 16-deep K step advances the start address by 16 rows (2 KB).
//   KIND 0 (rows):  C[r, n] = Σ_k A[r, k] · W_e[k, n]      A K-major rows, W row-major [K][N]
//                   (dA = dY·W_down with W_down [D][H]; dX = dGU·W13 with W13 [2H][D]); bf16 out
//   KIND 1 (wgrad): C_e[m, n] = Σ_{r in group e} A[r, m] · B[r, n]   both MN-major, K = tokens
//                   (dW_down = dYᵀ·a, dW13 = dGUᵀ·X); fp32 out per group
constexpr int kBwdBN = 256;
constexpr int kBwdA = BM * BK * 2;        // 16 KB (K-major 128 rows, or 2 MN chunks)
constexpr int kBwdB = kBwdBN * BK * 2;    // 32 KB (4 MN chunks)
constexpr int kBwdStage = kBwdA + kBwdB;
constexpr int kBwdStg = BM * 32 * 4;   // KIND 1 epilogue staging buffer: [128 rows][32 fp32]
constexpr int kBwdNStg = 4;            // KIND 1: staging buffers (stores in flight)
template <int KIND> struct BwdCfg {
  static constexpr int STAGES = KIND == 0 ? 4 : 3;
  static constexpr int SMEM = STAGES * kBwdStage + 1024 + (KIND == 1 ? kBwdNStg * kBwdStg : 0) + 1024;
};

struct BwdParams {
  CUtensorMap tmA, tmB, tmB1;   // tmB1: foreign-expert weights (KIND 0/2, groups with wslot < 0)
  CUtensorMap tmO, tmOF, tmWS;  // KIND 1 fp32 outputs, 3D {nout, mdim, slot}: out, out_foreign, ws
  const Group *groups;
  int32_t n_groups;
  int32_t kdim;          // KIND 0: contraction length (rows of W_e)
  int32_t mdim;          // KIND 1: output rows per group
  int32_t nout;          // output columns
  int32_t n_mt, n_nt;    // tiles per group (KIND 1: m x n) ; KIND 0: n tiles
  int32_t mblk_scale;    // KIND 0: 128-row blocks per Group.mblk_start unit
  void *out;
  void *out_foreign;     // KIND 1: output of foreign groups (wslot < 0), nullptr -> out[expert]
  float *ws;             // KIND 1: split-K partials
  int32_t num_sms;       // scheduling units for the split heuristic (SMs, or CTA pairs)
  CUtensorMap tmAs;      // KIND 0 pair kernel, swapped tiles: activation rows, 32-row boxes
  int32_t swap;          // KIND 0 pair kernel: groups of <= 64 rows as swapped tiles
  const __nv_bfloat16 *gu;   // KIND 2: [g | u] rows, gates, outputs w·a, [dg | du], partial dots
  const float *gate;
  __nv_bfloat16 *aw, *dgu;
  float *dotp;
};

__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((8192 >> 4) & 0x3FFF) << 16;     // LBO: next 64-wide MN chunk
  d |= (uint64_t)(1024 >> 4) << 32;                 // SBO: next 8-row K group
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

struct BwdTile {
  int row0, row_end, m0, n0, g, nk, split, nsplit;
  int half;   // pair kernel, kind 0: <= 128 rows left in the block -> M=128 pair MMA
  int swap;   // pair kernel, kind 0: <= 64 rows -> swapped tile D[features x tokens] (M=256, N=64)
};

template <int KIND>
__device__ __forceinline__ BwdTile decode_bwd(int t, const BwdParams &p, const int *s_mblk) {
  BwdTile ti;
  ti.half = 0;
  ti.swap = 0;
  if (KIND == 0) {
    const int mb = t / p.n_nt;
    ti.n0 = (t - mb * p.n_nt) * kBwdBN;
    int lo = 0, hi = p.n_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_mblk[mid] * p.mblk_scale <= mb) lo = mid;
      else hi = mid - 1;
    }
    const Group g = p.groups[lo];
    ti.g = lo;
    ti.row0 = g.row_base + (mb - s_mblk[lo] * p.mblk_scale) * BM;
    ti.row_end = g.row_base + g.n_rows;
    ti.m0 = 0;
    ti.nk = (p.kdim + BK - 1) / BK;
  } else {
    // s_mblk holds, in schedule order (split groups first), the first tile of each entry; the
    // group id of entry i is s_mblk[kMaxGroups / 2 + i] (KIND 1 uses two half-size arrays)
    const int per = p.n_mt * p.n_nt;
    int lo = 0, hi = p.n_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_mblk[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    ti.g = s_mblk[kMaxGroups / 2 + lo];
    const int rel = t - s_mblk[lo];
    ti.split = rel / per;
    const int r = rel - ti.split * per;
    const int mt = r / p.n_nt;
    ti.m0 = mt * BM;
    ti.n0 = (r - mt * p.n_nt) * kBwdBN;
    const Group g = p.groups[ti.g];
    ti.nsplit = wgrad_splits(g.n_rows, per, p.num_sms);
    const int ks = wgrad_split_rows(g.n_rows, ti.nsplit);
    // contract only up to the group's last 64-row K block (rows past n_rows are zero in both
    // operands): a 52-row group costs one K step, not four
    const int kend = (g.n_rows + BK - 1) / BK * BK;
    const int k0 = ti.split * ks;
    const int k1 = min(kend, k0 + ks);
    ti.row0 = g.row_base + k0;
    ti.row_end = g.row_base + g.n_rows;
    ti.nk = (k1 - k0) / BK;     // padded rows are zero in both operands
  }
  return ti;
}

template <int KIND>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_bwd_kernel(const __grid_constant__ BwdParams p) {
  constexpr int S = BwdCfg<KIND>::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + S * kBwdA;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * kBwdStage);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
  float *stg = reinterpret_cast<float *>(smem + S * kBwdStage + 1024);
  int ep_chunk = 0;
  __shared__ int s_mblk[kMaxGroups + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int total_tiles_k1 = 0;
  if (KIND == 0) {
    for (int g = threadIdx.x; g < p.n_groups; g += kGemmThreads) s_mblk[g] = p.groups[g].mblk_start;
  } else if (threadIdx.x == 0) {
    // schedule order: split groups (their many K-ranges) first, then the others
    const int per = p.n_mt * p.n_nt;
    int pos = 0, tile = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int g = 0; g < p.n_groups; ++g) {
        const int ns = wgrad_splits(p.groups[g].n_rows, per, p.num_sms);
        if ((ns > 1) != (pass == 0)) continue;
        s_mblk[pos] = tile;
        s_mblk[kMaxGroups / 2 + pos] = g;
        ++pos;
        tile += ns * per;
      }
    s_mblk[kMaxGroups / 2 - 1] = tile;
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(tfull + i), 1);
      mbar_init(smem_u32(tempty + i), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(2 * kAccCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  (void)total_tiles_k1;
  int total_tiles = 0;
  if (p.n_groups > 0) {
    if (KIND == 0) {
      const Group last = p.groups[p.n_groups - 1];
      total_tiles = (last.mblk_start * p.mblk_scale + (last.n_rows + BM - 1) / BM) * p.n_nt;
    } else {
      total_tiles = s_mblk[kMaxGroups / 2 - 1];
    }
  }
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const BwdTile ti = decode_bwd<KIND>(t, p, s_mblk);
        const int ws = KIND == 0 ? p.groups[ti.g].wslot : 0;
        const int wrow = (ws >= 0 ? ws : -1 - ws) * p.kdim;
        const CUtensorMap *bm = ws >= 0 ? &p.tmB : &p.tmB1;
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fb = smem_u32(full + stage);
          mbar_expect_tx(fb, kBwdStage);
          const uint32_t a_dst = smem_u32(sA + stage * kBwdA);
          const uint32_t b_dst = smem_u32(sB + stage * kBwdB);
          if (KIND == 0) {
            tma_load_2d(a_dst, &p.tmA, fb, kb * BK, ti.row0);                 // K-major rows
#pragma unroll
            for (int c = 0; c < kBwdBN / 64; ++c)                            // W_e[k, n] chunks
              tma_load_2d(b_dst + c * 8192, bm, fb, ti.n0 + c * 64, wrow + kb * BK);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_2d(a_dst + c * 8192, &p.tmA, fb, ti.m0 + c * 64, ti.row0 + kb * BK);
#pragma unroll
            for (int c = 0; c < kBwdBN / 64; ++c)
              tma_load_2d(b_dst + c * 8192, &p.tmB, fb, ti.n0 + c * 64, ti.row0 + kb * BK);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((KIND == 1 ? 1u : 0u) << 15) |
                             (1u << 16) | ((uint32_t)(kBwdBN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
        const BwdTile ti = decode_bwd<KIND>(t, p, s_mblk);
        const int acc = it & 1;
        mbar_wait(smem_u32(tempty + acc), ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kBwdA);
          const uint32_t b0 = smem_u32(sB + stage * kBwdB);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = KIND == 0 ? smem_desc(a0 + kk * 32) : smem_desc_mn(a0 + kk * 2048);
            tc_mma(d_tmem, ad, smem_desc_mn(b0 + kk * 2048), idesc, (kb | kk) != 0);
          }
          tc_commit(smem_u32(empty + stage));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(smem_u32(tfull + acc));
      }
    }
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const BwdTile ti = decode_bwd<KIND>(t, p, s_mblk);
      mbar_wait(smem_u32(tfull + acc), (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kAccCols;
      if (KIND == 0) {
        const int row = ti.row0 + q * 32 + lane;
        const bool ok = row < ti.row_end;
        __nv_bfloat16 *orow = reinterpret_cast<__nv_bfloat16 *>(p.out) + (size_t)row * p.nout + ti.n0;
#pragma unroll 1
        for (int j = 0; j < kBwdBN; j += 8) {
          float v[8];
          tmem_ld8(taddr + j, v);
          tmem_ld_wait();
          if (ok && ti.n0 + j < p.nout) {
            uint4 o;
            __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            *reinterpret_cast<uint4 *>(orow + j) = o;
          }
        }
      } else {
        // fp32 gradient tile -> shared memory (rows of 32 floats, 128-byte swizzle) -> TMA bulk
        // tensor stores of [128 rows x 32 cols] boxes (3D map: rows past mdim are clipped, not
        // written into the next expert's slot)
        const Group gg = p.groups[ti.g];
        const CUtensorMap *om = &p.tmO;
        int slot = gg.expert;
        if (p.out_foreign) {
          slot = gg.wslot >= 0 ? gg.wslot : -1 - gg.wslot;
          if (gg.wslot < 0) om = &p.tmOF;
        }
        if (ti.nsplit > 1) {  // partial of K-range ti.split -> workspace (groups in order, splits)
          int off = 0;
          const int per = p.n_mt * p.n_nt;
          for (int g2 = 0; g2 < ti.g; ++g2) {
            const int ns = wgrad_splits(p.groups[g2].n_rows, per, p.num_sms);
            if (ns > 1) off += ns;
          }
          om = &p.tmWS;
          slot = off + ti.split;
        }
        const int r = q * 32 + lane;
        const bool leader = threadIdx.x == 64;
#pragma unroll 1
        for (int c = 0; c < kBwdBN / 32; ++c, ++ep_chunk) {
          const int b = ep_chunk % kBwdNStg;
          if (leader) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");  // kBwdNStg - 1
          asm volatile("bar.sync 2, 128;" ::: "memory");
          float v[32];
#pragma unroll
          for (int i = 0; i < 4; ++i) tmem_ld8(taddr + c * 32 + 8 * i, v + 8 * i);
          tmem_ld_wait();
          float *rowp = stg + b * (BM * 32) + r * 32;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4 *>(rowp + ((i ^ (r & 7)) * 4)) =
                make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 2, 128;" ::: "memory");
          if (leader) {
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                         ::"l"(reinterpret_cast<uint64_t>(om)), "r"(ti.n0 + c * 32), "r"(ti.m0), "r"(slot),
                         "r"(smem_u32(stg + b * (BM * 32)))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      __syncwarp();
    }
  }
  if (KIND == 1 && threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * kAccCols) : "memory");
}


// ---------------------------------------------------------------- backward GEMMs, 2-CTA variant
// Same two kinds on CTA pairs (cta_group::2): a pair tile is 256 rows (KIND 0) / 256 output rows
// (KIND 1) x 256 columns; CTA r stages its 128 rows of A (K-major, or two 64-wide MN chunks) and
// the r-th 128-column half of B (two MN chunks), the leader issues M=256 N=256 MMAs.
constexpr int kPairA = BM * BK * 2;        // 16 KB per CTA
constexpr int kPairB = 128 * BK * 2;       // 16 KB per CTA (half of N)
constexpr int kPairStage = kPairA + kPairB;
// pair weight-gradient kernel: operand pipeline stages (64-deep, 32 KB each) and fp32 staging buffers
// (TMA stores in flight).  5 + 3 beat round 1's 4 + 4 by 6-8 % at base clocks on the P=8 critical-rank
// layout and at P=1 (tensor pipe 78 -> 84.5 %, profiles/r02_ab_wgrad_stages.txt)
#ifndef LLEP_WG_NSTG
#define LLEP_WG_NSTG 3
#endif
#ifndef LLEP_WG_STAGES
#define LLEP_WG_STAGES 5
#endif
constexpr int kPairNStg = LLEP_WG_NSTG;
#ifndef LLEP_BWD_KSUB
#define LLEP_BWD_KSUB 2   // A/B: build with -DLLEP_BWD_KSUB=1 for 64-deep stages in the row kinds
#endif
template <int KIND> struct BwdPairCfg {
  // row kinds: two 64-deep K sub-tiles per pipeline stage (8 MMAs per barrier round trip, as in the
  // forward); the weight-gradient kind keeps 64-deep stages (a small group is one K step)
  static constexpr int KSUB = KIND == 1 ? 1 : (LLEP_BWD_KSUB);
  static constexpr int STAGES = KIND == 1 ? LLEP_WG_STAGES : 6 / KSUB;
  static constexpr int SMEM = STAGES * KSUB * kPairStage + 1024 + (KIND == 1 ? kPairNStg * kBwdStg : kStoreStageBytes) + 1024;
};

template <int KIND>
__device__ __forceinline__ BwdTile decode_bwd_pair(int t, const BwdParams &p, const int *s_mblk) {
  BwdTile ti;
  ti.half = 0;
  ti.swap = 0;
  if (KIND != 1) {
    const int mb = t / p.n_nt;
    ti.n0 = (t - mb * p.n_nt) * kBwdBN;
    int lo = 0, hi = p.n_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_mblk[mid] <= mb) lo = mid;
      else hi = mid - 1;
    }
    const Group g = p.groups[lo];
    ti.g = lo;
    ti.row0 = g.row_base + (mb - s_mblk[lo]) * 2 * BM;
    ti.row_end = g.row_base + g.n_rows;
    ti.m0 = 0;
    ti.nk = (p.kdim + BK - 1) / BK;
    ti.half = ti.row_end - ti.row0 <= BM;
    ti.swap = KIND == 0 && p.swap && ti.row_end - ti.row0 <= 64;
  } else {
    const int per = p.n_mt * p.n_nt;
    int lo = 0, hi = p.n_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_mblk[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    ti.g = s_mblk[kMaxGroups / 2 + lo];
    const int rel = t - s_mblk[lo];
    ti.split = rel / per;
    const int r = rel - ti.split * per;
    const int mt = r / p.n_nt;
    ti.m0 = mt * 2 * BM;
    ti.n0 = (r - mt * p.n_nt) * kBwdBN;
    const Group g = p.groups[ti.g];
    ti.nsplit = wgrad_splits(g.n_rows, per, p.num_sms);
    const int ks = wgrad_split_rows(g.n_rows, ti.nsplit);
    // contract only up to the group's last 64-row K block (rows past n_rows are zero in both
    // operands): a 52-row group costs one K step, not four
    const int kend = (g.n_rows + BK - 1) / BK * BK;
    const int k0 = ti.split * ks;
    const int k1 = min(kend, k0 + ks);
    ti.row0 = g.row_base + k0;
    ti.row_end = g.row_base + g.n_rows;
    ti.nk = (k1 - k0) / BK;
  }
  return ti;
}

template <int KIND>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_bwd_pair_kernel(const __grid_constant__ BwdParams p) {
  constexpr int S = BwdPairCfg<KIND>::STAGES;
  constexpr int KS = BwdPairCfg<KIND>::KSUB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + S * KS * kPairA;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * KS * kPairStage);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
  float *stg = reinterpret_cast<float *>(smem + S * KS * kPairStage + 1024);
  int ep_chunk = 0;
  __shared__ int s_mblk[kMaxGroups + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  if (KIND != 1) {
    for (int g = threadIdx.x; g < p.n_groups; g += kGemmThreads) s_mblk[g] = p.groups[g].mblk_start;
  } else if (threadIdx.x == 0) {
    const int per = p.n_mt * p.n_nt;
    int pos = 0, tile = 0;
    // large (split) groups first; merging the small groups' write-bound tiles evenly among them
    // was measured 7-10 % slower (L2 pressure on the large groups' re-read operands)
    for (int pass = 0; pass < 2; ++pass) {
      for (int g = 0; g < p.n_groups; ++g) {
        const int ns = wgrad_splits(p.groups[g].n_rows, per, p.num_sms);
        if ((ns > 1) != (pass == 0)) continue;
        s_mblk[pos] = tile;
        s_mblk[kMaxGroups / 2 + pos] = g;
        ++pos;
        tile += ns * per;
      }
    }
    s_mblk[kMaxGroups / 2 - 1] = tile;
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(tfull + i), 1);
      mbar_init(smem_u32(tempty + i), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(2 * kAccCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  int total_tiles = 0;
  if (p.n_groups > 0) {
    if (KIND != 1) {
      const Group last = p.groups[p.n_groups - 1];
      total_tiles = (last.mblk_start + (last.n_rows + 2 * BM - 1) / (2 * BM)) * p.n_nt;
    } else {
      total_tiles = s_mblk[kMaxGroups / 2 - 1];
    }
  }
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < total_tiles; t += n_pairs) {
        const BwdTile ti = decode_bwd_pair<KIND>(t, p, s_mblk);
        const int ws = KIND != 1 ? p.groups[ti.g].wslot : 0;
        const int wrow = (ws >= 0 ? ws : -1 - ws) * p.kdim;
        const CUtensorMap *bm = (KIND != 1 && ws < 0) ? &p.tmB1 : &p.tmB;
        if (KIND == 0 && ti.swap) {
          // swapped tile, three 64-deep K sub-tiles per stage: this CTA's 128 weight features
          // (MN-major, the M operand; sub-tiles 0/1 in the stage's B slots, 2 in its second A slot)
          // and its 32 of the group's <= 64 token rows (K-major, the N operand; the first A slot)
          for (int kq = 0; kq * 3 < ti.nk; ++kq) {
            mbar_wait(smem_u32(empty + stage), phase ^ 1);
            const int nsub = min(3, ti.nk - kq * 3);
            const uint32_t fl = smem_u32(full + stage);
            if (leader) mbar_expect_tx(fl, 2 * nsub * (kPairB + 32 * 128));
            const uint32_t fb = mapa_shared(fl, 0);
            for (int s2 = 0; s2 < nsub; ++s2) {
              const int kb = kq * 3 + s2;
              const uint32_t w_dst = s2 < 2 ? smem_u32(sB + (stage * KS + s2) * kPairB)
                                            : smem_u32(sA + (stage * KS + 1) * kPairA);
#pragma unroll
              for (int c = 0; c < 2; ++c)
                tma_load_2d_pair(w_dst + c * 8192, bm, fb, ti.n0 + (int)crank * 128 + c * 64, wrow + kb * BK, pol);
              tma_load_2d_pair(smem_u32(sA + (stage * KS) * kPairA + s2 * (32 * 128)), &p.tmAs, fb, kb * BK,
                               ti.row0 + (int)crank * 32, pol);
            }
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          continue;
        }
        for (int kq = 0; kq * KS < ti.nk; ++kq) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const int nsub = min(KS, ti.nk - kq * KS);
          const uint32_t fl = smem_u32(full + stage);
          if (leader) mbar_expect_tx(fl, 2 * nsub * kPairStage);
          const uint32_t fb = mapa_shared(fl, 0);
          for (int s2 = 0; s2 < nsub; ++s2) {
          const int kb = kq * KS + s2;
          const uint32_t a_dst = smem_u32(sA + (stage * KS + s2) * kPairA);
          const uint32_t b_dst = smem_u32(sB + (stage * KS + s2) * kPairB);
          if (KIND != 1) {
            tma_load_2d_pair(a_dst, &p.tmA, fb, kb * BK, ti.row0 + (int)crank * (ti.half ? BM / 2 : BM), pol);
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(b_dst + c * 8192, bm, fb, ti.n0 + (int)crank * 128 + c * 64, wrow + kb * BK, pol);
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(a_dst + c * 8192, &p.tmA, fb, ti.m0 + (int)crank * BM + c * 64, ti.row0 + kb * BK, pol);
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(b_dst + c * 8192, &p.tmB, fb, ti.n0 + (int)crank * 128 + c * 64, ti.row0 + kb * BK, pol);
          }
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      const uint32_t idesc_full = (1u << 4) | (1u << 7) | (1u << 10) | ((KIND == 1 ? 1u : 0u) << 15) |
                                  (1u << 16) | ((uint32_t)(kBwdBN >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
      const uint32_t idesc_half = (idesc_full & ~(0x1Fu << 24)) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < total_tiles; t += n_pairs, ++it) {
        const BwdTile ti = decode_bwd_pair<KIND>(t, p, s_mblk);
        const uint32_t idesc = (KIND != 1 && ti.half) ? idesc_half : idesc_full;
        const int acc = it & 1;
        mbar_wait(smem_u32(tempty + acc), ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        if (KIND == 0 && ti.swap) {
          // A = weights (MN-major), B = tokens (K-major), M=256, N=64
          const uint32_t idesc_sw = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(64 >> 3) << 17) |
                                    ((uint32_t)((2 * BM) >> 4) << 24);
          for (int kq = 0; kq * 3 < ti.nk; ++kq) {
            mbar_wait(smem_u32(full + stage), phase);
            tc_fence_after();
            const int nsub = min(3, ti.nk - kq * 3);
            for (int s2 = 0; s2 < nsub; ++s2) {
              const uint32_t w0 = s2 < 2 ? smem_u32(sB + (stage * KS + s2) * kPairB) : smem_u32(sA + (stage * KS + 1) * kPairA);
              const uint32_t x0 = smem_u32(sA + (stage * KS) * kPairA + s2 * (32 * 128));
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                tc_mma_pair(d_tmem, smem_desc_mn(w0 + kk * 2048), smem_desc(x0 + kk * 32), idesc_sw,
                            ((kq * 3 + s2) | kk) != 0);
            }
            tc_commit_pair(smem_u32(empty + stage));
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc_commit_pair(smem_u32(tfull + acc));
          continue;
        }
        for (int kq = 0; kq * KS < ti.nk; ++kq) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          const int nsub = min(KS, ti.nk - kq * KS);
#pragma unroll
          for (int s2 = 0; s2 < KS; ++s2) {
            if (s2 < nsub) {
              const int kb = kq * KS + s2;
              const uint32_t a0 = smem_u32(sA + (stage * KS + s2) * kPairA);
              const uint32_t b0 = smem_u32(sB + (stage * KS + s2) * kPairB);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint64_t ad = KIND != 1 ? smem_desc(a0 + kk * 32) : smem_desc_mn(a0 + kk * 2048);
                tc_mma_pair(d_tmem, ad, smem_desc_mn(b0 + kk * 2048), idesc, (kb | kk) != 0);
              }
            }
          }
          tc_commit_pair(smem_u32(empty + stage));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair(smem_u32(tfull + acc));
      }
    }
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int t = pair; t < total_tiles; t += n_pairs, ++it) {
      const int acc = it & 1;
      const BwdTile ti = decode_bwd_pair<KIND>(t, p, s_mblk);
      mbar_wait(smem_u32(tfull + acc), (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kAccCols;
      if (KIND == 2) {
        // dA0 tile + SwiGLU backward (row f1): per element with g, u from GU and d = dA0 (fp32, TMEM)
        //   a = silu(g) u, da = w d, dg = da u sg (1 + g (1 - sg)), du = da silu(g), dot += a d
        // writes w·a, dg, du (bf16) and this thread's partial <a, dA0> over its columns
        const int L = q * 32 + lane;
        const int row = ti.half ? ti.row0 + (int)crank * (BM / 2) + (L & 63) : ti.row0 + (int)crank * BM + L;
        const int c0 = ti.half ? (L >> 6) * (kBwdBN / 2) : 0, cw = ti.half ? kBwdBN / 2 : kBwdBN;
        const bool ok = row < ti.row_end;
        const int H = p.nout;
        const float w = ok ? p.gate[row] : 0.f;
        const __nv_bfloat16 *gurow = p.gu + (size_t)row * 2 * H + ti.n0 + c0;
        __nv_bfloat16 *awrow = p.aw + (size_t)row * H + ti.n0 + c0;
        __nv_bfloat16 *dgrow = p.dgu + (size_t)row * 2 * H + ti.n0 + c0;
        uint8_t *wst = reinterpret_cast<uint8_t *>(stg) + q * (32 * 128);
        float dot = 0.f;
#pragma unroll 1
        for (int j = 0; j < cw; j += 32) {
          const int left = (H - ti.n0 - c0 - j) / 8;
          const int nv = left < 4 ? (left > 0 ? left : 0) : 4;
          float v[32];
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_ld8(taddr + j + 8 * c, v + 8 * c);
          uint4 gv[4], uv[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            gv[c] = make_uint4(0, 0, 0, 0);
            uv[c] = make_uint4(0, 0, 0, 0);
            if (ok && c < nv) {
              gv[c] = __ldg(reinterpret_cast<const uint4 *>(gurow + j + 8 * c));
              uv[c] = __ldg(reinterpret_cast<const uint4 *>(gurow + H + j + 8 * c));
            }
          }
          tmem_ld_wait();
          uint4 oa[8], og[8], ou[8];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gv[c]);
            const __nv_bfloat162 *u2 = reinterpret_cast<const __nv_bfloat162 *>(&uv[c]);
            __nv_bfloat162 *a2 = reinterpret_cast<__nv_bfloat162 *>(&oa[c]);
            __nv_bfloat162 *gg = reinterpret_cast<__nv_bfloat162 *>(&og[c]);
            __nv_bfloat162 *uu = reinterpret_cast<__nv_bfloat162 *>(&ou[c]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 gf = __bfloat1622float2(g2[i]), uf = __bfloat1622float2(u2[i]);
              const float gz[2] = {gf.x, gf.y}, uz[2] = {uf.x, uf.y};
              float ar[2], dgr[2], dur[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const float d = v[8 * c + 2 * i + e];
                const float sg = 1.f / (1.f + __expf(-gz[e]));
                const float si = gz[e] * sg;
                const float a = si * uz[e];
                const float da = w * d;
                ar[e] = w * a;
                dot += a * d;
                dgr[e] = da * uz[e] * sg * (1.f + gz[e] * (1.f - sg));
                dur[e] = da * si;
              }
              a2[i] = __floats2bfloat162_rn(ar[0], ar[1]);
              gg[i] = __floats2bfloat162_rn(dgr[0], dgr[1]);
              uu[i] = __floats2bfloat162_rn(dur[0], dur[1]);
            }
          }
          if (!ti.half) {
            const int k = ok ? 1 : 0;
            warp_store_rows(wst, lane, oa, nv, reinterpret_cast<unsigned long long>(awrow + j), k);
            warp_store_rows(wst, lane, og, nv, reinterpret_cast<unsigned long long>(dgrow + j), k);
            warp_store_rows(wst, lane, ou, nv, reinterpret_cast<unsigned long long>(dgrow + H + j), k);
          } else if (ok) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (c < nv) {
                *reinterpret_cast<uint4 *>(awrow + j + 8 * c) = oa[c];
                *reinterpret_cast<uint4 *>(dgrow + j + 8 * c) = og[c];
                *reinterpret_cast<uint4 *>(dgrow + H + j + 8 * c) = ou[c];
              }
          }
        }
        if (ok) {   // partial dots: slot 2·nb + (128-column half); a full tile leaves its second slot 0
          float *dp = p.dotp + (size_t)row * (2 * p.n_nt) + 2 * (ti.n0 / kBwdBN);
          if (ti.half) {
            dp[L >> 6] = dot;
          } else {
            dp[0] = dot;
            dp[1] = 0.f;
          }
        }
      } else if (KIND == 0 && ti.swap) {
        // swapped tile: TMEM lane = output column n0 + 128·crank + L, TMEM column j = token row0 + j
        const int n = ti.n0 + (int)crank * 128 + q * 32 + lane;
        __nv_bfloat16 *ocol = reinterpret_cast<__nv_bfloat16 *>(p.out) + n;
#pragma unroll 1
        for (int j = 0; j < 64; j += 8) {
          float v[8];
          tmem_ld8(taddr + j, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = ti.row0 + j + i;
            if (n < p.nout && row < ti.row_end) ocol[(size_t)row * p.nout] = __float2bfloat16_rn(v[i]);
          }
        }
      } else if (KIND == 0) {
        // full tile: lane = row of this CTA's 128; half tile (M=128 pair MMA): lanes 0-63 hold
        // columns [0, 128) and lanes 64-127 columns [128, 256) of the CTA's 64 rows
        const int L = q * 32 + lane;
        const int row = ti.half ? ti.row0 + (int)crank * (BM / 2) + (L & 63) : ti.row0 + (int)crank * BM + L;
        const int c0 = ti.half ? (L >> 6) * (kBwdBN / 2) : 0, cw = ti.half ? kBwdBN / 2 : kBwdBN;
        const bool ok = row < ti.row_end;
        __nv_bfloat16 *orow = reinterpret_cast<__nv_bfloat16 *>(p.out) + (size_t)row * p.nout + ti.n0 + c0;
        if (!ti.half) {   // full tile: coalesced row stores through the warp's smem stage
          uint8_t *wst = reinterpret_cast<uint8_t *>(stg) + q * (32 * 128);
#pragma unroll 1
          for (int j = 0; j < kBwdBN; j += 64) {
            const int left = (p.nout - ti.n0 - j) / 8;
            const int nv = left < 8 ? (left > 0 ? left : 0) : 8;
            float v[64];
#pragma unroll
            for (int c = 0; c < 8; ++c) tmem_ld8(taddr + j + 8 * c, v + 8 * c);
            tmem_ld_wait();
            uint4 o[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o[c]);
#pragma unroll
              for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[8 * c + 2 * i], v[8 * c + 2 * i + 1]);
            }
            warp_store_rows(wst, lane, o, nv, reinterpret_cast<unsigned long long>(orow + j), ok ? 1 : 0);
          }
        } else
#pragma unroll 1
        for (int j = 0; j < cw; j += 8) {
          float v[8];
          tmem_ld8(taddr + j, v);
          tmem_ld_wait();
          if (ok && ti.n0 + c0 + j < p.nout) {
            uint4 o;
            __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            *reinterpret_cast<uint4 *>(orow + j) = o;
          }
        }
      } else {
        const Group gg = p.groups[ti.g];
        const CUtensorMap *om = &p.tmO;
        int slot = gg.expert;
        if (p.out_foreign) {
          slot = gg.wslot >= 0 ? gg.wslot : -1 - gg.wslot;
          if (gg.wslot < 0) om = &p.tmOF;
        }
        if (ti.nsplit > 1) {
          int off = 0;
          const int per = p.n_mt * p.n_nt;
          for (int g2 = 0; g2 < ti.g; ++g2) {
            const int ns = wgrad_splits(p.groups[g2].n_rows, per, p.num_sms);
            if (ns > 1) off += ns;
          }
          om = &p.tmWS;
          slot = off + ti.split;
        }
        const int r = q * 32 + lane;
        const bool lead = threadIdx.x == 64;
        const int m0 = ti.m0 + (int)crank * BM;
#pragma unroll 1
        for (int c = 0; c < kBwdBN / 32; ++c, ++ep_chunk) {
          const int b = ep_chunk % kPairNStg;
          if (lead) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kPairNStg - 1) : "memory");
          asm volatile("bar.sync 2, 128;" ::: "memory");
          float v[32];
#pragma unroll
          for (int i = 0; i < 4; ++i) tmem_ld8(taddr + c * 32 + 8 * i, v + 8 * i);
          tmem_ld_wait();
          float *rowp = stg + b * (BM * 32) + r * 32;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4 *>(rowp + ((i ^ (r & 7)) * 4)) =
                make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 2, 128;" ::: "memory");
          if (lead) {
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                         ::"l"(reinterpret_cast<uint64_t>(om)), "r"(ti.n0 + c * 32), "r"(m0), "r"(slot),
                         "r"(smem_u32(stg + b * (BM * 32)))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty + acc), 0));
      __syncwarp();   // reconverge: named barriers (bar.sync) that follow require converged warps
    }
  }
  if (KIND == 1 && threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * kAccCols) : "memory");
}

bool make_map_box(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int box_cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

static bool make_map_out3d(CUtensorMap *m, const void *ptr, int nout, int mdim, int64_t slots) {
  auto enc = get_encode();
  if (!enc) return false;
  if (slots < 1) slots = 1;
  cuuint64_t dims[3] = {(cuuint64_t)nout, (cuuint64_t)mdim, (cuuint64_t)slots};
  cuuint64_t strides[2] = {(cuuint64_t)nout * 4, (cuuint64_t)mdim * nout * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)BM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t wgrad_workspace(const int32_t *n_rows, int n_groups, int mdim, int nout, int num_sms) {
  // num_sms > 0: 1-CTA tiles of 128 output rows over num_sms units; < 0: pair tiles of 256 rows
  // over -num_sms units (CTA pairs)
  const int tm = num_sms > 0 ? BM : 2 * BM;
  num_sms = num_sms > 0 ? num_sms : -num_sms;
  const int per = ((mdim + tm - 1) / tm) * ((nout + kBwdBN - 1) / kBwdBN);
  int64_t n = 0;
  for (int g = 0; g < n_groups; ++g) {
    const int ns = wgrad_splits(n_rows[g], per, num_sms);
    if (ns > 1) n += (int64_t)ns * mdim * nout;
  }
  return n;
}

__global__ void split_reduce_kernel(float *__restrict__ dst, const float *__restrict__ parts, int n_parts,
                                    int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4 *>(parts)[i];
    for (int s = 1; s < n_parts; ++s) {
      const float4 v = reinterpret_cast<const float4 *>(parts)[s * n4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4 *>(dst)[i] = acc;
  }
}

llep_status reduce_wgrad_splits(const BwdArgs &a, const int32_t *n_rows, const int32_t *wslots,
                                const int32_t *experts, int n_groups, cudaStream_t s) {
  const int tm = a.pair ? 2 * BM : BM;
  const int units = a.pair ? a.num_sms / 2 : a.num_sms;
  const int per = ((a.mdim + tm - 1) / tm) * ((a.nout + kBwdBN - 1) / kBwdBN);
  const int64_t mn = (int64_t)a.mdim * a.nout;
  int64_t off = 0;
  for (int g = 0; g < n_groups; ++g) {
    const int ns = wgrad_splits(n_rows[g], per, units);
    if (ns <= 1) continue;
    float *dst;
    if (a.out_foreign) {
      dst = wslots[g] >= 0 ? reinterpret_cast<float *>(a.out) + (int64_t)wslots[g] * mn
                           : reinterpret_cast<float *>(a.out_foreign) + (int64_t)(-1 - wslots[g]) * mn;
    } else {
      dst = reinterpret_cast<float *>(a.out) + (int64_t)experts[g] * mn;
    }
    split_reduce_kernel<<<296, 256, 0, s>>>(dst, a.ws + off * mn, ns, mn / 4);
    LLEP_CUDA(cudaGetLastError());
    off += ns;
  }
  return LLEP_OK;
}

llep_status run_gemm_bwd(const BwdArgs &a, cudaStream_t s) {
  if (a.nout % 8 || a.kdim % 8 || a.mdim % 8) {
    set_error("backward GEMM needs dims %% 8 == 0");
    return LLEP_ERR_INVALID;
  }
  if (a.kind == 1 && a.n_groups > kMaxGroups / 2 - 1) {   // the kernel's smem group table
    set_error("weight-gradient GEMM supports at most %d groups per device", kMaxGroups / 2 - 1);
    return LLEP_ERR_INVALID;
  }
  BwdParams p;
  memset(&p, 0, sizeof(p));
  p.groups = a.groups;
  p.n_groups = a.n_groups;
  p.kdim = a.kdim;
  p.mdim = a.mdim;
  p.nout = a.nout;
  p.n_nt = (a.nout + kBwdBN - 1) / kBwdBN;
  p.n_mt = (a.mdim + (a.pair ? 2 * BM : BM) - 1) / (a.pair ? 2 * BM : BM);
  p.mblk_scale = a.mblk_scale;
  p.out = a.out;
  p.out_foreign = a.out_foreign;
  p.ws = a.ws;
  p.num_sms = a.pair ? a.num_sms / 2 : a.num_sms;
  {
    const char *sw = getenv("LLEP_BWD_SWAP");   // A/B switch: swapped tiles in the row kind
    p.swap = a.pair ? (sw ? atoi(sw) : 1) : 0;
  }
  if (a.kind == 2) {
    if (!a.pair || !a.gu || !a.gate || !a.aw || !a.dgu || !a.dotp) {
      set_error("fused dA0 + SwiGLU-backward GEMM needs the pair kernel and all of gu, gate, aw, dgu, dotp");
      return LLEP_ERR_INVALID;
    }
    p.gu = reinterpret_cast<const __nv_bfloat16 *>(a.gu);
    p.gate = a.gate;
    p.aw = reinterpret_cast<__nv_bfloat16 *>(a.aw);
    p.dgu = reinterpret_cast<__nv_bfloat16 *>(a.dgu);
    p.dotp = a.dotp;
  }
  bool ok;
  if (a.kind != 1) {
    ok = make_map_box(&p.tmA, a.a, a.rows, a.kdim, BK, BM) && make_map_box(&p.tmAs, a.a, a.rows, a.kdim, BK, 32) &&
         make_map_box(&p.tmB, a.b, (int64_t)a.n_weights * a.kdim, a.nout, 64, BK) &&
         make_map_box(&p.tmB1, a.b_foreign ? a.b_foreign : a.b,
                      (int64_t)(a.b_foreign ? a.n_foreign : a.n_weights) * a.kdim, a.nout, 64, BK);
  } else {
    ok = make_map_box(&p.tmA, a.a, a.rows, a.mdim, 64, BK) &&
         make_map_box(&p.tmB, a.b, a.rows, a.nout, 64, BK) &&
         make_map_box(&p.tmB1, a.b, a.rows, a.nout, 64, BK) &&
         make_map_out3d(&p.tmO, a.out, a.nout, a.mdim, a.n_out_slots) &&
         make_map_out3d(&p.tmOF, a.out_foreign ? a.out_foreign : a.out, a.nout, a.mdim,
                        a.out_foreign ? a.n_foreign_slots : a.n_out_slots) &&
         make_map_out3d(&p.tmWS, a.ws ? (const void *)a.ws : a.out, a.nout, a.mdim,
                        a.ws ? a.n_ws_slots : a.n_out_slots);
  }
  if (!ok) {
    set_error("cuTensorMapEncodeTiled failed for a backward GEMM operand");
    return LLEP_ERR_CUDA;
  }
  if (a.pair) {
    static bool pattr[3] = {false, false, false};
    auto kern = a.kind == 0 ? gemm_bwd_pair_kernel<0> : a.kind == 1 ? gemm_bwd_pair_kernel<1> : gemm_bwd_pair_kernel<2>;
    const int smem = a.kind == 0 ? BwdPairCfg<0>::SMEM : a.kind == 1 ? BwdPairCfg<1>::SMEM : BwdPairCfg<2>::SMEM;
    if (!pattr[a.kind]) {
      LLEP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      pattr[a.kind] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.num_sms & ~1));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr2[1];
    attr2[0].id = cudaLaunchAttributeClusterDimension;
    attr2[0].val.clusterDim.x = 2;
    attr2[0].val.clusterDim.y = 1;
    attr2[0].val.clusterDim.z = 1;
    cfg.attrs = attr2;
    cfg.numAttrs = 1;
    LLEP_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
    return LLEP_OK;
  }
  static bool attr[2] = {false, false};
  if (!attr[a.kind]) {
    if (a.kind == 0)
      LLEP_CUDA(cudaFuncSetAttribute(gemm_bwd_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     BwdCfg<0>::SMEM));
    else
      LLEP_CUDA(cudaFuncSetAttribute(gemm_bwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     BwdCfg<1>::SMEM));
    attr[a.kind] = true;
  }
  if (a.kind == 0) gemm_bwd_kernel<0><<<a.num_sms, kGemmThreads, BwdCfg<0>::SMEM, s>>>(p);
  else gemm_bwd_kernel<1><<<a.num_sms, kGemmThreads, BwdCfg<1>::SMEM, s>>>(p);
  LLEP_CUDA(cudaGetLastError());
  return LLEP_OK;
}

namespace {}  // (run_grouped_gemm below)

bool tma_map_kmajor(CUtensorMap *m, const void *ptr, int64_t rows, int32_t kdim, int box_rows) {
  return make_map(m, ptr, rows, kdim, box_rows);
}

llep_status run_grouped_gemm(const GemmArgs &g, cudaStream_t s) {
  if (g.kdim % 8 != 0 || g.nout % 8 != 0) {
    set_error("grouped GEMM needs kdim %% 8 == 0 and nout %% 8 == 0");
    return LLEP_ERR_INVALID;
  }
  GemmParams prm;
  memset(&prm, 0, sizeof(prm));
  prm.groups = g.groups;
  prm.sched = g.sched;
  prm.wflags = g.wflags;
  prm.ep = g.ep;
  prm.err = g.err;
  prm.arrive = g.arrive;
  prm.mblk_src = g.mblk_src;
  prm.src_all = g.src_all;
  prm.row_src = g.row_src;
  prm.peer_slot = g.peer_slot;
  prm.n_groups_dev = g.n_groups_dev;
  prm.n_groups_host = g.n_groups_host;
  prm.kdim = g.kdim;
  prm.nout = g.nout;
  prm.gate = g.gate;
  prm.out = reinterpret_cast<__nv_bfloat16 *>(g.out);
  prm.out2 = reinterpret_cast<__nv_bfloat16 *>(g.out2);
  {
    const char *sw = getenv("LLEP_GEMM_SWAP");   // A/B switch: swapped tiles for groups of <= 64 rows
    prm.swap = sw ? atoi(sw) : 1;
  }
  if (g.mode == 3 && !g.out2) {
    set_error("grouped GEMM mode 3 needs the pre-activation output");
    return LLEP_ERR_INVALID;
  }
  if (g.row_align == 2 * BM) {   // 2-CTA pair tiles (groups 256-row aligned)
#ifdef LLEP_FWD_FORCE_BN192
    if (g.mode == 0 && g.nout % 96 == 0) return launch_pair<192, 0>(g, prm, s);
    if (g.mode == 1 && g.nout % 192 == 0) return launch_pair<192, 1>(g, prm, s);
#endif
    if (g.mode == 3) {
      if (g.nout % 128 == 0) return launch_pair<256, 3>(g, prm, s);
      if (g.nout % 120 == 0) return launch_pair<240, 3>(g, prm, s);
      if (g.nout % 96 == 0) return launch_pair<192, 3>(g, prm, s);
      return launch_pair<256, 3>(g, prm, s);
    }
    if (g.mode == 0) {
      if (g.nout % 128 == 0) return launch_pair<256, 0>(g, prm, s);
      if (g.nout % 120 == 0) return launch_pair<240, 0>(g, prm, s);
      if (g.nout % 96 == 0) return launch_pair<192, 0>(g, prm, s);
      return launch_pair<256, 0>(g, prm, s);
    }
    if (g.mode == 2) {
      if (g.nout % 128 == 0) return launch_pair<256, 2>(g, prm, s);
      if (g.nout % 120 == 0) return launch_pair<240, 2>(g, prm, s);
      if (g.nout % 96 == 0) return launch_pair<192, 2>(g, prm, s);
      return launch_pair<256, 2>(g, prm, s);
    }
    if (g.nout % 256 == 0) return launch_pair<256, 1>(g, prm, s);
    if (g.nout % 240 == 0) return launch_pair<240, 1>(g, prm, s);
    if (g.nout % 192 == 0) return launch_pair<192, 1>(g, prm, s);
    return launch_pair<256, 1>(g, prm, s);
  }
  if (g.mode == 3) {   // 1-CTA tiles: SwiGLU output, then the raw pre-activations (same MMAs)
    GemmArgs g0 = g;
    g0.mode = 0;
    llep_status st = run_grouped_gemm(g0, s);
    if (st != LLEP_OK) return st;
    g0.mode = 2;
    g0.out = g.out2;
    g0.out2 = nullptr;
    return run_grouped_gemm(g0, s);
  }
  // tile width: widest instantiated N that divides the output (else masked tail tiles)
  if (g.mode == 0) {
    if (g.nout % 128 == 0) return launch<256, 0>(g, prm, s);
    if (g.nout % 120 == 0) return launch<240, 0>(g, prm, s);
    if (g.nout % 96 == 0) return launch<192, 0>(g, prm, s);
    return launch<256, 0>(g, prm, s);
  }
  if (g.mode == 2) {
    if (g.nout % 128 == 0) return launch<256, 2>(g, prm, s);
    if (g.nout % 120 == 0) return launch<240, 2>(g, prm, s);
    if (g.nout % 96 == 0) return launch<192, 2>(g, prm, s);
    return launch<256, 2>(g, prm, s);
  }
  if (g.nout % 256 == 0) return launch<256, 1>(g, prm, s);
  if (g.nout % 240 == 0) return launch<240, 1>(g, prm, s);
  if (g.nout % 192 == 0) return launch<192, 1>(g, prm, s);
  return launch<256, 1>(g, prm, s);
}

}  // namespace llep
