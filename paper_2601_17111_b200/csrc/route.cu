// Routing-side kernels of the LLEP layer: load histogram (a1), load exchange + device barrier
// (a2), stable per-expert local ranks (a3), dispatch (a6) and combine (a10).
//
// The paper re-indexes with sort + index_select of the K-repeated tokens (Alg. 1/4, P:299-303,
// P:542-544) and calls that step memory-intensive.  Here the permutation is never
// materialised: a counting sort gives every flat slot j = t*K+k its stable rank r_j among this
// rank's slots of the same expert (P:282's order), dispatch turns (e, Σ_{q<p} C[q][e] + r_j)
// into a (device, row) through the replicated plan and copies the token row straight from the
// unsorted x into the destination's receive rows ("direct All-to-All on unsorted tensors",
// P:578), and combine pulls each slot's output row back and sums over K in slot order.
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

namespace llep {

namespace {

// ------------------------------------------------------------------------------ a1: histogram
constexpr int kCountThreads = 256;

__global__ void __launch_bounds__(kCountThreads) tile_count_kernel(
    const int32_t *__restrict__ ids, int64_t n_slots, int N, int32_t *__restrict__ tile_cnt,
    int32_t *__restrict__ err) {
  extern __shared__ int32_t hist[];
  for (int e = threadIdx.x; e < N; e += kCountThreads) hist[e] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTileSlots;
  const int64_t end = min(base + kTileSlots, n_slots);
  int bad = 0;
  for (int64_t j = base + threadIdx.x; j < end; j += kCountThreads) {
    const int e = ids[j];
    if (e >= 0 && e < N) atomicAdd(&hist[e], 1);
    else bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1);
  for (int e = threadIdx.x; e < N; e += kCountThreads)
    tile_cnt[(size_t)blockIdx.x * N + e] = hist[e];
}

// exclusive scan over tiles per expert -> tile offsets; totals = this rank's counts row.
// One block per 32 experts (lane = expert, coalesced), 8 warps each own a contiguous eighth of the
// tiles: pass 1 sums each warp's share, the warp bases are scanned in shared memory, pass 2 writes.
constexpr int kScanWarps = 8;

__global__ void __launch_bounds__(kScanWarps * 32) tile_scan_kernel(const int32_t *__restrict__ tile_cnt,
                                                                    int n_tiles, int N,
                                                                    int32_t *__restrict__ tile_off,
                                                                    int32_t *__restrict__ cnt) {
  __shared__ int part[kScanWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int per = (n_tiles + kScanWarps - 1) / kScanWarps;
  const int t0 = warp * per, t1 = min(n_tiles, t0 + per);
  int s = 0;
  if (e < N)
    for (int t = t0; t < t1; ++t) s += tile_cnt[(size_t)t * N + e];
  part[warp][lane] = s;
  __syncthreads();
  int run = 0;
  for (int w = 0; w < warp; ++w) run += part[w][lane];
  if (e < N) {
    for (int t = t0; t < t1; ++t) {
      const int v = tile_cnt[(size_t)t * N + e];
      tile_off[(size_t)t * N + e] = run;
      run += v;
    }
    if (warp == kScanWarps - 1) cnt[e] = run;
  }
}

// ----------------------------------------------------------------- a3: stable local ranks r_j
// One CTA per 1024-slot tile, 8 warps x 128 consecutive slots.  Pass 1 counts per warp with
// __match_any_sync (one smem update per distinct expert per 32 slots), an exclusive scan over
// the warps seeds each warp's counters with the tile offset, pass 2 re-walks the slots in order.
constexpr int kRankWarps = 8;
constexpr int kRankThreads = kRankWarps * 32;
constexpr int kSlotsPerWarp = kTileSlots / kRankWarps;

__global__ void __launch_bounds__(kRankThreads) local_rank_kernel(
    const int32_t *__restrict__ ids, int64_t n_slots, int N, const int32_t *__restrict__ tile_off,
    int32_t *__restrict__ local_rank, int32_t *__restrict__ prep_ids) {
  extern __shared__ int32_t wcnt[];  // [kRankWarps][N]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRankWarps * N; i += kRankThreads) wcnt[i] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kTileSlots + (int64_t)warp * kSlotsPerWarp;
  int32_t *mine = wcnt + warp * N;
  for (int i = 0; i < kSlotsPerWarp; i += 32) {
    const int64_t j = wbase + i + lane;
    int e = j < n_slots ? ids[j] : -1;
    if (e >= N) e = -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && lane == __ffs(peers) - 1) mine[e] += __popc(peers);
    __syncwarp();   // order this round's counter updates before the next round's (other lanes)
  }
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += kRankThreads) {
    int run = tile_off[(size_t)blockIdx.x * N + e];
    for (int w = 0; w < kRankWarps; ++w) {
      const int v = wcnt[w * N + e];
      wcnt[w * N + e] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int i = 0; i < kSlotsPerWarp; i += 32) {
    const int64_t j = wbase + i + lane;
    int e = j < n_slots ? ids[j] : -1;
    if (e >= N) e = -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int r = __popc(peers & ((1u << lane) - 1u));
    int base = 0;
    if (e >= 0) base = mine[e];
    __syncwarp();
    if (j < n_slots) {
      local_rank[j] = e >= 0 ? base + r : -1;
      prep_ids[j] = e;   // the ids this plan was built from: dispatch addresses with these (a5)
    }
    if (e >= 0 && lane == __ffs(peers) - 1) mine[e] = base + __popc(peers);
    __syncwarp();
  }
}

// ----------------------------------------------------------------- a2: exchange + barrier
__global__ void push_counts_kernel(const int32_t *__restrict__ cnt, int N, int rank, int P,
                                   int32_t *const *__restrict__ peer_lm) {
  for (int q = blockIdx.x; q < P; q += gridDim.x) {
    int32_t *dst = peer_lm[q] + (size_t)rank * N;
    for (int e = threadIdx.x; e < N; e += blockDim.x) dst[e] = cnt[e];
  }
}

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Every rank writes `epoch` into slot [rank] of every peer's flag array, then waits until all
// of its own slots reach `epoch`.  Writes of earlier kernels on this stream happen-before the
// release (stream order + cumulativity), so after the acquire every peer's earlier stores to
// this rank's arena are visible to the kernels that follow.  Bounded spin -> COMM error.
__global__ void barrier_kernel(uint32_t *const *__restrict__ peer_flags, int rank, int P,
                               uint32_t *__restrict__ ep, int32_t *__restrict__ err) {
  const int q = threadIdx.x;
  const uint32_t epoch = ep[kEpBarrier] + 1;   // this barrier's epoch (device-resident, see common.cuh)
  if (q < P) {
    __threadfence_system();
    st_release_sys(peer_flags[q] + rank, epoch);
    const uint32_t *mine = peer_flags[rank] + q;
    const long long t0 = clock64();
    long long spins = 0;
    while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
      if (((++spins) & 1023) == 0 && clock64() - t0 > 40000000000LL) {  // ~20 s
        atomicOr(err, 4);
        break;
      }
    }
  }
  __syncwarp();
  if (q == 0) ep[kEpBarrier] = epoch;
}

__global__ void advance_kernel(uint32_t *ep) {
  ep[kEpWeight] += 1;
  ep[kEpArrive] += 1;
}

// ----------------------------------------------------------------------------- a6: dispatch
// One warp per token: lanes k < K resolve slot (t,k) to its (device, row); then the warp streams
// x[t] once (16-byte loads) and stores it to each of the K destinations (peer-mapped rows).
constexpr int kDispatchWarps = 8;

__device__ __forceinline__ void dispatch_token(const DispatchArgs &a, int64_t t, int lane);

// Ordering of the peer stores (multi-GPU): every thread orders its own row / gate / source stores
// before the block's completion count with fence.acq_rel.sys; the last block acquires all counts
// (atom.acq_rel) and releases `epoch` into every destination's arrival flag [rank] at system scope, so
// a destination that acquires the flag sees every row this rank dispatched to it (cumulativity).
__global__ void __launch_bounds__(kDispatchWarps * 32) dispatch_kernel(DispatchArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kDispatchWarps + (threadIdx.x >> 5);
  if (t < a.B && !(a.skip && *a.skip)) dispatch_token(a, t, lane);
  if (!a.peer_flags) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.block_done) : "memory");
    if (prev == gridDim.x - 1) {
      *a.block_done = 0;   // next call's count (stream-ordered after this kernel)
      const uint32_t epoch = a.ep[kEpArrive];
      for (int q = 0; q < a.P; ++q) st_release_sys(a.peer_flags[q] + kArriveFlag0 + a.rank, epoch);
    }
  }
}

// P=1 or a rank without tokens: publish the arrival flags alone
__global__ void arrive_kernel(uint32_t *const *__restrict__ peer_flags, int rank, int P, const uint32_t *ep) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  const uint32_t epoch = ep[kEpArrive];
  for (int q = threadIdx.x; q < P; q += blockDim.x) st_release_sys(peer_flags[q] + kArriveFlag0 + rank, epoch);
}

__device__ __forceinline__ void dispatch_token(const DispatchArgs &a, int64_t t, int lane) {
  const int K = a.K, N = a.N, P = a.P, MC = P + 1;
  const uint8_t *plan = reinterpret_cast<const uint8_t *>(a.plan);
  const PlanLayout L = plan_layout(N, P);
  const int32_t *n_chunks = reinterpret_cast<const int32_t *>(plan + L.off_n_chunks);
  const llep_chunk *chunks = reinterpret_cast<const llep_chunk *>(plan + L.off_chunks);
  int dev = -1, row = 0, gathered = 0;
  if (lane < K) {
    const int64_t j = t * K + lane;
    // The plan, the load matrix and the local ranks all come from llep_prepare's ids, so the slot is
    // addressed with those (every planned receive row is written exactly once); a slot whose id
    // changed since then is dropped from the combine and reported (err[2], LLEP_ERR_PLAN).
    const int e = a.prep_ids[j];
    const bool changed = a.ids[j] != e;
    if (changed) atomicOr(a.err + 2, 1);
    if (e >= 0 && e < N) {
      const int nc = n_chunks[e];
      // global index within e: this source's block offset (R11 / R11') + the stable local rank (a3)
      const int g = a.local_rank[j] + (int)source_offset(chunks + (size_t)e * MC, nc, a.load_matrix, N, P, e,
                                                         a.rank, a.aligned);
      for (int c = 0; c < nc; ++c) {
        const llep_chunk ch = chunks[(size_t)e * MC + c];
        if (g >= ch.start && g < ch.end) {
          dev = ch.device;
          row = a.chunk_row[(size_t)e * MC + c] + (g - ch.start);
          break;
        }
      }
    }
    a.slot_dst[2 * j] = changed ? -1 : dev;
    a.slot_dst[2 * j + 1] = row;
    // local-row gather: GEMM1 reads this row from x[t] itself, nothing to copy
    if (dev == a.rank && a.rtok && a.mblk_src[row / a.row_align] == (1u << a.rank)) {
      a.rtok[row] = (int32_t)t;
      gathered = 1;
    }
    if (dev >= 0) {
      a.peer_g[dev][row] = changed ? 0.f : a.w[j];
      // (source rank, flat slot) of this receive row: the GEMM2 epilogue pushes the row's output
      // straight into slot j of this rank's slot buffer
      if (a.peer_rsrc) a.peer_rsrc[dev][row] = (int32_t)((j << 5) | a.rank);
    }
  }
  const int nv = a.D / 8;  // 16-byte vectors per row
  if (a.rtok) {   // drop the gathered slots from the copy; nothing left to copy -> skip the row load
    if (gathered) dev = -1;
    if (!__any_sync(0xffffffffu, dev >= 0)) return;
  }
  for (int src_i = 0; src_i < (a.x2 ? 2 : 1); ++src_i) {
    const int4 *src = reinterpret_cast<const int4 *>(src_i ? a.x2 : a.x) + t * nv;
    uint16_t *const *peer = src_i ? a.peer_x2 : a.peer_x;
    for (int i0 = 0; i0 < nv; i0 += 32 * 4) {
      int4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 32 + lane;
        if (i < nv) v[u] = __ldg(src + i);
      }
      for (int k = 0; k < K; ++k) {
        const int d = __shfl_sync(0xffffffffu, dev, k);
        const int r = __shfl_sync(0xffffffffu, row, k);
        if (d < 0) continue;
        int4 *dst = reinterpret_cast<int4 *>(peer[d]) + (int64_t)r * nv;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * 32 + lane;
          if (i < nv) dst[i] = v[u];
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------ a10: combine
// One warp per token: out[t] = Σ_{k=0..K-1} Y[dst(t,k)] in slot order, fp32 accumulation,
// one bf16 rounding (reverse All-to-All + reverse sort + sum over K).  The K source
// rows (local or peer-mapped) are resolved once per token; each lane then streams two 16-byte
// vectors of every source row per iteration (2K loads in flight per lane).
constexpr int kCombineWarps = 8;

__device__ __forceinline__ void acc_bf16x8(float *acc, const int4 &v) {
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    acc[2 * i] += f.x;
    acc[2 * i + 1] += f.y;
  }
}
__device__ __forceinline__ int4 pack_bf16x8(const float *acc) {
  int4 o;
  __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
  for (int u = 0; u < 4; ++u) h[u] = __floats2bfloat162_rn(acc[2 * u], acc[2 * u + 1]);
  return o;
}

template <int KM>  // compile-time bound on K (K <= KM)
__global__ void __launch_bounds__(kCombineWarps * 32) combine_kernel(CombineArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kCombineWarps + (threadIdx.x >> 5);
  if (t >= a.B) return;
  const int K = a.K;
  int dev = -1, row = 0;
  if (lane < K) {
    dev = a.slot_dst[2 * (t * K + lane)];
    row = a.slot_dst[2 * (t * K + lane) + 1];
  }
  if (a.peer_s && lane < K) a.slot_out[t * K + lane] = dev >= 0 ? a.peer_s[dev][row] : 0.f;
  const int nv = a.D / 8;
  const int4 *src[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const int d = __shfl_sync(0xffffffffu, dev, k & 31);
    const int r = __shfl_sync(0xffffffffu, row, k & 31);
    src[k] = (k < K && d >= 0) ? reinterpret_cast<const int4 *>(a.peer_y[d]) + (int64_t)r * nv : nullptr;
  }
  int4 *dst = reinterpret_cast<int4 *>(a.out) + t * nv;
  for (int i = lane; i < nv; i += 64) {
    const bool two = i + 32 < nv;
    int4 v0[KM], v1[KM];
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      v0[k] = make_int4(0, 0, 0, 0);
      v1[k] = make_int4(0, 0, 0, 0);
      if (src[k]) {
        v0[k] = __ldcs(src[k] + i);
        if (two) v1[k] = __ldcs(src[k] + i + 32);
      }
    }
    float acc0[8], acc1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc0[u] = acc1[u] = 0.f;
#pragma unroll
    for (int k = 0; k < KM; ++k) {   // slot order k = 0..K-1
      if (k < K) {
        acc_bf16x8(acc0, v0[k]);
        acc_bf16x8(acc1, v1[k]);
      }
    }
    __stcs(dst + i, pack_bf16x8(acc0));
    if (two) __stcs(dst + i + 32, pack_bf16x8(acc1));
  }
}

// -------------------------------------------------------------------------- backward (f1)
// Zero the padding rows of this device's groups (rows past n_rows up to the next multiple of 256)
// in up to two row buffers: the weight-gradient GEMMs contract over whole 256-row blocks.
__global__ void zero_pad_kernel(const Group *__restrict__ groups, int D, uint16_t *buf0, uint16_t *buf1) {
  const Group g = groups[blockIdx.x];
  const int pad_end = g.row_base + (g.n_rows + 255) / 256 * 256;
  const int nv = D / 8;
  for (int r = g.row_base + g.n_rows; r < pad_end; ++r) {
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      reinterpret_cast<int4 *>(buf0)[(int64_t)r * nv + i] = make_int4(0, 0, 0, 0);
      if (buf1) reinterpret_cast<int4 *>(buf1)[(int64_t)r * nv + i] = make_int4(0, 0, 0, 0);
    }
  }
}

// SwiGLU backward for one received row r (one warp per row), from the recomputed pre-activations
// GU[r] = [g | u], da0 = dY_unscaled · W_down and the row's gate w:
//   a = silu(g) u,  da = w da0,  dg = da u silu'(g),  du = da silu(g),  dw = <a, da0>
// writes A'[r] = w a (for dW_down = dO_rowsᵀ · A'), dGU[r] = [dg | du], and dw into gate[r].
// Padding rows of each group (up to 256) get zeros.
__global__ void bwd_swiglu_kernel(const Group *__restrict__ groups, int n_groups, int n_rows_total,
                                  int H, const uint16_t *__restrict__ GU, const uint16_t *__restrict__ dA0,
                                  float *__restrict__ gate_io, uint16_t *__restrict__ Aw,
                                  uint16_t *__restrict__ dGU) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= n_rows_total) return;
  int lo = 0, hi = n_groups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (groups[mid].row_base <= r) lo = mid;
    else hi = mid - 1;
  }
  const Group g = groups[lo];
  const bool real = r >= g.row_base && r < g.row_base + g.n_rows;
  const bool pad = r >= g.row_base + g.n_rows && r < g.row_base + (g.n_rows + 255) / 256 * 256;
  if (!real && !pad) return;
  const int nv = H / 8;
  const int4 *gu = reinterpret_cast<const int4 *>(GU) + (int64_t)r * 2 * nv;
  const int4 *d0 = reinterpret_cast<const int4 *>(dA0) + (int64_t)r * nv;
  int4 *aw = reinterpret_cast<int4 *>(Aw) + (int64_t)r * nv;
  int4 *dgu = reinterpret_cast<int4 *>(dGU) + (int64_t)r * 2 * nv;
  if (!real) {
    for (int i = lane; i < nv; i += 32) {
      aw[i] = make_int4(0, 0, 0, 0);
      dgu[i] = make_int4(0, 0, 0, 0);
      dgu[nv + i] = make_int4(0, 0, 0, 0);
    }
    return;
  }
  const float w = gate_io[r];
  float dot = 0.f;
  for (int i = lane; i < nv; i += 32) {
    const int4 gv = gu[i], uv = gu[nv + i], dv = d0[i];
    const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gv);
    const __nv_bfloat162 *u2 = reinterpret_cast<const __nv_bfloat162 *>(&uv);
    const __nv_bfloat162 *d2 = reinterpret_cast<const __nv_bfloat162 *>(&dv);
    int4 ao, go, uo;
    __nv_bfloat162 *a2 = reinterpret_cast<__nv_bfloat162 *>(&ao);
    __nv_bfloat162 *gg = reinterpret_cast<__nv_bfloat162 *>(&go);
    __nv_bfloat162 *uu = reinterpret_cast<__nv_bfloat162 *>(&uo);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 gf = __bfloat1622float2(g2[q]), uf = __bfloat1622float2(u2[q]), df = __bfloat1622float2(d2[q]);
      float ar[2], dgr[2], dur[2];
      const float gz[2] = {gf.x, gf.y}, uz[2] = {uf.x, uf.y}, dz[2] = {df.x, df.y};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float sg = 1.f / (1.f + __expf(-gz[c]));
        const float si = gz[c] * sg;
        const float a = si * uz[c];
        const float da = w * dz[c];
        ar[c] = a;
        dot += a * dz[c];
        dgr[c] = da * uz[c] * sg * (1.f + gz[c] * (1.f - sg));
        dur[c] = da * si;
      }
      a2[q] = __floats2bfloat162_rn(w * ar[0], w * ar[1]);
      gg[q] = __floats2bfloat162_rn(dgr[0], dgr[1]);
      uu[q] = __floats2bfloat162_rn(dur[0], dur[1]);
    }
    aw[i] = ao;
    dgu[i] = go;
    dgu[nv + i] = uo;
  }
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) gate_io[r] = dot;   // dL/dw of this (token, slot) row
}

// dst[i] += Σ_s src_s[i] in the listed order (the native device adds the weight-gradient partials
// its replicas returned, in ascending source-device order).
__global__ void grad_reduce_kernel(float *__restrict__ dst, const float *__restrict__ base, int n_src,
                                   int64_t stride4, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<float4 *>(dst)[i];
    for (int s = 0; s < n_src; ++s) {
      const float4 v = reinterpret_cast<const float4 *>(base)[s * stride4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4 *>(dst)[i] = acc;
  }
}

// Row f2: after the copy engine has written an expert's weights into a peer's foreign slot (same
// stream, so the copy completed first), publish `v` in that peer's weight flag with release
// semantics at system scope; the peer's GEMM producers acquire it before loading those weights.
__global__ void signal_kernel(uint32_t *flag, const uint32_t *ep) {
  __threadfence_system();
  st_release_sys(flag, ep[kEpWeight]);
}

// Row f2 broadcast tree: a replica forwards an expert's weights only after its own copy landed.
__global__ void wait_flag_kernel(const uint32_t *flag, const uint32_t *ep, int32_t *err) {
  const uint32_t v = ep[kEpWeight];
  const long long t0 = clock64();
  long long spins = 0;
  while ((int32_t)(ld_acquire_sys(flag) - v) < 0) {
    if (((++spins) & 1023) == 0 && clock64() - t0 > 40000000000LL) {
      atomicOr(err, 8);
      break;
    }
  }
  __threadfence_system();
}

// ------------------------------------------------------------------ a7 issued by the GPU (layer call)
// One launch per broadcast-tree level (PushArgs in common.cuh).  Items (expert, destination) of this
// rank's level are enumerated from the plan's replica bytes by warp 0 (ascending expert, then tree
// step); units = items x 2 MB chunks of the expert's [W13 | W2] bytes, spread over a fixed grid.
// Deadlock freedom: a level-l forward waits only for sends of lower levels, which other ranks issue
// from earlier launches of their side stream (each launch finishes before the next starts), and the
// grid is small (no shared memory beyond 16 KB, 256 threads) so it stays resident beside the GEMMs.
constexpr int kPushThreads = 256, kPushBlocks = 64;
constexpr int64_t kPushChunk = int64_t(1) << 21;

__device__ __forceinline__ int tree_holder(int native, uint32_t mask, int i) {
  if (i == 0) return native;
  uint32_t m = mask;
  for (int j = 1; j < i; ++j) m &= m - 1u;   // drop the i-1 lowest replicas
  return __ffs(m) - 1;
}

__global__ void __launch_bounds__(kPushThreads) push_level_kernel(PushArgs a) {
  __shared__ int32_t items[kMaxPushItems];   // (expert << 5) | destination device
  __shared__ int n_items, s_skip;
  const int tid = threadIdx.x, lane = tid & 31;
  const int N = a.N, P = a.P, M = a.M, rank = a.rank;
  const uint8_t *replica = reinterpret_cast<const uint8_t *>(a.plan) + plan_layout(N, P).off_replica;
  if (tid == 0) s_skip = a.skip && *a.skip;
  if (tid < 32) {
    int run = 0;
    for (int e0 = 0; e0 < N; e0 += 32) {
      const int e = e0 + lane;
      int cnt = 0, me = -1, k = 0, native = 0;
      uint32_t mask = 0;
      if (e < N) {
        native = e / M;
        for (int d = 0; d < P; ++d)
          if (replica[(size_t)e * P + d]) mask |= 1u << d;
        k = __popc(mask);
        if (native == rank) me = 0;
        else if ((mask >> rank) & 1u) me = 1 + __popc(mask & ((1u << rank) - 1u));
        const int lvl = me <= 0 ? 0 : 32 - __clz(me);   // floor(log2 me) + 1: first t with 2^t > me
        if (me >= 0 && k > 0 && lvl == a.level)
          for (int t = lvl; me + (1 << t) <= k; ++t) ++cnt;
      }
      int inc = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const int lvl = me <= 0 ? 0 : 32 - __clz(me);
      for (int i = 0; i < cnt; ++i) {
        const int pos = run + inc - cnt + i;
        if (pos < kMaxPushItems) items[pos] = (e << 5) | tree_holder(native, mask, me + (1 << (lvl + i)));
      }
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      n_items = run < kMaxPushItems ? run : kMaxPushItems;
      if (run > kMaxPushItems) atomicOr(a.err + 1, 64);
    }
  }
  __syncthreads();
  if (s_skip) return;
  const int64_t total = a.w13_bytes + a.w2_bytes;
  const int chunks = (int)((total + kPushChunk - 1) / kPushChunk);
  const int64_t units = (int64_t)n_items * chunks;
  const uint32_t epoch = a.ep[kEpWeight];
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int it = (int)(u / chunks), c = (int)(u % chunks);
    const int e = items[it] >> 5, d = items[it] & 31;
    const int fd = a.foreign_slot[(size_t)e * P + d];
    const uint8_t *src13, *src2;
    if (e / M == rank) {
      src13 = reinterpret_cast<const uint8_t *>(a.w13) + (size_t)(e - rank * M) * a.w13_bytes;
      src2 = reinterpret_cast<const uint8_t *>(a.w2) + (size_t)(e - rank * M) * a.w2_bytes;
    } else {
      // a forward: this rank's own copy of e must have landed (its parent's release)
      const int fm = a.foreign_slot[(size_t)e * P + rank];
      if (tid == 0) {
        const uint32_t *own = a.peer_flags[rank] + kWeightFlag0 + fm;
        const long long t0 = clock64();
        long long spins = 0;
        while ((int32_t)(ld_acquire_sys(own) - epoch) < 0) {
          if (((++spins) & 1023) == 0 &&
              (*reinterpret_cast<volatile int32_t *>(a.err + 1) != 0 || clock64() - t0 > 40000000000LL)) {
            atomicOr(a.err + 1, 8);
            break;
          }
        }
      }
      __syncthreads();
      src13 = a.peer_w13[rank] + (size_t)fm * a.w13_bytes;
      src2 = a.peer_w2[rank] + (size_t)fm * a.w2_bytes;
    }
    uint8_t *dst13 = a.peer_w13[d] + (size_t)fd * a.w13_bytes;
    uint8_t *dst2 = a.peer_w2[d] + (size_t)fd * a.w2_bytes;
    // bytes [b0, b1) of the concatenation [W13 | W2] (both multiples of 16 bytes)
    const int64_t b0 = (int64_t)c * kPushChunk, b1 = b0 + kPushChunk < total ? b0 + kPushChunk : total;
    for (int64_t b = b0 + (int64_t)tid * 64; b < b1; b += (int64_t)kPushThreads * 64) {
      int4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t o = b + q * 16;
        if (o < b1) v[q] = o < a.w13_bytes ? *reinterpret_cast<const int4 *>(src13 + o)
                                            : *reinterpret_cast<const int4 *>(src2 + (o - a.w13_bytes));
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t o = b + q * 16;
        if (o < b1) {
          if (o < a.w13_bytes) *reinterpret_cast<int4 *>(dst13 + o) = v[q];
          else *reinterpret_cast<int4 *>(dst2 + (o - a.w13_bytes)) = v[q];
        }
      }
    }
    // this thread's peer stores before the chunk count; the last chunk releases the slot's flag
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      uint32_t prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.counters + it) : "memory");
      if (prev == (uint32_t)chunks - 1) {
        a.counters[it] = 0;   // the next launch's count (stream-ordered after this kernel)
        st_release_sys(a.peer_flags[d] + kWeightFlag0 + fd, epoch);
      }
    }
    __syncthreads();
  }
}

// a10 with the pushed GEMM2 epilogue: every slot's gated output row already sits in this rank's
// slot buffer [B*K, D]; out[t] = Σ_{k} slotbuf[t*K + k] in slot order (fp32, one bf16 rounding).
template <int KM>
__global__ void __launch_bounds__(kCombineWarps * 32) combine_local_kernel(const uint16_t *__restrict__ slotbuf,
                                                                           int64_t B, int K, int D,
                                                                           const int32_t *__restrict__ slot_dst,
                                                                           uint16_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kCombineWarps + (threadIdx.x >> 5);
  if (t >= B) return;
  const int nv = D / 8;
  const int4 *src = reinterpret_cast<const int4 *>(slotbuf) + t * K * nv;
  int valid = 0;  // slots whose expert id was in range (others contribute nothing)
  if (lane < K) valid = slot_dst[2 * (t * K + lane)] >= 0;
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  int4 *dst = reinterpret_cast<int4 *>(out) + t * nv;
  for (int i = lane; i < nv; i += 64) {
    const bool two = i + 32 < nv;
    int4 v0[KM], v1[KM];
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      v0[k] = make_int4(0, 0, 0, 0);
      v1[k] = make_int4(0, 0, 0, 0);
      if (k < K && ((vm >> k) & 1)) {
        v0[k] = __ldcs(src + k * nv + i);
        if (two) v1[k] = __ldcs(src + k * nv + i + 32);
      }
    }
    float acc0[8], acc1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc0[u] = acc1[u] = 0.f;
#pragma unroll
    for (int k = 0; k < KM; ++k)
      if (k < K) {
        acc_bf16x8(acc0, v0[k]);
        acc_bf16x8(acc1, v1[k]);
      }
    __stcs(dst + i, pack_bf16x8(acc0));
    if (two) __stcs(dst + i + 32, pack_bf16x8(acc1));
  }
}

// ----------------------------------------------------------------------- host read-back
// Copies the plan blob, the layout summary and the error flags into mapped pinned host memory
// with plain stores (zero-copy), so the one host synchronisation of the layer never queues
// behind bulk copies that other streams have pending on the copy engines.
__global__ void mirror_kernel(const uint32_t *__restrict__ plan, int n_plan_words,
                              const uint32_t *__restrict__ summary, int n_sum_words,
                              const int32_t *__restrict__ err, uint32_t *__restrict__ host_plan,
                              uint32_t *__restrict__ host_sum, int32_t *__restrict__ host_err) {
  for (int i = threadIdx.x; i < n_plan_words; i += blockDim.x) host_plan[i] = plan[i];
  for (int i = threadIdx.x; i < n_sum_words; i += blockDim.x) host_sum[i] = summary[i];
  if (threadIdx.x < 4) host_err[threadIdx.x] = err[threadIdx.x];
}

}  // namespace

cudaError_t launch_zero_pad(const Group *groups, int n_groups, int D, uint16_t *buf0, uint16_t *buf1,
                            cudaStream_t s) {
  if (n_groups <= 0) return cudaSuccess;
  zero_pad_kernel<<<n_groups, 256, 0, s>>>(groups, D, buf0, buf1);
  return cudaGetLastError();
}

// dL/dw of each real received row from the fused dA0 + SwiGLU-backward epilogue's per-tile partial
// dot products <a, dA0> (nparts per row, summed in fixed order: deterministic); replaces the gate.
__global__ void dot_reduce_kernel(const Group *__restrict__ groups, int n_groups, int n_rows_total, int nparts,
                                  const float *__restrict__ dotp, float *__restrict__ gate_io) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows_total) return;
  int lo = 0, hi = n_groups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (groups[mid].row_base <= r) lo = mid;
    else hi = mid - 1;
  }
  const Group g = groups[lo];
  if (r < g.row_base || r >= g.row_base + g.n_rows) return;
  const float *q = dotp + (int64_t)r * nparts;
  float acc = 0.f;
  for (int j = 0; j < nparts; ++j) acc += q[j];
  gate_io[r] = acc;
}

cudaError_t launch_dot_reduce(const Group *groups, int n_groups, int n_rows_total, int nparts, const float *dotp,
                              float *gate_io, cudaStream_t s) {
  if (n_rows_total <= 0 || n_groups <= 0) return cudaSuccess;
  dot_reduce_kernel<<<(n_rows_total + 255) / 256, 256, 0, s>>>(groups, n_groups, n_rows_total, nparts, dotp,
                                                               gate_io);
  return cudaGetLastError();
}

cudaError_t launch_bwd_swiglu(const Group *groups, int n_groups, int n_rows_total, int H, const uint16_t *GU,
                              const uint16_t *dA0, float *gate_io, uint16_t *Aw, uint16_t *dGU, cudaStream_t s) {
  if (n_rows_total <= 0 || n_groups <= 0) return cudaSuccess;
  const int warps = 8;
  bwd_swiglu_kernel<<<(n_rows_total + warps - 1) / warps, warps * 32, 0, s>>>(groups, n_groups, n_rows_total, H,
                                                                            GU, dA0, gate_io, Aw, dGU);
  return cudaGetLastError();
}

cudaError_t launch_grad_reduce(float *dst, const float *base, int n_src, int64_t stride_floats, int64_t n_floats,
                               cudaStream_t s) {
  if (n_src <= 0) return cudaSuccess;
  grad_reduce_kernel<<<296, 256, 0, s>>>(dst, base, n_src, stride_floats / 4, n_floats / 4);
  return cudaGetLastError();
}

cudaError_t launch_signal(uint32_t *flag, const uint32_t *ep, cudaStream_t s) {
  signal_kernel<<<1, 1, 0, s>>>(flag, ep);
  return cudaGetLastError();
}

cudaError_t launch_wait_flag(const uint32_t *flag, const uint32_t *ep, int32_t *err, cudaStream_t s) {
  wait_flag_kernel<<<1, 1, 0, s>>>(flag, ep, err);
  return cudaGetLastError();
}

cudaError_t launch_push_level(const PushArgs &a, cudaStream_t s) {
  push_level_kernel<<<kPushBlocks, kPushThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_advance(uint32_t *ep, cudaStream_t s) {
  advance_kernel<<<1, 1, 0, s>>>(ep);
  return cudaGetLastError();
}

cudaError_t launch_combine_local(const uint16_t *slotbuf, int64_t B, int K, int D, const int32_t *slot_dst,
                                 uint16_t *out, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((B + kCombineWarps - 1) / kCombineWarps);
  if (K <= 2) combine_local_kernel<2><<<blocks, kCombineWarps * 32, 0, s>>>(slotbuf, B, K, D, slot_dst, out);
  else if (K <= 4) combine_local_kernel<4><<<blocks, kCombineWarps * 32, 0, s>>>(slotbuf, B, K, D, slot_dst, out);
  else if (K <= 8) combine_local_kernel<8><<<blocks, kCombineWarps * 32, 0, s>>>(slotbuf, B, K, D, slot_dst, out);
  else if (K <= 16) combine_local_kernel<16><<<blocks, kCombineWarps * 32, 0, s>>>(slotbuf, B, K, D, slot_dst, out);
  else combine_local_kernel<32><<<blocks, kCombineWarps * 32, 0, s>>>(slotbuf, B, K, D, slot_dst, out);
  return cudaGetLastError();
}

cudaError_t launch_mirror(const void *plan, size_t plan_bytes, const void *summary, size_t sum_bytes,
                          const int32_t *err, void *host_plan, void *host_sum, int32_t *host_err,
                          cudaStream_t s) {
  mirror_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const uint32_t *>(plan), (int)(plan_bytes / 4),
                                  reinterpret_cast<const uint32_t *>(summary), (int)(sum_bytes / 4), err,
                                  reinterpret_cast<uint32_t *>(host_plan), reinterpret_cast<uint32_t *>(host_sum),
                                  host_err);
  return cudaGetLastError();
}

cudaError_t launch_tile_count(const int32_t *ids, int64_t n_slots, int32_t N, int32_t *tile_cnt,
                              int32_t *err, cudaStream_t s) {
  const int n_tiles = (int)((n_slots + kTileSlots - 1) / kTileSlots);
  if (n_tiles == 0) return cudaSuccess;
  tile_count_kernel<<<n_tiles, kCountThreads, sizeof(int32_t) * N, s>>>(ids, n_slots, N, tile_cnt, err);
  return cudaGetLastError();
}

cudaError_t launch_tile_scan(const int32_t *tile_cnt, int32_t n_tiles, int32_t N, int32_t *tile_off,
                             int32_t *cnt, cudaStream_t s) {
  tile_scan_kernel<<<(N + 31) / 32, kScanWarps * 32, 0, s>>>(tile_cnt, n_tiles, N, tile_off, cnt);
  return cudaGetLastError();
}

cudaError_t launch_local_rank(const int32_t *ids, int64_t n_slots, int32_t N, const int32_t *tile_off,
                              int32_t *local_rank, int32_t *prep_ids, cudaStream_t s) {
  const int n_tiles = (int)((n_slots + kTileSlots - 1) / kTileSlots);
  if (n_tiles == 0) return cudaSuccess;
  const size_t smem = sizeof(int32_t) * kRankWarps * N;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(local_rank_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  local_rank_kernel<<<n_tiles, kRankThreads, smem, s>>>(ids, n_slots, N, tile_off, local_rank, prep_ids);
  return cudaGetLastError();
}

cudaError_t launch_push_counts(const int32_t *cnt, int32_t N, int32_t rank, int32_t P,
                               int32_t *const *peer_lm, cudaStream_t s) {
  push_counts_kernel<<<P, 256, 0, s>>>(cnt, N, rank, P, peer_lm);
  return cudaGetLastError();
}

cudaError_t launch_barrier(uint32_t *const *peer_flags, int32_t rank, int32_t P, uint32_t *ep,
                           int32_t *err, cudaStream_t s) {
  barrier_kernel<<<1, 32, 0, s>>>(peer_flags, rank, P, ep, err);
  return cudaGetLastError();
}

cudaError_t launch_arrive(uint32_t *const *peer_flags, int32_t rank, int32_t P, const uint32_t *ep, cudaStream_t s) {
  arrive_kernel<<<1, 32, 0, s>>>(peer_flags, rank, P, ep);
  return cudaGetLastError();
}

cudaError_t launch_dispatch(const DispatchArgs &a, cudaStream_t s) {
  if (a.B == 0) return a.peer_flags ? launch_arrive(a.peer_flags, a.rank, a.P, a.ep, s) : cudaSuccess;
  const int64_t blocks = (a.B + kDispatchWarps - 1) / kDispatchWarps;
  dispatch_kernel<<<(unsigned)blocks, kDispatchWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_combine(const CombineArgs &a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((a.B + kCombineWarps - 1) / kCombineWarps);
  if (a.K <= 2) combine_kernel<2><<<blocks, kCombineWarps * 32, 0, s>>>(a);
  else if (a.K <= 4) combine_kernel<4><<<blocks, kCombineWarps * 32, 0, s>>>(a);
  else if (a.K <= 8) combine_kernel<8><<<blocks, kCombineWarps * 32, 0, s>>>(a);
  else if (a.K <= 16) combine_kernel<16><<<blocks, kCombineWarps * 32, 0, s>>>(a);
  else combine_kernel<32><<<blocks, kCombineWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace llep
