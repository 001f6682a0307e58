// Device planner (Alg. 4 head + Alg. 2 LLA + Alg. 3 LLAS + 𝒲) and the per-device group layout.
//
// The planner is tiny (N <= 1024 experts, P <= 32 devices) but sits on the critical path of
// every layer, so it runs on the GPU next to the load exchange instead of on the host as in the
// paper's pure-Python LLA: one CTA sorts the experts (rank sort, all threads), then one
// warp runs the sequential LLA loop with device d's (g_a, g_p) held in lane d, so each LLAS
// candidate choice is a warp arg-min over lanes.  The only floating-point operations
// are m_α = (α·S)/P and the λ ratio max/(S/N), done with __dmul_rn/__ddiv_rn
// so they round exactly like the host planner (bit-identical plans, R1/R9).
#include <stdint.h>

#include <climits>

#include "common.cuh"

namespace llep {

namespace {

__device__ __forceinline__ long long warp_sum_ll(long long v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_max_ll(long long v) {
  for (int o = 16; o > 0; o >>= 1) {
    long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}
// arg-min of (key, lane) over the warp; lanes that do not compete pass key = LLONG_MAX.
__device__ __forceinline__ int warp_argmin(long long key) {
  int id = threadIdx.x & 31;
  for (int o = 16; o > 0; o >>= 1) {
    long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    int id2 = __shfl_xor_sync(0xffffffffu, id, o);
    if (k2 < key || (k2 == key && id2 < id)) {
      key = k2;
      id = id2;
    }
  }
  return id;
}

constexpr int kPlanThreads = 256;

__global__ void __launch_bounds__(kPlanThreads) planner_kernel(
    const int32_t *__restrict__ C, int N, int P, double alpha, long long m, double lambda,
    int force_ep, uint8_t *__restrict__ plan) {
  extern __shared__ long long sm_l[];           // l[N]
  int *sm_order = reinterpret_cast<int *>(sm_l + N);
  __shared__ long long red[2][kPlanThreads / 32];
  __shared__ unsigned long long sm_assigned[kMaxWorld];
  __shared__ int sm_ntransfer;

  const PlanLayout L = plan_layout(N, P);
  llep_plan_header *hdr = reinterpret_cast<llep_plan_header *>(plan);
  long long *assigned = reinterpret_cast<long long *>(plan + L.off_assigned);
  int32_t *n_chunks = reinterpret_cast<int32_t *>(plan + L.off_n_chunks);
  llep_chunk *chunks = reinterpret_cast<llep_chunk *>(plan + L.off_chunks);
  uint8_t *replica = plan + L.off_replica;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int MC = P + 1;
  const int M = N / P;

  // zero the plan body
  for (size_t i = tid * 4; i < L.bytes; i += kPlanThreads * 4)
    *reinterpret_cast<uint32_t *>(plan + i) = 0u;
  if (tid < kMaxWorld) sm_assigned[tid] = 0ull;
  if (tid == 0) sm_ntransfer = 0;
  // l <- sum of loads of global experts across all GPUs (Alg. 4)
  long long s_loc = 0, m_loc = 0;
  for (int e = tid; e < N; e += kPlanThreads) {
    long long v = 0;
    for (int p = 0; p < P; ++p) v += C[(size_t)p * N + e];
    sm_l[e] = v;
    s_loc += v;
    m_loc = v > m_loc ? v : m_loc;
  }
  s_loc = warp_sum_ll(s_loc);
  m_loc = warp_max_ll(m_loc);
  if (lane == 0) {
    red[0][warp] = s_loc;
    red[1][warp] = m_loc;
  }
  __syncthreads();
  long long S = 0, maxl = 0;
  for (int w = 0; w < kPlanThreads / 32; ++w) {
    S += red[0][w];
    maxl = red[1][w] > maxl ? red[1][w] : maxl;
  }
  // m_α = α × (1/P) × Σ l, evaluated (α·S)/P and floored once (R1)
  const long long cap = (long long)floor(__ddiv_rn(__dmul_rn(alpha, (double)S), (double)P));
  // λ test: balanced iff max(l)/mean(l) < λ; S == 0 counts as balanced (R9)
  bool fallback = (S == 0) ||
                  (__ddiv_rn((double)maxl, __ddiv_rn((double)S, (double)N)) < lambda);
  // If cap >= every device's native load, every expert is Case 1 of Alg. 2: LLA's plan
  // is the all-native one (exactly; the sequential loop is skipped).  Not a λ fallback.
  bool all_case1 = false;
  if (!force_ep && !fallback) {
    long long gmax = 0;
    for (int d = 0; d < P; ++d) {
      long long gn = 0;
      for (int e = d * M; e < (d + 1) * M; ++e) gn += sm_l[e];
      gmax = gn > gmax ? gn : gmax;
    }
    all_case1 = cap >= gmax;
  }
  const bool native_only = force_ep || fallback || all_case1;

  if (native_only) {
    // standard EP (Alg. 1) / λ fallback: every expert's load on its native device
    for (int e = tid; e < N; e += kPlanThreads) {
      long long le = sm_l[e];
      if (le > 0) {
        llep_chunk c;
        c.device = e / M;
        c.start = 0;
        c.end = (int32_t)le;
        chunks[(size_t)e * MC] = c;
        n_chunks[e] = 1;
        atomicAdd(&sm_assigned[e / M], (unsigned long long)le);
      }
    }
    __syncthreads();
  } else {
    // sort(l, decreasing), ties -> lower expert id (R5): rank sort
    for (int e = tid; e < N; e += kPlanThreads) {
      long long le = sm_l[e];
      int r = 0;
      for (int j = 0; j < N; ++j) {
        long long lj = sm_l[j];
        r += (lj > le) || (lj == le && j < e);
      }
      sm_order[r] = e;
    }
    __syncthreads();
    if (warp == 0) {
      // lane d holds device d's native-pending g_p and assigned g_a
      long long gp = 0, ga = 0;
      if (lane < P)
        for (int e = lane * M; e < (lane + 1) * M; ++e) gp += sm_l[e];
      int forces = 0;
      for (int idx = 0; idx < N; ++idx) {
        const int e = sm_order[idx];
        const long long le = sm_l[e];
        if (le == 0) break;                                   // R6: zero-load experts, no chunk
        const int ng = e / M;
        if (lane == ng) gp -= le;
        const long long na = cap - __shfl_sync(0xffffffffu, ga, ng) -
                             __shfl_sync(0xffffffffu, gp, ng);
        llep_chunk *A = chunks + (size_t)e * MC;
        int nc = 0;
        long long r, to;
        if (na >= le) {                                       // Case 1
          if (lane == 0) A[0] = llep_chunk{ng, 0, (int32_t)le};
          if (lane == ng) ga += le;
          nc = 1;
          r = 0;
          to = le;
        } else if (na > 0) {                                  // Case 2, R2
          if (lane == 0) A[0] = llep_chunk{ng, 0, (int32_t)na};
          if (lane == ng) ga += na;
          nc = 1;
          r = le - na;
          to = na;
        } else {                                              // Case 3
          r = le;
          to = 0;
        }
        // LLAS (Alg. 3)
        while (r > 0) {
          const bool cand = lane < P && lane != ng;
          const long long load = ga + gp;                     // sort key of P:492
          long long c = cap - load;
          c = c < r ? c : r;
          const bool ok = cand && c > 0 && !(c < m && r > c); // R3
          const unsigned okmask = __ballot_sync(0xffffffffu, ok);
          int sel;
          long long csel;
          if (okmask) {                                       // first acceptable in order (R4)
            sel = warp_argmin(ok ? load : LLONG_MAX);
            csel = __shfl_sync(0xffffffffu, c, sel);
          } else {                                            // force-assign o[0]
            sel = warp_argmin(cand ? load : LLONG_MAX);
            csel = r;
            ++forces;
          }
          if (lane == 0) A[nc] = llep_chunk{sel, (int32_t)to, (int32_t)(to + csel)};
          if (lane == sel) ga += csel;
          ++nc;
          r -= csel;
          to += csel;
        }
        if (lane == 0) n_chunks[e] = nc;
      }
      if (lane < P) sm_assigned[lane] = (unsigned long long)ga;
      if (lane == 0) hdr->force_count = forces;
    }
    __syncthreads();
  }
  // 𝒲: replica[e][d] = 1 iff e has a chunk on d != native(e)
  for (int e = tid; e < N; e += kPlanThreads) {
    const int ng = e / M;
    int cnt = 0;
    for (int c = 0; c < n_chunks[e]; ++c) {
      int d = chunks[(size_t)e * MC + c].device;
      if (d != ng && !replica[(size_t)e * P + d]) {
        replica[(size_t)e * P + d] = 1;
        ++cnt;
      }
    }
    if (cnt) atomicAdd(&sm_ntransfer, cnt);
  }
  __syncthreads();
  if (tid == 0) {
    long long mx = 0;
    for (int d = 0; d < P; ++d) {
      long long a = (long long)sm_assigned[d];
      assigned[d] = a;
      mx = a > mx ? a : mx;
    }
    hdr->n_experts = N;
    hdr->world_size = P;
    hdr->max_chunks = MC;
    hdr->fallback_ep = (!force_ep && fallback) ? 1 : 0;
    if (native_only) hdr->force_count = 0;
    hdr->n_transfers = sm_ntransfer;
    hdr->total = S;
    hdr->capacity = cap;
    hdr->max_assigned = mx;
    hdr->off_assigned = L.off_assigned;
    hdr->off_n_chunks = L.off_n_chunks;
    hdr->off_chunks = L.off_chunks;
    hdr->off_replica = L.off_replica;
  }
}

// ---------------------------------------------------------------------------------- layout
// Per device d: expert groups = native experts of d with rows on d (ascending id), then the
// foreign experts S_d (ascending id); each group's rows = e's chunks on d concatenated in plan
// order, starting at a 128-aligned row base.  Every rank computes every device's layout from
// the replicated plan, so dispatch can address peers' receive rows without a handshake.
constexpr int kLayoutThreads = 1024;

__global__ void __launch_bounds__(kLayoutThreads) layout_kernel(LayoutArgs a) {
  const int N = a.N, P = a.P, M = a.M, MC = P + 1;
  const uint8_t *plan = reinterpret_cast<const uint8_t *>(a.plan);
  const PlanLayout L = plan_layout(N, P);
  const llep_plan_header *hdr = reinterpret_cast<const llep_plan_header *>(plan);
  const int32_t *n_chunks = reinterpret_cast<const int32_t *>(plan + L.off_n_chunks);
  const llep_chunk *chunks = reinterpret_cast<const llep_chunk *>(plan + L.off_chunks);
  const long long *assigned = reinterpret_cast<const long long *>(plan + L.off_assigned);
  __shared__ int sm_err;
  __shared__ int sm_groups, sm_mblocks;
  __shared__ int sm_before[kMaxGroups];  // blocks of the same class in earlier groups
  __shared__ int sm_nbig, sm_nsmall;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) sm_err = 0;
  __syncthreads();
  // rows of e on each device + plan/load consistency (chunk totals == l_e)
  for (int e = tid; e < N; e += kLayoutThreads) {
    int32_t *ro = a.rows_on + (size_t)e * P;
    for (int d = 0; d < P; ++d) ro[d] = 0;
    long long le = 0;
    for (int p = 0; p < P; ++p) le += a.load_matrix[(size_t)p * N + e];
    long long tot = 0, expect = 0;
    const int nc = n_chunks[e];
    bool bad = nc < 0 || nc > MC;
    for (int c = 0; c < nc && !bad; ++c) {
      llep_chunk ch = chunks[(size_t)e * MC + c];
      if (ch.device < 0 || ch.device >= P || ch.start != expect || ch.end <= ch.start) bad = true;
      else {
        ro[ch.device] += ch.end - ch.start;
        tot += ch.end - ch.start;
        expect = ch.end;
      }
    }
    if (bad || tot != le) atomicOr(&sm_err, 1);
  }
  __syncthreads();
  // group scan, one warp per device
  for (int d = warp; d < P; d += kLayoutThreads / 32) {
    int run_rows = 0, run_groups = 0, run_mblk = 0, n_foreign = 0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int base = 0; base < N; base += 32) {
        const int e = base + lane;
        const bool native = (e / M) == d;
        const bool in = e < N && (pass == 0 ? native : !native);
        const int rows = in ? a.rows_on[(size_t)e * P + d] : 0;
        const bool has = rows > 0;
        const int ra = a.row_align;
        const int padded = (rows + ra - 1) / ra * ra;
        const int mblk = padded / ra;
        int inc = padded, incm = mblk;
        for (int o = 1; o < 32; o <<= 1) {
          int u = __shfl_up_sync(0xffffffffu, inc, o);
          int um = __shfl_up_sync(0xffffffffu, incm, o);
          if (lane >= o) {
            inc += u;
            incm += um;
          }
        }
        const unsigned hm = __ballot_sync(0xffffffffu, has);
        const int gidx = run_groups + __popc(hm & ((1u << lane) - 1u));
        const int row_base = run_rows + inc - padded;
        const int fslot = n_foreign + __popc(hm & ((1u << lane) - 1u));
        if (e < N && in) {
          a.foreign_slot[(size_t)e * P + d] = (pass == 1 && has) ? fslot : -1;
        }
        if (has && d == a.rank && gidx < kMaxGroups) {
          Group g;
          g.expert = e;
          g.wslot = pass == 0 ? e - d * M : -1 - fslot;
          g.row_base = row_base;
          g.n_rows = rows;
          g.mblk_start = run_mblk + incm - mblk;
          g.pad[0] = g.pad[1] = g.pad[2] = 0;
          a.groups[gidx] = g;
        }
        // rows_on[e][d] is not needed past this point: keep the group's row base there, encoded
        // as -(base+1) so chunk_row below can read it
        if (has) a.rows_on[(size_t)e * P + d] = -(row_base + 1);
        run_rows += __shfl_sync(0xffffffffu, inc, 31);
        run_mblk += __shfl_sync(0xffffffffu, incm, 31);
        run_groups += __popc(hm);
        if (pass == 1) n_foreign += __popc(hm);
      }
    }
    if (lane == 0) {
      a.dev_padded[d] = run_rows;
      a.dev_foreign[d] = n_foreign;
      if (d == a.rank) {
        sm_groups = run_groups;
        sm_mblocks = run_mblk;
      }
    }
  }
  __syncthreads();
  // m-block schedule of this rank's grouped GEMMs: small groups interleaved among big ones.
  // Warp 0 scans the groups' block counts per class (big / small) 32 groups at a time.
  if (warp == 0) {
    const int G = sm_groups < kMaxGroups ? sm_groups : kMaxGroups;
    int nb = 0, ns = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      int mb = 0;
      bool big = false;
      if (g < G) {
        mb = (a.groups[g].n_rows + a.row_align - 1) / a.row_align;
        big = mb * a.row_align > kSmallGroupRows;
      }
      int ib = big ? mb : 0, is = big ? 0 : mb;
      for (int o = 1; o < 32; o <<= 1) {
        const int ub = __shfl_up_sync(0xffffffffu, ib, o), us = __shfl_up_sync(0xffffffffu, is, o);
        if (lane >= o) {
          ib += ub;
          is += us;
        }
      }
      if (g < G) sm_before[g] = big ? nb + ib - mb : ns + is - mb;
      nb += __shfl_sync(0xffffffffu, ib, 31);
      ns += __shfl_sync(0xffffffffu, is, 31);
    }
    if (lane == 0) {
      sm_nbig = nb;
      sm_nsmall = ns;
    }
  }
  __syncthreads();
  if (sm_mblocks <= a.sched_cap && sm_groups <= kMaxGroups) {
    for (int mb = tid; mb < sm_mblocks; mb += kLayoutThreads) {
      int lo = 0, hi = sm_groups - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.groups[mid].mblk_start <= mb) lo = mid;
        else hi = mid - 1;
      }
      const Group g = a.groups[lo];
      const int m = mb - g.mblk_start;
      const bool big = (g.n_rows + a.row_align - 1) / a.row_align * a.row_align > kSmallGroupRows;
      const int64_t pos = interleave_pos(big, sm_before[lo] + m, sm_nbig, sm_nsmall);
      a.sched[pos] = sched_pack(lo, m);
    }
  }
  // row f2: sources of every m-block of this rank (group order).  Group rows are e's chunks on this
  // device in plan order; a chunk (d, s, t) holds global indices [s, t) of e, and source q owns
  // [off_q, off_q + C[q][e]) of them (off_q = source_offset: rank-major R11 or chunk-aligned R11'), so the
  // block's rows map to
  // global ranges whose overlap with each source's range decides the mask.
  if (a.mblk_src && sm_mblocks <= a.sched_cap && sm_groups <= kMaxGroups) {
    for (int mb = tid; mb < sm_mblocks; mb += kLayoutThreads) {
      int lo = 0, hi = sm_groups - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.groups[mid].mblk_start <= mb) lo = mid;
        else hi = mid - 1;
      }
      const Group g = a.groups[lo];
      const int r0 = (mb - g.mblk_start) * a.row_align;
      const int r1 = min(r0 + a.row_align, g.n_rows);
      const int e = g.expert;
      uint32_t mask = 0;
      int off = 0;
      for (int c = 0; c < n_chunks[e] && c < MC; ++c) {
        const llep_chunk ch = chunks[(size_t)e * MC + c];
        if (ch.device != a.rank) continue;
        const int len = ch.end - ch.start;
        const int x0 = max(r0, off), x1 = min(r1, off + len);
        if (x0 < x1) {
          const long long g0 = ch.start + (x0 - off), g1 = ch.start + (x1 - off);   // global [g0, g1)
          for (int q = 0; q < P; ++q) {
            const long long nq = a.load_matrix[(size_t)q * N + e];
            const long long cum = source_offset(chunks + (size_t)e * MC, n_chunks[e], a.load_matrix, N, P, e, q,
                                                a.aligned);
            if (nq > 0 && cum < g1 && cum + nq > g0) mask |= 1u << q;
          }
        }
        off += len;
      }
      a.mblk_src[mb] = mask;
    }
  }
  // destination row of each chunk's first token: group base + rows of e's earlier chunks on d
  for (int e = tid; e < N; e += kLayoutThreads) {
    const int nc = n_chunks[e];
    for (int c = 0; c < nc && c < MC; ++c) {
      llep_chunk ch = chunks[(size_t)e * MC + c];
      if (ch.device < 0 || ch.device >= P) continue;
      int off = 0;
      for (int c2 = 0; c2 < c; ++c2) {
        llep_chunk q = chunks[(size_t)e * MC + c2];
        if (q.device == ch.device) off += q.end - q.start;
      }
      const int enc = a.rows_on[(size_t)e * P + ch.device];
      a.chunk_row[(size_t)e * MC + c] = (-enc - 1) + off;
    }
  }
  __syncthreads();
  if (tid == 0) {
    LayoutSummary s;
    long long mx = 0;
    int mf = 0;
    for (int d = 0; d < P; ++d) {
      mx = a.dev_padded[d] > mx ? a.dev_padded[d] : mx;
      mf = a.dev_foreign[d] > mf ? a.dev_foreign[d] : mf;
    }
    s.rows_needed = mx;
    s.my_rows = assigned[a.rank];
    s.my_padded = a.dev_padded[a.rank];
    s.foreign_needed = mf;
    s.my_groups = sm_groups;
    s.my_mblocks = sm_mblocks;
    s.fallback_ep = hdr->fallback_ep;
    s.force_count = hdr->force_count;
    s.n_transfers = hdr->n_transfers;
    s.error = sm_err | (sm_groups > kMaxGroups ? 2 : 0) | (sm_mblocks > a.sched_cap ? 8 : 0);
    // capture-safe layer: the arena this call runs in must hold every device's rows (same on all ranks)
    if (a.arena_rows > 0 && (mx > a.arena_rows || mf > a.arena_foreign)) s.error |= 16;
    s.pad = 0;
    *a.summary = s;
    if (a.n_groups_dev) *a.n_groups_dev = s.error ? 0 : sm_groups;
    if (a.err && s.error) atomicOr(a.err + 3, (s.error & 16) ? 1 : 2);
  }
}

}  // namespace

cudaError_t launch_planner(const int32_t *load_matrix, int32_t N, int32_t P, double alpha,
                           int64_t min_chunk, double lambda, int32_t force_ep, void *plan,
                           cudaStream_t s) {
  size_t smem = sizeof(long long) * N + sizeof(int) * N;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(planner_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  planner_kernel<<<1, kPlanThreads, smem, s>>>(load_matrix, N, P, alpha, (long long)min_chunk,
                                               lambda, force_ep, reinterpret_cast<uint8_t *>(plan));
  return cudaGetLastError();
}

cudaError_t launch_layout(const LayoutArgs &a, cudaStream_t s) {
  layout_kernel<<<1, kLayoutThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace llep
