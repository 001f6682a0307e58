// C ABI of the LLEP hot path (include/llep.h): host planner, per-rank context with a CUDA-IPC
// symmetric arena, and the two stream-ordered calls llep_prepare / llep_moe_forward.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"

namespace llep {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

llep_status cuda_status(cudaError_t e, const char *what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? LLEP_ERR_NOMEM : LLEP_ERR_CUDA;
}

static llep_status invalid(const char *msg) {
  set_error("%s", msg);
  return LLEP_ERR_INVALID;
}

static llep_status check_params(const llep_params *p) {
  if (!p) return invalid("params is null");
  if (!(p->alpha >= 1.0)) return invalid("alpha < 1");
  if (!(p->lambda >= 1.0)) return invalid("lambda < 1");
  if (p->min_chunk < 0) return invalid("min_chunk < 0");
  return LLEP_OK;
}

static llep_status check_np(int32_t N, int32_t P) {
  if (P < 1 || N < 1) return invalid("N and P must be >= 1");
  if (N % P != 0) return invalid("N not divisible by P");
  if (N > kMaxGroups) return invalid("N > 1024 experts is not supported");
  return LLEP_OK;
}

// ------------------------------------------------------------------ host planner
// Sequential twin of planner_kernel (plan.cu); same decisions, same IEEE double operations.
static void host_plan(const int64_t *l, int32_t N, int32_t P, const llep_params *prm,
                      bool force_ep, uint8_t *blob) {
  const PlanLayout L = plan_layout(N, P);
  memset(blob, 0, L.bytes);
  llep_plan_header *hdr = reinterpret_cast<llep_plan_header *>(blob);
  int64_t *assigned = reinterpret_cast<int64_t *>(blob + L.off_assigned);
  int32_t *n_chunks = reinterpret_cast<int32_t *>(blob + L.off_n_chunks);
  llep_chunk *chunks = reinterpret_cast<llep_chunk *>(blob + L.off_chunks);
  uint8_t *replica = blob + L.off_replica;
  const int MC = P + 1, M = N / P;
  int64_t S = 0, maxl = 0;
  for (int e = 0; e < N; ++e) {
    S += l[e];
    maxl = std::max(maxl, l[e]);
  }
  volatile double prod = prm->alpha * (double)S;  // volatile: one rounding per operation
  volatile double mal = prod / (double)P;
  const int64_t cap = (int64_t)std::floor((double)mal);
  bool fallback = (S == 0);
  if (!fallback) {
    volatile double mean = (double)S / (double)N;
    volatile double ratio = (double)maxl / (double)mean;
    fallback = ratio < prm->lambda;
  }
  int forces = 0;
  std::vector<int64_t> ga(P, 0), gp(P, 0);
  if (force_ep || fallback) {
    for (int e = 0; e < N; ++e)
      if (l[e] > 0) {
        chunks[(size_t)e * MC] = llep_chunk{e / M, 0, (int32_t)l[e]};
        n_chunks[e] = 1;
        ga[e / M] += l[e];
      }
  } else {
    std::vector<int> order(N);
    for (int e = 0; e < N; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return l[a] > l[b]; });
    for (int e = 0; e < N; ++e) gp[e / M] += l[e];
    for (int idx = 0; idx < N; ++idx) {
      const int e = order[idx];
      const int64_t le = l[e];
      if (le == 0) break;
      const int ng = e / M;
      gp[ng] -= le;
      const int64_t na = cap - ga[ng] - gp[ng];
      llep_chunk *A = chunks + (size_t)e * MC;
      int nc = 0;
      int64_t r, to;
      if (na >= le) {
        A[nc++] = llep_chunk{ng, 0, (int32_t)le};
        ga[ng] += le;
        r = 0;
        to = le;
      } else if (na > 0) {
        A[nc++] = llep_chunk{ng, 0, (int32_t)na};
        ga[ng] += na;
        r = le - na;
        to = na;
      } else {
        r = le;
        to = 0;
      }
      while (r > 0) {
        int sel = -1, force_sel = -1;
        int64_t csel = 0, best = 0, fbest = 0;
        for (int o = 0; o < P; ++o) {
          if (o == ng) continue;
          const int64_t load = ga[o] + gp[o];
          if (force_sel < 0 || load < fbest) {
            force_sel = o;
            fbest = load;
          }
          const int64_t c = std::min(r, cap - load);
          if (c <= 0 || (c < prm->min_chunk && r > c)) continue;
          if (sel < 0 || load < best) {
            sel = o;
            best = load;
            csel = c;
          }
        }
        if (sel < 0) {
          sel = force_sel;
          csel = r;
          ++forces;
        }
        A[nc++] = llep_chunk{sel, (int32_t)to, (int32_t)(to + csel)};
        ga[sel] += csel;
        r -= csel;
        to += csel;
      }
      n_chunks[e] = nc;
    }
  }
  int ntr = 0;
  for (int e = 0; e < N; ++e)
    for (int c = 0; c < n_chunks[e]; ++c) {
      const int d = chunks[(size_t)e * MC + c].device;
      if (d != e / M && !replica[(size_t)e * P + d]) {
        replica[(size_t)e * P + d] = 1;
        ++ntr;
      }
    }
  int64_t mx = 0;
  for (int d = 0; d < P; ++d) {
    assigned[d] = ga[d];
    mx = std::max(mx, ga[d]);
  }
  hdr->n_experts = N;
  hdr->world_size = P;
  hdr->max_chunks = MC;
  hdr->fallback_ep = (!force_ep && fallback) ? 1 : 0;
  hdr->force_count = (force_ep || fallback) ? 0 : forces;
  hdr->n_transfers = ntr;
  hdr->total = S;
  hdr->capacity = cap;
  hdr->max_assigned = mx;
  hdr->off_assigned = L.off_assigned;
  hdr->off_n_chunks = L.off_n_chunks;
  hdr->off_chunks = L.off_chunks;
  hdr->off_replica = L.off_replica;
}

}  // namespace llep

using namespace llep;

// ====================================================================== context
struct llep_context {
  int32_t N, K, D, H, P, M, rank, device, num_sms;
  int32_t row_align = 256;  // 256: 2-CTA GEMM tiles; 128: 1-CTA tiles (LLEP_ROW_ALIGN=128)
  int32_t token_order = LLEP_ORDER_CHUNK_ALIGNED;   // a3/a5 global token order (llep_context_set_token_order)
  int64_t mem_cap = 0;      // 0: no cap on scratch + arena + activations
  int64_t max_tokens;
  // rank-local scratch
  int32_t *tile_cnt = nullptr, *tile_off = nullptr, *cnt = nullptr, *local_rank = nullptr;
  int32_t *slot_dst = nullptr, *err = nullptr, *lm_local = nullptr;
  int32_t *prep_ids = nullptr;            // [max_tokens*K] the ids of the last llep_prepare
  int32_t *rows_on = nullptr, *chunk_row = nullptr, *foreign_slot = nullptr;
  int32_t *dev_padded = nullptr, *dev_foreign = nullptr;
  Group *groups = nullptr;
  int32_t *sched = nullptr;
  uint32_t *mblk_src = nullptr;           // [sched_cap] row f2: sources of each m-block
  uint32_t *block_done = nullptr;         // dispatch_kernel's finished-block count
  int64_t sched_cap = 0;
  LayoutSummary *summary = nullptr;
  LayoutSummary *summary_host = nullptr;  // mapped pinned (written by mirror_kernel)
  int32_t *err_host = nullptr;            // mapped pinned
  uint8_t *plan_mirror = nullptr;         // mapped pinned, plan blob bytes
  uint16_t *act = nullptr;                // A [arena_rows, H]
  int32_t *rtok = nullptr;                // [arena_rows] token of each gathered receive row (a6 local rows)
  size_t scratch_bytes = 0;
  // symmetric arena
  uint8_t *arena = nullptr;
  size_t arena_bytes = 0;
  int64_t arena_rows = 0;
  int32_t arena_foreign = 0;
  size_t off_flags = 0, off_lm = 0, off_x = 0, off_g = 0, off_w13 = 0, off_w2 = 0;
  size_t off_rsrc = 0, off_slot = 0;   // receive-row sources; slot buffer [max_tokens*K, D] (last)
  // backward (row f1): arena regions O [R, D] bf16 + returned weight-gradient slots, local buffers
  bool backward = false;
  int32_t arena_grad = 0;
  size_t off_o = 0, off_grad = 0;
  uint16_t *gu = nullptr, *da0 = nullptr, *aw = nullptr, *dgu = nullptr;
  float *stage13 = nullptr, *stage2 = nullptr;
  float *dotp = nullptr;    // fused dA0 + SwiGLU backward: partial <a, dA0> per (row, half tile)
  int64_t dotp_cap = 0;     // floats
  float *wsbuf = nullptr;   // split-K partials of the weight-gradient GEMMs
  int64_t ws_cap = 0;       // floats
  uint8_t *peer_base[kMaxWorld] = {};
  bool peer_opened[kMaxWorld] = {};
  bool peers_ready = false;
  void **d_ptrs = nullptr;  // device: flags[P], lm[P], x[P], g[P], o[P], grad[P], rsrc[P], slot[P], w13[P], w2[P]
  uint32_t *ep = nullptr;   // device epochs [4] (common.cuh kEp*): barrier, weight flags, dispatch arrivals
  int32_t *ngroups_dev = nullptr;   // capture-safe layer: this rank's group count (0 on arena overflow)
  uint32_t *push_cnt = nullptr;     // capture-safe layer: [kMaxPushItems] chunk counts of the GPU weight push
  // host copy of the last prepared plan
  std::vector<uint8_t> plan_host;
  const void *plan_dev_cached = nullptr;
  int64_t prepared_tokens = -1;
  const int32_t *prepared_ids = nullptr;  // caller's topk_ids pointer of the last llep_prepare
  size_t lazy_bytes = 0;                  // backward workspaces grown on demand (wsbuf, dotp)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // measurement
  bool timing = false, pending = false;
  bool in_layer = false;    // inside llep_moe_layer (capture-safe: no phase events, no host reads)
  cudaEvent_t mark[9] = {};
  double phase_ms[LLEP_NUM_PHASES] = {};
  int64_t calls = 0, launches = 0, gemm_rows = 0, pending_rows = 0;
};

static void mark(llep_context *c, int i, cudaStream_t s) {
  if (c->timing && !c->in_layer) cudaEventRecord(c->mark[i], s);
}

// fold the events of the last completed prepare+forward into the totals
static void collect(llep_context *c) {
  if (!c->pending) return;
  cudaEventSynchronize(c->mark[8]);
  static const int from[LLEP_NUM_PHASES] = {0, 1, 2, 4, 5, 6, 7};
  for (int p = 0; p < LLEP_NUM_PHASES; ++p) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->mark[from[p]], c->mark[from[p] + 1]);
    c->phase_ms[p] += ms;
  }
  c->calls += 1;
  c->gemm_rows += c->pending_rows;
  c->pending = false;
}

// Geometry record at the start of every arena.  Peers address each other's regions with their OWN
// offsets, so every rank's arena must have the same geometry; llep_context_open_peers reads each peer's
// record through the peer mapping and refuses asymmetric arenas (different max_tokens, shape, reserve
// or backward setting on some rank) instead of letting peer stores land at wrong addresses.
struct ArenaGeometry {
  int64_t arena_bytes, arena_rows, max_tokens;
  int32_t arena_foreign, arena_grad, backward, N, K, D, H, P, row_align, magic;
};
constexpr int32_t kGeomMagic = 0x4c4c4550;   // "LLEP"
constexpr size_t kGeomBytes = 256;

static ArenaGeometry geometry(const llep_context *c);

static void layout_offsets(llep_context *c, int64_t rows, int32_t foreign) {
  size_t off = kGeomBytes;
  c->off_flags = off;
  off += 4 * kFlagWords;
  c->off_lm = off;
  off = align8(off + sizeof(int32_t) * (size_t)c->P * c->N);
  off = (off + 1023) & ~size_t(1023);
  c->off_x = off;
  off += (size_t)rows * c->D * 2;
  off = (off + 1023) & ~size_t(1023);
  c->off_g = off;
  off += (size_t)rows * 4;
  off = (off + 1023) & ~size_t(1023);
  c->off_rsrc = off;
  off += (size_t)rows * 4;
  off = (off + 1023) & ~size_t(1023);
  c->off_w13 = off;
  off += (size_t)foreign * 2 * c->H * c->D * 2;
  off = (off + 1023) & ~size_t(1023);
  c->off_w2 = off;
  off += (size_t)foreign * c->D * c->H * 2;
  off = (off + 1023) & ~size_t(1023);
  c->off_o = off;
  if (c->backward) off += (size_t)rows * c->D * 2;
  off = (off + 1023) & ~size_t(1023);
  c->off_grad = off;
  if (c->backward) off += (size_t)c->arena_grad * 3 * c->H * c->D * 4;
  off = (off + 1023) & ~size_t(1023);
  c->off_slot = off;   // slot buffer [max_tokens*K, D] (max_tokens is identical on every rank)
  off += (size_t)std::max<int64_t>(c->max_tokens, 1) * c->K * c->D * 2;
  c->arena_bytes = (off + 4095) & ~size_t(4095);
}

static size_t bwd_local_bytes(const llep_context *c, int64_t rows, int32_t foreign) {
  if (!c->backward) return 0;
  return (size_t)rows * c->H * 2 * 6 + (size_t)foreign * 3 * c->H * c->D * 4;
}

static ArenaGeometry geometry(const llep_context *c) {
  ArenaGeometry g;
  memset(&g, 0, sizeof(g));
  g.arena_bytes = (int64_t)c->arena_bytes;
  g.arena_rows = c->arena_rows;
  g.max_tokens = c->max_tokens;
  g.arena_foreign = c->arena_foreign;
  g.arena_grad = c->arena_grad;
  g.backward = c->backward ? 1 : 0;
  g.N = c->N; g.K = c->K; g.D = c->D; g.H = c->H; g.P = c->P;
  g.row_align = c->row_align;
  g.magic = kGeomMagic;
  return g;
}

// every device byte the context holds: arena + scratch + activations + backward buffers + lazily
// grown backward workspaces
static size_t held_bytes(const llep_context *c) {
  return c->arena_bytes + c->scratch_bytes + (size_t)c->arena_rows * (c->H * 2 + 4) +
         bwd_local_bytes(c, c->arena_rows, c->arena_foreign) + c->lazy_bytes;
}

static void close_peers(llep_context *c) {
  for (int q = 0; q < c->P; ++q) {
    if (c->peer_opened[q] && c->peer_base[q]) cudaIpcCloseMemHandle(c->peer_base[q]);
    c->peer_opened[q] = false;
    c->peer_base[q] = nullptr;
  }
  c->peers_ready = false;
}

constexpr int kPeerPtrArrays = 10;

static llep_status upload_peer_ptrs(llep_context *c) {
  std::vector<void *> h(kPeerPtrArrays * c->P);
  for (int q = 0; q < c->P; ++q) {
    uint8_t *b = c->peer_base[q];
    h[q] = b + c->off_flags;
    h[c->P + q] = b + c->off_lm;
    h[2 * c->P + q] = b + c->off_x;
    h[3 * c->P + q] = b + c->off_g;
    h[4 * c->P + q] = b + c->off_o;
    h[5 * c->P + q] = b + c->off_grad;
    h[6 * c->P + q] = b + c->off_rsrc;
    h[7 * c->P + q] = b + c->off_slot;
    h[8 * c->P + q] = b + c->off_w13;
    h[9 * c->P + q] = b + c->off_w2;
  }
  LLEP_CUDA(cudaMemcpy(c->d_ptrs, h.data(), sizeof(void *) * kPeerPtrArrays * c->P, cudaMemcpyHostToDevice));
  return LLEP_OK;
}

static llep_status alloc_arena(llep_context *c, int64_t rows, int32_t foreign) {
  rows = std::max<int64_t>(rows, kRowAlign);
  foreign = std::max(foreign, 1);
  if (c->mem_cap > 0) {
    llep_context probe_sizes;  // offsets only
    probe_sizes.N = c->N; probe_sizes.D = c->D; probe_sizes.H = c->H; probe_sizes.P = c->P;
    probe_sizes.K = c->K; probe_sizes.max_tokens = c->max_tokens;
    layout_offsets(&probe_sizes, rows, foreign);
    probe_sizes.backward = c->backward;
    probe_sizes.arena_grad = c->arena_grad;
    layout_offsets(&probe_sizes, rows, foreign);
    const int64_t need = (int64_t)(probe_sizes.arena_bytes + c->scratch_bytes + (size_t)rows * (c->H * 2 + 4) +
                                   bwd_local_bytes(c, rows, foreign) + c->lazy_bytes);
    if (need > c->mem_cap) {
      set_error("memory cap: the plan needs %.2f GB on this device (arena + activations + scratch), "
                "cap %.2f GB", need / 1e9, c->mem_cap / 1e9);
      return LLEP_ERR_NOMEM;
    }
  }
  close_peers(c);
  if (c->arena) cudaFree(c->arena);
  if (c->act) cudaFree(c->act);
  if (c->rtok) cudaFree(c->rtok);
  c->rtok = nullptr;
  void *bufs[] = {c->gu, c->da0, c->aw, c->dgu, c->stage13, c->stage2};
  for (void *b : bufs)
    if (b) cudaFree(b);
  c->gu = c->da0 = c->aw = c->dgu = nullptr;
  c->stage13 = c->stage2 = nullptr;
  c->arena = nullptr;
  c->act = nullptr;
  layout_offsets(c, rows, foreign);
  LLEP_CUDA(cudaMalloc(&c->arena, c->arena_bytes));
  LLEP_CUDA(cudaMemset(c->arena, 0, c->off_x));  // geometry + flags + load matrix
  LLEP_CUDA(cudaMalloc(&c->act, (size_t)rows * c->H * 2));
  LLEP_CUDA(cudaMalloc(&c->rtok, (size_t)rows * 4));
  if (c->backward) {
    LLEP_CUDA(cudaMalloc(&c->gu, (size_t)rows * 2 * c->H * 2));
    LLEP_CUDA(cudaMalloc(&c->da0, (size_t)rows * c->H * 2));
    LLEP_CUDA(cudaMalloc(&c->aw, (size_t)rows * c->H * 2));
    LLEP_CUDA(cudaMalloc(&c->dgu, (size_t)rows * 2 * c->H * 2));
    LLEP_CUDA(cudaMalloc(&c->stage13, (size_t)foreign * 2 * c->H * c->D * 4));
    LLEP_CUDA(cudaMalloc(&c->stage2, (size_t)foreign * c->H * c->D * 4));
  }
  c->arena_rows = rows;
  c->arena_foreign = foreign;
  {
    const ArenaGeometry g = geometry(c);
    LLEP_CUDA(cudaMemcpy(c->arena, &g, sizeof(g), cudaMemcpyHostToDevice));
  }
  c->peer_base[c->rank] = c->arena;
  if (c->P == 1) {
    c->peers_ready = true;
    return upload_peer_ptrs(c);
  }
  return LLEP_OK;
}

extern "C" {

const char *llep_last_error(void) { return g_err; }
const char *llep_version(void) { return "llep-b200 0.1 (sm_100a)"; }

size_t llep_plan_bytes(int32_t n_experts, int32_t world_size) {
  if (n_experts < 1 || world_size < 1) return 0;
  return plan_layout(n_experts, world_size).bytes;
}

static llep_status plan_common(const int64_t *loads, int32_t N, int32_t P, const llep_params *p,
                               void *out, bool force_ep) {
  llep_status st;
  if ((st = check_np(N, P)) != LLEP_OK) return st;
  if ((st = check_params(p)) != LLEP_OK) return st;
  if (!loads || !out) return invalid("null pointer");
  int64_t S = 0;
  for (int e = 0; e < N; ++e) {
    if (loads[e] < 0) return invalid("negative load");
    S += loads[e];
  }
  if (S > INT32_MAX) return invalid("total load exceeds int32 chunk bounds");
  host_plan(loads, N, P, p, force_ep, reinterpret_cast<uint8_t *>(out));
  return LLEP_OK;
}

llep_status llep_plan(const int64_t *loads, int32_t n_experts, int32_t world_size,
                      const llep_params *params, void *plan_out) {
  return plan_common(loads, n_experts, world_size, params, plan_out, false);
}

llep_status llep_plan_ep(const int64_t *loads, int32_t n_experts, int32_t world_size,
                         const llep_params *params, void *plan_out) {
  return plan_common(loads, n_experts, world_size, params, plan_out, true);
}

llep_status llep_plan_device(const int32_t *load_matrix, int32_t N, int32_t P,
                             const llep_params *params, int32_t force_ep, void *plan_out,
                             void *stream) {
  llep_status st;
  if ((st = check_np(N, P)) != LLEP_OK) return st;
  if ((st = check_params(params)) != LLEP_OK) return st;
  if (P > kMaxWorld) return invalid("device planner supports P <= 32");
  if (!load_matrix || !plan_out) return invalid("null pointer");
  LLEP_CUDA(launch_planner(load_matrix, N, P, params->alpha, params->min_chunk, params->lambda,
                           force_ep, plan_out, (cudaStream_t)stream));
  return LLEP_OK;
}

llep_status llep_context_create(const llep_shape *s, int32_t rank, int32_t device,
                                int64_t max_tokens, llep_context **out) {
  if (!s || !out) return invalid("null pointer");
  llep_status st;
  if ((st = check_np(s->n_experts, s->world_size)) != LLEP_OK) return st;
  if (s->world_size > kMaxWorld) return invalid("P > 32 is not supported");
  if (s->top_k < 1 || s->top_k > s->n_experts) return invalid("K not in [1, N]");
  if (s->top_k > 32) return invalid("K > 32 is not supported");
  if (s->d_model < 8 || s->d_ff < 8 || s->d_model % 8 || s->d_ff % 8)
    return invalid("D and H must be positive multiples of 8");
  if (rank < 0 || rank >= s->world_size) return invalid("rank out of range");
  if (max_tokens < 0) return invalid("max_tokens < 0");
  LLEP_CUDA(cudaSetDevice(device));
  llep_context *c = new llep_context();
  c->N = s->n_experts;
  c->K = s->top_k;
  c->D = s->d_model;
  c->H = s->d_ff;
  c->P = s->world_size;
  c->M = c->N / c->P;
  c->rank = rank;
  c->device = device;
  c->max_tokens = max_tokens;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (const char *ra = getenv("LLEP_ROW_ALIGN")) c->row_align = atoi(ra) == 128 ? 128 : 256;
  const int64_t slots = std::max<int64_t>(1, max_tokens * c->K);
  const int64_t tiles = (slots + kTileSlots - 1) / kTileSlots;
  auto A = [&](auto **p, size_t bytes) -> cudaError_t {
    c->scratch_bytes += bytes;
    return cudaMalloc(reinterpret_cast<void **>(p), bytes);
  };
  cudaError_t e = cudaSuccess;
  const int N = c->N, P = c->P;
  if (!e) e = A(&c->tile_cnt, sizeof(int32_t) * tiles * N);
  if (!e) e = A(&c->tile_off, sizeof(int32_t) * tiles * N);
  if (!e) e = A(&c->cnt, sizeof(int32_t) * N);
  if (!e) e = A(&c->local_rank, sizeof(int32_t) * slots);
  if (!e) e = A(&c->prep_ids, sizeof(int32_t) * slots);
  if (!e) e = A(&c->slot_dst, sizeof(int32_t) * 2 * slots);
  if (!e) e = A(&c->err, sizeof(int32_t) * 4);
  if (!e) e = A(&c->lm_local, sizeof(int32_t) * P * N);
  if (!e) e = A(&c->rows_on, sizeof(int32_t) * N * P);
  if (!e) e = A(&c->chunk_row, sizeof(int32_t) * N * (P + 1));
  if (!e) e = A(&c->foreign_slot, sizeof(int32_t) * N * P);
  if (!e) e = A(&c->dev_padded, sizeof(int32_t) * P);
  if (!e) e = A(&c->dev_foreign, sizeof(int32_t) * P);
  if (!e) e = A(&c->groups, sizeof(Group) * kMaxGroups);
  // worst case: every slot of every rank lands on this device, plus one partial block per group
  c->sched_cap = ((int64_t)P * slots + kRowAlign - 1) / kRowAlign + kMaxGroups;
  if (!e) e = A(&c->sched, sizeof(int32_t) * c->sched_cap);
  if (!e) e = A(&c->mblk_src, sizeof(uint32_t) * c->sched_cap);
  if (!e) e = A(&c->block_done, sizeof(uint32_t));
  if (!e) e = cudaMemset(c->block_done, 0, sizeof(uint32_t));
  if (!e) e = A(&c->summary, sizeof(LayoutSummary));
  if (!e) e = A(&c->d_ptrs, sizeof(void *) * kPeerPtrArrays * P);
  if (!e) e = A(&c->ep, sizeof(uint32_t) * 4);
  if (!e) e = cudaMemset(c->ep, 0, sizeof(uint32_t) * 4);
  if (!e) e = A(&c->ngroups_dev, sizeof(int32_t));
  if (!e) e = A(&c->push_cnt, sizeof(uint32_t) * kMaxPushItems);
  if (!e) e = cudaMemset(c->push_cnt, 0, sizeof(uint32_t) * kMaxPushItems);
  if (!e) e = cudaMemset(c->err, 0, sizeof(int32_t) * 4);
  if (!e) e = cudaHostAlloc(&c->summary_host, sizeof(LayoutSummary), cudaHostAllocMapped);
  if (!e) e = cudaHostAlloc(&c->err_host, sizeof(int32_t) * 4, cudaHostAllocMapped);
  if (!e) e = cudaHostAlloc(&c->plan_mirror, plan_layout(c->N, c->P).bytes, cudaHostAllocMapped);
  if (!e) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (!e) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  if (!e) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  for (int i = 0; i < 9 && !e; ++i) e = cudaEventCreate(&c->mark[i]);
  if (e) {
    llep_context_destroy(c);
    return cuda_status(e, "llep_context_create");
  }
  // initial arena: every rank's local slots, room for the balanced case
  const int64_t rows0 = (max_tokens * c->K + (int64_t)c->M * c->row_align);
  if ((st = alloc_arena(c, rows0, 1)) != LLEP_OK) {
    llep_context_destroy(c);
    return st;
  }
  *out = c;
  return LLEP_OK;
}

void llep_context_destroy(llep_context *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  close_peers(c);
  void *ptrs[] = {c->tile_cnt, c->tile_off, c->cnt, c->local_rank, c->prep_ids, c->slot_dst, c->err,
                  c->lm_local, c->rows_on, c->chunk_row, c->foreign_slot, c->dev_padded,
                  c->dev_foreign, c->groups, c->sched, c->mblk_src, c->block_done, c->summary, c->d_ptrs, c->ep, c->ngroups_dev, c->push_cnt, c->act, c->rtok, c->arena,
                  c->gu, c->da0, c->aw, c->dgu, c->stage13, c->stage2, c->wsbuf, c->dotp};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (c->summary_host) cudaFreeHost(c->summary_host);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->plan_mirror) cudaFreeHost(c->plan_mirror);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (int i = 0; i < 9; ++i)
    if (c->mark[i]) cudaEventDestroy(c->mark[i]);
  delete c;
}

llep_status llep_context_ipc_handle(llep_context *c, void *handle64) {
  if (!c || !handle64) return invalid("null pointer");
  cudaIpcMemHandle_t h;
  LLEP_CUDA(cudaIpcGetMemHandle(&h, c->arena));
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  memcpy(handle64, &h, 64);
  return LLEP_OK;
}

llep_status llep_context_open_peers(llep_context *c, const void *handles, int32_t n) {
  if (!c || !handles) return invalid("null pointer");
  if (n != c->P) return invalid("need one handle per rank");
  close_peers(c);
  for (int q = 0; q < c->P; ++q) {
    if (q == c->rank) {
      c->peer_base[q] = c->arena;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, reinterpret_cast<const uint8_t *>(handles) + 64 * q, 64);
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      set_error("cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
      close_peers(c);
      return LLEP_ERR_COMM;
    }
    c->peer_base[q] = reinterpret_cast<uint8_t *>(p);
    c->peer_opened[q] = true;
  }
  const ArenaGeometry mine = geometry(c);
  for (int q = 0; q < c->P; ++q) {
    ArenaGeometry g;
    cudaError_t e = cudaMemcpy(&g, c->peer_base[q], sizeof(g), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      close_peers(c);
      return cuda_status(e, "reading a peer's arena geometry");
    }
    if (memcmp(&g, &mine, sizeof(g)) != 0) {
      set_error("asymmetric arenas: rank %d has max_tokens %lld, rows %lld, foreign %d, grad %d, backward %d; "
                "rank %d has %lld, %lld, %d, %d, %d (every rank must create its context with the same shape and "
                "max_tokens and call llep_context_reserve / enable_backward with the same arguments)",
                q, (long long)g.max_tokens, (long long)g.arena_rows, g.arena_foreign, g.arena_grad, g.backward,
                c->rank, (long long)mine.max_tokens, (long long)mine.arena_rows, mine.arena_foreign,
                mine.arena_grad, mine.backward);
      close_peers(c);
      return LLEP_ERR_INVALID;
    }
  }
  c->peers_ready = true;
  return upload_peer_ptrs(c);
}

llep_status llep_context_reserve(llep_context *c, int64_t rows, int32_t foreign, int32_t grad_slots) {
  if (!c) return invalid("null context");
  if (rows <= c->arena_rows && foreign <= c->arena_foreign && grad_slots <= c->arena_grad && c->peers_ready)
    return LLEP_OK;
  LLEP_CUDA(cudaSetDevice(c->device));
  LLEP_CUDA(cudaDeviceSynchronize());
  const int32_t old_grad = c->arena_grad;
  c->arena_grad = std::max(grad_slots, c->arena_grad);
  llep_status st = alloc_arena(c, std::max(rows, c->arena_rows), std::max(foreign, c->arena_foreign));
  if (st != LLEP_OK) c->arena_grad = old_grad;
  return st;
}

llep_status llep_context_enable_backward(llep_context *c) {
  if (!c) return invalid("null context");
  if (c->row_align != 256) return invalid("the backward pass needs the 256-row (2-CTA) group layout");
  if (c->backward) return LLEP_OK;
  LLEP_CUDA(cudaSetDevice(c->device));
  LLEP_CUDA(cudaDeviceSynchronize());
  c->backward = true;
  // regions change: collective like llep_context_reserve (re-exchange the IPC handles for P > 1)
  return alloc_arena(c, c->arena_rows, c->arena_foreign);
}

llep_status llep_context_set_token_order(llep_context *c, int32_t order) {
  if (!c) return invalid("null context");
  if (order != LLEP_ORDER_RANK_MAJOR && order != LLEP_ORDER_CHUNK_ALIGNED) return invalid("unknown token order");
  c->token_order = order;
  c->plan_dev_cached = nullptr;   // the layout (source masks) depends on it: recompute for the next call
  return LLEP_OK;
}

llep_status llep_context_set_memory_cap(llep_context *c, int64_t bytes) {
  if (!c || bytes < 0) return invalid("null context or negative cap");
  c->mem_cap = bytes;
  return LLEP_OK;
}

int64_t llep_context_device_bytes(const llep_context *c) {
  if (!c) return 0;
  return (int64_t)held_bytes(c);
}

static uint32_t *const *peer_flags(llep_context *c) { return reinterpret_cast<uint32_t *const *>(c->d_ptrs); }
static int32_t *const *peer_lm(llep_context *c) { return reinterpret_cast<int32_t *const *>(c->d_ptrs + c->P); }
static uint16_t *const *peer_x(llep_context *c) { return reinterpret_cast<uint16_t *const *>(c->d_ptrs + 2 * c->P); }
static float *const *peer_g(llep_context *c) { return reinterpret_cast<float *const *>(c->d_ptrs + 3 * c->P); }

static llep_status barrier(llep_context *c, cudaStream_t s) {
  if (c->P == 1) return LLEP_OK;
  ++c->launches;
  LLEP_CUDA(launch_barrier(peer_flags(c), c->rank, c->P, c->ep, c->err + 1, s));
  return LLEP_OK;
}

// max over devices of the weight-gradient partials returned to it (𝒲 entries with src = device)
static int32_t grad_slots_needed(const llep_context *c) {
  const PlanLayout L = plan_layout(c->N, c->P);
  const uint8_t *rep = c->plan_host.data() + L.off_replica;
  int32_t mx = 0;
  for (int n = 0; n < c->P; ++n) {
    int32_t k = 0;
    for (int e = n * c->M; e < (n + 1) * c->M; ++e)
      for (int d = 0; d < c->P; ++d) k += rep[(size_t)e * c->P + d];
    mx = std::max(mx, k);
  }
  return mx;
}

static void fill_req(llep_context *c, llep_requirements *req) {
  const LayoutSummary &s = *c->summary_host;
  req->rows_needed = s.rows_needed;
  req->foreign_needed = s.foreign_needed;
  req->grad_slots_needed = c->backward ? grad_slots_needed(c) : 0;
  req->fits = (s.rows_needed <= c->arena_rows && s.foreign_needed <= c->arena_foreign &&
               req->grad_slots_needed <= c->arena_grad) ? 1 : 0;
  req->my_rows = s.my_rows;
  req->my_groups = s.my_groups;
  req->fallback_ep = s.fallback_ep;
  req->force_count = s.force_count;
  req->n_transfers = s.n_transfers;
}

static llep_status run_layout(llep_context *c, const void *plan, cudaStream_t s, bool layer = false) {
  LayoutArgs la;
  la.arena_rows = layer ? c->arena_rows : 0;   // the layer call checks the arena fit on the device
  la.arena_foreign = c->arena_foreign;
  la.n_groups_dev = layer ? c->ngroups_dev : nullptr;
  la.err = layer ? c->err : nullptr;
  la.plan = plan;
  la.load_matrix = c->lm_local;
  la.N = c->N;
  la.P = c->P;
  la.M = c->M;
  la.rank = c->rank;
  la.rows_on = c->rows_on;
  la.chunk_row = c->chunk_row;
  la.foreign_slot = c->foreign_slot;
  la.groups = c->groups;
  la.dev_padded = c->dev_padded;
  la.dev_foreign = c->dev_foreign;
  la.summary = c->summary;
  la.sched = c->sched;
  la.sched_cap = c->sched_cap;
  la.row_align = c->row_align;
  la.mblk_src = c->mblk_src;
  la.aligned = c->token_order == LLEP_ORDER_CHUNK_ALIGNED;
  LLEP_CUDA(launch_layout(la, s));
  ++c->launches;
  return LLEP_OK;
}

// Sticky device error words (err[4]): [0] a router index outside [0, N) (a1); [1] a device barrier (4),
// weight-flag wait (8), GEMM weight wait (16) or source wait (32) timed out, or too many GPU weight pushes
// (64); [2] topk_ids changed between llep_prepare and the forward / backward call (those slots were
// dropped); [3] capture-safe layer: the plan did not fit the arena (1) or was inconsistent (2).
// Reported once, then cleared.
static llep_status decode_err(llep_context *c, const int32_t *e, cudaStream_t s) {
  if (!(e[0] | e[1] | e[2] | e[3])) return LLEP_OK;
  cudaMemsetAsync(c->err, 0, sizeof(int32_t) * 4, s);
  if (e[0]) {
    set_error("router index outside [0, N)");
    return LLEP_ERR_ROUTING;
  }
  if (e[1]) {
    set_error("device barrier or weight-flag wait timed out (a peer did not arrive), code %d", e[1]);
    return LLEP_ERR_COMM;
  }
  if (e[3]) {
    set_error(e[3] & 1 ? "llep_moe_layer: the plan needs more receive rows or foreign-weight slots than the arena "
                         "holds (llep_context_reserve more); that call computed nothing"
                       : "llep_moe_layer: plan inconsistent with the load matrix or too many groups");
    return LLEP_ERR_PLAN;
  }
  set_error("topk_ids changed between llep_prepare and llep_moe_forward/backward: the changed slots were "
            "dropped from that call's output");
  return LLEP_ERR_PLAN;
}

// one host synchronisation: plan blob + layout summary + error flags
static llep_status read_back(llep_context *c, const void *plan, cudaStream_t s) {
  const size_t pb = plan_layout(c->N, c->P).bytes;
  void *dp = nullptr, *ds = nullptr, *de = nullptr;
  LLEP_CUDA(cudaHostGetDevicePointer(&dp, c->plan_mirror, 0));
  LLEP_CUDA(cudaHostGetDevicePointer(&ds, c->summary_host, 0));
  LLEP_CUDA(cudaHostGetDevicePointer(&de, c->err_host, 0));
  LLEP_CUDA(launch_mirror(plan, pb, c->summary, sizeof(LayoutSummary), c->err, dp, ds,
                          reinterpret_cast<int32_t *>(de), s));
  ++c->launches;
  LLEP_CUDA(cudaStreamSynchronize(s));
  c->plan_host.assign(c->plan_mirror, c->plan_mirror + pb);
  c->plan_dev_cached = plan;
  llep_status st = decode_err(c, c->err_host, s);
  if (st != LLEP_OK) return st;
  if (c->summary_host->error) {
    set_error("plan inconsistent with the load matrix (chunk totals != l_e) or too many groups");
    return LLEP_ERR_PLAN;
  }
  return LLEP_OK;
}

// a1 -> a2 -> a4 -> a5 on the stream (no host synchronisation): histogram and local ranks, counts
// pushed into every rank's load matrix + barrier, device planner, layout
static llep_status prepare_kernels(llep_context *c, const int32_t *ids, int64_t B, const llep_params *prm,
                                   int32_t force_ep, void *plan_out, cudaStream_t s, bool layer) {
  llep_status st;
  const int N = c->N, P = c->P;
  const int64_t slots = B * c->K;
  const int n_tiles = (int)((slots + kTileSlots - 1) / kTileSlots);
  mark(c, 0, s);
  // a1: per-tile histogram + scan -> counts row; a3: stable local ranks
  LLEP_CUDA(launch_tile_count(ids, slots, N, c->tile_cnt, c->err, s));
  if (n_tiles > 0) {
    LLEP_CUDA(launch_tile_scan(c->tile_cnt, n_tiles, N, c->tile_off, c->cnt, s));
    c->launches += 3;
  } else {
    LLEP_CUDA(cudaMemsetAsync(c->cnt, 0, sizeof(int32_t) * N, s));
  }
  LLEP_CUDA(launch_local_rank(ids, slots, N, c->tile_off, c->local_rank, c->prep_ids, s));
  mark(c, 1, s);
  // a2: push the counts row into every rank's load matrix, barrier, keep a local copy
  LLEP_CUDA(launch_push_counts(c->cnt, N, c->rank, P, peer_lm(c), s));
  ++c->launches;
  if ((st = barrier(c, s)) != LLEP_OK) return st;
  LLEP_CUDA(cudaMemcpyAsync(c->lm_local, c->arena + c->off_lm, sizeof(int32_t) * P * N,
                            cudaMemcpyDeviceToDevice, s));
  mark(c, 2, s);
  // a4: planner; a5: layout
  LLEP_CUDA(launch_planner(c->lm_local, N, P, prm->alpha, prm->min_chunk, prm->lambda, force_ep,
                           plan_out, s));
  ++c->launches;
  if ((st = run_layout(c, plan_out, s, layer)) != LLEP_OK) return st;
  mark(c, 3, s);
  return LLEP_OK;
}

llep_status llep_prepare(llep_context *c, const int32_t *ids, int64_t B, const llep_params *prm,
                         int32_t force_ep, void *plan_out, llep_requirements *req, void *stream) {
  if (!c || !prm || !plan_out || (B > 0 && !ids)) return invalid("null pointer");
  llep_status st;
  if ((st = check_params(prm)) != LLEP_OK) return st;
  if (B < 0 || B > c->max_tokens) return invalid("n_tokens outside [0, max_tokens]");
  if (c->P > 1 && !c->peers_ready) {
    set_error("peers not opened (llep_context_open_peers)");
    return LLEP_ERR_COMM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  collect(c);
  c->pending = false;
  c->prepared_tokens = -1;   // a failed prepare leaves nothing for llep_moe_forward to use
  c->prepared_ids = nullptr;
  if ((st = prepare_kernels(c, ids, B, prm, force_ep, plan_out, s, false)) != LLEP_OK) return st;
  if ((st = read_back(c, plan_out, s)) != LLEP_OK) return st;
  c->prepared_tokens = B;
  c->prepared_ids = ids;
  if (req) fill_req(c, req);
  return LLEP_OK;
}

// a7: weight migration as a binomial broadcast tree per expert.  Holders of expert e are
// h_0 = native(e) followed by its replica devices in ascending order; holder i sends to holders
// i + 2^t for every 2^t > i (h_0 to 1, 2, 4, ...), so the native device's egress is ceil(log2(k+1))
// copies instead of k.  A replica forwards from its own foreign slot after waiting for that slot's
// flag; every copy is followed by a release-signal of the destination slot's flag (epoch `ep`).
// f(e, d) = position of e among d's foreign experts (ascending id).  Side stream, copy engines.
static llep_status push_weights(llep_context *c, const uint16_t *w13, const uint16_t *w2, cudaStream_t s,
                                bool *any_copy) {
  const int N = c->N, P = c->P, M = c->M, D = c->D, H = c->H;
  const PlanLayout L = plan_layout(N, P);
  const uint8_t *replica = c->plan_host.data() + L.off_replica;
  const size_t w13_bytes = (size_t)2 * H * D * 2, w2_bytes = (size_t)D * H * 2;
  *any_copy = false;
  if (P == 1) return LLEP_OK;
  std::vector<int> fslot((size_t)N * P, -1), cnt(P, 0);
  for (int e = 0; e < N; ++e)
    for (int d = 0; d < P; ++d)
      if (replica[(size_t)e * P + d]) fslot[(size_t)e * P + d] = cnt[d]++;
  std::vector<int> holders;
  for (int e = 0; e < N; ++e) {
    holders.assign(1, e / M);
    for (int d = 0; d < P; ++d)
      if (replica[(size_t)e * P + d]) holders.push_back(d);
    const int k = (int)holders.size() - 1;
    int me = -1;
    for (int i = 0; i <= k; ++i)
      if (holders[i] == c->rank) me = i;
    if (k == 0 || me < 0) continue;
    int hb = 0;                                   // highest power of two <= me (0 for the native)
    while (me > 0 && (2 << hb) <= me) ++hb;
    const int t0 = me == 0 ? 0 : hb + 1;
    if (me + (1 << t0) > k) continue;             // a leaf of the tree
    if (!*any_copy) {
      LLEP_CUDA(cudaEventRecord(c->ev_fork, s));
      LLEP_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
      *any_copy = true;
    }
    const uint8_t *src13, *src2;
    if (me == 0) {
      const int el = e - c->rank * M;
      src13 = reinterpret_cast<const uint8_t *>(w13 + (size_t)el * 2 * H * D);
      src2 = reinterpret_cast<const uint8_t *>(w2 + (size_t)el * D * H);
    } else {
      const int f = fslot[(size_t)e * P + c->rank];
      const uint32_t *own = reinterpret_cast<const uint32_t *>(c->arena + c->off_flags) + kWeightFlag0 + f;
      LLEP_CUDA(launch_wait_flag(own, c->ep, c->err + 1, c->side));
      ++c->launches;
      src13 = c->arena + c->off_w13 + (size_t)f * w13_bytes;
      src2 = c->arena + c->off_w2 + (size_t)f * w2_bytes;
    }
    for (int t = t0; me + (1 << t) <= k; ++t) {
      const int d = holders[me + (1 << t)];
      const int f = fslot[(size_t)e * P + d];
      LLEP_CUDA(cudaMemcpyAsync(c->peer_base[d] + c->off_w13 + (size_t)f * w13_bytes, src13, w13_bytes,
                                cudaMemcpyDeviceToDevice, c->side));
      LLEP_CUDA(cudaMemcpyAsync(c->peer_base[d] + c->off_w2 + (size_t)f * w2_bytes, src2, w2_bytes,
                                cudaMemcpyDeviceToDevice, c->side));
      uint32_t *flag = reinterpret_cast<uint32_t *>(c->peer_base[d] + c->off_flags) + kWeightFlag0 + f;
      LLEP_CUDA(launch_signal(flag, c->ep, c->side));
      ++c->launches;
    }
  }
  return LLEP_OK;
}

// The forward kernels (a7, a6, a8, a9, a10).  layer = false: the two-call path, planned on the host copy
// of the plan (group count, arena check, copy-engine weight pushes).  layer = true (llep_moe_layer): the
// plan never leaves the device -- group count from the layout kernel, arena fit checked there, weight
// pushes issued by the GPU -- so the call is capture-safe.
static llep_status moe_forward(llep_context *c, const uint16_t *x, const int32_t *ids,
                               const float *topk_w, int64_t B, const uint16_t *w13,
                               const uint16_t *w2, const void *plan, uint16_t *out, uint16_t *gu_save,
                               int64_t gu_rows, void *stream, bool layer = false) {
  if (!c || !plan || !w13 || !w2 || (B > 0 && (!x || !ids || !topk_w || !out)))
    return invalid("null pointer");
  if (B != c->prepared_tokens) return invalid("n_tokens differs from the last llep_prepare");
  if (B > 0 && ids != c->prepared_ids) {
    set_error("topk_ids is not the buffer passed to the last llep_prepare (the plan, load matrix and local "
              "ranks were computed from that one)");
    return LLEP_ERR_PLAN;
  }
  cudaStream_t s = (cudaStream_t)stream;
  llep_status st;
  if (!layer && plan != c->plan_dev_cached) {
    if ((st = run_layout(c, plan, s)) != LLEP_OK) return st;
    if ((st = read_back(c, plan, s)) != LLEP_OK) return st;
  }
  LayoutSummary sum_dev_planned;
  memset(&sum_dev_planned, 0, sizeof(sum_dev_planned));
  const LayoutSummary &sum = layer ? sum_dev_planned : *c->summary_host;
  if (!layer && (sum.rows_needed > c->arena_rows || sum.foreign_needed > c->arena_foreign)) {
    set_error("plan needs %lld rows / %d foreign experts, arena holds %lld / %d: call "
              "llep_context_reserve", (long long)sum.rows_needed, sum.foreign_needed,
              (long long)c->arena_rows, c->arena_foreign);
    return LLEP_ERR_PLAN;
  }
  const int N = c->N, P = c->P, M = c->M, D = c->D, H = c->H;
  (void)H;
  if (gu_save && gu_rows < sum.my_padded) {
    set_error("gu_save holds %lld rows, this rank's layout needs %lld (llep_requirements.rows_needed "
              "is always enough)", (long long)gu_rows, (long long)sum.my_padded);
    return LLEP_ERR_INVALID;
  }
  // a7: weight migration, pushed by the native device on a side stream (copy engines); row f2: each
  // destination's GEMM waits for a foreign slot's flag only when it reaches that slot's tiles
  bool any_copy = false;
  if (P > 1) {   // this call's weight-flag and arrival epochs (device-resident, same on every rank)
    LLEP_CUDA(launch_advance(c->ep, s));
    ++c->launches;
  }
  if (!layer) {
    if ((st = push_weights(c, w13, w2, s, &any_copy)) != LLEP_OK) return st;
  } else if (P > 1) {
    // a7 issued by the GPU from the device plan: one launch per broadcast-tree level on the side stream
    LLEP_CUDA(cudaEventRecord(c->ev_fork, s));
    LLEP_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    any_copy = true;
    PushArgs pa;
    pa.plan = plan;
    pa.foreign_slot = c->foreign_slot;
    pa.N = N;
    pa.P = P;
    pa.M = M;
    pa.rank = c->rank;
    pa.w13 = w13;
    pa.w2 = w2;
    pa.peer_w13 = reinterpret_cast<uint8_t *const *>(c->d_ptrs + 8 * P);
    pa.peer_w2 = reinterpret_cast<uint8_t *const *>(c->d_ptrs + 9 * P);
    pa.peer_flags = peer_flags(c);
    pa.w13_bytes = (int64_t)2 * H * D * 2;
    pa.w2_bytes = (int64_t)D * H * 2;
    pa.ep = c->ep;
    pa.counters = c->push_cnt;
    pa.err = c->err;
    pa.skip = &c->summary->error;
    for (int lvl = 0; (1 << lvl) < P; ++lvl) {
      pa.level = lvl;
      LLEP_CUDA(launch_push_level(pa, c->side));
      ++c->launches;
    }
  }
  mark(c, 4, s);
  if (any_copy) LLEP_CUDA(cudaEventRecord(c->ev_join, c->side));
  // a6: dispatch (gather-on-send into every destination's receive rows)
  DispatchArgs da{};
  da.x = x;
  da.ids = ids;
  da.w = topk_w;
  da.local_rank = c->local_rank;
  da.prep_ids = c->prep_ids;
  da.err = c->err;
  da.load_matrix = c->lm_local;
  da.plan = plan;
  da.chunk_row = c->chunk_row;
  da.B = B;
  da.K = c->K;
  da.D = D;
  da.N = N;
  da.P = P;
  da.rank = c->rank;
  da.peer_x = peer_x(c);
  da.peer_g = peer_g(c);
  da.slot_dst = c->slot_dst;
  da.x2 = nullptr;
  da.peer_x2 = nullptr;
  da.peer_rsrc = reinterpret_cast<int32_t *const *>(c->d_ptrs + 6 * P);
  // row f2: no barrier between the dispatch and GEMM1.  The dispatch publishes a per-source arrival
  // flag on every device once all of its rows are stored; GEMM1's producers wait, per m-block, only
  // for the sources of that block's rows (and, per foreign group, for its weight flag), so tiles start
  // as their inputs land instead of after the slowest rank (LLEP_DISPATCH_BARRIER=1: old barrier)
  const bool overlap = P > 1 && !getenv("LLEP_DISPATCH_BARRIER");
  da.peer_flags = overlap ? peer_flags(c) : nullptr;
  da.ep = c->ep;
  da.block_done = c->block_done;
  da.skip = layer ? &c->summary->error : nullptr;   // arena overflow: store nothing (flags still go out)
  // a6 local rows, opt-in (LLEP_GATHER=1): rows this rank routes to itself, in m-blocks fed by this rank
  // alone, are gathered by GEMM1 from x with TMA gather4 instead of copied.  Bit-identical, but OFF by
  // default: gather4 moves ~22 cycles per 128-byte row per SM (1.7 TB/s over 148 SMs, any row order,
  // profiles/r02_gather4_probe.jsonl), 4x short of what the A operand of a re-used tile needs, so GEMM1
  // took 10.2 ms instead of 3.6 ms at G120 P=1 to save the 0.18 ms copy
  const char *gv = getenv("LLEP_GATHER");
  const bool gather = c->row_align == 256 && gv && atoi(gv) == 1;
  da.rtok = gather ? c->rtok : nullptr;
  da.mblk_src = c->mblk_src;
  da.row_align = c->row_align;
  da.aligned = c->token_order == LLEP_ORDER_CHUNK_ALIGNED;
  LLEP_CUDA(launch_dispatch(da, s));
  c->launches += B > 0 || overlap;
  if (!overlap && (st = barrier(c, s)) != LLEP_OK) return st;   // dispatched rows landed
  mark(c, 5, s);
  // a8: GEMM1 + SwiGLU   X [rows, D] -> A [rows, H]
  uint16_t *X = reinterpret_cast<uint16_t *>(c->arena + c->off_x);
  GemmArgs g1;
  memset(&g1, 0, sizeof(g1));
  g1.mode = gu_save ? 3 : 0;   // training forward: also save the raw [g | u] for the backward
  g1.out2 = gu_save;
  g1.a = X;
  g1.a_rows = c->arena_rows;
  g1.kdim = D;
  g1.w_native = w13;
  g1.n_native = M;
  g1.w_foreign = reinterpret_cast<const uint16_t *>(c->arena + c->off_w13);
  g1.n_foreign = c->arena_foreign;
  g1.nout = H;
  g1.groups = c->groups;
  g1.sched = getenv("LLEP_GEMM_GROUP_ORDER") ? nullptr : c->sched;
  g1.n_groups_dev = layer ? c->ngroups_dev : nullptr;   // layer: the count never leaves the device
  g1.n_groups_host = sum.my_groups;
  g1.gate = nullptr;
  g1.out = c->act;
  g1.wflags = P > 1 ? reinterpret_cast<const uint32_t *>(c->arena + c->off_flags) + kWeightFlag0 : nullptr;
  g1.ep = c->ep;
  g1.err = c->err;
  g1.arrive = overlap ? reinterpret_cast<const uint32_t *>(c->arena + c->off_flags) + kArriveFlag0 : nullptr;
  g1.mblk_src = c->mblk_src;
  g1.src_all = P >= 32 ? 0xffffffffu : (1u << P) - 1u;
  g1.row_src = nullptr;
  g1.peer_slot = nullptr;
  g1.num_sms = c->num_sms;
  g1.row_align = c->row_align;
  g1.xg = gather ? x : nullptr;
  g1.xg_rows = B;
  g1.rtok = gather ? c->rtok : nullptr;
  g1.self_mask = 1u << c->rank;
  const bool gemms = layer || sum.my_groups > 0;
  if (gemms && (st = run_grouped_gemm(g1, s)) != LLEP_OK) return st;
  c->launches += gemms;
  mark(c, 6, s);
  // a9: GEMM2 + gate   A [rows, H] -> Y [rows, D]  (Y reuses X's rows: X is dead after GEMM1)
  GemmArgs g2 = g1;
  g2.mode = 1;
  g2.out2 = nullptr;
  g2.xg = nullptr;
  g2.rtok = nullptr;
  g2.a = c->act;
  g2.kdim = H;
  g2.w_native = w2;
  g2.w_foreign = reinterpret_cast<const uint16_t *>(c->arena + c->off_w2);
  g2.nout = D;
  g2.gate = reinterpret_cast<const float *>(c->arena + c->off_g);
  g2.out = X;
  // a9 + a10 fused: the epilogue pushes each gated row into its home rank's slot buffer (NVLink
  // peer stores for remote rows, overlapped with the MMAs of later tiles)
  g2.row_src = reinterpret_cast<const int32_t *>(c->arena + c->off_rsrc);
  g2.peer_slot = reinterpret_cast<uint16_t *const *>(c->d_ptrs + 7 * P);
  if (gemms && (st = run_grouped_gemm(g2, s)) != LLEP_OK) return st;
  c->launches += gemms;
  mark(c, 7, s);
  if ((st = barrier(c, s)) != LLEP_OK) return st;
  // a10: local K-sum of the slot buffer the GEMM2 epilogues (this rank's and every peer's) filled
  LLEP_CUDA(launch_combine_local(reinterpret_cast<const uint16_t *>(c->arena + c->off_slot), B, c->K, D,
                                 c->slot_dst, out, s));
  c->launches += B > 0;
  if (any_copy) LLEP_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));   // keep the side stream joined
  mark(c, 8, s);
  if (c->timing && !layer) {
    c->pending = true;
    c->pending_rows = sum.my_rows;
  }
  return LLEP_OK;
}

llep_status llep_moe_layer(llep_context *c, const uint16_t *x, const int32_t *ids, const float *topk_w,
                           int64_t B, const uint16_t *w13, const uint16_t *w2, const llep_params *prm,
                           int32_t force_ep, void *plan_out, uint16_t *out, void *stream) {
  if (!c || !prm || !plan_out || !w13 || !w2 || (B > 0 && (!x || !ids || !topk_w || !out)))
    return invalid("null pointer");
  llep_status st;
  if ((st = check_params(prm)) != LLEP_OK) return st;
  if (B < 0 || B > c->max_tokens) return invalid("n_tokens outside [0, max_tokens]");
  if (c->P > 1 && !c->peers_ready) {
    set_error("peers not opened (llep_context_open_peers)");
    return LLEP_ERR_COMM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  c->in_layer = true;   // (pending phase events of an earlier two-call forward stay pending)
  st = prepare_kernels(c, ids, B, prm, force_ep, plan_out, s, true);
  if (st == LLEP_OK) {
    c->prepared_tokens = B;
    c->prepared_ids = ids;
    st = moe_forward(c, x, ids, topk_w, B, w13, w2, plan_out, out, nullptr, 0, stream, true);
  }
  // the host copy of the plan (plan_host / summary_host) is not this call's: a later llep_moe_forward or
  // llep_moe_backward re-reads the plan it is given
  c->plan_dev_cached = nullptr;
  c->in_layer = false;
  return st;
}


llep_status llep_moe_forward(llep_context *c, const uint16_t *x, const int32_t *ids, const float *topk_w,
                             int64_t B, const uint16_t *w13, const uint16_t *w2, const void *plan,
                             uint16_t *out, void *stream) {
  return moe_forward(c, x, ids, topk_w, B, w13, w2, plan, out, nullptr, 0, stream);
}

llep_status llep_moe_forward_train(llep_context *c, const uint16_t *x, const int32_t *ids,
                                   const float *topk_w, int64_t B, const uint16_t *w13, const uint16_t *w2,
                                   const void *plan, uint16_t *out, uint16_t *gu_save, int64_t gu_rows,
                                   void *stream) {
  if (!gu_save) return invalid("null pointer (gu_save)");
  return moe_forward(c, x, ids, topk_w, B, w13, w2, plan, out, gu_save, gu_rows, stream);
}

// Grow a lazily sized backward workspace (floats), counted in llep_context_device_bytes and checked
// against the memory cap like the arena.
static llep_status grow_lazy(llep_context *c, float **buf, int64_t *cap, int64_t need, cudaStream_t s) {
  const size_t add = (size_t)(need - *cap) * 4;
  if (c->mem_cap > 0 && (int64_t)(held_bytes(c) + add) > c->mem_cap) {
    set_error("memory cap: the backward workspace needs %.2f GB more on this device, cap %.2f GB", add / 1e9,
              c->mem_cap / 1e9);
    return LLEP_ERR_NOMEM;
  }
  LLEP_CUDA(cudaStreamSynchronize(s));
  if (*buf) cudaFree(*buf);
  c->lazy_bytes -= (size_t)*cap * 4;
  *buf = nullptr;
  *cap = 0;
  LLEP_CUDA(cudaMalloc(buf, (size_t)need * 4));
  *cap = need;
  c->lazy_bytes += (size_t)need * 4;
  return LLEP_OK;
}

// This rank's expert groups in the layout kernel's order (native with rows, then foreign, ascending
// ids), from the host copy of the plan: rows, weight slot (>= 0 native, -1-f foreign), expert.
static void my_groups_host(const llep_context *c, std::vector<int32_t> &rows, std::vector<int32_t> &wslot,
                           std::vector<int32_t> &expert) {
  const PlanLayout L = plan_layout(c->N, c->P);
  const llep_chunk *chunks = reinterpret_cast<const llep_chunk *>(c->plan_host.data() + L.off_chunks);
  const int32_t *n_chunks = reinterpret_cast<const int32_t *>(c->plan_host.data() + L.off_n_chunks);
  rows.clear();
  wslot.clear();
  expert.clear();
  int f = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int e = 0; e < c->N; ++e) {
      const bool native = e / c->M == c->rank;
      if (native != (pass == 0)) continue;
      int r = 0;
      for (int k = 0; k < n_chunks[e]; ++k) {
        const llep_chunk ch = chunks[(size_t)e * (c->P + 1) + k];
        if (ch.device == c->rank) r += ch.end - ch.start;
      }
      if (r == 0) continue;
      rows.push_back(r);
      wslot.push_back(native ? e - c->rank * c->M : -1 - f);
      expert.push_back(e);
      if (!native) ++f;
    }
}

static llep_status moe_backward(llep_context *c, const uint16_t *x, const int32_t *ids,
                                const float *topk_w, const uint16_t *dout, int64_t B,
                                const uint16_t *w13, const uint16_t *w2, const void *plan, uint16_t *dx,
                                float *dgates, float *dw13, float *dw2, const uint16_t *gu_saved,
                                int64_t gu_rows, void *stream) {
  if (!c || !plan || !w13 || !w2 || !dw13 || !dw2 ||
      (B > 0 && (!x || !ids || !topk_w || !dout || !dx || !dgates)))
    return invalid("null pointer");
  if (!c->backward) return invalid("call llep_context_enable_backward first");
  if (B != c->prepared_tokens) return invalid("n_tokens differs from the last llep_prepare");
  if (B > 0 && ids != c->prepared_ids) {
    set_error("topk_ids is not the buffer passed to the last llep_prepare (the plan, load matrix and local "
              "ranks were computed from that one)");
    return LLEP_ERR_PLAN;
  }
  cudaStream_t s = (cudaStream_t)stream;
  llep_status st;
  if (plan != c->plan_dev_cached) {
    if ((st = run_layout(c, plan, s)) != LLEP_OK) return st;
    if ((st = read_back(c, plan, s)) != LLEP_OK) return st;
  }
  const LayoutSummary &sum = *c->summary_host;
  const int32_t gslots = grad_slots_needed(c);
  if (sum.rows_needed > c->arena_rows || sum.foreign_needed > c->arena_foreign || gslots > c->arena_grad) {
    set_error("plan needs %lld rows / %d foreign / %d gradient slots, arena holds %lld / %d / %d: call "
              "llep_context_reserve", (long long)sum.rows_needed, sum.foreign_needed, gslots,
              (long long)c->arena_rows, c->arena_foreign, c->arena_grad);
    return LLEP_ERR_PLAN;
  }
  if (gu_saved && gu_rows < sum.my_padded) {
    set_error("gu_saved holds %lld rows, this rank's layout needs %lld", (long long)gu_rows,
              (long long)sum.my_padded);
    return LLEP_ERR_INVALID;
  }
  const int N = c->N, P = c->P, M = c->M, D = c->D, H = c->H;
  const PlanLayout L = plan_layout(N, P);
  const uint8_t *replica = c->plan_host.data() + L.off_replica;
  const llep_chunk *chunks = reinterpret_cast<const llep_chunk *>(c->plan_host.data() + L.off_chunks);
  const int32_t *n_chunks = reinterpret_cast<const int32_t *>(c->plan_host.data() + L.off_n_chunks);
  const size_t slot13 = (size_t)2 * H * D, slot2 = (size_t)D * H, slot_all = slot13 + slot2;
  uint16_t *X = reinterpret_cast<uint16_t *>(c->arena + c->off_x);
  uint16_t *O = reinterpret_cast<uint16_t *>(c->arena + c->off_o);
  float *G = reinterpret_cast<float *>(c->arena + c->off_g);
  // a7 + a6: weights to the replicas, x and dout rows + gates to their destinations
  bool any_copy = false;
  if (P > 1) {
    LLEP_CUDA(launch_advance(c->ep, s));
    ++c->launches;
  }
  if ((st = push_weights(c, w13, w2, s, &any_copy)) != LLEP_OK) return st;
  if (any_copy) LLEP_CUDA(cudaEventRecord(c->ev_join, c->side));
  DispatchArgs da{};
  da.x = x;
  da.ids = ids;
  da.w = topk_w;
  da.local_rank = c->local_rank;
  da.prep_ids = c->prep_ids;
  da.err = c->err;
  da.load_matrix = c->lm_local;
  da.plan = plan;
  da.chunk_row = c->chunk_row;
  da.B = B;
  da.K = c->K;
  da.D = D;
  da.N = N;
  da.P = P;
  da.rank = c->rank;
  da.peer_x = peer_x(c);
  da.peer_g = peer_g(c);
  da.slot_dst = c->slot_dst;
  da.x2 = dout;
  da.peer_x2 = reinterpret_cast<uint16_t *const *>(c->d_ptrs + 4 * P);
  da.peer_rsrc = nullptr;
  da.peer_flags = nullptr;   // the backward keeps its barrier (weights and rows joined before the GEMMs)
  da.ep = c->ep;
  da.skip = nullptr;
  da.block_done = c->block_done;
  da.rtok = nullptr;         // the backward GEMMs read every row from the receive buffer
  da.mblk_src = nullptr;
  da.row_align = c->row_align;
  da.aligned = c->token_order == LLEP_ORDER_CHUNK_ALIGNED;
  LLEP_CUDA(launch_dispatch(da, s));
  c->launches += B > 0;
  if (any_copy) LLEP_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
  if ((st = barrier(c, s)) != LLEP_OK) return st;
  const int G_ = sum.my_groups;
  // native experts without rows here: their gradient (before returned partials) is zero
  for (int el = 0; el < M; ++el) {
    const int e = c->rank * M + el;
    bool has = false;
    for (int k = 0; k < n_chunks[e] && !has; ++k) has = chunks[(size_t)e * (P + 1) + k].device == c->rank;
    if (!has) {
      LLEP_CUDA(cudaMemsetAsync(dw13 + (size_t)el * slot13, 0, slot13 * 4, s));
      LLEP_CUDA(cudaMemsetAsync(dw2 + (size_t)el * slot2, 0, slot2 * 4, s));
    }
  }
  if (G_ > 0) {
    LLEP_CUDA(launch_zero_pad(c->groups, G_, D, X, O, s));
    ++c->launches;
    // GU = X · W13ᵀ (raw gate / up pre-activations): recomputed, unless the training forward saved
    // them under this plan (bit-identical: same kernel, same K order)
    const uint16_t *GU = gu_saved ? gu_saved : c->gu;
    GemmArgs g1;
    memset(&g1, 0, sizeof(g1));
    g1.mode = 2;
    g1.a = X;
    g1.a_rows = c->arena_rows;
    g1.kdim = D;
    g1.w_native = w13;
    g1.n_native = M;
    g1.w_foreign = reinterpret_cast<const uint16_t *>(c->arena + c->off_w13);
    g1.n_foreign = c->arena_foreign;
    g1.nout = H;
    g1.groups = c->groups;
    g1.sched = c->sched;
    g1.n_groups_host = G_;
    g1.out = c->gu;
    g1.num_sms = c->num_sms;
    g1.row_align = c->row_align;
    if (!gu_saved) {
      if ((st = run_grouped_gemm(g1, s)) != LLEP_OK) return st;
      ++c->launches;
    }
    // dA0 = dO · W_down  (W_down [D][H] row-major: MN-major B)
    BwdArgs b;
    memset(&b, 0, sizeof(b));
    b.kind = 0;
    b.a = O;
    b.b = w2;
    b.rows = c->arena_rows;
    b.kdim = D;
    b.mdim = 8;
    b.nout = H;
    b.n_weights = M;
    b.b_foreign = reinterpret_cast<const uint16_t *>(c->arena + c->off_w2);
    b.n_foreign = c->arena_foreign;
    b.groups = c->groups;
    b.n_groups = G_;
    b.mblk_scale = 2;
    b.out = c->da0;
    b.num_sms = c->num_sms;
    b.pair = getenv("LLEP_BWD_1CTA") ? 0 : 1;
    // opt-in: dA0 GEMM with the SwiGLU backward fused into its epilogue.  Measured 11-15 % SLOWER per
    // training step than dA0 + bwd_swiglu (its epilogue's per-row GU loads are latency-bound and
    // outlast the tile's MMAs), so the separate kernel is the default
    const char *fz = getenv("LLEP_BWD_FUSED");
    const bool fuse = b.pair && fz && atoi(fz);
    if (fuse) {
      // dA0 GEMM with the SwiGLU backward in its epilogue (dA0 never reaches HBM): w·a, [dg | du] and
      // per-tile partial dots; padding rows zeroed separately; dL/dw = fixed-order sum of the partials
      const int nparts = 2 * ((H + 255) / 256);
      const int64_t need = c->arena_rows * nparts;
      if (need > c->dotp_cap) {
        if ((st = grow_lazy(c, &c->dotp, &c->dotp_cap, need, s)) != LLEP_OK) return st;
      }
      b.kind = 2;
      b.gu = GU;
      b.gate = G;
      b.aw = c->aw;
      b.dgu = c->dgu;
      b.dotp = c->dotp;
      if ((st = run_gemm_bwd(b, s)) != LLEP_OK) return st;
      LLEP_CUDA(launch_zero_pad(c->groups, G_, H, c->aw, nullptr, s));
      LLEP_CUDA(launch_zero_pad(c->groups, G_, 2 * H, c->dgu, nullptr, s));
      LLEP_CUDA(launch_dot_reduce(c->groups, G_, (int)sum.my_padded, nparts, c->dotp, G, s));
      c->launches += 4;
      b.kind = 0;
    } else {
      if ((st = run_gemm_bwd(b, s)) != LLEP_OK) return st;
      ++c->launches;
      // SwiGLU backward per row; dL/dw replaces the gate in G
      LLEP_CUDA(launch_bwd_swiglu(c->groups, G_, (int)sum.my_padded, H, GU, c->da0, G, c->aw, c->dgu, s));
      ++c->launches;
    }
    // dW_down = dOᵀ · (w a)   and   dW13 = [dg|du]ᵀ · X   (native -> dw2/dw13, foreign -> staging);
    // large groups are split along their rows, partials summed in fixed order (deterministic)
    std::vector<int32_t> grows, gslot, gexp;
    my_groups_host(c, grows, gslot, gexp);
    const int bwd_pair = getenv("LLEP_BWD_1CTA") ? 0 : 1;   // 2-CTA backward GEMMs (A/B switch)
    const int units = bwd_pair ? -(c->num_sms / 2) : c->num_sms;
    const int64_t need_ws = std::max(wgrad_workspace(grows.data(), (int)grows.size(), D, H, units),
                                     wgrad_workspace(grows.data(), (int)grows.size(), 2 * H, D, units));
    if (need_ws > c->ws_cap) {
      if ((st = grow_lazy(c, &c->wsbuf, &c->ws_cap, need_ws, s)) != LLEP_OK) return st;
    }
    BwdArgs w;
    memset(&w, 0, sizeof(w));
    w.kind = 1;
    w.n_out_slots = M;
    w.n_foreign_slots = c->arena_foreign;
    w.rows = c->arena_rows;
    w.kdim = 8;
    w.groups = c->groups;
    w.n_groups = G_;
    w.mblk_scale = 2;
    w.num_sms = c->num_sms;
    w.pair = bwd_pair;
    w.ws = c->wsbuf;
    w.a = O;
    w.b = c->aw;
    w.mdim = D;
    w.nout = H;
    w.n_ws_slots = c->ws_cap / ((int64_t)D * H);
    w.out = dw2;
    w.out_foreign = c->stage2;
    if ((st = run_gemm_bwd(w, s)) != LLEP_OK) return st;
    if ((st = reduce_wgrad_splits(w, grows.data(), gslot.data(), gexp.data(), (int)grows.size(), s)) != LLEP_OK)
      return st;
    w.a = c->dgu;
    w.b = X;
    w.mdim = 2 * H;
    w.nout = D;
    w.n_ws_slots = c->ws_cap / ((int64_t)2 * H * D);
    w.out = dw13;
    w.out_foreign = c->stage13;
    if ((st = run_gemm_bwd(w, s)) != LLEP_OK) return st;
    if ((st = reduce_wgrad_splits(w, grows.data(), gslot.data(), gexp.data(), (int)grows.size(), s)) != LLEP_OK)
      return st;
    c->launches += 2;
    // dX = [dg|du] · W13   (W13 [2H][D] row-major: MN-major B), into X's rows (X is dead now)
    b.a = c->dgu;
    b.b = w13;
    b.kdim = 2 * H;
    b.nout = D;
    b.b_foreign = reinterpret_cast<const uint16_t *>(c->arena + c->off_w13);
    b.out = X;
    if ((st = run_gemm_bwd(b, s)) != LLEP_OK) return st;
    ++c->launches;
  }
  // push the weight-gradient partials of foreign experts to their native devices; the slot on
  // device n of (e, d) is the position of (e, d) among n's 𝒲 entries ordered by (e, d)
  bool any_push = false;
  if (P > 1) {
    int f = 0;
    for (int e = 0; e < N; ++e) {
      if (!replica[(size_t)e * P + c->rank]) continue;
      const int n = e / M;
      int slot = 0;
      for (int e2 = n * M; e2 < (n + 1) * M; ++e2)
        for (int d2 = 0; d2 < P; ++d2)
          if (replica[(size_t)e2 * P + d2] && (e2 < e || (e2 == e && d2 < c->rank))) ++slot;
      if (!any_push) {
        LLEP_CUDA(cudaEventRecord(c->ev_fork, s));
        LLEP_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        any_push = true;
      }
      uint8_t *dst = c->peer_base[n] + c->off_grad + (size_t)slot * slot_all * 4;
      LLEP_CUDA(cudaMemcpyAsync(dst, c->stage13 + (size_t)f * slot13, slot13 * 4, cudaMemcpyDeviceToDevice, c->side));
      LLEP_CUDA(cudaMemcpyAsync(dst + slot13 * 4, c->stage2 + (size_t)f * slot2, slot2 * 4,
                                cudaMemcpyDeviceToDevice, c->side));
      ++f;
    }
  }
  if (any_push) {
    LLEP_CUDA(cudaEventRecord(c->ev_join, c->side));
    LLEP_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
  }
  if ((st = barrier(c, s)) != LLEP_OK) return st;
  // dx[t] = Σ_k dX[dst(t,k)] (slot order), dgates[t,k] = dL/dw of that row
  CombineArgs ca;
  ca.slot_dst = c->slot_dst;
  ca.peer_y = peer_x(c);
  ca.B = B;
  ca.K = c->K;
  ca.D = D;
  ca.out = dx;
  ca.peer_s = reinterpret_cast<const float *const *>(c->d_ptrs + 3 * P);
  ca.slot_out = dgates;
  LLEP_CUDA(launch_combine(ca, s));
  c->launches += B > 0;
  // native device: add the returned partials, ascending source device (slots are (e, d)-ordered)
  if (P > 1) {
    int slot = 0;
    for (int e = c->rank * M; e < (c->rank + 1) * M; ++e) {
      int cnt = 0;
      for (int d2 = 0; d2 < P; ++d2) cnt += replica[(size_t)e * P + d2];
      if (cnt) {
        const int el = e - c->rank * M;
        const float *base = reinterpret_cast<const float *>(c->arena + c->off_grad) + (size_t)slot * slot_all;
        LLEP_CUDA(launch_grad_reduce(dw13 + (size_t)el * slot13, base, cnt, slot_all, slot13, s));
        LLEP_CUDA(launch_grad_reduce(dw2 + (size_t)el * slot2, base + slot13, cnt, slot_all, slot2, s));
        c->launches += 2;
      }
      slot += cnt;
    }
  }
  return LLEP_OK;
}

llep_status llep_moe_backward(llep_context *c, const uint16_t *x, const int32_t *ids, const float *topk_w,
                              const uint16_t *dout, int64_t B, const uint16_t *w13, const uint16_t *w2,
                              const void *plan, uint16_t *dx, float *dgates, float *dw13, float *dw2,
                              void *stream) {
  return moe_backward(c, x, ids, topk_w, dout, B, w13, w2, plan, dx, dgates, dw13, dw2, nullptr, 0, stream);
}

llep_status llep_moe_backward_saved(llep_context *c, const uint16_t *x, const int32_t *ids,
                                    const float *topk_w, const uint16_t *dout, int64_t B, const uint16_t *w13,
                                    const uint16_t *w2, const void *plan, const uint16_t *gu_saved,
                                    int64_t gu_rows, uint16_t *dx, float *dgates, float *dw13, float *dw2,
                                    void *stream) {
  if (!gu_saved) return invalid("null pointer (gu_saved)");
  return moe_backward(c, x, ids, topk_w, dout, B, w13, w2, plan, dx, dgates, dw13, dw2, gu_saved, gu_rows,
                      stream);
}

llep_status llep_context_check(llep_context *c, void *stream) {
  if (!c) return invalid("null context");
  cudaStream_t s = (cudaStream_t)stream;
  LLEP_CUDA(cudaStreamSynchronize(s));
  int32_t e[4];
  LLEP_CUDA(cudaMemcpy(e, c->err, sizeof(e), cudaMemcpyDeviceToHost));
  llep_status st = decode_err(c, e, s);
  LLEP_CUDA(cudaStreamSynchronize(s));
  return st;
}

llep_status llep_context_set_timing(llep_context *c, int32_t enable) {
  if (!c) return invalid("null context");
  collect(c);
  c->timing = enable != 0;
  return LLEP_OK;
}

llep_status llep_context_stats(llep_context *c, llep_stats *out, int32_t reset) {
  if (!c || !out) return invalid("null pointer");
  collect(c);
  for (int p = 0; p < LLEP_NUM_PHASES; ++p) out->ms[p] = c->phase_ms[p];
  out->calls = c->calls;
  out->kernel_launches = c->launches;
  out->gemm_rows = c->gemm_rows;
  if (reset) {
    for (int p = 0; p < LLEP_NUM_PHASES; ++p) c->phase_ms[p] = 0.0;
    c->calls = c->launches = c->gemm_rows = 0;
  }
  return LLEP_OK;
}

llep_status llep_debug_copy(llep_context *c, int32_t what, void *dst, int64_t n, void *stream) {
  if (!c || !dst) return invalid("null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const void *src = nullptr;
  size_t esz = 4, avail = 0;
  const int64_t slots = std::max<int64_t>(0, c->prepared_tokens) * c->K;
  switch (what) {
    case LLEP_DBG_LOAD_MATRIX: src = c->lm_local; avail = (size_t)c->P * c->N; break;
    case LLEP_DBG_SLOT_DST: src = c->slot_dst; avail = 2 * slots; break;
    case LLEP_DBG_GROUPS: src = c->groups; avail = (size_t)kMaxGroups * 8; break;
    case LLEP_DBG_RECV_X: src = c->arena + c->off_x; esz = 2; avail = (size_t)c->arena_rows * c->D; break;
    case LLEP_DBG_Y: src = c->arena + c->off_x; esz = 2; avail = (size_t)c->arena_rows * c->D; break;
    case LLEP_DBG_ACT: src = c->act; esz = 2; avail = (size_t)c->arena_rows * c->H; break;
    case LLEP_DBG_LOCAL_RANK: src = c->local_rank; avail = slots; break;
    case LLEP_DBG_RECV_G: src = c->arena + c->off_g; avail = c->arena_rows; break;
    default: return invalid("unknown debug buffer");
  }
  if (n < 0 || (size_t)n > avail) return invalid("n_elems exceeds the buffer");
  LLEP_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * esz, cudaMemcpyDeviceToDevice, s));
  return LLEP_OK;
}

llep_status llep_router(const uint16_t *x, const uint16_t *w_router, int64_t n_tokens, int32_t d_model,
                        int32_t n_experts, int32_t top_k, int32_t *topk_ids, float *topk_w,
                        float *logits, void *stream) {
  if (n_tokens < 0) return invalid("n_tokens < 0");
  if (n_experts < 1 || n_experts > 512) return invalid("router: n_experts must be in [1, 512]");
  if (top_k < 1 || top_k > 16 || top_k > n_experts) return invalid("router: top_k must be in [1, min(16, N)]");
  if (d_model < 8 || d_model % 8) return invalid("router: d_model must be a positive multiple of 8");
  if (n_tokens == 0) return LLEP_OK;
  if (!x || !w_router || !topk_ids || !topk_w) return invalid("null pointer");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w_router)) & 15)
    return invalid("router: x and w_router must be 16-byte aligned");
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    LLEP_CUDA(cudaGetDevice(&dev));
    LLEP_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  RouterArgs a{x, w_router, n_tokens, d_model, n_experts, top_k, topk_ids, topk_w, logits, num_sms};
  return run_router(a, (cudaStream_t)stream);
}

llep_status llep_grouped_gemm(int32_t mode, const uint16_t *a, int64_t rows, int32_t kdim,
                              const uint16_t *w, int32_t n_weights, int32_t nout,
                              const int32_t *groups, int32_t n_groups, const float *gate,
                              uint16_t *out, void *stream) {
  if (mode < 0 || mode > 3) return invalid("mode must be 0..3");
  const int ra = (mode & 2) ? 256 : kRowAlign;   // mode bit 1: 2-CTA (cta_group::2) tiles
  mode &= 1;
  if (!a || !w || !groups || !out || (mode == 1 && !gate)) return invalid("null pointer");
  if (n_groups < 0 || n_groups > kMaxGroups) return invalid("n_groups out of range");
  std::vector<Group> g(std::max(n_groups, 1));
  int mb = 0;
  for (int i = 0; i < n_groups; ++i) {
    const int32_t *q = groups + 4 * i;
    if (q[0] < 0 || q[0] >= n_weights) return invalid("group expert out of range");
    if (q[1] % ra || q[2] < 1 || q[1] + (int64_t)q[2] > rows)
      return invalid("group rows must start tile-aligned (128, or 256 for 2-CTA), be nonempty and fit");
    if (i > 0 && q[1] < g[i - 1].row_base + ((g[i - 1].n_rows + ra - 1) / ra) * ra)
      return invalid("groups must be in increasing, non-overlapping row order");
    g[i] = Group{q[0], q[0], q[1], q[2], mb, {0, 0, 0}};
    mb += (q[2] + ra - 1) / ra;
    // mblk_start counts only this group's blocks: rows between groups are skipped
  }
  // m-block schedule, same interleave as the layout kernel
  int64_t nb = 0, ns = 0;
  std::vector<int64_t> before(std::max(n_groups, 1));
  for (int i = 0; i < n_groups; ++i) {
    const int b = (g[i].n_rows + ra - 1) / ra;
    if (b * ra > kSmallGroupRows) { before[i] = nb; nb += b; }
    else { before[i] = ns; ns += b; }
  }
  std::vector<int32_t> sched(std::max<int64_t>(mb, 1));
  for (int i = 0; i < n_groups; ++i) {
    const int b = (g[i].n_rows + ra - 1) / ra;
    for (int m = 0; m < b; ++m)
      sched[interleave_pos(b * ra > kSmallGroupRows, before[i] + m, nb, ns)] = sched_pack(i, m);
  }
  cudaStream_t s = (cudaStream_t)stream;
  Group *dg = nullptr;
  int32_t *dsched = nullptr;
  LLEP_CUDA(cudaMallocAsync(&dg, sizeof(Group) * g.size(), s));
  LLEP_CUDA(cudaMemcpyAsync(dg, g.data(), sizeof(Group) * g.size(), cudaMemcpyHostToDevice, s));
  LLEP_CUDA(cudaMallocAsync(&dsched, sizeof(int32_t) * sched.size(), s));
  LLEP_CUDA(cudaMemcpyAsync(dsched, sched.data(), sizeof(int32_t) * sched.size(), cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GemmArgs ga;
  memset(&ga, 0, sizeof(ga));
  ga.mode = mode;
  ga.a = a;
  ga.a_rows = rows;
  ga.kdim = kdim;
  ga.w_native = w;
  ga.n_native = n_weights;
  ga.w_foreign = nullptr;
  ga.n_foreign = 0;
  ga.nout = nout;
  ga.groups = dg;
  ga.sched = getenv("LLEP_GEMM_GROUP_ORDER") ? nullptr : dsched;  // A/B switch for the schedule
  ga.n_groups_dev = nullptr;
  ga.n_groups_host = n_groups;
  ga.gate = gate;
  ga.out = out;
  ga.num_sms = sms;
  ga.row_align = ra;
  llep_status st = n_groups > 0 ? run_grouped_gemm(ga, s) : LLEP_OK;
  cudaFreeAsync(dg, s);
  cudaFreeAsync(dsched, s);
  return st;
}

llep_status llep_gemm_bwd(int32_t kind, const uint16_t *a, const uint16_t *w_or_b, int64_t rows,
                          int32_t kdim_or_mdim, int32_t nout, int32_t n_weights, const int32_t *groups,
                          int32_t n_groups, void *out, void *stream) {
  const int pair = (kind & 2) ? 1 : 0;   // kind bit 1: 2-CTA (cta_group::2) variant
  kind &= 1;
  if (!a || !w_or_b || !groups || !out) return invalid("null pointer");
  if (n_groups < 0 || n_groups > kMaxGroups) return invalid("n_groups out of range");
  std::vector<Group> g(std::max(n_groups, 1));
  int mb = 0;
  for (int i = 0; i < n_groups; ++i) {
    const int32_t *q = groups + 4 * i;
    if (q[0] < 0 || q[0] >= n_weights) return invalid("group expert out of range");
    if (q[1] % 256 || q[2] < 1 || q[1] + (int64_t)((q[2] + 255) / 256 * 256) > rows)
      return invalid("group rows must start 256-aligned, be nonempty and fit (padded to 256)");
    g[i] = Group{q[0], q[0], q[1], q[2], mb, {0, 0, 0}};
    mb += (q[2] + 255) / 256;
  }
  cudaStream_t s = (cudaStream_t)stream;
  Group *dg = nullptr;
  LLEP_CUDA(cudaMallocAsync(&dg, sizeof(Group) * g.size(), s));
  LLEP_CUDA(cudaMemcpyAsync(dg, g.data(), sizeof(Group) * g.size(), cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  BwdArgs ba;
  memset(&ba, 0, sizeof(ba));
  ba.kind = kind;
  ba.a = a;
  ba.b = w_or_b;
  ba.rows = rows;
  ba.kdim = kind == 0 ? kdim_or_mdim : 8;
  ba.mdim = kind == 1 ? kdim_or_mdim : 8;
  ba.nout = nout;
  ba.n_weights = n_weights;
  ba.groups = dg;
  ba.n_groups = n_groups;
  ba.mblk_scale = 2;   // Group.mblk_start counts 256-row blocks
  ba.out = out;
  ba.num_sms = sms;
  if (const char *o = getenv("LLEP_GEMM_SMS")) ba.num_sms = std::max(2, std::min(sms, atoi(o)));   // experiments
  ba.pair = pair;
  std::vector<int32_t> nr(n_groups), ex(n_groups);
  for (int i = 0; i < n_groups; ++i) {
    nr[i] = groups[4 * i + 2];
    ex[i] = groups[4 * i];
  }
  float *ws = nullptr;
  if (kind == 1) {
    const int64_t need = wgrad_workspace(nr.data(), n_groups, ba.mdim, nout, pair ? -(sms / 2) : sms);
    if (need > 0) LLEP_CUDA(cudaMallocAsync(&ws, (size_t)need * 4, s));
    ba.n_ws_slots = need / ((int64_t)ba.mdim * nout);
    ba.n_out_slots = n_weights;
  }
  ba.ws = ws;
  llep_status st = n_groups > 0 ? run_gemm_bwd(ba, s) : LLEP_OK;
  if (st == LLEP_OK && kind == 1 && n_groups > 0)
    st = reduce_wgrad_splits(ba, nr.data(), nr.data(), ex.data(), n_groups, s);
  if (ws) cudaFreeAsync(ws, s);
  cudaFreeAsync(dg, s);
  return st;
}

}  // extern "C"
