// Internal declarations shared by the LLEP CUDA translation units (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "llep.h"

namespace llep {

constexpr int kMaxWorld = 32;     // device planner keeps one device per lane
constexpr int kRowAlign = 128;    // group row bases are aligned to the GEMM M tile
constexpr int kTileSlots = 1024;  // slots per histogram / local-rank tile
constexpr int kMaxGroups = 1024;  // expert groups one rank may compute

void set_error(const char *fmt, ...);
llep_status cuda_status(cudaError_t e, const char *what);

#define LLEP_CUDA(call)                                                    \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) return ::llep::cuda_status(_e, #call);          \
  } while (0)

// Plan blob field offsets (see llep.h "plan blob").
struct PlanLayout {
  int32_t off_assigned, off_n_chunks, off_chunks, off_replica;
  size_t bytes;
};
__host__ __device__ inline size_t align8(size_t x) { return (x + 7) & ~size_t(7); }
__host__ __device__ inline PlanLayout plan_layout(int32_t N, int32_t P) {
  PlanLayout L;
  size_t off = align8(sizeof(llep_plan_header));
  L.off_assigned = (int32_t)off;
  off = align8(off + sizeof(int64_t) * P);
  L.off_n_chunks = (int32_t)off;
  off = align8(off + sizeof(int32_t) * N);
  L.off_chunks = (int32_t)off;
  off = align8(off + sizeof(llep_chunk) * (size_t)N * (P + 1));
  L.off_replica = (int32_t)off;
  off = align8(off + (size_t)N * P);
  L.bytes = off;
  return L;
}

// GEMM m-block schedule.  Groups with few 128-row blocks stream a whole expert's weights for
// little work (weight-bandwidth bound); their blocks are spread evenly among the blocks of large
// groups so the persistent GEMM overlaps that streaming with compute-bound tiles.
#ifndef LLEP_SMALL_GROUP_ROWS
// 512: at the G120 P=8 critical-rank layout the 15 native groups of 416 rows (512 padded) are then
// spread among the spilled chunk's blocks (and their weights read evict-first): GEMM1 -0.6 %, GEMM2
// -0.7 % at base clocks vs 256; P=1 unchanged (profiles/r02_ab_small_group_rows.txt)
#define LLEP_SMALL_GROUP_ROWS 512
#endif
constexpr int kSmallGroupRows = LLEP_SMALL_GROUP_ROWS;  // groups of at most this many padded rows are "small"
// Position of the idx-th block of its class when nb "big" and ns "small" blocks are merged
// evenly: keys (2k+1)*ns for big block k, (2j+1)*nb for small block j, ties -> big first.
__host__ __device__ inline int64_t interleave_pos(bool big, int64_t idx, int64_t nb, int64_t ns) {
  if (big) {
    if (ns == 0) return idx;
    const int64_t c = ((2 * idx + 1) * ns - 1) / nb;
    const int64_t cnt = (c + 1) / 2;
    return idx + (cnt < ns ? cnt : ns);
  }
  if (nb == 0) return idx;
  const int64_t c = ((2 * idx + 1) * nb) / ns;
  const int64_t cnt = (c + 1) / 2;
  return idx + (cnt < nb ? cnt : nb);
}
__host__ __device__ inline int32_t sched_pack(int32_t g, int32_t m) { return (g << 20) | m; }

// Split-K of the weight-gradient GEMMs (contraction over a group's rows): a group with many rows is
// cut into K ranges so its output tiles fill the SMs in several waves; each range writes an fp32
// partial into a workspace and the partials are summed in fixed order (deterministic).
constexpr int kSplitMinRows = 4096;
__host__ __device__ inline int wgrad_splits(int n_rows, int tiles_per_split, int num_sms) {
  const int padded = (n_rows + 255) / 256 * 256;
  if (n_rows < kSplitMinRows) return 1;
  int want = (4 * num_sms + tiles_per_split - 1) / tiles_per_split;   // >= ~4 waves per group
  const int cap = padded / 1024;                                       // >= 1024 rows per split
  if (want > cap) want = cap;
  if (want < 1) want = 1;
#ifndef LLEP_WG_WAVEFIT
#define LLEP_WG_WAVEFIT 1
#endif
  if (LLEP_WG_WAVEFIT) {
    // the tiles are scheduled statically over the units, so a last wave that is only partly full
    // leaves units idle for one (long) tile: take up to 2x the splits if that fills the waves >= 2 %
    // better (waves per split, ceil(tiles / units) / splits).  G120 P=8 dW13: 276 tiles per split on
    // 74 CTA pairs -> 2 splits = 7.46 waves run as 8, 4 splits = 14.92 as 15: dW13 + its reduce
    // -0.3..-2 % (P=8 layout) and -3 % (P=1) at base clocks (profiles/r02_ab_wgrad_wavefit.txt); the
    // small groups' tiles that follow already fill most of the idle tail
    const int w0 = want;
    float best = (float)((tiles_per_split * w0 + num_sms - 1) / num_sms) / w0;
    for (int sp = w0 + 1; sp <= 2 * w0 && sp <= cap; ++sp) {
      const float c = (float)((tiles_per_split * sp + num_sms - 1) / num_sms) / sp;
      if (c < 0.98f * best) {
        best = c;
        want = sp;
      }
    }
  }
  const int ks = ((padded + want - 1) / want + 255) / 256 * 256;       // 256-row aligned K range
  return (padded + ks - 1) / ks;
}
__host__ __device__ inline int wgrad_split_rows(int n_rows, int splits) {
  const int padded = (n_rows + 255) / 256 * 256;
  return ((padded + splits - 1) / splits + 255) / 256 * 256;
}

// Offset of source rank p's block in expert e's global token range (a3/a5).  aligned = 0: rank-major,
// Σ_{q<p} C[q][e] (reading R11).  aligned = 1 (R11', the default): for an expert with more than one chunk
// the blocks follow e's chunk devices in plan order (first appearance), then the other ranks ascending,
// so a spill device's chunk holds its own rows wherever the counts allow.  A: e's chunks, nc of them;
// C: the [P, N] load matrix.  Identical on every rank (replicated plan and C).
__device__ __forceinline__ int64_t source_offset(const llep_chunk *A, int nc, const int32_t *C, int N, int P,
                                                 int e, int p, int aligned) {
  int64_t off = 0;
  if (!aligned || nc <= 1) {
    for (int q = 0; q < p; ++q) off += C[(size_t)q * N + e];
    return off;
  }
  uint32_t seen = 0;
  for (int c = 0; c < nc; ++c) {
    const int d = A[c].device;
    if ((seen >> d) & 1u) continue;
    if (d == p) return off;
    seen |= 1u << d;
    off += C[(size_t)d * N + e];
  }
  for (int q = 0; q < p; ++q)
    if (!((seen >> q) & 1u)) off += C[(size_t)q * N + e];
  return off;
}

// Group table entry (8 int32) of one expert group a device computes.
struct Group {
  int32_t expert;      // global expert id
  int32_t wslot;       // >= 0: native slot (e - rank*M);  < 0: foreign slot f = -1 - wslot
  int32_t row_base;    // first receive row (multiple of kRowAlign)
  int32_t n_rows;      // rows of this expert on this device
  int32_t mblk_start;  // prefix sum of ceil(n_rows / 128) over earlier groups
  int32_t pad[3];
};

// Summary written by the layout kernel, read back once by the host.
struct LayoutSummary {
  int64_t rows_needed;   // max_d padded rows
  int64_t my_rows;       // g_a[rank]
  int64_t my_padded;     // padded rows of this rank
  int32_t foreign_needed;
  int32_t my_groups;
  int32_t my_mblocks;
  int32_t fallback_ep, force_count, n_transfers;
  int32_t error;         // nonzero: plan/load inconsistency
  int32_t pad;
};

// Device workspace pointers of the layout step (rank-local).
struct LayoutArgs {
  const void *plan;
  const int32_t *load_matrix;  // [P, N]
  int32_t N, P, M, rank;
  int32_t *rows_on;            // [N*P] rows of e on d
  int32_t *chunk_row;          // [N*(P+1)] destination row of each chunk's first token
  int32_t *foreign_slot;       // [N*P] foreign slot of e on d, -1 if none
  Group *groups;               // [kMaxGroups] this rank's groups
  int32_t *dev_padded;         // [P] padded rows per device
  int32_t *dev_foreign;        // [P] |S_d|
  LayoutSummary *summary;
  int32_t *sched;              // [sched_cap] this rank's m-block order (sched_pack)
  int64_t sched_cap;
  int32_t row_align;           // group row bases / GEMM M tile: 128 or 256
  uint32_t *mblk_src;          // [sched_cap] per m-block (group order) of this rank: bit q set iff the
                               // block holds rows dispatched by source rank q (row f2 arrival waits)
  int32_t aligned;             // token order (source_offset): 0 rank-major (R11), 1 chunk-aligned (R11')
  // capture-safe layer (llep_moe_layer) only: the arena this call must fit.  A plan that needs more rows
  // or foreign slots on ANY device (the same decision on every rank) sets summary->error |= 16,
  // err[3] |= 1 and *n_groups_dev = 0, so no kernel of that call writes past the arena.
  int64_t arena_rows;          // 0: no check (the two-call path checks on the host)
  int32_t arena_foreign;
  int32_t *n_groups_dev;       // this rank's group count for the GEMMs (0 on overflow)
  int32_t *err;
};

// Device-resident epochs (one word each, zero at context creation).  Every synchronising kernel reads
// its epoch from here instead of a launch argument, so a captured CUDA graph replays correctly: the
// barrier kernel advances kEpBarrier itself; advance_kernel bumps kEpWeight and kEpArrive once at the
// start of every forward / backward call (P > 1).  All ranks run the same sequence -> same values.
constexpr int kEpBarrier = 0, kEpWeight = 1, kEpArrive = 2;

// kernel launchers (route.cu / plan.cu / gemm.cu)
cudaError_t launch_tile_count(const int32_t *ids, int64_t n_slots, int32_t N, int32_t *tile_cnt,
                              int32_t *err, cudaStream_t s);
cudaError_t launch_tile_scan(const int32_t *tile_cnt, int32_t n_tiles, int32_t N, int32_t *tile_off,
                             int32_t *cnt_out, cudaStream_t s);
cudaError_t launch_local_rank(const int32_t *ids, int64_t n_slots, int32_t N, const int32_t *tile_off,
                              int32_t *local_rank, int32_t *prep_ids, cudaStream_t s);
cudaError_t launch_push_counts(const int32_t *cnt, int32_t N, int32_t rank, int32_t P,
                               int32_t *const *peer_lm, cudaStream_t s);
cudaError_t launch_barrier(uint32_t *const *peer_flags, int32_t rank, int32_t P, uint32_t *ep,
                           int32_t *err, cudaStream_t s);
cudaError_t launch_advance(uint32_t *ep, cudaStream_t s);
cudaError_t launch_planner(const int32_t *load_matrix, int32_t N, int32_t P, double alpha,
                           int64_t min_chunk, double lambda, int32_t force_ep, void *plan,
                           cudaStream_t s);
cudaError_t launch_layout(const LayoutArgs &a, cudaStream_t s);
cudaError_t launch_zero_pad(const Group *groups, int n_groups, int D, uint16_t *buf0, uint16_t *buf1,
                            cudaStream_t s);
cudaError_t launch_dot_reduce(const Group *groups, int n_groups, int n_rows_total, int nparts, const float *dotp,
                              float *gate_io, cudaStream_t s);
cudaError_t launch_bwd_swiglu(const Group *groups, int n_groups, int n_rows_total, int H, const uint16_t *GU,
                              const uint16_t *dA0, float *gate_io, uint16_t *Aw, uint16_t *dGU, cudaStream_t s);
cudaError_t launch_grad_reduce(float *dst, const float *base, int n_src, int64_t stride_floats, int64_t n_floats,
                               cudaStream_t s);
cudaError_t launch_signal(uint32_t *flag, const uint32_t *ep, cudaStream_t s);
cudaError_t launch_wait_flag(const uint32_t *flag, const uint32_t *ep, int32_t *err, cudaStream_t s);
constexpr int kWeightFlag0 = 32;   // arena flag words: [0, 32) barrier, [32, 32 + kMaxGroups) weight slots,
constexpr int kArriveFlag0 = kWeightFlag0 + kMaxGroups;   // then [32) dispatch arrivals (one per source)
constexpr int kFlagWords = kArriveFlag0 + kMaxWorld;
cudaError_t launch_arrive(uint32_t *const *peer_flags, int32_t rank, int32_t P, const uint32_t *ep, cudaStream_t s);
cudaError_t launch_combine_local(const uint16_t *slotbuf, int64_t B, int K, int D, const int32_t *slot_dst,
                                 uint16_t *out, cudaStream_t s);
cudaError_t launch_mirror(const void *plan, size_t plan_bytes, const void *summary, size_t sum_bytes,
                          const int32_t *err, void *host_plan, void *host_sum, int32_t *host_err,
                          cudaStream_t s);

struct DispatchArgs {
  const uint16_t *x;        // [B, D]
  const int32_t *ids;       // [B, K]
  const float *w;           // [B, K]
  const int32_t *local_rank;
  const int32_t *prep_ids;  // [B, K] the ids llep_prepare planned with (addressing uses these)
  int32_t *err;             // err[2] |= 1: a slot's id differs from the prepared one (slot dropped)
  const int32_t *load_matrix;
  const void *plan;
  const int32_t *chunk_row;
  int64_t B;
  int32_t K, D, N, P, rank;
  uint16_t *const *peer_x;  // [P] receive rows base of each device (peer-mapped)
  float *const *peer_g;     // [P]
  int32_t *slot_dst;        // [2*B*K] (device, row)
  const uint16_t *x2;       // optional second row source (backward: the upstream gradient dOut)
  uint16_t *const *peer_x2; // [P] its receive rows
  int32_t *const *peer_rsrc;  // optional [P] per receive row: (flat slot << 5) | source rank
  // row f2 (dispatch overlapped with the GEMMs): when peer_flags is set, the last block to finish
  // publishes `epoch` into arrival flag [rank] of every device (release, system scope) once all of this
  // rank's rows are stored; block_done counts finished blocks (rank-local, returns to 0)
  uint32_t *const *peer_flags;
  const uint32_t *ep;       // device epochs: the arrival value is ep[kEpArrive]
  uint32_t *block_done;
  const int32_t *skip;      // capture-safe layer: nonzero (arena overflow, LayoutSummary.error bit 16)
                            // -> the kernel stores nothing but still publishes its arrival flags
  // row a6 local-row gather: a row this rank sends to ITSELF, in an m-block whose rows all come from
  // this rank (mblk_src[row / row_align] == 1 << rank), is not copied: rtok[row] = its token index and
  // GEMM1 gathers x[t] straight from the caller's tokens with TMA (nullptr: copy every row)
  int32_t *rtok;
  const uint32_t *mblk_src;
  int32_t row_align;
  int32_t aligned;          // token order of the global index (source_offset)
};
cudaError_t launch_dispatch(const DispatchArgs &a, cudaStream_t s);

struct CombineArgs {
  const int32_t *slot_dst;
  const uint16_t *const *peer_y;  // [P]
  int64_t B;
  int32_t K, D;
  uint16_t *out;
  const float *const *peer_s;  // optional per-row scalar to pull per slot (backward: dL/dgate)
  float *slot_out;             // [B*K]
};
cudaError_t launch_combine(const CombineArgs &a, cudaStream_t s);

// grouped GEMM (gemm.cu).  mode 0: SwiGLU epilogue; mode 1: gate-scale epilogue.
struct GemmArgs {
  int32_t mode;
  const uint16_t *a;         // [rows, kdim]
  int64_t a_rows;
  int32_t kdim;
  const uint16_t *w_native;  // [n_native * wrows, kdim]
  int32_t n_native;
  const uint16_t *w_foreign; // [n_foreign * wrows, kdim]
  int32_t n_foreign;
  int32_t nout;              // output columns: H (mode 0) or D (mode 1)
  const Group *groups;       // device
  const int32_t *sched;      // device m-block order (sched_pack), or nullptr = group order
  const int32_t *n_groups_dev;  // device int (may be nullptr -> n_groups_host)
  int32_t n_groups_host;
  const float *gate;         // [rows] (mode 1)
  uint16_t *out;             // [rows, nout]
  uint16_t *out2;            // mode 3 (GEMM1 + SwiGLU that also saves [g | u]): [rows, 2*nout]
  const uint32_t *wflags;    // row f2: foreign slot f's weights landed when wflags[f] >= ep[kEpWeight]
  const uint32_t *ep;        //         (nullptr: weights already resident); device epochs
  int32_t *err;              //         err[1] |= 16 if a weight wait times out (~20 s); waits are
                             //         skipped once err[1] is set (a peer failed: no hang)
  const uint32_t *arrive;    // row f2: this rank's dispatch arrival flags [P] (nullptr: rows resident)
                             //         source q's rows landed when arrive[q] >= ep[kEpArrive]
  const uint32_t *mblk_src;  //         per m-block (group order): mask of the sources of its rows
  uint32_t src_all;          //         mask of every source rank: once all have arrived, skip the lookups
  const int32_t *row_src;    // mode 1 push epilogue: (slot << 5) | rank of each receive row, and
  uint16_t *const *peer_slot;//   [P] slot buffers [B*K, nout]: the row's output goes to
                             //   peer_slot[rank] + slot*nout (nullptr: write `out` rows)
  int32_t num_sms;
  int32_t row_align;         // 128: 1-CTA M=128 tiles; 256: 2-CTA (cta_group::2) M=256 tiles
  // modes 0/3, pair tiles: m-blocks with mblk_src[mblk] == self_mask read their A rows straight from
  // the tokens xg [xg_rows, kdim] (TMA gather4 of rows rtok[row]) instead of a (nullptr: off)
  const uint16_t *xg;
  int64_t xg_rows;
  const int32_t *rtok;
  uint32_t self_mask;
};
llep_status run_grouped_gemm(const GemmArgs &g, cudaStream_t s);

// a7 weight migration issued by the GPU (capture-safe layer): one launch per level of the binomial
// broadcast tree of every replicated expert (holders h_0 = native, then the replicas ascending; holder i
// sends to i + 2^t for 2^t > i).  Level 0 = the native sends, level l >= 1 = forwards by holders
// 2^(l-1) <= i < 2^l, each after acquiring its own slot's flag.  Every launch enumerates this rank's
// sends of its level from the plan, splits them into chunks over a fixed grid (16-byte loads, NVLink
// peer stores), and the last chunk of a send releases the destination slot's weight flag.
struct PushArgs {
  const void *plan;
  const int32_t *foreign_slot;      // [N*P] layout: position of e among d's foreign experts, -1 if none
  int32_t N, P, M, rank, level;
  const uint16_t *w13, *w2;         // this rank's native weights [M][2H][D], [M][D][H]
  uint8_t *const *peer_w13;         // [P] foreign-weight regions of every arena (w13 slots, then w2)
  uint8_t *const *peer_w2;
  uint32_t *const *peer_flags;      // [P] flag words of every arena
  int64_t w13_bytes, w2_bytes;      // per expert
  const uint32_t *ep;               // ep[kEpWeight]: the release value
  uint32_t *counters;               // [kMaxPushItems] chunk completion counts (return to 0)
  int32_t *err;                     // err[1] |= 8 when a forward's wait times out
  const int32_t *skip;              // arena overflow: no pushes (every rank decides the same)
};
constexpr int kMaxPushItems = 4096;
cudaError_t launch_push_level(const PushArgs &a, cudaStream_t s);

// backward GEMMs (gemm.cu).  kind 0: out[r] = a[r, 0:kdim] · W_e[kdim, nout] (bf16 out, grouped by rows,
// Group.mblk_start counted in units of mblk_scale 128-row blocks); kind 1: out[e] = a[rows_e]ᵀ · b[rows_e]
// (fp32 [mdim, nout] per group, K = the group's rows padded to 256, padding rows zero)
struct BwdArgs {
  int32_t kind;
  const uint16_t *a;
  const uint16_t *b;
  int64_t rows;
  int32_t kdim, mdim, nout, n_weights;
  const uint16_t *b_foreign;  // kind 0: foreign-expert weights (groups with wslot < 0)
  int32_t n_foreign;
  void *out_foreign;          // kind 1: output of groups with wslot < 0 (slot -1 - wslot); nullptr:
                              // every group writes `out` at slot Group.expert
  float *ws;                  // kind 1: split-K partials (wgrad_workspace floats)
  int64_t n_out_slots, n_foreign_slots, n_ws_slots;  // kind 1: [mdim x nout] slots behind each
  const Group *groups;
  int32_t n_groups;
  int32_t mblk_scale;
  void *out;
  int32_t num_sms;
  int32_t pair;               // 1: 2-CTA (cta_group::2) variant, 256-row / 256-output-row pair tiles
  // kind 2 (= kind 0 for dA0 = dY·W_down, with the SwiGLU backward fused into the epilogue; pair only):
  const uint16_t *gu;         //   [rows, 2*nout] saved / recomputed pre-activations [g | u]
  const float *gate;          //   [rows] the row's gate w
  uint16_t *aw, *dgu;         //   out: w·a [rows, nout], [dg | du] [rows, 2*nout]
  float *dotp;                //   out: partial <a, dA0> per (row, 128-column half tile) [rows, 2*ceil(nout/256)]
};
llep_status run_gemm_bwd(const BwdArgs &a, cudaStream_t s);

// router of Eq. 2 (row f4, router.cu)
struct RouterArgs {
  const void *x, *w_router;
  int64_t n_tokens;
  int32_t d_model, n_experts, top_k;
  int32_t *ids;
  float *gates, *logits;
  int32_t num_sms;
};
llep_status run_router(const RouterArgs &a, cudaStream_t s);
// host: workspace floats of a kind-1 launch over groups with these row counts; reduce the partials
int64_t wgrad_workspace(const int32_t *n_rows, int n_groups, int mdim, int nout, int num_sms);
llep_status reduce_wgrad_splits(const BwdArgs &a, const int32_t *n_rows, const int32_t *wslots,
                                const int32_t *experts, int n_groups, cudaStream_t s);

}  // namespace llep
