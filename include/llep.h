/*
 * llep.h -- C ABI of the B200-native Least-Loaded Expert Parallelism (LLEP) hot path.
 *
 * Paper: "Least-Loaded Expert Parallelism", arxiv 2601.17111 (text in PAPER.md; P:n = line n).
 * The problem as the paper states it: per device p, tokens B_p, router weights G_p and indices
 * I_p, and the local expert weights W_i, i in [pM, (p+1)M) -> the MoE output H'_p
 * (Alg. 4 header/output).  The planner takes the global loads l, M (hence P), α, m
 * (Alg. 2 input) and λ (Alg. 4).
 *
 * Conventions
 *   - Every pointer is plain host or device memory as stated per argument; no framework types.
 *   - Tensors are caller-owned.  The library never frees a caller pointer and keeps none past
 *     the call, except the context's OWN symmetric arena (see llep_context_*).
 *   - Device calls are stream-ordered on the caller's `stream` (a cudaStream_t passed as void*).
 *   - Return codes only; no exception crosses the ABI.  llep_last_error() gives a message
 *     (thread-local) naming the first violated condition.
 *   - Layouts are row-major.  bf16 = IEEE bfloat16 bit patterns (uint16_t).
 *   - Shapes: N experts, K = top-k, D = d_model, H = d_ff, P = EP world size, M = N / P,
 *     B = tokens on this rank.  Expert e is native to device floor(e / M) (Alg. 2).
 */
#ifndef LLEP_H
#define LLEP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status codes */
typedef enum {
  LLEP_OK = 0,
  LLEP_ERR_INVALID = 1,  /* bad argument: N % P != 0, K not in [1,N], D/H/P < 1, α < 1, λ < 1,
                            m < 0, negative load, misaligned / null pointer, unsupported shape  */
  LLEP_ERR_PLAN = 2,     /* plan inconsistent with the loads (chunk totals != l_e), or too
                            large for the context's arena (call llep_context_reserve first)     */
  LLEP_ERR_ROUTING = 3,  /* a router index outside [0, N) (detected on device, reported by the
                            next call that synchronises: llep_prepare)                          */
  LLEP_ERR_NOMEM = 4,    /* device allocation failed                                           */
  LLEP_ERR_CUDA = 5,     /* CUDA runtime / driver error                                        */
  LLEP_ERR_COMM = 6      /* peer mapping or device-barrier failure (timeout)                    */
} llep_status;

const char *llep_last_error(void);
const char *llep_version(void);

/* ------------------------------------------------------------------ parameters */
/* Planner constraints (§4 "Constraints"): α >= 1 scales the per-device capacity
 * m_α = α·Σl/P; m >= 0 is the minimum tokens per spilled GEMM chunk; λ >= 1 is the imbalance
 * threshold below which standard EP runs (max(l)/mean(l) < λ, Alg. 4).  The paper's
 * settings are α=1, m=1024, λ=1.3. */
typedef struct {
  double alpha;
  int64_t min_chunk;
  double lambda;
} llep_params;

/* ------------------------------------------------------------------ plan blob
 * A plan is one contiguous, caller-owned buffer of llep_plan_bytes(N, P) bytes, identical in
 * host and device memory, laid out as:
 *
 *   offset 0                 llep_plan_header
 *   hdr.off_assigned         int64_t    assigned[P]        g_a: rows device d computes
 *   hdr.off_n_chunks         int32_t    n_chunks[N]        chunks of expert e (0 if l_e == 0)
 *   hdr.off_chunks           llep_chunk chunks[N][P+1]     𝒜[e] in plan order; unused slots 0
 *   hdr.off_replica          uint8_t    replica[N][P]      𝒲: 1 iff e has a chunk on d != native
 *
 * 𝒜 (Alg. 2 output): expert e's global token range [0, l_e) is split into chunks
 * (device, start, end), in the order LLA/LLAS appended them; the native chunk (Case 1/2) first.
 * An expert can hold two chunks on one device (accepted spill + force-assign), and never more
 * than P+1 chunks (each non-final LLAS chunk fills a distinct device to capacity).
 * 𝒲: transfer of W_e from native(e) to every d with replica[e][d] = 1.
 * Two plans for the same inputs are bit-identical (host and device planners included). */
typedef struct {
  int32_t device, start, end;
} llep_chunk;

typedef struct {
  int32_t n_experts, world_size, max_chunks; /* max_chunks = P + 1                          */
  int32_t fallback_ep;   /* 1 iff S == 0 or max(l)/(S/N) < λ -> all-native plan  */
  int32_t force_count;   /* LLAS force-assigns; if > 0 a device may exceed cap   */
  int32_t n_transfers;   /* |𝒲|                                                             */
  int64_t total;         /* S = Σ l                                                          */
  int64_t capacity;      /* cap = floor((α·S)/P) in IEEE double, no FMA (m_α)         */
  int64_t max_assigned;  /* max_d g_a[d]                                                     */
  int32_t off_assigned, off_n_chunks, off_chunks, off_replica;
} llep_plan_header;

size_t llep_plan_bytes(int32_t n_experts, int32_t world_size);

/* llep_plan -- the LLEP planner on the host (Alg. 4 head P:537-541, Alg. 2 P:382-423,
 * Alg. 3, 𝒲 P:420).
 *   loads     [N] int64, host: global per-expert loads l (slot counts summed over ranks)
 *   plan_out  host buffer of llep_plan_bytes(N, P) bytes (written completely)
 * Readings of the paper's silent points are listed in DESIGN.md §Readings (R1-R9): integer
 * capacity, no empty chunks, skip of c <= 0 candidates, ties by (load desc, id asc) and
 * (g_a+g_p asc, id asc), whole-remainder force-assign.
 * Errors: LLEP_ERR_INVALID (N % P, α < 1, λ < 1, m < 0, negative load, null). Pure, re-entrant. */
llep_status llep_plan(const int64_t *loads, int32_t n_experts, int32_t world_size,
                      const llep_params *params, void *plan_out);

/* llep_plan_ep -- the all-native plan of standard EP (Alg. 1) on the host;
 * fallback_ep = 0 (it is the baseline, not the λ fallback). */
llep_status llep_plan_ep(const int64_t *loads, int32_t n_experts, int32_t world_size,
                         const llep_params *params, void *plan_out);

/* llep_plan_device -- the same planner as a one-warp device kernel (bit-identical blob).
 *   load_matrix  [P, N] int32, device: C[q][e] = rank q's slots routed to e; l = column sums
 *   plan_out     device buffer of llep_plan_bytes(N, P) bytes
 *   force_ep     0: LLEP (λ test + LLA); 1: standard-EP plan
 * Requires P <= 32.  Errors: LLEP_ERR_INVALID, LLEP_ERR_CUDA. */
llep_status llep_plan_device(const int32_t *load_matrix, int32_t n_experts, int32_t world_size,
                             const llep_params *params, int32_t force_ep, void *plan_out,
                             void *stream);

/* ------------------------------------------------------------------ context (one per rank)
 * The context owns this rank's symmetric arena: load-matrix slots, barrier flags, receive rows
 * X [R, D] bf16 + gates [R] fp32, expert-FFN outputs Y [R, D] bf16, activations A [R, H] bf16
 * and imported (foreign) expert weights.  Peers map each other's arenas through CUDA IPC so
 * the dispatch stores and combine loads go straight over NVLink (no staging copies). */
typedef struct llep_context llep_context;

typedef struct {
  int32_t n_experts, top_k, d_model, d_ff, world_size;
} llep_shape;

/* Create the context for `rank` on CUDA device `device` (the caller's current device).
 * max_tokens: largest B any rank will pass -- the SAME value on every rank (the arenas are symmetric:
 * peers address each other's regions with their own offsets; llep_context_open_peers compares every
 * peer's arena geometry and fails with LLEP_ERR_INVALID if it differs).  Allocates the rank-local
 * scratch and an initial arena (grown by llep_context_reserve).  Errors: INVALID (shape rules above;
 * D, H % 8 != 0; P > 32), NOMEM, CUDA. */
llep_status llep_context_create(const llep_shape *shape, int32_t rank, int32_t device,
                                int64_t max_tokens, llep_context **out);
void llep_context_destroy(llep_context *ctx);

/* Symmetric-arena bootstrap.  Every rank calls get_handle, the caller all-gathers the P
 * 64-byte handles (any transport; the library needs only the bytes), and every rank calls
 * open_peers with the gathered [P][64] array.  P == 1 needs neither call.  open_peers reads the
 * geometry record at the start of every peer's arena and returns LLEP_ERR_INVALID when a peer's
 * differs from this rank's (asymmetric max_tokens / reserve / backward setting). */
llep_status llep_context_ipc_handle(llep_context *ctx, void *handle64);
llep_status llep_context_open_peers(llep_context *ctx, const void *handles, int32_t n);

/* Grow the arena so every rank can receive `rows` padded rows, `foreign` imported experts and (with
 * the backward pass enabled) `grad_slots` returned weight-gradient partials.  Collective: all ranks
 * must call it with the same arguments, then redo the handle exchange.  The numbers come from
 * llep_requirements (identical on every rank). */
llep_status llep_context_reserve(llep_context *ctx, int64_t rows, int32_t foreign, int32_t grad_slots);

/* Enable the backward pass (row f1): the arena gains the upstream-gradient rows and the slots that
 * receive spilled experts' weight-gradient partials, plus rank-local buffers.  Collective
 * like llep_context_reserve (re-exchange the IPC handles afterwards for P > 1). */
llep_status llep_context_enable_backward(llep_context *ctx);

/* Bytes the context currently holds on the device: arena, scratch, activations, backward buffers and
 * the lazily grown backward workspaces (every cudaMalloc the context made). */
int64_t llep_context_device_bytes(const llep_context *ctx);

/* Global token order of an expert's routed slots (a3, the index the plan's chunk ranges [start, end)
 * refer to; the paper leaves it open, "build chunks of B̄_p from 𝒜"):
 *   LLEP_ORDER_RANK_MAJOR     rank 0's slots of e in flat order t*K+k, then rank 1's, ... (reading R11,
 *                             SPEC S:247-255)
 *   LLEP_ORDER_CHUNK_ALIGNED  (default) for an expert with more than one chunk the sources' blocks follow
 *                             its chunk devices in plan order (first appearance), then the other ranks
 *                             ascending (reading R11'): a spill device's chunk holds its own rows wherever
 *                             the counts allow, so they cross no link.  Experts with <= 1 chunk: rank-major.
 * Outputs are identical under both (every row is computed alone; the K-sum is in slot order); the plan
 * is unchanged; receive rows, slot destinations and NVLink bytes differ.  Every rank must use the same
 * order.  Takes effect at the next llep_prepare / llep_moe_layer.  Errors: INVALID. */
enum { LLEP_ORDER_RANK_MAJOR = 0, LLEP_ORDER_CHUNK_ALIGNED = 1 };
llep_status llep_context_set_token_order(llep_context *ctx, int32_t order);

/* Per-GPU memory cap for the context's device allocations (0 = none).  A llep_context_reserve that
 * would take the context above `bytes` fails with LLEP_ERR_NOMEM and leaves the arena unchanged:
 * the "tight per-GPU memory cap" of the Qwen3-shaped benchmark (BASELINE.json), under which standard
 * EP's hot device cannot hold its receive rows while LLEP's capacity-bounded plan fits (§4). */
llep_status llep_context_set_memory_cap(llep_context *ctx, int64_t bytes);

/* Needs of one plan, identical on every rank (the plan is replicated and deterministic). */
typedef struct {
  int64_t rows_needed;     /* max_d padded receive rows of device d (groups 128-row aligned)  */
  int32_t foreign_needed;  /* max_d |S_d|                                                      */
  int32_t fits;            /* 1 iff both fit this context's current arena                      */
  int64_t my_rows;         /* g_a[rank]                                                         */
  int32_t my_groups;       /* expert groups this rank computes (native with rows + foreign)    */
  int32_t fallback_ep, force_count, n_transfers;
  int32_t grad_slots_needed; /* backward: max_d weight-gradient partials returned to device d   */
} llep_requirements;

/* ------------------------------------------------------------------ the hot path
 * llep_prepare -- steps 1-2 of the path for this rank (Alg. 4):
 *   a1  local load histogram of topk_ids (per-tile counts, stable per-expert local ranks)
 *   a2  exchange: push this rank's counts row to every peer, device barrier -> C [P, N]
 *   a4  planner kernel on C (λ test, LLA, LLAS, 𝒲) -> plan_out (device blob)
 *   a5  layout: per-device expert groups (native first, then foreign), 128-row aligned bases
 * then one device->host read of the requirements (needed to size the arena; the only host
 * synchronisation of the layer).  The context keeps the prepared ids (a device copy) and the
 * topk_ids pointer: the following llep_moe_forward / backward must pass the same buffer unchanged.
 *   topk_ids   [B, K] int32, device.  Ids outside [0, N) -> LLEP_ERR_ROUTING.
 *   force_ep   1 -> standard EP plan on the same kernels (Alg. 1); 0 -> LLEP.
 *   plan_out   device buffer, llep_plan_bytes(N, P).
 *   req        host, may be NULL.
 * All ranks must call llep_prepare and llep_moe_forward the same number of times (barriers). */
llep_status llep_prepare(llep_context *ctx, const int32_t *topk_ids, int64_t n_tokens,
                         const llep_params *params, int32_t force_ep, void *plan_out,
                         llep_requirements *req, void *stream);

/* llep_moe_forward -- steps 3-4 (Alg. 4) with the plan from llep_prepare:
 *   a6  dispatch: gather-on-send of x rows + gates straight from the unsorted inputs into the
 *       destination device's receive rows (NVLink peer stores; local rows stay in HBM)
 *   a7  weight migration: copy-engine push of W13_e, W2_e native(e) -> d for every 𝒲 entry
 *   a8  grouped GEMM1 + SwiGLU: A = silu(X W_gateᵀ) ⊙ (X W_upᵀ)   (tcgen05/TMEM/TMA)
 *   a9  grouped GEMM2 + gate:   Y = diag(g) · (A W_downᵀ)          (Ĥ = Ĝ ⊙ B̂W)
 *   a10 combine: out[t] = Σ_{k=0..K-1} Y[dst(t,k)] in slot order, fp32, one bf16 rounding
 *       (reverse All-to-All + reverse sort + sum over K), pulled over NVLink.
 *   x          [B, D] bf16, device      topk_ids [B, K] int32     topk_w [B, K] fp32
 *   w13        [M, 2H, D] bf16: rows 0..H-1 = W_gate,e, rows H..2H-1 = W_up,e (native experts)
 *   w2         [M, D, H] bf16 = W_down,e
 *   plan       device blob from llep_prepare of these topk_ids.  The context caches the host copy
 *              and the layout of the last plan by ADDRESS: a plan at another address is laid out
 *              and validated again (chunk totals == loads, else LLEP_ERR_PLAN); do not overwrite
 *              a prepared plan in place between llep_prepare and llep_moe_forward/backward
 *   out        [B, D] bf16, device
 * The plan, load matrix and stable local ranks belong to the ids of the last llep_prepare, so:
 *   - topk_ids must be the buffer passed to that llep_prepare (else LLEP_ERR_PLAN, immediately) and
 *     B must equal its n_tokens (else LLEP_ERR_INVALID);
 *   - if that buffer's contents changed since, the dispatch addresses every slot with the prepared
 *     ids (every planned row is still written exactly once), drops the slots whose id changed from
 *     the output and raises a sticky device flag reported as LLEP_ERR_PLAN by llep_context_check or
 *     the next llep_prepare.
 * Errors: INVALID, PLAN (plan larger than the arena; ids buffer not the prepared one), CUDA, COMM. */
llep_status llep_moe_forward(llep_context *ctx, const uint16_t *x, const int32_t *topk_ids,
                             const float *topk_w, int64_t n_tokens, const uint16_t *w13,
                             const uint16_t *w2, const void *plan, uint16_t *out, void *stream);

/* llep_moe_forward_train -- llep_moe_forward for a training step (row f1): identical outputs,
 * and GEMM1's epilogue also stores this rank's raw gate / up pre-activations
 *   gu_save [gu_rows, 2H] bf16, device, caller-owned: row r of this rank's receive layout holds
 *           [X_r W_gateᵀ | X_r W_upᵀ] (bf16 of the fp32 tensor-core accumulator; padding rows of a
 *           group are left untouched).  gu_rows >= this rank's padded layout rows, which
 *           llep_requirements.rows_needed of the same llep_prepare always covers.
 * Pass the buffer and the same plan to llep_moe_backward_saved, which then skips recomputing
 * X·W13ᵀ.  Errors: as llep_moe_forward; INVALID if gu_save is NULL or gu_rows is too small. */
llep_status llep_moe_forward_train(llep_context *ctx, const uint16_t *x, const int32_t *topk_ids,
                                   const float *topk_w, int64_t n_tokens, const uint16_t *w13,
                                   const uint16_t *w2, const void *plan, uint16_t *out, uint16_t *gu_save,
                                   int64_t gu_rows, void *stream);

/* llep_moe_layer -- the whole layer of Alg. 4 in ONE stream-ordered call with NO host
 * synchronisation and no host reads of device data: llep_prepare's kernels (a1 histogram + local
 * ranks, a2 count push + barrier, a4 device planner into plan_out, a5 layout) followed by
 * llep_moe_forward's (a7, a6, a8, a9, a10).  The launch sequence depends only on (ctx, n_tokens), so
 * the call can be captured in a CUDA graph and replayed with new x / topk_ids / topk_w contents: the
 * plan is recomputed on the device every replay.  Differences from the two-call path:
 *   - the group count of the GEMMs stays on the device (layout kernel);
 *   - a7 is issued by the GPU (one small kernel per broadcast-tree level on a side stream, NVLink
 *     peer stores, release flags per foreign slot) instead of copy engines planned on the host;
 *   - the arena must already hold the plan (llep_context_reserve beforehand, with every rank's
 *     rows / foreign slots, e.g. from an earlier llep_prepare's llep_requirements or a bound).  A plan
 *     that does not fit is detected on the device identically on every rank: that call writes no
 *     receive rows and computes no tiles (its `out` is undefined) and the next llep_context_check
 *     returns LLEP_ERR_PLAN.  Other device errors are sticky in the same way.
 *   - no per-phase timing (llep_context_set_timing covers the two-call path only).
 * Arguments as llep_prepare + llep_moe_forward (plan_out: device buffer of llep_plan_bytes, written).
 * Every output equals the two-call path's bit for bit.  Synchronous errors: INVALID, COMM, CUDA. */
llep_status llep_moe_layer(llep_context *ctx, const uint16_t *x, const int32_t *topk_ids, const float *topk_w,
                           int64_t n_tokens, const uint16_t *w13, const uint16_t *w2, const llep_params *params,
                           int32_t force_ep, void *plan_out, uint16_t *out, void *stream);

/* llep_moe_backward -- the backward pass of the layer (row f1) under the plan of
 * llep_prepare for these topk_ids, recomputing the forward internals (nothing is kept from a
 * forward call), for the loss L with dL/dout = dout:
 *   dispatch x and dout rows + gates (a6) ‖ weight pushes (a7) -> barrier
 *   GU = X·W13ᵀ (gate/up pre-activations, tcgen05)       dA0 = dO·W_down   (MN-major tcgen05 GEMM)
 *   per row: a = silu(g)u, da = w·dA0, dg = da·u·silu'(g), du = da·silu(g), dL/dw = <a, dA0>
 *   dW_down = dOᵀ·(w·a), dW13 = [dg|du]ᵀ·X (per expert, contraction over its rows), dX = [dg|du]·W13
 *   replicas push the weight-gradient partials of spilled experts to the native device, which adds
 *   them in ascending source-device order -> barrier -> combine dX rows (Σ_K, slot order)
 *   dout     [B, D] bf16          dx [B, D] bf16         dgates [B, K] fp32 (dL/dtopk_w)
 *   dw13     [M, 2H, D] fp32 (dL/dW_gate rows 0..H-1, dL/dW_up rows H..2H-1)   dw2 [M, D, H] fp32
 * Requires llep_context_enable_backward and the arena of llep_requirements.fits.
 * Errors: INVALID, PLAN, CUDA, COMM. */
llep_status llep_moe_backward(llep_context *ctx, const uint16_t *x, const int32_t *topk_ids,
                              const float *topk_w, const uint16_t *dout, int64_t n_tokens,
                              const uint16_t *w13, const uint16_t *w2, const void *plan, uint16_t *dx,
                              float *dgates, float *dw13, float *dw2, void *stream);

/* llep_moe_backward_saved -- llep_moe_backward with the pre-activations saved by
 * llep_moe_forward_train under the SAME plan (gu_saved [gu_rows, 2H] bf16, device, read only): the
 * GU = X·W13ᵀ recompute is skipped; every output is bit-identical to llep_moe_backward's (the saved
 * values come from the same kernel with the same K order).  Errors: as llep_moe_backward; INVALID if
 * gu_saved is NULL or gu_rows is smaller than this rank's padded layout rows. */
llep_status llep_moe_backward_saved(llep_context *ctx, const uint16_t *x, const int32_t *topk_ids,
                                    const float *topk_w, const uint16_t *dout, int64_t n_tokens,
                                    const uint16_t *w13, const uint16_t *w2, const void *plan,
                                    const uint16_t *gu_saved, int64_t gu_rows, uint16_t *dx, float *dgates,
                                    float *dw13, float *dw2, void *stream);

/* ------------------------------------------------------------------ measurement
 * Per-phase device time, from CUDA events recorded on the caller's stream at the phase
 * boundaries of llep_prepare / llep_moe_forward, accumulated over calls while timing is on:
 *   ROUTE    a1 + a3 (histogram, scan, stable local ranks)
 *   EXCHANGE a2 (count push + device barrier + local copy of C)
 *   PLAN     a4 + a5 (planner kernel + layout kernel)
 *   DISPATCH a6 + a7 (dispatch kernel, weight pushes joined, device barrier)
 *   GEMM1    a8 (grouped GEMM + SwiGLU)      GEMM2  a9 (grouped GEMM + gate)
 *   COMBINE  a10 (device barrier + combine kernel)
 * kernel_launches counts every kernel the library launched (timing on or off). */
enum {
  LLEP_PH_ROUTE = 0,
  LLEP_PH_EXCHANGE = 1,
  LLEP_PH_PLAN = 2,
  LLEP_PH_DISPATCH = 3,
  LLEP_PH_GEMM1 = 4,
  LLEP_PH_GEMM2 = 5,
  LLEP_PH_COMBINE = 6,
  LLEP_NUM_PHASES = 7
};
typedef struct {
  double ms[LLEP_NUM_PHASES];
  int64_t calls;            /* completed prepare+forward pairs timed */
  int64_t kernel_launches;  /* kernels launched since the last reset */
  int64_t gemm_rows;        /* Σ over timed calls of real rows this rank's GEMMs processed */
} llep_stats;
llep_status llep_context_set_timing(llep_context *ctx, int32_t enable);

/* Synchronise `stream` and return (then clear) the sticky device-side error of the context's calls so
 * far: LLEP_ERR_ROUTING (an id outside [0, N)), LLEP_ERR_COMM (a device barrier or weight-flag wait timed
 * out, ~20 s), LLEP_ERR_PLAN (topk_ids changed between llep_prepare and llep_moe_forward/backward; those
 * slots were dropped).  LLEP_OK if none.  The hot path itself never synchronises for these. */
llep_status llep_context_check(llep_context *ctx, void *stream);
/* Synchronises the pending events, writes the totals, resets them if `reset`. */
llep_status llep_context_stats(llep_context *ctx, llep_stats *out, int32_t reset);

/* ------------------------------------------------------------------ inspection (tests)
 * Copy the last prepare/forward intermediates to caller DEVICE buffers (sizes in elements):
 *   LLEP_DBG_LOAD_MATRIX  int32 [P*N]        LLEP_DBG_SLOT_DST  int32 [2*B*K] (device,row)
 *   LLEP_DBG_GROUPS       int32 [G*8]        (expert, weight slot (-1-f = foreign f), row_base,
 *                                             n_rows, mblk_start, 0, 0, 0), G = my_groups
 *   LLEP_DBG_RECV_X       bf16 [rows*D]      LLEP_DBG_ACT bf16 [rows*H]   LLEP_DBG_Y bf16 [rows*D]
 *                         (RECV_X: every received row; under the opt-in LLEP_GATHER=1 the rows this
 *                         rank sends to itself in all-local m-blocks are read from x instead and
 *                         are not in RECV_X)
 *   LLEP_DBG_LOCAL_RANK   int32 [B*K]  (r_j: rank of slot j among this rank's slots of ids[j]) */
enum {
  LLEP_DBG_LOAD_MATRIX = 1,
  LLEP_DBG_SLOT_DST = 2,
  LLEP_DBG_GROUPS = 3,
  LLEP_DBG_RECV_X = 4,
  LLEP_DBG_ACT = 5,
  LLEP_DBG_Y = 6,
  LLEP_DBG_LOCAL_RANK = 7,
  LLEP_DBG_RECV_G = 8
};
llep_status llep_debug_copy(llep_context *ctx, int32_t what, void *dst, int64_t n_elems,
                            void *stream);

/* Standalone grouped-GEMM entry (kernel tests / micro-bench, the paper's F-gemm shape P:1127):
 * rows of group g occupy [row_base[g], row_base[g]+n_rows[g]) of a, with row_base % 128 == 0
 * (% 256 when mode bit 1 is set: 2-CTA cta_group::2 M=256 tiles; mode & 1 selects the epilogue).
 *   mode 0: out[r, 0:Hn] = silu(a W[e][0:Hn]ᵀ) ⊙ (a W[e][Hn:2Hn]ᵀ),  W [E, 2Hn, Kd], out [R, Hn]
 *   mode 1: out[r, 0:Nn] = gate[r] · (a W[e]ᵀ),                      W [E, Nn, Kd],  out [R, Nn]
 * groups: HOST int32 [G*4] = (expert, row_base, n_rows, 0), increasing non-overlapping rows.
 * Errors: INVALID (mode, ranges, alignment), CUDA. */
llep_status llep_grouped_gemm(int32_t mode, const uint16_t *a, int64_t rows, int32_t kdim,
                              const uint16_t *w, int32_t n_weights, int32_t nout,
                              const int32_t *groups, int32_t n_groups, const float *gate,
                              uint16_t *out, void *stream);

/* Standalone backward-pass GEMMs (row f1; kernel tests / micro-bench), MN-major tcgen05 operands:
 *   kind 0: out[r, 0:nout] = a[r, 0:kdim] · w[e][kdim, nout] for r in group rows (bf16 out [rows, nout]);
 *           a [rows, kdim] bf16, w [E, kdim, nout] bf16 row-major (e.g. W_down [D][H], W13 [2H][D])
 *   kind 1: out[e][mdim, nout] = Σ_{r in group} a[r, 0:mdim] ⊗ b[r, 0:nout]  (fp32 out [E, mdim, nout]);
 *           a [rows, mdim], b [rows, nout] bf16; rows past a group's end up to the next multiple of
 *           256 must be zero in a and b (the contraction runs over whole 256-row blocks)
 * groups: HOST int32 [G*4] = (expert / output slot, row_base, n_rows, 0), row_base % 256 == 0. */
llep_status llep_gemm_bwd(int32_t kind, const uint16_t *a, const uint16_t *w_or_b, int64_t rows,
                          int32_t kdim_or_mdim, int32_t nout, int32_t n_weights, const int32_t *groups,
                          int32_t n_groups, void *out, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Router (row f4): Eq. 2 of PAPER.md for one rank's tokens, producing the top-K ids and
 * gates that llep_prepare / llep_moe_forward consume.
 *   z[t, i]  = Σ_d x[t, d] · w_router[i, d]        (w_router [N, D] = W_rᵀ, one row per expert)
 *   s[t, :]  = softmax(z[t, :]) over all N experts (fp32, max-subtracted; Σ accumulated online in
 *              expert order, rescaled to the running max once per 64 experts)
 *   topk_ids[t, k]  = the k-th largest s[t, :], descending, ties -> lower expert id (DESIGN R31/R32)
 *   topk_w[t, k]    = s[t, topk_ids[t, k]]          (no renormalisation over the K: Eq. 2 writes none)
 * x: DEVICE bf16 [n_tokens, d_model] row-major; w_router: DEVICE bf16 [n_experts, d_model];
 * topk_ids: DEVICE int32 [n_tokens, top_k]; topk_w: DEVICE fp32 [n_tokens, top_k];
 * logits: DEVICE fp32 [n_tokens, n_experts] or NULL (a copy of z, for tests).  Caller-owned; the
 * library keeps no pointer.  z accumulates in fp32 on the tensor cores (bf16 products are exact).
 * Limits: 1 <= n_experts <= 512, 1 <= top_k <= min(16, n_experts), d_model % 8 == 0, 16-byte
 * aligned x / w_router.  n_tokens == 0 is a no-op.  Stream-ordered on `stream`.
 * Errors: INVALID (limits, null pointers, alignment), CUDA. */
llep_status llep_router(const uint16_t *x, const uint16_t *w_router, int64_t n_tokens, int32_t d_model,
                        int32_t n_experts, int32_t top_k, int32_t *topk_ids, float *topk_w,
                        float *logits, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LLEP_H */
