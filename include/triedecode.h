/*
 * triedecode.h -- C ABI of libtriedecode.so, the B200 (sm_100a) hot path of trie-based
 * parallel beam decoding (arXiv 2502.00085, "PAPER.md").
 *
 * Citations: "P:<n>" = /root/reference/PAPER.md line n (section / algorithm named),
 * "S:<n>" = SPEC.md line n.  Readings of silent or ambiguous passages: DESIGN.md "Readings".
 *
 * CONVENTIONS (apply to every entry point)
 *  - Pointers are DEVICE pointers unless the name ends in `_host`.
 *  - Every call is asynchronous on the caller's cudaStream_t and performs no host
 *    synchronisation, except trie_create / trie_read_hyps / trie_status (documented).
 *  - Ownership: the caller owns every buffer (Q, K/V pools, outputs, the workspace and
 *    the attention scratch).  The library never calls cudaMalloc; the handle is a small
 *    host struct holding pointers into the caller's workspace.  trie_destroy frees only
 *    that host struct.
 *  - Errors: each call returns TRIE_OK (0) or a negative code; a human-readable detail
 *    is available from trie_last_error() (thread-local).  Faults that can only be
 *    detected on the device latch bits into a device status word (TRIE_ST_*), read with
 *    trie_status().
 *  - Threading: a handle is bound to one stream at a time and is not thread-safe;
 *    distinct handles are independent ("distinct sessions may run in
 *    parallel").
 *  - CUDA graphs: all trie STATE (metadata, N, leaves, scores, tickets, page counters,
 *    gather sequence numbers) lives on the device, so captured calls replay correctly at
 *    any later step.  Two host-side quantities fix a call's LAUNCH SHAPE only: b_live
 *    (1 until the first trie_beam_step / trie_append after trie_create / trie_reset, b
 *    from then on) and, for trie_attn_decode_rope, whether the call recomputes the
 *    (cos, sin) table of the leaves' depths (the first fused call after each beam step /
 *    append does; the step counter `steps` is host-tracked for that).  Hence: capture
 *    steady-state steps (b_live = b) as "beam step + the step's attention calls", and the
 *    first step of a job (b_live = 1) as its own graph starting at trie_reset (bench.py's
 *    "first" / "steady" graphs); do not replay a graph captured at b_live = 1 later in a
 *    job, nor a graph holding only non-first fused attention calls of a step after a
 *    beam step that was not replayed with it.
 *
 * DATA LAYOUT
 *  - KV pool, per layer: [R][Hkv][capacity][D], kv_dtype elements, head-major so that a
 *    tile of consecutive slots of one (request, KV head) is one contiguous region (one
 *    TMA box).  Slot n of request r holds trie node n (the prompt occupies slots 0..t-1).
 *    Rows at slots >= N must hold FINITE values (zero-initialise pools once).
 *  - Q / attention output: [R][b_live][Hq][D] (the QKV GEMM's row layout).
 *  - New K/V rows for rope_kv_append: [R][b_live][Hkv][D].
 *  - Trie metadata (inside the workspace, trie_get_arrays): token/parent/depth int32
 *    [R][capacity], beam_mask uint32 [R][capacity] (bit r of word n <=> node n is on
 *    the root-to-leaf path of beam r, generated nodes only), leaf int32 [R][32],
 *    score float [R][32], n_nodes int32 [R], prompt_len int32 [R].
 *    Invariants kept by the library: parent[n] < n; depth[] non-decreasing in slot
 *    order; the b_live leaves are the last b_live slots after every append.
 */
#ifndef TRIEDECODE_H
#define TRIEDECODE_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define TRIE_OK 0
#define TRIE_EINVAL (-1)    /* bad shape or argument */
#define TRIE_ESTATE (-2)    /* call-order violation (e.g. prune before any append) */
#define TRIE_ECUDA (-3)     /* CUDA launch / runtime failure (detail in trie_last_error) */
#define TRIE_ECAPACITY (-4) /* workspace or scratch too small */

/* device status bits (latched; trie_status) */
#define TRIE_ST_CAPACITY 0x1u    /* an append would exceed `capacity` slots */
#define TRIE_ST_PARENT 0x2u      /* broken parent chain: parent[n] >= n or out of range */
#define TRIE_ST_EMPTY_ROW 0x4u   /* attention row with no allowed key */
#define TRIE_ST_LEAF 0x8u        /* leaf id outside [0, N) */

/* kv_dtype */
#define TRIE_F32 0
#define TRIE_BF16 1

typedef struct trie_cfg {
  int32_t n_requests;     /* R: independent requests on this GPU (the data-parallel unit, §8(e)) */
  int32_t beam_width;     /* b: 1..32 (b <= vocab)                                         */
  int32_t max_prompt_len; /* t_max: row stride of the prompt token matrix                  */
  int32_t capacity;       /* slots per request (>= t_max + b * steps without GC)           */
  int32_t n_layers;       /* L                                                             */
  int32_t n_q_heads;      /* Hq (local to this GPU)                                        */
  int32_t n_kv_heads;     /* Hkv (local); Hq % Hkv == 0 (GQA)                       */
  int32_t head_dim;       /* D: multiple of 16, <= 256                                     */
  int32_t vocab;          /* V                                                             */
  int32_t window;         /* W: sliding window in keys incl. self along the branch; 0 = dense */
  int32_t gc_interval;    /* g: informational (the caller schedules trie_prune_compact)    */
  int32_t kv_dtype;       /* TRIE_F32 or TRIE_BF16 (also the dtype of Q, new K/V, output)  */
  int32_t n_pages;        /* 0: dense pools; > 0: paged pools of n_pages 64-slot pages (below) */
} trie_cfg;

/*
 * KV pool layouts (per layer; K and V alike).
 *   dense  (n_pages == 0): [R][Hkv][capacity][D] -- slot n of request r, KV head h at row
 *          (r * Hkv + h) * capacity + n.
 *   paged  (n_pages  > 0; physical memory follows the live trie):
 *          [n_pages][Hkv][64][D] -- slot n of request r at row (page * Hkv + h) * 64 + n % 64
 *          with page = page_table[r][n / 64] (trie_arrays.page_table, [R][capacity / 64]
 *          int32; capacity % 64 == 0).  Request r's prompt occupies the fixed pages
 *          off_r .. off_r + ceil(t_r / 64) - 1, off_r = sum_{q < r} ceil(t_q / 64) (the
 *          caller's prefill writes them); every other page sits in a device free queue.
 *          trie_beam_step / trie_append take pages from it when N grows into a new 64-slot
 *          block (TRIE_ST_CAPACITY latches when it is empty); trie_prune_compact returns
 *          the pages above the compacted N (§3.5: pruned rows free their memory).
 *          trie_arrays.page_ctr [4] uint32: pops, pushes, peak pages in use (since trie_create),
 *          n_pages; pages
 *          in use = n_pages - (pushes + free_at_create - pops) (see trie_page_stats).
 *          Paged pools are supported by the handle's calls (trie_rope_kv_append,
 *          trie_attn_decode_rope, trie_prune_compact); the handle-less trie_attn_decode
 *          addresses dense pools only.
 */

typedef struct trie_handle trie_handle;

/* device pointers into the workspace, for passing to the pure entry points */
typedef struct trie_arrays {
  int32_t* token;
  int32_t* parent;
  int32_t* depth;
  uint32_t* beam_mask;
  int32_t* leaf;
  float* score;
  int32_t* n_nodes;
  int32_t* prompt_len;
  uint32_t* status;
  int32_t b_live; /* live beams: 1 before the first append, then b (host-tracked) */
  int32_t steps;  /* appends done since create/reset (host-tracked) */
  uint32_t* finished; /* [R][32]: beam j's last generated token is the EOS id (trie_set_eos) */
  int32_t* page_table; /* paged pools: [R][capacity / 64] page of each 64-slot block (else NULL) */
  uint32_t* page_ctr;  /* paged pools: [4] = pops, pushes, peak pages in use, n_pages */
} trie_arrays;

/*
 * SURVEY §8(f) NEXT-3, sliding-window eviction (paged pools, cfg.window > 0; the paper
 * evaluates SWA models, and keeps their whole cache): return to the free queue
 * the page of every 64-slot block of each request that holds only prompt rows below
 * min_j (depth[leaf_j] - W + 1) -- rows outside every live beam's window (reading R14) for
 * the rest of the job, since leaf depths only grow.  Attention never reads them again and
 * GC never moves prompt rows.  Contract: after trie_reset the prompt maps to its original
 * pages again and the caller must re-write (prefill) their K/V before the first attention.
 * Async on stream; EINVAL for dense pools or window == 0.
 */
int trie_swa_evict(trie_handle* h, cudaStream_t stream);

/* Paged pools: host copy of {pages in use, peak pages in use, n_pages} (synchronises). */
int trie_page_stats(trie_handle* h, int32_t* stats_host, cudaStream_t stream);

/* Workspace bytes for a configuration (metadata + scratch of beam_step / prune). */
int trie_workspace_bytes(const trie_cfg* cfg, size_t* bytes);

/*
 * Alg. 2 l.1 initialize_trie(prompt): for every request r the prompt
 * becomes a chain: token[i] = prompt[r][i], parent[i] = i-1 (-1 for i = 0), depth[i] = i
 * (§3.4 positions), leaf = [t_r - 1], score = [0], N = t_r.
 * prompt_lens_host [R] (host): 1 <= t_r <= t_max (EINVAL otherwise: empty prompt).
 * prompt_tokens [R][t_max] int32 (device), copied into the workspace (trie_reset reuses it).
 * Synchronises the stream once (validation of sizes).  Prompt K/V are the caller's
 * (prefill is model context, not part of this library).
 */
int trie_create(const trie_cfg* cfg, void* workspace, size_t workspace_bytes,
                const int32_t* prompt_lens_host, const int32_t* prompt_tokens,
                trie_handle** out, cudaStream_t stream);

/* Re-initialise the metadata from the stored prompts (same as trie_create, async; the
 * latched status word is cleared too). */
int trie_reset(trie_handle* h, cudaStream_t stream);

int trie_destroy(trie_handle* h);

int trie_get_arrays(const trie_handle* h, trie_arrays* out);

/*
 * a-1: position-integrity RoPE + write-before-read KV append (§3.4; Alg. 3 l.7
 * "allow attention to current node" P:175).  For request r, live beam j:
 * pos = depth[leaf[r][j]]; q[r][j] (all Hq heads) and k_new[r][j] are rotated in place
 * (rotate-half pairs (i, i+D/2), theta_i = rope_theta^(-2i/D), angle evaluated in fp64)
 * and k, v are stored at slot leaf[r][j] of the layer's pools.
 * q: [R][b_live][Hq][D] in/out; k_new, v_new: [R][b_live][Hkv][D] (k_new is rotated in
 * place as well); k_pool, v_pool: the layer's [R][Hkv][capacity][D] pools.
 */
int trie_rope_kv_append(trie_handle* h, void* q, void* k_new, const void* v_new,
                        void* k_pool, void* v_pool, float rope_theta, cudaStream_t stream);

/*
 * a-3: trie attention decode (§3.3 P:188-196 tree attention; Alg. 3 mask P:165-186).
 * Pure function of its arguments.  For request r, live beam j, query head hq
 * (KV head hq / (Hq/Hkv)):
 *   o = sum_{n in A_rj} softmax_n(q . k_n / sqrt(D)) v_n,
 *   A_rj = { n < N_r : (n < t_r or bit j of beam_mask[r][n]) and
 *            (window == 0 or depth[r][n] >= depth[r][leaf_rj] - window + 1) }.
 * Masked keys are excluded exactly (weight 0, reading R22).  Every unique KV row is
 * read from HBM once per (request, KV head) and serves all b_live * (Hq/Hkv) queries.
 * beam_mask == NULL: the mask is derived from parent[] by per-leaf walks (Alg. 3) into
 * the scratch; otherwise parent may be NULL.
 * q, out: [R][b_live][Hq][D]; lse (optional, may be NULL): [R][b_live][Hq] float,
 * natural-log sum of exp of the scaled scores.  rows_hint: expected max N over requests
 * (sizes the split-K grid; 0 = capacity).  scratch: >= trie_attn_scratch_bytes().
 * status (optional device word, may be NULL): TRIE_ST_EMPTY_ROW is OR-ed in when a query
 * row has no allowed key (its output row is then 0 and its lse -inf).
 */
size_t trie_attn_scratch_bytes(const trie_cfg* cfg, int32_t b_live, int32_t rows_hint);
int trie_attn_decode(const trie_cfg* cfg, int32_t b_live, const void* q, const void* k_pool,
                     const void* v_pool, const int32_t* prompt_len, const int32_t* parent,
                     const int32_t* depth, const int32_t* leaf_ids, const int32_t* n_nodes,
                     const uint32_t* beam_mask, int32_t window, int32_t rows_hint, void* out,
                     float* lse, void* scratch, size_t scratch_bytes, uint32_t* status,
                     cudaStream_t stream);

/*
 * Which attention kernel a configuration uses (host only): info_host[0] = path (0 CUDA-core
 * fp32/other, 1 narrow mma.sync, 2 wide mma.sync, 3 tcgen05/TMEM),
 * [1] = split-K count, [2] = 1 if trie_attn_decode_rope fuses into one launch, [3] = Qg.
 */
int trie_attn_plan_info(const trie_cfg* cfg, int32_t b_live, int32_t rows_hint,
                        int32_t* info_host);

/*
 * a-1 + a-3 fused (one launch when a tensor-core kernel applies: bf16, D in {64, 96, 128},
 * Qg = b_live * Hq/Hkv <= 32 (narrow for Qg <= 8, wide above) or the tcgen05 kernel for
 * Qg >= 33; trie_attn_plan_info [2]): the same result as trie_rope_kv_append followed
 * by trie_attn_decode over the handle's trie (window = cfg.window), except that q and
 * k_new are read un-rotated and not written back.  Each attention CTA rotates its own
 * query heads at the beams' depths and, if its tiles contain leaf slots, rotates and
 * appends those leaves' K/V rows (write-before-read, §3.4 / Alg. 3 l.7) before loading
 * the tile.  Other shapes run the two steps as two launches (q, k_new then hold their
 * rotated values).  Arguments as in the two calls; scratch >= trie_attn_scratch_bytes.
 * Ordering contract: the prompt rows [0, t_r - 1) of the pools (the caller's prefill) must
 * be written before trie_create / trie_reset and not rewritten while the handle decodes --
 * the fused kernel may load the tiles below the shortest prompt before its programmatic
 * dependency wait (prompt nodes never move or change, §3.5 invariant 3; row t_r - 1, the
 * prompt leaf, is appended by the first call after create / reset).
 */
int trie_attn_decode_rope(trie_handle* h, const void* q, const void* k_new, const void* v_new,
                          void* k_pool, void* v_pool, float rope_theta, int32_t rows_hint,
                          void* out, float* lse, void* scratch, size_t scratch_bytes,
                          cudaStream_t stream);

/*
 * a-4 + a-5 (+ a-2 update): one beam step (Alg. 2 l.9-11; Alg. 1 l.6 P:116).
 * logits [R][b_live][V] fp32 (b_live = 1 on the first call).  Per request:
 *   lp_j[v] = x_j[v] - lse_j,  lse_j = max + log sum exp(x_j - max);
 *   the b best candidates (score_j + lp_j[v], v, j) in the total order score desc,
 *   token asc, beam asc (readings R1, R3) are selected, in rank order;
 *   rank r is appended at slot N + r with token v, parent leaf[j], depth[parent] + 1
 *   (§3.4), leaves := the new slots, scores := the new scores, N += b;
 *   beam_mask: new[n] bit r = old[n] bit j_r for every generated node (update_mask,
 *   P:197-198), new leaf r gets bit r.
 * Outputs (optional, may be NULL): sel_parent_beam, sel_token int32 [R][b], new_score
 * float [R][b].
 */
int trie_beam_step(trie_handle* h, const float* logits, int32_t* sel_parent_beam,
                   int32_t* sel_token, float* new_score, cudaStream_t stream);

/*
 * SURVEY §8(f) NEXT-3, EOS (reading R5b; the paper is silent): EOS is an ABSORBING
 * token.  A beam whose last generated token is eos_id is finished: in every later
 * trie_beam_step its next-token distribution is one-hot at eos_id (log-prob 0: one
 * candidate, score unchanged, no logits read), so finished hypotheses keep competing for
 * the b beams by cumulative score.  A request is done when all b beams are finished: from
 * then on trie_beam_step returns the identity selection (parent j = rank j, token eos_id,
 * score unchanged) and appends nothing, so its trie and hypotheses stay fixed; the fused
 * trie_attn_decode_rope then skips the request entirely -- no K/V
 * append, its output rows are NOT written (their logits are never read again).
 * eos_id = -1 (default) disables it.
 * Host-side setting; EINVAL for eos_id outside [-1, V).  trie_append marks finished beams
 * the same way; trie_create / trie_reset clear the flags.
 */
int trie_set_eos(trie_handle* h, int32_t eos_id);

/* a-5 alone (teacher forcing): append the given selections [R][b] exactly as above. */
int trie_append(trie_handle* h, const int32_t* sel_parent_beam, const int32_t* sel_token,
                const float* new_score, cudaStream_t stream);

/*
 * a-6: garbage collection (§3.5 Marking / Pruning / Compaction; Alg. 2 l.5-7).
 * keep[n] = n < t or beam_mask[n] != 0 (= n is an ancestor-or-self of a live leaf);
 * new[n] = exclusive prefix sum of keep (stable, the paper's index_select order);
 * token/depth/beam_mask move to new[n], parent' = new[parent], leaf' = new[leaf],
 * N' = sum keep; in every layer the K/V rows of moved nodes are copied n -> new[n].
 * k_pools_host / v_pools_host: host arrays of L device pointers (each layer's pool).
 * The caller decides the schedule (every g steps; the hot path uses g = 1).
 */
int trie_prune_compact(trie_handle* h, void* const* k_pools_host, void* const* v_pools_host,
                       cudaStream_t stream);

/*
 * Alg. 2 l.14 / Alg. 1 l.8: read every live hypothesis (rank order; rank 0
 * is the best).  tokens_host [R][b][max_len] (root-to-leaf tokens, prompt included,
 * padded with -1), len_host [R][b], score_host [R][b].  Synchronises the stream.
 */
int trie_read_hyps(trie_handle* h, int32_t max_len, int32_t* tokens_host, int32_t* len_host,
                   float* score_host, void* scratch, size_t scratch_bytes, cudaStream_t stream);

/*
 * Measurement baseline, not part of the trie path: the cache reorder
 * of conventional batch beam search (Alg. 1; HF _reorder_cache, the paper's
 * comparison system).  Every beam owns a private cache; after top-b, beam r of request i
 * continues parent beam j = sel_parent_beam[i*b + r] (Alg. 1 l.6-7), so for every layer l
 * and KV head h:
 *   dst_l[i*b + r][h][n] = src_l[i*b + j][h][n]   for prompt_len[i*b + r] <= n < n_rows[i*b + j].
 * The prompt rows (identical in every beam's cache) are not copied.  Pools per layer:
 * [R*b][Hkv][capacity][head_dim] elements of elem_bytes (2 = bf16, 4 = fp32); the *_host
 * arguments are host arrays of n_layers device pointers; src and dst must be distinct.
 * prompt_len, n_rows: [R*b] int32 (device); sel_parent_beam: [R][b] int32 (device); status:
 * optional device word, TRIE_ST_PARENT latched for a parent index outside [0, b).
 * Async on stream; EINVAL for bad shapes or null / in-place pools.
 */
int trie_batch_reorder_kv(int32_t n_requests, int32_t beam_width, int32_t n_layers,
                          int32_t n_kv_heads, int32_t head_dim, int32_t capacity,
                          int32_t elem_bytes, const int32_t* sel_parent_beam,
                          const int32_t* prompt_len, const int32_t* n_rows,
                          void* const* src_k_host, void* const* src_v_host,
                          void* const* dst_k_host, void* const* dst_v_host, uint32_t* status,
                          cudaStream_t stream);

/*
 * the KV-head shard's per-layer all-gather of attention
 * outputs FUSED into trie_attn_decode_rope (BASELINE.json configs[3]; the paper's
 * multi-GPU run, states no mechanism).  World W <= 8 ranks hold the same requests
 * and trie (identical logits -> identical selections) but each only its KV heads
 * [rank*Hkv, (rank+1)*Hkv) and their Hq query heads (cfg.n_q_heads / n_kv_heads are the
 * LOCAL counts).  Every rank owns a gather buffer of 2 halves, each [R][b_live][W*Hq][D]
 * (dtype of the pools), and a flag array uint32 [W]; both are exchanged between the
 * processes (trie_ipc_alloc / trie_ipc_open: CUDA IPC -- peer-mapped over NVLink on an
 * 8-GPU box, the same device on a one-GPU test box).
 *
 * trie_gather_setup registers, for every rank p, this process's pointer to p's gather
 * buffer and to p's flag array (peer_out_host[rank] / peer_flags_host[rank] = the local
 * ones).  From then on every trie_attn_decode_rope call on the handle, in the epilogue of
 * the kernel that produces the output rows (the attention kernel, or the split-K combine),
 * also stores every output row of its heads into EVERY rank's gather buffer (head block
 * `rank`, half = the call's sequence number mod 2; the local `out` is written as before)
 * with plain peer stores as each CTA finishes, then -- after the last output row of the
 * launch -- publishes the launch's sequence number e (1, 2, ...) to flags[rank] of every
 * rank (release, system scope).  Every rank must make the same sequence of calls.
 * trie_gather_wait enqueues a wait until every rank's flag in the LOCAL flag array reaches
 * this rank's own e (acquire, system scope) and then copies half (e - 1) mod 2 of the local
 * gather buffer -- every rank's heads of call e, [R][b_live][W*Hq][D] -- into gathered_out
 * (device; NULL: wait only).  Two halves (each R*beam_width*W*Hq*D elements): a rank can
 * run one call ahead of a slower peer still reading the previous call's half; it cannot
 * run two ahead, since its next wait needs that peer's next call.  Both the sequence
 * number and the half are device-side, so the calls are CUDA-graph replayable.
 * Supported on the fused bf16 tensor-core paths (trie_attn_plan_info [2] = 1); EINVAL
 * otherwise.  world = 1 (or setup never called) disables the gather.
 */
int trie_gather_setup(trie_handle* h, int32_t world, int32_t rank, void* const* peer_out_host,
                      uint32_t* const* peer_flags_host);
int trie_gather_wait(trie_handle* h, void* gathered_out, cudaStream_t stream);

/*
 * CUDA IPC helpers for the gather buffers: trie_ipc_alloc = cudaMalloc (zeroed) + its
 * 64-byte cudaIpcMemHandle_t in handle_out; trie_ipc_open maps a peer's handle into this
 * process (cudaIpcMemLazyEnablePeerAccess); trie_ipc_close / trie_ipc_free undo them.
 */
int trie_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
int trie_ipc_open(const void* handle, void** dev_ptr);
int trie_ipc_close(void* dev_ptr);
int trie_ipc_free(void* dev_ptr);

/* Read (and keep) the latched device status bits.  Synchronises the stream. */
int trie_status(trie_handle* h, uint32_t* bits_host, cudaStream_t stream);

const char* trie_last_error(void);

/* library version (major << 16 | minor) */
int trie_version(void);

/* Number of kernels this process has launched through the library (all entry points;
 * used by bench.py to report the launches inside its timed region). */
unsigned long long trie_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TRIEDECODE_H */
