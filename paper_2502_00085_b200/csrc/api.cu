// C ABI glue of libtriedecode: argument validation, workspace carving, dispatch.
// Every step of the hot path runs in the kernels of this library; there is no CPU path.
#include <stdlib.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <new>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

int trie_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int trie_check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);  // one call per kernel launch site
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return trie_set_error(TRIE_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return TRIE_OK;
}

static int validate(const trie_cfg* c) {
  if (!c) return trie_set_error(TRIE_EINVAL, "null cfg");
  if (c->n_requests < 1) return trie_set_error(TRIE_EINVAL, "n_requests < 1");
  if (c->beam_width < 1 || c->beam_width > TRIE_MAX_BEAMS)
    return trie_set_error(TRIE_EINVAL, "beam_width %d not in [1, 32]", c->beam_width);
  if (c->vocab < c->beam_width) return trie_set_error(TRIE_EINVAL, "beam_width > vocab");
  if (c->max_prompt_len < 1) return trie_set_error(TRIE_EINVAL, "max_prompt_len < 1");
  if (c->capacity < c->max_prompt_len + c->beam_width)
    return trie_set_error(TRIE_EINVAL, "capacity < max_prompt_len + beam_width");
  if (c->n_layers < 0 || c->n_layers > TRIE_MAX_LAYERS)
    return trie_set_error(TRIE_EINVAL, "n_layers not in [0, %d]", TRIE_MAX_LAYERS);
  if (c->n_q_heads < 1 || c->n_kv_heads < 1 || c->n_q_heads % c->n_kv_heads)
    return trie_set_error(TRIE_EINVAL, "n_q_heads %% n_kv_heads != 0 (GQA, S:104)");
  if (c->beam_width * (c->n_q_heads / c->n_kv_heads) > 128)
    return trie_set_error(TRIE_EINVAL, "beam_width * (n_q_heads / n_kv_heads) = %d > 128 queries per KV head",
                          c->beam_width * (c->n_q_heads / c->n_kv_heads));
  if (c->head_dim < 16 || c->head_dim > 256 || c->head_dim % 16)
    return trie_set_error(TRIE_EINVAL, "head_dim must be a multiple of 16 in [16, 256]");
  if (c->window < 0) return trie_set_error(TRIE_EINVAL, "window < 0");
  if (c->kv_dtype != TRIE_F32 && c->kv_dtype != TRIE_BF16)
    return trie_set_error(TRIE_EINVAL, "kv_dtype");
  if (c->n_pages < 0) return trie_set_error(TRIE_EINVAL, "n_pages < 0");
  if (c->n_pages > 0 && c->capacity % 64)
    return trie_set_error(TRIE_EINVAL, "paged pools need capacity %% 64 == 0");
  return TRIE_OK;
}

bool trie::pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// pre-wait prefetch of prompt tiles in the fused attention (TRIE_PREFETCH=0 disables)
static bool prefetch_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_PREFETCH");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t trie_layout(const trie_cfg* c, trie_handle* h, char* base) {
  const size_t R = c->n_requests, cap = c->capacity, b = c->beam_width;
  const size_t chunks = (c->vocab + TRIE_BEAM_CHUNK - 1) / TRIE_BEAM_CHUNK;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  char* token = take(R * cap * 4);
  char* parent = take(R * cap * 4);
  char* depth = take(R * cap * 4);
  char* mask = take(R * cap * 4);
  char* leaf = take(R * TRIE_MAX_BEAMS * 4);
  char* score = take(R * TRIE_MAX_BEAMS * 4);
  char* nn = take(R * 4);
  char* nkv = take(R * 4);
  char* tlen = take(R * 4);
  char* status = take(4);
  char* prompts = take(R * c->max_prompt_len * 4);
  char* newidx = take(R * cap * 4);
  char* moves = take(R * cap * 4);
  char* mdst = take(R * cap * 4);
  char* nmoves = take(R * 4);
  char* cmax = take(R * b * chunks * 4);
  char* csum = take(R * b * chunks * 4);
  char* ctop = take(R * b * chunks * b * 8);
  char* rlse = take(R * TRIE_MAX_BEAMS * 4);
  char* rtop = take(R * TRIE_MAX_BEAMS * TRIE_MAX_BEAMS * 8);
  char* tickets = take(R * (TRIE_MAX_BEAMS + 1) * 4);
  char* sp = take(R * b * 4);
  char* st = take(R * b * 4);
  char* ss = take(R * b * 4);
  char* rtab = take(R * TRIE_MAX_BEAMS * (c->head_dim / 2) * 8);
  char* fin = take(R * TRIE_MAX_BEAMS * 4);
  char* gat = take(64);  // gather ticket + completed-launch counter (NEXT-4)
  // paged pools (NEXT-2): page table, pages per request, prompt page base, free queue, counters
  const size_t np = c->n_pages > 0 ? (size_t)c->n_pages : 0;
  char* pt = take(np ? R * (cap / 64) * 4 : 0);
  char* pused = take(np ? R * 4 : 0);
  char* pbase = take(np ? R * 4 : 0);
  char* fq = take(np * 4);
  char* pctr = take(np ? 64 : 0);
  if (h) {
    h->token = (int32_t*)token;
    h->parent = (int32_t*)parent;
    h->depth = (int32_t*)depth;
    h->mask = (uint32_t*)mask;
    h->leaf = (int32_t*)leaf;
    h->score = (float*)score;
    h->n_nodes = (int32_t*)nn;
    h->n_kv = (int32_t*)nkv;
    h->tlen = (int32_t*)tlen;
    h->status = (uint32_t*)status;
    h->prompts = (int32_t*)prompts;
    h->newidx = (int32_t*)newidx;
    h->moves = (int32_t*)moves;
    h->moves_dst = (int32_t*)mdst;
    h->n_moves = (int32_t*)nmoves;
    h->chunk_max = (float*)cmax;
    h->chunk_sum = (float*)csum;
    h->chunk_top = (uint64_t*)ctop;
    h->row_lse = (float*)rlse;
    h->row_top = (uint64_t*)rtop;
    h->cnt_row = (uint32_t*)tickets;
    h->cnt_req = (uint32_t*)tickets + R * TRIE_MAX_BEAMS;
    h->sel_parent = (int32_t*)sp;
    h->sel_token = (int32_t*)st;
    h->sel_score = (float*)ss;
    h->rope_tab = (float2*)rtab;
    h->fin = (uint32_t*)fin;
    h->g_ticket = (uint32_t*)gat;
    h->g_epoch = (uint32_t*)gat + 1;
    h->page_table = np ? (int32_t*)pt : nullptr;
    h->pages_used = np ? (int32_t*)pused : nullptr;
    h->page_base = np ? (int32_t*)pbase : nullptr;
    h->free_q = np ? (int32_t*)fq : nullptr;
    h->page_ctr = np ? (uint32_t*)pctr : nullptr;
    h->chunks = (int32_t)chunks;
  }
  return off;
}

extern "C" {

int trie_version(void) { return (1 << 16) | 0; }

unsigned long long trie_launch_count(void) { return g_launches.load(); }

const char* trie_last_error(void) { return g_err; }

int trie_workspace_bytes(const trie_cfg* cfg, size_t* bytes) {
  int rc = validate(cfg);
  if (rc) return rc;
  if (!bytes) return trie_set_error(TRIE_EINVAL, "null bytes");
  *bytes = trie_layout(cfg, nullptr, nullptr);
  return TRIE_OK;
}

int trie_create(const trie_cfg* cfg, void* workspace, size_t workspace_bytes,
                const int32_t* prompt_lens_host, const int32_t* prompt_tokens,
                trie_handle** out, cudaStream_t stream) {
  int rc = validate(cfg);
  if (rc) return rc;
  if (!workspace || !prompt_lens_host || !prompt_tokens || !out)
    return trie_set_error(TRIE_EINVAL, "null argument");
  const size_t need = trie_layout(cfg, nullptr, nullptr);
  if (workspace_bytes < need)
    return trie_set_error(TRIE_ECAPACITY, "workspace %zu < %zu bytes", workspace_bytes, need);
  if ((uintptr_t)workspace % 256)
    return trie_set_error(TRIE_EINVAL, "workspace must be 256-byte aligned");
  for (int r = 0; r < cfg->n_requests; ++r) {
    const int t = prompt_lens_host[r];
    if (t < 1) return trie_set_error(TRIE_EINVAL, "empty prompt for request %d (S:260)", r);
    if (t > cfg->max_prompt_len)
      return trie_set_error(TRIE_EINVAL, "prompt %d longer than max_prompt_len", r);
  }
  trie_handle* h = new (std::nothrow) trie_handle();
  if (!h) return trie_set_error(TRIE_EINVAL, "out of host memory");
  h->cfg = *cfg;
  h->ws = (char*)workspace;
  h->ws_bytes = workspace_bytes;
  trie_layout(cfg, h, (char*)workspace);
  h->host_tlen.assign(prompt_lens_host, prompt_lens_host + cfg->n_requests);
  std::vector<int32_t> pbase(cfg->n_requests, 0);
  if (cfg->n_pages > 0) {  // fixed prompt pages: request r from off_r = sum_{q<r} ceil(t_q/64)
    int off = 0;
    for (int r = 0; r < cfg->n_requests; ++r) {
      pbase[r] = off;
      off += (prompt_lens_host[r] + 63) / 64;
    }
    if (off > cfg->n_pages) {
      delete h;
      return trie_set_error(TRIE_ECAPACITY, "n_pages %d < %d prompt pages", cfg->n_pages, off);
    }
    h->prompt_pages = off;
  }
  cudaError_t e = cudaMemcpyAsync(h->tlen, prompt_lens_host, cfg->n_requests * 4,
                                  cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess && cfg->n_pages > 0)
    e = cudaMemcpyAsync(h->page_base, pbase.data(), cfg->n_requests * 4, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h->prompts, prompt_tokens,
                        (size_t)cfg->n_requests * cfg->max_prompt_len * 4,
                        cudaMemcpyDeviceToDevice, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->status, 0, 4, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->g_ticket, 0, 8, stream);  // ticket, epoch
  if (e == cudaSuccess && h->page_ctr) e = cudaMemsetAsync(h->page_ctr, 0, 16, stream);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(h->cnt_row, 0, (size_t)cfg->n_requests * (TRIE_MAX_BEAMS + 1) * 4, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // prompt_lens_host may be freed
  if (e != cudaSuccess) {
    delete h;
    return trie_set_error(TRIE_ECUDA, "trie_create: %s", cudaGetErrorString(e));
  }
  rc = trie::launch_init(h, stream);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return TRIE_OK;
}

int trie_reset(trie_handle* h, cudaStream_t stream) {
  if (!h) return trie_set_error(TRIE_EINVAL, "null handle");
  h->b_live = 1;
  h->steps = 0;
  h->rope_tab_steps = -1;
  const cudaError_t e = cudaMemsetAsync(h->status, 0, 4, stream);  // a new job: clear latched faults
  if (e != cudaSuccess) return trie_set_error(TRIE_ECUDA, "trie_reset: %s", cudaGetErrorString(e));
  return trie::launch_init(h, stream);
}

int trie_destroy(trie_handle* h) {
  delete h;
  return TRIE_OK;
}

int trie_swa_evict(trie_handle* h, cudaStream_t stream) {
  if (!h) return trie_set_error(TRIE_EINVAL, "null handle");
  if (h->cfg.n_pages <= 0 || h->cfg.window <= 0)
    return trie_set_error(TRIE_EINVAL, "trie_swa_evict: paged pools with a window only");
  return trie::launch_swa_evict(h, stream);
}

int trie_page_stats(trie_handle* h, int32_t* stats_host, cudaStream_t stream) {
  if (!h || !stats_host) return trie_set_error(TRIE_EINVAL, "null argument");
  if (h->cfg.n_pages <= 0) return trie_set_error(TRIE_EINVAL, "dense pools: no pages");
  uint32_t c[4];
  cudaError_t e = cudaMemcpyAsync(c, h->page_ctr, 16, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return trie_set_error(TRIE_ECUDA, "trie_page_stats: %s", cudaGetErrorString(e));
  const uint32_t free0 = (uint32_t)(h->cfg.n_pages - h->prompt_pages);
  stats_host[0] = h->cfg.n_pages - (int32_t)(c[1] + free0 - c[0]);
  stats_host[1] = (int32_t)c[2];
  stats_host[2] = h->cfg.n_pages;
  return TRIE_OK;
}

int trie_get_arrays(const trie_handle* h, trie_arrays* o) {
  if (!h || !o) return trie_set_error(TRIE_EINVAL, "null argument");
  o->token = h->token;
  o->parent = h->parent;
  o->depth = h->depth;
  o->beam_mask = h->mask;
  o->leaf = h->leaf;
  o->score = h->score;
  o->n_nodes = h->n_nodes;
  o->prompt_len = h->tlen;
  o->status = h->status;
  o->b_live = h->b_live;
  o->steps = h->steps;
  o->finished = h->fin;
  o->page_table = h->page_table;
  o->page_ctr = h->page_ctr;
  return TRIE_OK;
}

int trie_set_eos(trie_handle* h, int32_t eos_id) {
  if (!h) return trie_set_error(TRIE_EINVAL, "null handle");
  if (eos_id < -1 || eos_id >= h->cfg.vocab) return trie_set_error(TRIE_EINVAL, "eos_id not in [-1, V)");
  h->eos = eos_id;
  return TRIE_OK;
}

int trie_rope_kv_append(trie_handle* h, void* q, void* k_new, const void* v_new, void* k_pool,
                        void* v_pool, float rope_theta, cudaStream_t stream) {
  if (!h || !q || !k_new || !v_new || !k_pool || !v_pool)
    return trie_set_error(TRIE_EINVAL, "null argument");
  if (!(rope_theta > 1.f)) return trie_set_error(TRIE_EINVAL, "rope_theta must be > 1");
  return trie::launch_rope_append(h, q, k_new, v_new, k_pool, v_pool, rope_theta, stream);
}

// ---- attention ------------------------------------------------------------------------
static trie::AttnParams shape_params(const trie_cfg* cfg, int b_live) {
  trie::AttnParams p{};
  p.R = cfg->n_requests;
  p.b_live = b_live;
  p.Hq = cfg->n_q_heads;
  p.Hkv = cfg->n_kv_heads;
  p.D = cfg->head_dim;
  p.cap = cfg->capacity;
  p.bf16 = cfg->kv_dtype == TRIE_BF16;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)cfg->head_dim);
  return p;
}

static int sm_count() {
  static int sm_cache[64] = {0};
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess && dev < 64) {
    if (!sm_cache[dev]) cudaDeviceGetAttribute(&sm_cache[dev], cudaDevAttrMultiProcessorCount, dev);
    if (sm_cache[dev]) sms = sm_cache[dev];
  }
  return sms;
}

static size_t part_bytes(const trie_cfg* c, int b_live, int splits) {
  if (splits <= 1) return 0;
  const size_t Qg = (size_t)b_live * (c->n_q_heads / c->n_kv_heads);
  return (size_t)c->n_requests * c->n_kv_heads * splits * Qg * (c->head_dim + 2) * 4;
}

// Attention plan: split count and scratch layout [counters | split partials | derived
// beam mask].  A pure function of the shapes, so trie_attn_scratch_bytes and
// trie_attn_decode agree.  (The opt-in persistent work-queue kernel of r08 was slower
// everywhere and is kept only as profiles/r08_experiments/attn_persist.patch.)
struct AttnPlan {
  int splits;
  size_t counter_bytes, part_bytes, mask_bytes;
};

static AttnPlan attn_plan(const trie_cfg* c, int b_live, int rows_hint, bool rope = false) {
  AttnPlan pl{};
  const int rows = rows_hint > 0 ? rows_hint : c->capacity;
  trie::AttnParams sp = shape_params(c, b_live);
  sp.rope = rope ? 1 : 0;
  sp.rows_hint = rows;
  pl.splits = trie::attn_plan_splits(sp, rows, sm_count());
  pl.part_bytes = align_up(part_bytes(c, b_live, pl.splits));
  pl.mask_bytes = align_up((size_t)c->n_requests * c->capacity * 4);
  return pl;
}

size_t trie_attn_scratch_bytes(const trie_cfg* cfg, int32_t b_live, int32_t rows_hint) {
  if (validate(cfg)) return 0;
  // the larger of the plain plan (+ the derived mask of beam_mask == NULL) and the fused
  // trie_attn_decode_rope plan: the kernels of the two may differ in occupancy
  const AttnPlan pl = attn_plan(cfg, b_live, rows_hint);
  const AttnPlan pr = attn_plan(cfg, b_live, rows_hint, true);
  const size_t a = pl.counter_bytes + pl.part_bytes + pl.mask_bytes;
  const size_t b = pr.counter_bytes + pr.part_bytes;
  return (a > b ? a : b) + 256;
}

// pt: the handle's page table for paged pools (NEXT-2), NULL for dense pools
static int attn_decode_impl(const trie_cfg* cfg, int32_t b_live, const void* q, const void* k_pool,
                            const void* v_pool, const int32_t* prompt_len, const int32_t* parent,
                            const int32_t* depth, const int32_t* leaf_ids, const int32_t* n_nodes,
                            const uint32_t* beam_mask, int32_t window, int32_t rows_hint, void* out,
                            float* lse, void* scratch, size_t scratch_bytes, uint32_t* status,
                            cudaStream_t stream, const int32_t* pt);

int trie_attn_decode(const trie_cfg* cfg, int32_t b_live, const void* q, const void* k_pool,
                     const void* v_pool, const int32_t* prompt_len, const int32_t* parent,
                     const int32_t* depth, const int32_t* leaf_ids, const int32_t* n_nodes,
                     const uint32_t* beam_mask, int32_t window, int32_t rows_hint, void* out,
                     float* lse, void* scratch, size_t scratch_bytes, uint32_t* status,
                     cudaStream_t stream) {
  if (cfg && cfg->n_pages > 0)
    return trie_set_error(TRIE_EINVAL, "trie_attn_decode addresses dense pools; paged pools go "
                                       "through the handle (trie_attn_decode_rope)");
  return attn_decode_impl(cfg, b_live, q, k_pool, v_pool, prompt_len, parent, depth, leaf_ids, n_nodes,
                          beam_mask, window, rows_hint, out, lse, scratch, scratch_bytes, status, stream,
                          nullptr);
}

static int attn_decode_impl(const trie_cfg* cfg, int32_t b_live, const void* q, const void* k_pool,
                            const void* v_pool, const int32_t* prompt_len, const int32_t* parent,
                            const int32_t* depth, const int32_t* leaf_ids, const int32_t* n_nodes,
                            const uint32_t* beam_mask, int32_t window, int32_t rows_hint, void* out,
                            float* lse, void* scratch, size_t scratch_bytes, uint32_t* status,
                            cudaStream_t stream, const int32_t* pt) {
  int rc = validate(cfg);
  if (rc) return rc;
  if (b_live < 1 || b_live > cfg->beam_width) return trie_set_error(TRIE_EINVAL, "b_live");
  if (!q || !k_pool || !v_pool || !prompt_len || !depth || !leaf_ids || !n_nodes || !out)
    return trie_set_error(TRIE_EINVAL, "null argument");
  if (window < 0) return trie_set_error(TRIE_EINVAL, "window < 0");
  const AttnPlan pl = attn_plan(cfg, b_live, rows_hint);
  const size_t pb = pl.counter_bytes + pl.part_bytes;
  const size_t need = pb + (beam_mask ? 0 : pl.mask_bytes);
  if (need > 0 && (!scratch || scratch_bytes < need))
    return trie_set_error(TRIE_ECAPACITY, "attention scratch %zu < %zu", scratch_bytes, need);
  if (!beam_mask) {
    if (!parent) return trie_set_error(TRIE_EINVAL, "beam_mask == NULL needs parent[]");
    uint32_t* derived = (uint32_t*)((char*)scratch + pb);
    rc = trie::launch_mask_walk(cfg, b_live, prompt_len, parent, leaf_ids, n_nodes, derived,
                                nullptr, stream);
    if (rc) return rc;
    beam_mask = derived;
  }
  trie::AttnParams p = shape_params(cfg, b_live);
  p.rows_hint = rows_hint > 0 ? rows_hint : cfg->capacity;
  p.q = q;
  p.k = k_pool;
  p.v = v_pool;
  p.out = out;
  p.lse = lse;
  p.tlen = prompt_len;
  p.depth = depth;
  p.leaf = leaf_ids;
  p.nn = n_nodes;
  p.mask = beam_mask;
  p.aux = scratch;
  p.part = (float*)((char*)scratch + pl.counter_bytes);
  p.status = status;
  p.window = window;
  p.splits = pl.splits;
  if (pt) {
    p.pt = pt;
    p.pt_stride = cfg->capacity / 64;
    p.n_pages = cfg->n_pages;
  }
  if (trie::attn_tc_supported(p))
    return trie::launch_attn_tc(p, stream);
  return trie::launch_attn_v1(p, stream);
}

int trie_attn_plan_info(const trie_cfg* cfg, int32_t b_live, int32_t rows_hint,
                        int32_t* info_host) {
  int rc = validate(cfg);
  if (rc) return rc;
  if (!info_host || b_live < 1 || b_live > cfg->beam_width)
    return trie_set_error(TRIE_EINVAL, "bad argument");
  trie::AttnParams p = shape_params(cfg, b_live);
  p.rows_hint = rows_hint > 0 ? rows_hint : cfg->capacity;
  const AttnPlan pl = attn_plan(cfg, b_live, rows_hint);
  const int Qg = b_live * (cfg->n_q_heads / cfg->n_kv_heads);
  int path = 0;
  if (trie::attn_tc_shape_ok(p))
    path = trie::attn_umma_eligible(p) ? 3 : trie::attn_tc_variant(p);
  p.k = p.v = (const void*)(uintptr_t)256;  // aligned placeholders for the shape test
  const bool fused = trie::attn_rope_fusable(p);
  info_host[0] = path;
  info_host[1] = fused ? attn_plan(cfg, b_live, rows_hint, true).splits : pl.splits;
  info_host[2] = fused ? 1 : 0;
  info_host[3] = Qg;
  return TRIE_OK;
}

// ---- fused a-1 + a-3 -------------------------------------------------------------------
int trie_attn_decode_rope(trie_handle* h, const void* q, const void* k_new, const void* v_new,
                          void* k_pool, void* v_pool, float rope_theta, int32_t rows_hint,
                          void* out, float* lse, void* scratch, size_t scratch_bytes,
                          cudaStream_t stream) {
  if (!h || !q || !k_new || !v_new || !k_pool || !v_pool || !out)
    return trie_set_error(TRIE_EINVAL, "null argument");
  if (!(rope_theta > 1.f)) return trie_set_error(TRIE_EINVAL, "rope_theta must be > 1");
  const trie_cfg* cfg = &h->cfg;
  const int b_live = h->b_live;
  trie::AttnParams p = shape_params(cfg, b_live);
  p.rows_hint = rows_hint > 0 ? rows_hint : cfg->capacity;
  p.q = q;
  p.k = k_pool;
  p.v = v_pool;
  p.out = out;
  p.lse = lse;
  p.tlen = h->tlen;
  p.depth = h->depth;
  p.leaf = h->leaf;
  p.nn = h->n_nodes;
  p.mask = h->mask;
  p.status = h->status;
  p.window = cfg->window;
  p.rope = 1;
  p.k_new = k_new;
  p.v_new = v_new;
  p.rope_tab = h->rope_tab;
  if (cfg->n_pages > 0) {  // paged pools (NEXT-2)
    p.pt = h->page_table;
    p.pt_stride = cfg->capacity / 64;
    p.n_pages = cfg->n_pages;
  }
  const bool fuse = trie::attn_rope_fusable(p) &&
                    (((uintptr_t)q | (uintptr_t)k_new | (uintptr_t)v_new) & 3) == 0;
  if (h->g_world > 1 && !fuse)
    return trie_set_error(TRIE_EINVAL, "gather: needs the fused bf16 tensor-core path");
  if (!fuse) {  // two launches: rotate + append, then attention over the handle's trie
    int rc = trie::launch_rope_append(h, const_cast<void*>(q), const_cast<void*>(k_new), v_new,
                                      k_pool, v_pool, rope_theta, stream);
    if (rc) return rc;
    return attn_decode_impl(cfg, b_live, q, k_pool, v_pool, h->tlen, h->parent, h->depth, h->leaf,
                            h->n_nodes, h->mask, cfg->window, rows_hint, out, lse, scratch,
                            scratch_bytes, h->status, stream, h->page_table);
  }
  if (h->rope_tab_steps != h->steps || h->rope_tab_theta != rope_theta ||
      h->rope_tab_blive != b_live) {  // once per step, shared by all layers
    int rc = trie::launch_rope_table(h, rope_theta, stream);
    if (rc) return rc;
    h->rope_tab_steps = h->steps;
    h->rope_tab_theta = rope_theta;
    h->rope_tab_blive = b_live;
  }
  const AttnPlan pl = attn_plan(cfg, b_live, rows_hint, true);
  const size_t need = pl.counter_bytes + pl.part_bytes;
  if (need > 0 && (!scratch || scratch_bytes < need))
    return trie_set_error(TRIE_ECAPACITY, "attention scratch %zu < %zu", scratch_bytes, need);
  p.aux = scratch;
  p.part = (float*)((char*)scratch + pl.counter_bytes);
  p.splits = pl.splits;
  // NEXT-3: with an EOS id, the fused kernels skip requests whose beams all finished
  if (h->eos >= 0) p.fin = h->fin;
  if (h->g_world > 1) {  // NEXT-4: the output rows also go to every rank's gather buffer
    p.ga = trie_gather_args(h);
    const uint32_t items = (uint32_t)(cfg->n_requests * cfg->n_kv_heads);
    p.ga.expected = pl.splits == 1 ? items : items * (uint32_t)(b_live * (cfg->n_q_heads / cfg->n_kv_heads));
  }
  if (cfg->window == 0 && prefetch_enabled()) {
    // tiles below the shortest prompt's last row hold prompt rows that no kernel of the
    // library writes (AttnParams::pre_tiles); row t - 1 is excluded: it is the first
    // step's leaf, appended by the b_live = 1 call.  Only split 0 prefetches; its range
    // ceil(tiles / splits) >= ceil((pre + 1) / splits) tiles bounds the count.
    int t_min = INT32_MAX;
    for (int32_t t : h->host_tlen) t_min = t < t_min ? t : t_min;
    const int pre = (t_min - 1) / 64;
    const int per_min = (pre + 1 + pl.splits - 1) / pl.splits;
    p.pre_tiles = pre < per_min ? pre : per_min;
  }
  return trie::launch_attn_tc(p, stream);
}

// ---- beam step / append / prune --------------------------------------------------------
int trie_beam_step(trie_handle* h, const float* logits, int32_t* sel_parent_beam,
                   int32_t* sel_token, float* new_score, cudaStream_t stream) {
  if (!h || !logits) return trie_set_error(TRIE_EINVAL, "null argument");
  int rc = trie::launch_beam_step(h, logits, sel_parent_beam, sel_token, new_score, stream);
  if (rc) return rc;
  h->b_live = h->cfg.beam_width;
  h->steps += 1;
  return TRIE_OK;
}

int trie_append(trie_handle* h, const int32_t* sel_parent_beam, const int32_t* sel_token,
                const float* new_score, cudaStream_t stream) {
  if (!h || !sel_parent_beam || !sel_token) return trie_set_error(TRIE_EINVAL, "null argument");
  int rc = trie::launch_append(h, sel_parent_beam, sel_token, new_score, stream);
  if (rc) return rc;
  h->b_live = h->cfg.beam_width;
  h->steps += 1;
  return TRIE_OK;
}

int trie_prune_compact(trie_handle* h, void* const* k_pools_host, void* const* v_pools_host,
                       cudaStream_t stream) {
  if (!h) return trie_set_error(TRIE_EINVAL, "null handle");
  if (h->cfg.n_layers > 0 && (!k_pools_host || !v_pools_host))
    return trie_set_error(TRIE_EINVAL, "null pool pointer arrays");
  if (h->steps == 0) return TRIE_OK;  // nothing appended yet: the prompt chain is all live
  return trie::launch_prune(h, k_pools_host, v_pools_host, stream);
}

int trie_read_hyps(trie_handle* h, int32_t max_len, int32_t* tokens_host, int32_t* len_host,
                   float* score_host, void* scratch, size_t scratch_bytes, cudaStream_t stream) {
  if (!h || max_len < 1) return trie_set_error(TRIE_EINVAL, "bad argument");
  const int R = h->cfg.n_requests, b = h->b_live;
  const size_t need = (size_t)R * b * (max_len + 1) * 4;
  if (!scratch || scratch_bytes < need)
    return trie_set_error(TRIE_ECAPACITY, "read_hyps scratch %zu < %zu", scratch_bytes, need);
  int rc = trie::launch_read_hyps(h, max_len, (int32_t*)scratch, stream);
  if (rc) return rc;
  int32_t* tmp = new (std::nothrow) int32_t[(size_t)R * b * (max_len + 1)];
  float* sc = new (std::nothrow) float[(size_t)R * TRIE_MAX_BEAMS];
  if (!tmp || !sc) {
    delete[] tmp;
    delete[] sc;
    return trie_set_error(TRIE_EINVAL, "out of host memory");
  }
  cudaError_t e = cudaMemcpyAsync(tmp, scratch, need, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(sc, h->score, (size_t)R * TRIE_MAX_BEAMS * 4, cudaMemcpyDeviceToHost,
                        stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e == cudaSuccess) {
    for (int r = 0; r < R; ++r)
      for (int j = 0; j < b; ++j) {
        const int32_t* src = tmp + ((size_t)r * b + j) * (max_len + 1);
        if (len_host) len_host[r * b + j] = src[0];
        if (tokens_host) memcpy(tokens_host + ((size_t)r * b + j) * max_len, src + 1, max_len * 4);
        if (score_host) score_host[r * b + j] = sc[r * TRIE_MAX_BEAMS + j];
      }
  }
  delete[] tmp;
  delete[] sc;
  if (e != cudaSuccess) return trie_set_error(TRIE_ECUDA, "read_hyps: %s", cudaGetErrorString(e));
  return TRIE_OK;
}

int trie_status(trie_handle* h, uint32_t* bits_host, cudaStream_t stream) {
  if (!h || !bits_host) return trie_set_error(TRIE_EINVAL, "null argument");
  cudaError_t e = cudaMemcpyAsync(bits_host, h->status, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return trie_set_error(TRIE_ECUDA, "status: %s", cudaGetErrorString(e));
  return TRIE_OK;
}

}  // extern "C"
