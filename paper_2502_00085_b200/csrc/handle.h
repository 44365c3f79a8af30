// Internal: the host-side handle and workspace carving of libtriedecode.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <vector>

#include "../../include/triedecode.h"

struct trie_handle {
  trie_cfg cfg;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  // trie metadata, SoA [R][cap]
  int32_t* token = nullptr;
  int32_t* parent = nullptr;
  int32_t* depth = nullptr;
  uint32_t* mask = nullptr;
  int32_t* leaf = nullptr;    // [R][32]
  float* score = nullptr;     // [R][32]
  int32_t* n_nodes = nullptr; // [R]
  int32_t* n_kv = nullptr;    // [R] slots [0, n_kv) hold K/V (pending leaves do not)
  int32_t* tlen = nullptr;    // [R]
  uint32_t* status = nullptr; // [1]
  int32_t* prompts = nullptr; // [R][t_max]
  // prune scratch
  int32_t* newidx = nullptr;  // [R][cap]
  int32_t* moves = nullptr;   // [R][cap] source slots of the moved K/V rows (ascending)
  int32_t* moves_dst = nullptr;  // [R][cap] their destination slots
  int32_t* n_moves = nullptr; // [R]
  // beam-step scratch
  float* chunk_max = nullptr;     // [R][b][chunks]
  float* chunk_sum = nullptr;     // [R][b][chunks]
  uint64_t* chunk_top = nullptr;  // [R][b][chunks][b]  key = ord(x) << 32 | ~v
  float* row_lse = nullptr;       // [R][32]
  uint64_t* row_top = nullptr;    // [R][32][32] each row's top-b keys
  uint32_t* cnt_row = nullptr;    // [R][32] beam-step tickets (zeroed at create)
  uint32_t* cnt_req = nullptr;    // [R]
  int32_t* sel_parent = nullptr;  // [R][b]
  int32_t* sel_token = nullptr;   // [R][b]
  float* sel_score = nullptr;     // [R][b]
  float2* rope_tab = nullptr;     // [R][b_live][D/2] (cos, sin) at the leaves' depths
  uint32_t* fin = nullptr;        // [R][32] beam finished (its last token is eos; NEXT-3)
  int32_t eos = -1;               // trie_set_eos; -1 = no EOS (the hot path)
  int32_t rope_tab_steps = -1;    // host: step count the table was computed for
  float rope_tab_theta = 0.f;
  int32_t rope_tab_blive = 0;
  int32_t chunks = 1;
  // NEXT-4 fused all-gather (trie_gather_setup): every rank's gather buffer / flag array as
  // mapped in this process; ticket + completed-launch counter in the workspace
  int32_t g_world = 0, g_rank = 0;
  void* g_out[8] = {};
  uint32_t* g_flags[8] = {};
  uint32_t* g_ticket = nullptr;
  uint32_t* g_epoch = nullptr;
  // paged pools (cfg.n_pages > 0, NEXT-2)
  int32_t* page_table = nullptr;  // [R][cap/64]
  int32_t* pages_used = nullptr;  // [R] pages mapped (blocks [0, used) of the table)
  int32_t* page_base = nullptr;   // [R] first prompt page (fixed)
  int32_t* free_q = nullptr;      // [n_pages] ring of free pages
  uint32_t* page_ctr = nullptr;   // [0] pops, [1] pushes, [2] peak in use, [3] n_pages
  int32_t prompt_pages = 0;       // host: sum over requests of ceil(t_r / 64)
  // host-tracked state
  int32_t b_live = 1;
  int32_t steps = 0;
  std::vector<int32_t> host_tlen;
};

// logits per beam-step chunk CTA (beam_step.cu)
constexpr int TRIE_BEAM_CHUNK = 8192;

// the kernels' view of the handle's gather registration (attn_common.cuh GatherArgs)
#include "attn_common.cuh"
inline trie::GatherArgs trie_gather_args(const trie_handle* h) {
  trie::GatherArgs ga = {};
  ga.world = h->g_world;
  ga.rank = h->g_rank;
  for (int q = 0; q < h->g_world && q < 8; ++q) {
    ga.out[q] = h->g_out[q];
    ga.flag[q] = h->g_flags[q];
  }
  ga.ticket = h->g_ticket;
  ga.epoch = h->g_epoch;
  ga.half_stride = (size_t)h->cfg.n_requests * h->cfg.beam_width * h->g_world * h->cfg.n_q_heads *
                   h->cfg.head_dim;
  return ga;
}

// Paged pools (NEXT-2): the kernels' view of the page state.  Free queue: logical entry i
// lives at fq[i % n_pages]; entries [0, n_pages - prompt_pages) are filled by k_init, pushes
// append at n_pages - prompt_pages + ctr[1], pops take entry ctr[0].
struct PageArgs {
  int32_t* pt;          // [R][cap/64]
  int32_t* used;        // [R]
  const int32_t* base;  // [R]
  int32_t* fq;          // [n_pages]
  uint32_t* ctr;        // [4] pops, pushes, peak in use, n_pages
  int n_pages, prompt_pages;
};
inline PageArgs page_args(const trie_handle* h) {
  PageArgs a = {};
  a.n_pages = h->cfg.n_pages > 0 ? h->cfg.n_pages : 0;
  a.pt = h->page_table;
  a.used = h->pages_used;
  a.base = h->page_base;
  a.fq = h->free_q;
  a.ctr = h->page_ctr;
  a.prompt_pages = h->prompt_pages;
  return a;
}

// carve the workspace; with h == nullptr only computes the size
size_t trie_layout(const trie_cfg* cfg, trie_handle* h, char* base);

// launchers (defined in the .cu files)
namespace trie {
int launch_init(trie_handle* h, cudaStream_t s);
int launch_append(trie_handle* h, const int32_t* par, const int32_t* tok, const float* sc,
                  cudaStream_t s);
int launch_beam_step(trie_handle* h, const float* logits, int32_t* out_par, int32_t* out_tok,
                     float* out_sc, cudaStream_t s);
int launch_prune(trie_handle* h, void* const* kp, void* const* vp, cudaStream_t s);
int launch_swa_evict(trie_handle* h, cudaStream_t s);
int launch_rope_append(trie_handle* h, void* q, void* k_new, const void* v_new, void* kpool,
                       void* vpool, float theta, cudaStream_t s);
int launch_read_hyps(trie_handle* h, int32_t max_len, int32_t* out_dev, cudaStream_t s);
int launch_rope_table(trie_handle* h, float theta, cudaStream_t s);
int launch_mask_walk(const trie_cfg* cfg, int32_t b_live, const int32_t* tlen,
                     const int32_t* parent, const int32_t* leaf, const int32_t* nn,
                     uint32_t* mask_out, uint32_t* status, cudaStream_t s);
}  // namespace trie
