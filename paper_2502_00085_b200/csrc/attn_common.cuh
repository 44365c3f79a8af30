// Parameters shared by the trie attention kernels (attn_decode.cu, attn_decode_tc.cu).
#pragma once
#include <stdint.h>

namespace trie {

// NEXT-4 fused all-gather of the KV-head shard (trie_gather_setup): every output row is
// also stored into every rank's gather buffer; the last item of the launch publishes the
// launch's sequence number to every rank's flag array.  world == 0: disabled.
struct GatherArgs {
  void* out[8];       // per rank: its gather buffer [2][R][b_live][world*Hq][D] (bf16)
  uint32_t* flag[8];  // per rank: its flag array [world]
  uint32_t* ticket;   // this handle's arrival counter (zero between launches)
  uint32_t* epoch;    // this handle's completed-launch counter
  int world, rank;
  uint32_t expected;  // arrivals per launch (items, or rows for the split-K combine)
  size_t half_stride; // elements per half: R * beam_width * world * Hq * D
};

struct AttnParams {
  const void* q;       // [R][b_live][Hq][D]
  const void* k;       // [R][Hkv][cap][D]
  const void* v;       // [R][Hkv][cap][D]
  void* out;           // [R][b_live][Hq][D]
  float* lse;          // [R][b_live][Hq] or null
  const int32_t* tlen; // [R]
  const int32_t* depth;   // [R][cap]
  const int32_t* leaf;    // [R][32]
  const int32_t* nn;      // [R]
  const uint32_t* mask;   // [R][cap]
  float* part;            // split partials
  void* aux;              // scratch base (counters, if any, precede the split partials)
  uint32_t* status;
  int R, b_live, Hq, Hkv, D, cap, window, splits;
  int rows_hint;          // expected rows per request (planning only; 0 = capacity)
  float scale_log2;       // log2(e) / sqrt(D)
  int bf16;
  // fused RoPE + KV append (trie_attn_decode_rope): q is read un-rotated, the leaves'
  // k_new/v_new rows are rotated/appended into the pools by the CTA owning their tile
  int rope;
  const void* k_new;      // [R][b_live][Hkv][D]
  const void* v_new;      // [R][b_live][Hkv][D]
  const float2* rope_tab; // [R][b_live][D/2] (cos, sin) of the leaves' depths (per step)
  // pre_tiles > 0: the first pre_tiles 64-slot tiles of every request hold prompt rows
  // below t - 1 only (host-known minimum prompt length, no window, one split).  Those rows
  // are written by the caller's prefill before trie_create / trie_reset and never again by
  // any kernel of the library (the prompt never moves, invariant 3; row t - 1 is excluded,
  // the first step appends it as the prompt leaf), so their K/V may be loaded BEFORE
  // griddepcontrol.wait: the first ring stages fill while the predecessor drains.
  int pre_tiles;
  int half_tiles;         // narrow / wide: the last tile of an item loads 32-row boxes when <= 32 rows remain
  // NEXT-3 (narrow / wide, handle path with an EOS id): fin [R][32] finished flags; a
  // request whose b_live beams are all finished is done -- its CTAs read and write nothing
  const uint32_t* fin;
  GatherArgs ga;
  // paged pools (cfg.n_pages > 0, NEXT-2): page table [R][pt_stride]; NULL = dense pools
  const int32_t* pt;
  int pt_stride;
  int n_pages;
};

// Pool row of slot n of request r, KV head h (include/triedecode.h "KV pool layouts").
__device__ __forceinline__ long attn_row(const AttnParams& p, int r, int h, int n) {
  if (p.pt) return ((long)__ldg(p.pt + r * p.pt_stride + (n >> 6)) * p.Hkv + h) * 64 + (n & 63);
  return ((long)r * p.Hkv + h) * p.cap + n;
}
// rows of the 2-D [rows][D] view of a pool
inline long attn_pool_rows(const AttnParams& p) {
  return p.pt ? (long)p.n_pages * p.Hkv * 64 : (long)p.R * p.Hkv * p.cap;
}

int launch_attn_v1(const AttnParams& p, cudaStream_t s);
int launch_gather_wait(const GatherArgs& ga, int R, int b_live, int Hq, int D, void* dst, cudaStream_t s);
int launch_attn_tc(const AttnParams& p, cudaStream_t s);
bool attn_rope_fusable(const AttnParams& p);
bool attn_tc_supported(const AttnParams& p);
int launch_attn_combine_bf16(const AttnParams& p, cudaStream_t s);
int attn_plan_splits(const AttnParams& p, int rows_est, int sms);
bool attn_tc_shape_ok(const AttnParams& p);
int attn_tc_variant(const AttnParams& p);  // 1 = narrow, 2 = wide (mma.sync kernels)
bool attn_umma_eligible(const AttnParams& p);
int attn_umma_occ(const AttnParams& p);
int launch_attn_umma(const AttnParams& p, cudaStream_t s);

}  // namespace trie
