// trie_beam_step: log-softmax + global top-b over b x V logits (Alg. 2 l.9 argsort_b,
// P:146; Alg. 1 l.6 top-b), then update_trie / update_mask (Alg. 2 l.10-11,
// P:147-148; §3.3; §3.4 positions P:206).
//
// Stage A (k_row_chunk): one CTA per (request, beam row, chunk of CHUNK logits): chunk
//   max, chunk sum exp(x - max) and the chunk's top-b by (x desc, v asc), from registers
//   (one HBM pass over the fp32 logits, 16-byte loads).
// Stage B (k_select_append): one CTA per request: combine chunk (max, sum) into each row's
//   lse; reduce every row's chunk lists to the row's top-b; score the <= b*b survivors
//   cs = score_j + (x - lse_j) and take the global top-b in the total order
//   (cs desc, v asc, j asc) (readings R1, R3); then append (token/parent/depth, leaves,
//   scores, N) and the bitset update new[n] bit r = old[n] bit j_r.
// Keys: 64-bit, larger = better.  Row stage: ord(x) << 32 | ~v.  Global stage:
//   ord(cs) << 32 | ~(v * b_live + j).  A row's top-b by x contains that row's top-b by
//   cs (cs is monotone in x within a row); fp32 rounding of cs can only reorder
//   candidates whose cs differ by <= 1 ulp -- the near-tie case of the parity protocol.
#include <float.h>

#include "common.cuh"
#include "handle.h"

namespace trie {

constexpr int BS_A = 256;
constexpr int ITEMS_A = 16;  // CHUNK = BS_A * ITEMS_A = 4096 logits per CTA
constexpr int CHUNK = BS_A * ITEMS_A;

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

// Warp-cooperative top-k by repeated arg-max over ITEMS keys per lane (keys are unique).
// Selected keys are written (descending) to out[0..k) by lane 0; items are consumed.
template <int ITEMS>
__device__ __forceinline__ void warp_topk(uint64_t (&key)[ITEMS], int k, uint64_t* out) {
  const int lane = threadIdx.x & 31;
  for (int s = 0; s < k; ++s) {
    uint64_t best = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) best = key[i] > best ? key[i] : best;
    uint64_t wb = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      uint64_t y = shfl_xor_u64(wb, o);
      wb = y > wb ? y : wb;
    }
    if (lane == 0) out[s] = wb;
    if (wb == 0) continue;  // fewer than k real items
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (key[i] == wb) key[i] = 0;  // unique keys: exactly one lane clears it
  }
}

// ---- Stage A --------------------------------------------------------------------------
__global__ void __launch_bounds__(BS_A) k_row_chunk(const float* __restrict__ logits, int V,
                                                    int b_live, int b, int chunks,
                                                    float* chunk_max, float* chunk_sum,
                                                    uint64_t* chunk_top) {
  __shared__ float sm_red[BS_A / 32];
  __shared__ uint64_t sm_top[BS_A / 32][TRIE_MAX_BEAMS];
  const int c = blockIdx.x, row = blockIdx.y;  // row = r * b_live + j
  const float* x = logits + (size_t)row * V;
  const int v0 = c * CHUNK;
  float val[ITEMS_A];
  // coalesced: item i of thread tid is element v0 + i*BS_A + tid
#pragma unroll
  for (int i = 0; i < ITEMS_A; ++i) {
    const int v = v0 + i * BS_A + threadIdx.x;
    val[i] = v < V ? __ldg(x + v) : -INFINITY;
  }
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < ITEMS_A; ++i) m = fmaxf(m, val[i]);
  m = warp_max(m);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm_red[w] = m;
  __syncthreads();
  m = sm_red[0];
#pragma unroll
  for (int i = 1; i < BS_A / 32; ++i) m = fmaxf(m, sm_red[i]);
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ITEMS_A; ++i) s += (val[i] == -INFINITY) ? 0.f : expf(val[i] - m);
  s = warp_sum(s);
  if (lane == 0) sm_red[w] = s;
  // top-b keys of this chunk
  uint64_t key[ITEMS_A];
#pragma unroll
  for (int i = 0; i < ITEMS_A; ++i) {
    const int v = v0 + i * BS_A + threadIdx.x;
    key[i] = v < V ? ((uint64_t)f2ord(val[i]) << 32) | (uint32_t)(~(uint32_t)v) : 0ull;
  }
  const int k = min(b, CHUNK);
  warp_topk<ITEMS_A>(key, k, sm_top[w]);
  __syncthreads();
  const size_t o = (size_t)row * chunks + c;
  if (w == 0) {
    // merge the 8 warp lists (8*k <= 256 keys, 8 per lane)
    uint64_t kk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = i * 32 + lane;
      const int ww = idx / TRIE_MAX_BEAMS, pos = idx % TRIE_MAX_BEAMS;
      kk[i] = (ww < BS_A / 32 && pos < k) ? sm_top[ww][pos] : 0ull;
    }
    uint64_t* dst = chunk_top + o * b;
    warp_topk<8>(kk, k, dst);
    if (lane == 0) {
      float tot = 0.f;
      for (int i = 0; i < BS_A / 32; ++i) tot += sm_red[i];
      chunk_max[o] = m;
      chunk_sum[o] = tot;
    }
  }
}

// ---- append (Alg. 2 l.10-11) -----------------------------------------------------------
// Called by all threads of a CTA for request r with the selection in shared memory.
__device__ void append_sel(int r, int b_new, int b_old, const int* sp, const int* st,
                           const float* ss, int32_t* token, int32_t* parent, int32_t* depth,
                           uint32_t* mask, int32_t* leaf, float* score, int32_t* nn,
                           int32_t* nkv, const int32_t* tlen, int cap, uint32_t* status) {
  __shared__ int sm_old_leaf[TRIE_MAX_BEAMS];
  const size_t base = (size_t)r * cap;
  const int N = nn[r], t = tlen[r];
  if (threadIdx.x < b_old) sm_old_leaf[threadIdx.x] = leaf[r * TRIE_MAX_BEAMS + threadIdx.x];
  __syncthreads();
  const bool fits = N + b_new <= cap;
  if (!fits) {
    if (threadIdx.x == 0) latch(status, TRIE_ST_CAPACITY);
    return;
  }
  // update_mask over generated nodes: new bit r = old bit j_r
  for (int n = t + threadIdx.x; n < N; n += blockDim.x) {
    const uint32_t w = mask[base + n];
    uint32_t nw = 0u;
    for (int q = 0; q < b_new; ++q) nw |= ((w >> sp[q]) & 1u) << q;
    mask[base + n] = nw;
  }
  if (threadIdx.x < b_new) {
    const int q = threadIdx.x;
    const int j = sp[q];
    const int p = (j >= 0 && j < b_old) ? sm_old_leaf[j] : -1;
    const int slot = N + q;
    if (p < 0 || p >= N) latch(status, TRIE_ST_LEAF);
    token[base + slot] = st[q];
    parent[base + slot] = p;
    depth[base + slot] = (p >= 0 && p < N) ? depth[base + p] + 1 : 0;  // §3.4
    mask[base + slot] = 1u << q;
  }
  __syncthreads();
  if (threadIdx.x < b_new) {
    leaf[r * TRIE_MAX_BEAMS + threadIdx.x] = N + threadIdx.x;
    score[r * TRIE_MAX_BEAMS + threadIdx.x] = ss[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    nn[r] = N + b_new;
    nkv[r] = N;  // the new leaves are pending: their K/V arrive with the next forward
  }
}

__global__ void k_append(const int32_t* par, const int32_t* tok, const float* sc, int b_new,
                         int b_old, int32_t* token, int32_t* parent, int32_t* depth,
                         uint32_t* mask, int32_t* leaf, float* score, int32_t* nn, int32_t* nkv,
                         const int32_t* tlen, int cap, uint32_t* status) {
  __shared__ int sp[TRIE_MAX_BEAMS], st[TRIE_MAX_BEAMS];
  __shared__ float ss[TRIE_MAX_BEAMS];
  const int r = blockIdx.x;
  if (threadIdx.x < b_new) {
    sp[threadIdx.x] = par[r * b_new + threadIdx.x];
    st[threadIdx.x] = tok[r * b_new + threadIdx.x];
    ss[threadIdx.x] = sc ? sc[r * b_new + threadIdx.x] : 0.f;
  }
  __syncthreads();
  append_sel(r, b_new, b_old, sp, st, ss, token, parent, depth, mask, leaf, score, nn, nkv,
             tlen, cap, status);
}

// ---- Stage B ---------------------------------------------------------------------------
constexpr int BS_B = 256;
__global__ void __launch_bounds__(BS_B) k_select_append(
    const float* chunk_max, const float* chunk_sum, const uint64_t* chunk_top, int b_live,
    int b, int chunks, int32_t* token, int32_t* parent, int32_t* depth, uint32_t* mask,
    int32_t* leaf, float* score, int32_t* nn, int32_t* nkv, const int32_t* tlen, int cap,
    uint32_t* status, int32_t* out_par, int32_t* out_tok, float* out_sc) {
  __shared__ float sm_lse[TRIE_MAX_BEAMS];
  __shared__ uint64_t sm_row[TRIE_MAX_BEAMS][TRIE_MAX_BEAMS];  // each row's top-b by x
  __shared__ uint64_t sm_sel[TRIE_MAX_BEAMS];
  __shared__ int sp[TRIE_MAX_BEAMS], st[TRIE_MAX_BEAMS];
  __shared__ float ss[TRIE_MAX_BEAMS];
  const int r = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = b;  // candidates needed per row (b <= V guaranteed by the host)
  // (1) per row: lse from chunk (max, sum); the row's top-k from its chunk lists
  for (int j = w; j < b_live; j += BS_B / 32) {
    const size_t rowi = (size_t)r * b_live + j;
    float M = -INFINITY;
    for (int c = lane; c < chunks; c += 32) M = fmaxf(M, chunk_max[rowi * chunks + c]);
    M = warp_max(M);
    float S = 0.f;
    for (int c = lane; c < chunks; c += 32) {
      const float cm = chunk_max[rowi * chunks + c];
      S += chunk_sum[rowi * chunks + c] * expf(cm - M);
    }
    S = warp_sum(S);
    if (lane == 0) sm_lse[j] = M + logf(S);
    // chunks * k keys; process in slices of 32*ITEMS and keep a running top-k
    constexpr int IT = 8;
    uint64_t best[IT];  // running top-k held in the first k of a 32*IT pool
    const int total = chunks * k;
    const uint64_t* src = chunk_top + rowi * chunks * b;
    // pool = running list (k <= 32, lane-distributed at item 0) + next slice
    uint64_t run = 0ull;  // lane l holds running[l] (l < k)
    for (int s0 = 0; s0 < total; s0 += 32 * (IT - 1)) {
      best[0] = run;
#pragma unroll
      for (int i = 1; i < IT; ++i) {
        const int idx = s0 + (i - 1) * 32 + lane;
        best[i] = 0ull;
        if (idx < total) {
          const int c = idx / k, pos = idx % k;
          best[i] = src[(size_t)c * b + pos];
        }
      }
      uint64_t* dst = &sm_row[j][0];
      warp_topk<IT>(best, k, dst);
      __syncwarp();
      run = lane < k ? dst[lane] : 0ull;
      __syncwarp();
    }
  }
  __syncthreads();
  // (2) global: b_live * k candidates keyed by (cs, ~(v*b_live + j))
  {
    constexpr int IT = 32;  // b_live*k <= 1024 = 32 lanes * 32 items, handled by warp 0
    if (w == 0) {
      uint64_t key[IT];
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        const int idx = i * 32 + lane;
        key[i] = 0ull;
        const int j = idx / k, pos = idx % k;
        if (j < b_live) {
          const uint64_t rk = sm_row[j][pos];
          if (rk != 0ull) {
            const float x = ord2f((uint32_t)(rk >> 32));
            const uint32_t v = ~(uint32_t)rk;
            const float cs = score[r * TRIE_MAX_BEAMS + j] + (x - sm_lse[j]);
            key[i] = ((uint64_t)f2ord(cs) << 32) | (uint32_t)(~(v * (uint32_t)b_live + j));
          }
        }
      }
      warp_topk<IT>(key, b, sm_sel);
    }
  }
  __syncthreads();
  if (threadIdx.x < b) {
    const uint64_t kk = sm_sel[threadIdx.x];
    const uint32_t id = ~(uint32_t)kk;
    sp[threadIdx.x] = (int)(id % (uint32_t)b_live);
    st[threadIdx.x] = (int)(id / (uint32_t)b_live);
    ss[threadIdx.x] = ord2f((uint32_t)(kk >> 32));
    if (out_par) out_par[r * b + threadIdx.x] = sp[threadIdx.x];
    if (out_tok) out_tok[r * b + threadIdx.x] = st[threadIdx.x];
    if (out_sc) out_sc[r * b + threadIdx.x] = ss[threadIdx.x];
  }
  __syncthreads();
  append_sel(r, b, b_live, sp, st, ss, token, parent, depth, mask, leaf, score, nn, nkv, tlen,
             cap, status);
}

int launch_beam_step(trie_handle* h, const float* logits, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  const int chunks = (c.vocab + CHUNK - 1) / CHUNK;
  dim3 ga(chunks, c.n_requests * h->b_live);
  k_row_chunk<<<ga, BS_A, 0, s>>>(logits, c.vocab, h->b_live, c.beam_width, chunks,
                                  h->chunk_max, h->chunk_sum, h->chunk_top);
  int rc = trie_check_launch("k_row_chunk");
  if (rc) return rc;
  k_select_append<<<c.n_requests, BS_B, 0, s>>>(
      h->chunk_max, h->chunk_sum, h->chunk_top, h->b_live, c.beam_width, chunks, h->token,
      h->parent, h->depth, h->mask, h->leaf, h->score, h->n_nodes, h->n_kv, h->tlen, c.capacity,
      h->status, h->sel_parent, h->sel_token, h->sel_score);
  return trie_check_launch("k_select_append");
}

int launch_append(trie_handle* h, const int32_t* par, const int32_t* tok, const float* sc,
                  cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  k_append<<<c.n_requests, 256, 0, s>>>(par, tok, sc, c.beam_width, h->b_live, h->token,
                                        h->parent, h->depth, h->mask, h->leaf, h->score,
                                        h->n_nodes, h->n_kv, h->tlen, c.capacity, h->status);
  return trie_check_launch("k_append");
}

}  // namespace trie
