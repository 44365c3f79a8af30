// trie_beam_step: log-softmax + global top-b over b x V logits (Alg. 2 l.9 argsort_b,
// P:146; Alg. 1 l.6 top-b), then update_trie / update_mask (Alg. 2 l.10-11,
// P:147-148; §3.3; §3.4 positions P:206).
//
// ONE launch, k_beam_step, grid (chunks, R * b_live), 256 threads per CTA:
//   chunk stage (every CTA): 8192 logits of one (request, beam row) from HBM once
//     (16-byte streaming loads, 32 per thread in registers), chunk max and sum
//     exp(x - max) (packed FFMA2 + MUFU.EX2), and the chunk's top-b by (x desc, v asc).
//     The top-b is THRESHOLD + SORT: every warp has ceil(b/8) lanes whose maximum is
//     >= its ceil(b/8)-th largest lane maximum (redux.sync rounds), so the chunk has >= b
//     elements >= T = the minimum of that over the 8 warps; only elements >= T (a few x b)
//     are pushed to shared memory and sorted (one warp bitonic sort when <= 32, rank
//     counting up to 512).  If ties overflow the buffer, warp arg-max rounds instead.
//   row stage (the LAST chunk CTA of a row, acq_rel atomic ticket): row lse from the
//     chunk (max, sum) pairs; the row's top-b by a bitonic merge tree of the chunk lists
//     (top-32 of two sorted lists = one bitonic merge of max(A[i], B[31-i])).
//   request stage (the LAST row CTA of a request): candidate scores
//     cs = score_j + (x - lse_j) of the b_live x b survivors, global top-b in the total
//     order (cs desc, v asc, j asc) (readings R1, R3) by the same merge tree, then append
//     (token/parent/depth, leaves, scores, N) and the bitset update
//     new[n] bit r = old[n] bit j_r.
// Keys: 64-bit, larger = better.  Row stage: ord(x) << 32 | ~v.  Global stage:
//   ord(cs) << 32 | ~(v * b_live + j).  A row's top-b by x contains that row's top-b by
//   cs (cs is monotone in x within a row); fp32 rounding of cs can only reorder
//   candidates whose cs differ by <= 1 ulp -- the near-tie case of the parity protocol.
// The tickets (cnt_row, cnt_req) are zeroed by trie_create and re-zeroed by the CTA that
// takes the last ticket, so the kernel is CUDA-graph replayable.
#include <float.h>

#include "common.cuh"
#include "handle.h"

namespace trie {

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

// ---- selection helpers ------------------------------------------------------------------
constexpr int BS = 256;
constexpr int ITEMS = 32;            // logits per thread
constexpr int CHUNK = BS * ITEMS;    // 8192 logits per CTA
static_assert(CHUNK == TRIE_BEAM_CHUNK, "workspace sizing (handle.h)");
constexpr int CAND_CAP = 512;        // candidate keys buffered by the chunk stage
constexpr int RANK_MAX = 128;        // row / request stage: rank counting up to this many keys

// Descending top-k of n unique keys (0 = empty) by rank counting: out[rank(x)] = x for
// rank < k, out[] zero-filled first.  Block-wide; src may be shared or global memory.
__device__ __forceinline__ void block_rank_topk(const uint64_t* src, int n, int k, uint64_t* out) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t x = src[i];
    if (x == 0ull) continue;
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += src[j] > x ? 1 : 0;
    if (rank < k) out[rank] = x;
  }
  __syncthreads();
}

// One value per lane -> the warp's values sorted descending (lane i holds the i-th largest):
// bitonic sort over shuffles.
__device__ __forceinline__ float warp_sort_desc(float v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const float o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool desc = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      v = (lower == desc) ? fmaxf(v, o) : fminf(v, o);
    }
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_sort_desc_u64(uint64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = shfl_xor_u64(v, stride);
      const bool desc = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      v = (lower == desc) ? (o > v ? o : v) : (o < v ? o : v);
    }
  }
  return v;
}

// Top-32 of two descending 32-lists (lane i holds the i-th entry; 0 pads): C[i] =
// max(A[i], B[31 - i]) holds the top 32 of A u B and is bitonic, so one bitonic merge
// (5 shuffle stages) sorts it descending.
__device__ __forceinline__ uint64_t warp_merge_top32(uint64_t a, uint64_t b) {
  const int lane = threadIdx.x & 31;
  const uint64_t br = shfl_u64(b, 31 - lane);
  uint64_t c = a > br ? a : br;
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const uint64_t o = shfl_xor_u64(c, stride);
    c = ((lane & stride) == 0) ? (o > c ? o : c) : (o < c ? o : c);
  }
  return c;
}

// Every warp holds a descending 32-list in `acc`; merge the 8 lists pairwise (3 levels)
// through `buf` [8][32]; the block's top-32 ends in buf[0][0..32).
__device__ __forceinline__ void block_merge_tree(uint64_t acc, uint64_t (*buf)[32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  buf[w][lane] = acc;
  __syncthreads();
#pragma unroll
  for (int n = 4; n >= 1; n >>= 1) {
    uint64_t m = 0ull;
    if (w < n) m = warp_merge_top32(buf[w][lane], buf[w + n][lane]);
    __syncthreads();
    if (w < n) buf[w][lane] = m;
    __syncthreads();
  }
}


// ticket counter increment with release + acquire semantics at gpu scope: the barrier
// before it orders the CTA's writes; the barrier after it publishes the acquire
__device__ __forceinline__ uint32_t ticket_acq_rel(uint32_t* p) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}

__device__ __forceinline__ uint64_t row_key(float x, int v) {
  return ((uint64_t)f2ord(x) << 32) | (uint32_t)(~(uint32_t)v);
}

// ---- paged pools (NEXT-2): map pages until request r's table covers n_slots ----------
// One thread per request.  Pops take free-queue entry ctr[0]; the queue is empty when that
// entry has not been pushed yet (pushes happen only in k_page_release, another launch).
__device__ void page_grow(const PageArgs& pg, int r, int cap, int n_slots, uint32_t* status) {
  const int stride = cap / 64, need = (n_slots + 63) / 64;
  const uint32_t nfree0 = (uint32_t)(pg.n_pages - pg.prompt_pages);
  int used = pg.used[r];
  while (used < need) {
    const uint32_t i = atomicAdd(&pg.ctr[0], 1u);
    const uint32_t pushes = *(volatile uint32_t*)&pg.ctr[1];
    if (i >= nfree0 + pushes) {  // out of pages
      latch(status, TRIE_ST_CAPACITY);
      break;
    }
    pg.pt[r * stride + used] = pg.fq[i % (uint32_t)pg.n_pages];
    ++used;
    atomicMax(&pg.ctr[2], (uint32_t)pg.n_pages - (nfree0 + pushes - (i + 1u)));  // peak in use
  }
  pg.used[r] = used;
}

// ---- append (Alg. 2 l.10-11) -----------------------------------------------------------
// Called by all threads of a CTA for request r with the selection in shared memory.
__device__ void append_sel(int r, int b_new, int b_old, const int* sp, const int* st,
                           const float* ss, int32_t* token, int32_t* parent, int32_t* depth,
                           uint32_t* mask, int32_t* leaf, float* score, int32_t* nn,
                           int32_t* nkv, const int32_t* tlen, int cap, uint32_t* status,
                           uint32_t* fin, int eos, const PageArgs& pg) {
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
  if (pg.n_pages > 0 && threadIdx.x == 0) page_grow(pg, r, cap, N + b_new, status);
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
    if (fin) fin[r * TRIE_MAX_BEAMS + q] = (eos >= 0 && st[q] == eos) ? 1u : 0u;  // NEXT-3
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
                         const int32_t* tlen, int cap, uint32_t* status, uint32_t* fin, int eos,
                         PageArgs pg) {
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
             tlen, cap, status, fin, eos, pg);
}

// ---- the fused beam step ----------------------------------------------------------------
struct BeamStepArgs {
  const float* logits;
  int V, b_live, b, chunks;
  float* chunk_max;
  float* chunk_sum;
  uint64_t* chunk_top;   // [R * b_live][chunks][b]
  float* row_lse;        // [R][32]
  uint64_t* row_top;     // [R][32][32]
  uint32_t* cnt_row;     // [R * 32]
  uint32_t* cnt_req;     // [R]
  int32_t *token, *parent, *depth;
  uint32_t* mask;
  int32_t* leaf;
  float* score;
  int32_t *nn, *nkv;
  const int32_t* tlen;
  int cap;
  uint32_t* status;
  int32_t *sel_par, *sel_tok;
  float* sel_sc;
  int32_t *out_par, *out_tok;
  float* out_sc;
  // NEXT-3 (reading R5b): EOS as an absorbing state.  A beam whose last generated token is
  // eos (fin[r][j] != 0) continues only with eos at log-probability 0 (its row is treated
  // as one-hot at eos: lse 0, one candidate, score unchanged); eos < 0 disables.
  int eos;
  uint32_t* fin;  // [R][32]
  PageArgs pg;    // paged pools (NEXT-2): pages mapped as N grows
};

// element index of item i of this thread within the row
template <bool VEC>
__device__ __forceinline__ int item_v(int v0, int i) {
  return VEC ? v0 + 4 * ((i >> 2) * BS + (int)threadIdx.x) + (i & 3) : v0 + i * BS + (int)threadIdx.x;
}

// One work item = one chunk of one (request, beam) row, then (ticket) its row stage, then
// (ticket) its request stage.  val[] holds the chunk's logits (-inf padding); with sval
// != nullptr the same values are also in shared memory in load order (element v0 + e at
// sval[e]), which the candidate push reads by index.
template <bool VEC>
__device__ __forceinline__ void beam_item(const BeamStepArgs& a, int row, int c,
                                          const float (&val)[ITEMS], const float* sval,
                                          bool finrow = false) {
  __shared__ uint32_t sm_red[BS / 32], sm_tb[BS / 32];
  __shared__ float sm_sum[BS / 32];
  __shared__ __align__(16) float sm_stage[BS * ITEMS];
  __shared__ uint64_t sm_cand[CAND_CAP];
  __shared__ uint64_t sm_wtop[BS / 32][TRIE_MAX_BEAMS];
  __shared__ uint64_t sm_mrg[BS / 32][32];
  __shared__ float sm_lse[TRIE_MAX_BEAMS];
  __shared__ int sm_n, sm_last;
  __shared__ int sp[TRIE_MAX_BEAMS], st[TRIE_MAX_BEAMS];
  __shared__ float ss[TRIE_MAX_BEAMS];
  const int r = row / a.b_live, j_row = row % a.b_live;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int V = a.V, k = a.b;  // candidates kept per chunk / row (b <= V, b <= 32)
  const int v0 = c * CHUNK;

  // ---- chunk stage ----------------------------------------------------------------------
  if (threadIdx.x == 0) sm_n = 0;
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) m = fmaxf(m, val[i]);  // padding items are -inf
  // threshold T with >= k elements of the chunk >= T: every warp has >= mk = ceil(k/8)
  // lanes whose maximum is >= its mk-th largest lane maximum tb_w (redux rounds, one lane
  // excluded per round), so T = min over the 8 warps of tb_w
  const uint32_t mkey = f2ord(m);
  const uint32_t wmax = __reduce_max_sync(0xffffffffu, mkey);
  uint32_t tb = wmax;
  {
    uint32_t kk = mkey;
    for (int q = 1; q < (k + BS / 32 - 1) / (BS / 32); ++q) {
      const uint32_t who = __ballot_sync(0xffffffffu, kk == tb);
      if (lane == __ffs(who) - 1) kk = 0u;
      tb = __reduce_max_sync(0xffffffffu, kk);
    }
  }
  if (lane == 0) { sm_red[w] = wmax; sm_tb[w] = tb; }
  __syncthreads();
  uint32_t mo = sm_red[0], to = sm_tb[0];
#pragma unroll
  for (int i = 1; i < BS / 32; ++i) {
    mo = max(mo, sm_red[i]);
    to = min(to, sm_tb[i]);
  }
  m = ord2f(mo);
  const float T = ord2f(to);
  // sum exp(x - m) = sum 2^(x log2e - m log2e): packed FFMA2 / FADD2 + one MUFU.EX2 per
  // logit (ex2.approx: ~2 ulp, far inside the 1e-4 score tolerance); padding -> 2^-inf = 0
  const float l2e = 1.4426950408889634f;
  const float nml = m == -INFINITY ? 0.f : -m * l2e;
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < ITEMS; i += 2) {
    const float2 y = ffma2(make_float2(val[i], val[i + 1]), make_float2(l2e, l2e), make_float2(nml, nml));
    acc = fadd2(acc, make_float2(ex2_approx(y.x), ex2_approx(y.y)));
  }
  float s = warp_sum(acc.x + acc.y);
  if (lane == 0) sm_sum[w] = s;
  // candidates: one compare per logit into a bit set; lanes with set bits stage their
  // values in shared memory and push (value, index) keys
  uint32_t bits = 0u;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) bits |= (val[i] >= T ? 1u : 0u) << i;
  if (T == -INFINITY) {  // too few finite logits: drop the -inf padding items
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (item_v<VEC>(v0, i) >= V) bits &= ~(1u << i);
  }
  if (finrow) {  // absorbing eos: the row's only candidate is eos itself
    bits = 0u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (item_v<VEC>(v0, i) == a.eos) bits |= 1u << i;
  }
  if (bits) {
    float* stg = sm_stage + threadIdx.x * ITEMS;
    if (!sval) {
#pragma unroll
      for (int q = 0; q < ITEMS / 4; ++q)
        reinterpret_cast<float4*>(stg)[q] = make_float4(val[4 * q], val[4 * q + 1], val[4 * q + 2], val[4 * q + 3]);
    }
    do {
      const int i = __ffs(bits) - 1;
      bits &= bits - 1;
      const int v = item_v<VEC>(v0, i);
      const int pos = atomicAdd(&sm_n, 1);
      if (pos < CAND_CAP) sm_cand[pos] = row_key(sval ? sval[v - v0] : stg[i], v);
    } while (bits);
  }
  __syncthreads();
  const size_t o = (size_t)row * a.chunks + c;
  uint64_t* ctop = a.chunk_top + o * a.b;
  const int n_cand = sm_n;
  if (n_cand <= 32) {  // common case: one warp ranks the candidates (unique keys) by
    // counting larger ones with broadcast shared-memory reads -- no dependent shuffle chain
    if (w == 0) {
      const uint64_t key = lane < n_cand ? sm_cand[lane] : 0ull;
      int rank = 0;
      for (int j = 0; j < n_cand; ++j) rank += sm_cand[j] > key ? 1 : 0;
      if (lane < n_cand && rank < k) ctop[rank] = key;
      if (lane >= n_cand && lane < k) ctop[lane] = 0ull;  // fewer than k candidates
    }
  } else if (n_cand <= CAND_CAP) {
    block_rank_topk(sm_cand, n_cand, k, ctop);
  } else {  // ties overflowed the buffer: warp arg-max rounds over the registers
    // k rounds of warp arg-max; keys are rebuilt from val[] (a taken-bit per item)
    uint32_t taken = 0u;
    for (int q = 0; q < k; ++q) {
      uint64_t best = 0ull;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int v = item_v<VEC>(v0, i);
        const uint64_t key = (v < V && !((taken >> i) & 1u)) ? row_key(val[i], v) : 0ull;
        best = key > best ? key : best;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const uint64_t y = shfl_xor_u64(best, off);
        best = y > best ? y : best;
      }
      if (lane == 0) sm_wtop[w][q] = best;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (best != 0ull && item_v<VEC>(v0, i) < V && row_key(val[i], item_v<VEC>(v0, i)) == best)
          taken |= 1u << i;
    }
    __syncthreads();
    if (w == 0) {
      uint64_t kk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = i * 32 + lane;
        const int ww = idx / TRIE_MAX_BEAMS, pos = idx % TRIE_MAX_BEAMS;
        kk[i] = (ww < BS / 32 && pos < k) ? sm_wtop[ww][pos] : 0ull;
      }
      warp_topk<8>(kk, k, ctop);
    }
  }
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int i = 0; i < BS / 32; ++i) tot += sm_sum[i];
    a.chunk_max[o] = m;
    a.chunk_sum[o] = tot;
  }
  // ---- ticket: the last chunk CTA of this row continues --------------------------------
  __syncthreads();
  if (threadIdx.x == 0)  // release: the CTA's writes (ordered by the barrier) before the ticket
    sm_last = ticket_acq_rel(&a.cnt_row[row]) == (unsigned)(a.chunks - 1);
  __syncthreads();
  if (!sm_last) return;
  if (threadIdx.x == 0) a.cnt_row[row] = 0u;

  // ---- row stage: lse and the row's top-b ------------------------------------------------
  const size_t rowi = (size_t)row * a.chunks;
  if (w == 0) {
    float M = -INFINITY;
    for (int cc = lane; cc < a.chunks; cc += 32) M = fmaxf(M, __ldcg(a.chunk_max + rowi + cc));
    M = warp_max(M);
    float S = 0.f;
    for (int cc = lane; cc < a.chunks; cc += 32)
      S += __ldcg(a.chunk_sum + rowi + cc) * expf(__ldcg(a.chunk_max + rowi + cc) - M);
    S = warp_sum(S);
    if (lane == 0) a.row_lse[r * TRIE_MAX_BEAMS + j_row] = M + logf(S);
  }
  // the chunk lists (sorted descending, zero padded) merged: each warp folds chunks
  // w, w + 8, ... into a running top-32, then a 3-level tree over the warps
  // (up to RANK_MAX keys: staged in shared memory and ranked by counting, one key per
  // thread, instead of the 3-level merge tree's dependent shuffle / barrier chain; r2s5:
  // Phi 18.2 -> 17.4 us, but 256 / 512 keys (b = 16 / 32) are slower than the tree)
  const uint64_t* lists = a.chunk_top + rowi * a.b;
  if (a.chunks * k <= RANK_MAX) {
    const int n = a.chunks * k;
    for (int i = threadIdx.x; i < n; i += BS) sm_cand[i] = __ldcg(lists + (size_t)(i / k) * a.b + i % k);
    __syncthreads();
    block_rank_topk(sm_cand, n, k, sm_mrg[0]);
  } else {
    uint64_t acc = 0ull;
    for (int cc = w; cc < a.chunks; cc += BS / 32) {
      const uint64_t x = lane < k ? __ldcg(lists + (size_t)cc * a.b + lane) : 0ull;
      acc = warp_merge_top32(acc, x);
    }
    block_merge_tree(acc, sm_mrg);
  }
  uint64_t* rtop = a.row_top + ((size_t)r * TRIE_MAX_BEAMS + j_row) * TRIE_MAX_BEAMS;
  if (threadIdx.x < k) rtop[threadIdx.x] = sm_mrg[0][threadIdx.x];
  // ---- ticket: the last row CTA of this request continues --------------------------------
  __syncthreads();
  if (threadIdx.x == 0) sm_last = ticket_acq_rel(&a.cnt_req[r]) == (unsigned)(a.b_live - 1);
  __syncthreads();
  if (!sm_last) return;
  if (threadIdx.x == 0) a.cnt_req[r] = 0u;

  // ---- request stage: global top-b over b_live x k survivors ------------------------------
  const int b_live = a.b_live;
  if (a.eos >= 0 && b_live == a.b) {  // NEXT-3: every beam finished -> the request is done:
    // identity selection (each beam keeps its EOS-terminated hypothesis and score), no append
    __shared__ int sm_done;
    if (threadIdx.x == 0) {
      int all = 1;
      for (int j = 0; j < b_live; ++j) all &= a.fin[r * TRIE_MAX_BEAMS + j] != 0u;
      sm_done = all;
    }
    __syncthreads();
    if (sm_done) {
      if (threadIdx.x < a.b) {
        const int q = threadIdx.x, o2 = r * a.b + q;
        const float scq = a.score[r * TRIE_MAX_BEAMS + q];
        a.sel_par[o2] = q; a.sel_tok[o2] = a.eos; a.sel_sc[o2] = scq;
        if (a.out_par) a.out_par[o2] = q;
        if (a.out_tok) a.out_tok[o2] = a.eos;
        if (a.out_sc) a.out_sc[o2] = scq;
      }
      return;
    }
  }
  if (threadIdx.x < b_live) sm_lse[threadIdx.x] = __ldcg(a.row_lse + r * TRIE_MAX_BEAMS + threadIdx.x);
  __syncthreads();
  // each warp takes rows w, w + 8, ...: lane = position in the row's list.  The row list
  // is in (x desc, v asc) order, which is (cs desc) order up to fp32 ties of cs; re-sort
  // only if a tie left it out of global-key order, then merge (as in the row stage)
  if (b_live * k <= RANK_MAX) {  // all b_live x k global keys ranked by counting (as above)
    const int n = b_live * k;
    for (int i = threadIdx.x; i < n; i += BS) {
      const int j = i / k;
      uint64_t gk = 0ull;
      const uint64_t rk = __ldcg(a.row_top + ((size_t)r * TRIE_MAX_BEAMS + j) * TRIE_MAX_BEAMS + i % k);
      if (rk != 0ull) {
        const float xv = ord2f((uint32_t)(rk >> 32));
        const uint32_t v = ~(uint32_t)rk;
        const float cs = a.score[r * TRIE_MAX_BEAMS + j] + (xv - sm_lse[j]);
        gk = ((uint64_t)f2ord(cs) << 32) | (uint32_t)(~(v * (uint32_t)b_live + j));
      }
      sm_cand[i] = gk;
    }
    __syncthreads();
    block_rank_topk(sm_cand, n, k, sm_mrg[0]);
  } else {
    uint64_t acc = 0ull;
    for (int j = w; j < b_live; j += BS / 32) {
      uint64_t gk = 0ull;
      if (lane < k) {
        const uint64_t rk = __ldcg(a.row_top + ((size_t)r * TRIE_MAX_BEAMS + j) * TRIE_MAX_BEAMS + lane);
        if (rk != 0ull) {
          const float xv = ord2f((uint32_t)(rk >> 32));
          const uint32_t v = ~(uint32_t)rk;
          const float cs = a.score[r * TRIE_MAX_BEAMS + j] + (xv - sm_lse[j]);
          gk = ((uint64_t)f2ord(cs) << 32) | (uint32_t)(~(v * (uint32_t)b_live + j));
        }
      }
      const uint64_t nxt = shfl_u64(gk, (lane + 1) & 31);
      if (!__all_sync(0xffffffffu, lane == 31 || gk >= nxt)) gk = warp_sort_desc_u64(gk);
      acc = warp_merge_top32(acc, gk);
    }
    block_merge_tree(acc, sm_mrg);
  }
  const uint64_t* sel = sm_mrg[0];
  if (threadIdx.x < a.b) {
    const uint64_t kk = sel[threadIdx.x];
    const uint32_t id = ~(uint32_t)kk;
    const int q = threadIdx.x;
    sp[q] = (int)(id % (uint32_t)b_live);
    st[q] = (int)(id / (uint32_t)b_live);
    ss[q] = ord2f((uint32_t)(kk >> 32));
    const int o2 = r * a.b + q;
    a.sel_par[o2] = sp[q]; a.sel_tok[o2] = st[q]; a.sel_sc[o2] = ss[q];
    if (a.out_par) a.out_par[o2] = sp[q];
    if (a.out_tok) a.out_tok[o2] = st[q];
    if (a.out_sc) a.out_sc[o2] = ss[q];
  }
  __syncthreads();
  append_sel(r, a.b, b_live, sp, st, ss, a.token, a.parent, a.depth, a.mask, a.leaf, a.score,
             a.nn, a.nkv, a.tlen, a.cap, a.status, a.fin, a.eos, a.pg);
}

// Register-path kernel: grid (chunks, rows), one item per CTA (any V; the TMA kernel
// below needs V % 4 == 0 and 16-byte aligned rows).
template <bool VEC>
#ifndef TRIE_BEAM_MINB
#define TRIE_BEAM_MINB 4  // CTAs per SM the register budget is sized for (64 regs, small spill):
                          // r64 microbench, Llama shape: 4 -> 41.2 us, 3 -> 47.5, 2 -> 62.4
#endif
__global__ void __launch_bounds__(BS, TRIE_BEAM_MINB) k_beam_step(const BeamStepArgs a) {
  pdl_trigger();
  pdl_wait();
  const int c = blockIdx.x, row = blockIdx.y;
  const int V = a.V, v0 = c * CHUNK;
  const float* x = a.logits + (size_t)row * V;
  float val[ITEMS];
  const bool finrow = a.eos >= 0 && a.fin[(row / a.b_live) * TRIE_MAX_BEAMS + row % a.b_live] != 0u;
  if (finrow) {  // one-hot at eos (log-prob 0): no logits are read
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) val[i] = item_v<VEC>(v0, i) == a.eos ? 0.f : -INFINITY;
  } else if (VEC) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int q = 0; q < ITEMS / 4; ++q) {
      const int e = item_v<true>(v0, 4 * q);
      float4 f = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (e < V) f = __ldcs(x4 + (e >> 2));  // V % 4 == 0: all four valid
      val[4 * q + 0] = f.x; val[4 * q + 1] = f.y; val[4 * q + 2] = f.z; val[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = item_v<false>(v0, i);
      val[i] = e < V ? __ldcs(x + e) : -INFINITY;
    }
  }
  beam_item<VEC>(a, row, c, val, nullptr, finrow);
}

int launch_beam_step(trie_handle* h, const float* logits, int32_t* out_par, int32_t* out_tok,
                     float* out_sc, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  BeamStepArgs a;
  a.logits = logits;
  a.V = c.vocab;
  a.b_live = h->b_live;
  a.b = c.beam_width;
  a.chunks = (c.vocab + CHUNK - 1) / CHUNK;
  const bool vec = (c.vocab % 4 == 0) && ((uintptr_t)logits % 16 == 0);
  a.chunk_max = h->chunk_max;
  a.chunk_sum = h->chunk_sum;
  a.chunk_top = h->chunk_top;
  a.row_lse = h->row_lse;
  a.row_top = h->row_top;
  a.cnt_row = h->cnt_row;
  a.cnt_req = h->cnt_req;
  a.token = h->token; a.parent = h->parent; a.depth = h->depth; a.mask = h->mask;
  a.leaf = h->leaf; a.score = h->score; a.nn = h->n_nodes; a.nkv = h->n_kv; a.tlen = h->tlen;
  a.cap = c.capacity;
  a.status = h->status;
  a.sel_par = h->sel_parent; a.sel_tok = h->sel_token; a.sel_sc = h->sel_score;
  a.out_par = out_par; a.out_tok = out_tok; a.out_sc = out_sc;
  a.eos = h->eos;
  a.fin = h->fin;
  a.pg = page_args(h);
  dim3 grid(a.chunks, c.n_requests * h->b_live);
  if (vec)
    launch_k(k_beam_step<true>, grid, dim3(BS), 0, s, a);
  else
    launch_k(k_beam_step<false>, grid, dim3(BS), 0, s, a);
  return trie_check_launch("k_beam_step");
}

int launch_append(trie_handle* h, const int32_t* par, const int32_t* tok, const float* sc,
                  cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  k_append<<<c.n_requests, 256, 0, s>>>(par, tok, sc, c.beam_width, h->b_live, h->token,
                                        h->parent, h->depth, h->mask, h->leaf, h->score,
                                        h->n_nodes, h->n_kv, h->tlen, c.capacity, h->status, h->fin,
                                        h->eos, page_args(h));
  return trie_check_launch("k_append");
}

}  // namespace trie
