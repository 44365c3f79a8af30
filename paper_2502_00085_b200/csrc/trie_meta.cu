// Trie metadata kernels: initialize_trie (Alg. 2 l.1), garbage collection (§3.5:
// marking / pruning / compaction), hypothesis read-out (Alg. 2 l.14) and the
// Alg. 3 parent walk that derives beam bitsets when the caller passes no beam_mask.
#include <stdio.h>

#include "common.cuh"
#include "handle.h"

namespace trie {

// exclusive block scan of one int per thread; returns prefix, writes block total
template <int BS>
__device__ __forceinline__ int block_excl_scan(int v, int* total, int* sm_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < BS / 32 ? sm_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < BS / 32) sm_warp[lane] = s;  // inclusive warp-total prefix
  }
  __syncthreads();
  int before = (w > 0 ? sm_warp[w - 1] : 0) + x - v;
  *total = sm_warp[BS / 32 - 1];
  __syncthreads();
  return before;
}

// ---- Alg. 2 l.1 initialize_trie(prompt) --------------------------------------------------
// Paged pools (NEXT-2): request r's prompt keeps its fixed pages page_base[r] + i; every
// other page goes into the free queue (pages prompt_pages .. n_pages - 1, in order); the
// counters restart (pops 0, pushes 0, peak = the prompt pages).

__global__ void k_init(int32_t* token, int32_t* parent, int32_t* depth, uint32_t* mask,
                       int32_t* leaf, float* score, int32_t* nn, int32_t* nkv,
                       const int32_t* tlen, const int32_t* prompts, int t_max, int cap,
                       uint32_t* fin, PageArgs pg) {
  const int r = blockIdx.x;
  const int t = tlen[r];
  const size_t base = (size_t)r * cap;
  if (pg.n_pages > 0) {
    const int np = (t + 63) / 64, stride = cap / 64;
    for (int i = threadIdx.x; i < stride; i += blockDim.x) pg.pt[r * stride + i] = i < np ? pg.base[r] + i : -1;
    if (threadIdx.x == 0) pg.used[r] = np;
    const int nfree = pg.n_pages - pg.prompt_pages;
    for (int i = r * blockDim.x + threadIdx.x; i < nfree; i += gridDim.x * blockDim.x)
      pg.fq[i] = pg.prompt_pages + i;
    if (r == 0 && threadIdx.x == 0) {
      pg.ctr[0] = 0u;
      pg.ctr[1] = 0u;
      pg.ctr[2] = max(pg.ctr[2], (uint32_t)pg.prompt_pages);  // peak since trie_create
      pg.ctr[3] = (uint32_t)pg.n_pages;
    }
  }
  for (int i = threadIdx.x; i < t; i += blockDim.x) {
    token[base + i] = prompts[(size_t)r * t_max + i];
    parent[base + i] = i - 1;
    depth[base + i] = i;  // §3.4: position of the conventional sequence
    mask[base + i] = 0u;  // prompt columns are implicitly allowed for every beam
  }
  if (threadIdx.x < TRIE_MAX_BEAMS) fin[r * TRIE_MAX_BEAMS + threadIdx.x] = 0u;  // no beam finished
  if (threadIdx.x == 0) {
    leaf[r * TRIE_MAX_BEAMS] = t - 1;
    score[r * TRIE_MAX_BEAMS] = 0.f;
    nn[r] = t;
    nkv[r] = t;  // the prompt's K/V come from the caller's prefill
  }
}


int launch_init(trie_handle* h, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  k_init<<<c.n_requests, 256, 0, s>>>(h->token, h->parent, h->depth, h->mask, h->leaf, h->score,
                                      h->n_nodes, h->n_kv, h->tlen, h->prompts,
                                      c.max_prompt_len, c.capacity, h->fin, page_args(h));
  return trie_check_launch("k_init");
}

// ---- §3.5 GC: keep-scan + stable metadata compaction + move list ----------------------
// One CTA per request.  keep[n] = n < t or beam_mask[n] != 0 (n is an ancestor-or-self
// of a live leaf: the bits are exactly Alg. 3's rows, see beam_step.cu).  new[n] =
// exclusive prefix sum of keep.  In-place compaction moves every kept row to a lower or
// equal slot; processing rows in ascending batches, each batch read-all -> barrier ->
// write-all, is race free (a write target new[n] <= n never belongs to a later batch).
constexpr int PRUNE_BS = 512;
__global__ void __launch_bounds__(PRUNE_BS) k_prune_scan(
    int32_t* token, int32_t* parent, int32_t* depth, uint32_t* mask, int32_t* leaf,
    int32_t* nn, const int32_t* nkv, const int32_t* tlen, int32_t* newidx, int32_t* moves,
    int32_t* moves_dst, int32_t* n_moves, int b_live, int cap, uint32_t* status) {
  __shared__ int sm_warp[32];
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int N = nn[r], t = tlen[r], n_kv = nkv[r];
  const size_t base = (size_t)r * cap;
  int32_t* nidx = newidx + base;
  // pass 1: scan
  int carry = t;
  for (int b0 = t; b0 < N; b0 += PRUNE_BS) {
    const int n = b0 + threadIdx.x;
    const int keep = (n < N && mask[base + n] != 0u) ? 1 : 0;
    int tot;
    const int pre = block_excl_scan<PRUNE_BS>(keep, &tot, sm_warp);
    if (n < N) nidx[n] = keep ? carry + pre : -1;
    carry += tot;
  }
  const int N_new = carry;
  __syncthreads();
  // pass 2: compaction in ascending batches + ordered move list
  int mcarry = 0;
  for (int b0 = t; b0 < N; b0 += PRUNE_BS) {
    const int n = b0 + threadIdx.x;
    int dst = -1, tok = 0, par = 0, dep = 0;
    uint32_t msk = 0;
    if (n < N) {
      dst = nidx[n];
      if (dst >= 0) {
        tok = token[base + n];
        const int p = parent[base + n];
        dep = depth[base + n];
        msk = mask[base + n];
        if (p < 0 || p >= n) {
          latch(status, TRIE_ST_PARENT);
          par = -1;
        } else {
          par = p < t ? p : nidx[p];
          if (par < 0) latch(status, TRIE_ST_PARENT);  // kept node with a dropped parent
        }
      }
    }
    const int mv = (dst >= 0 && dst != n && n < n_kv) ? 1 : 0;
    int mtot;
    const int mpre = block_excl_scan<PRUNE_BS>(mv, &mtot, sm_warp);  // contains barriers
    if (dst >= 0) {
      token[base + dst] = tok;
      parent[base + dst] = par;
      depth[base + dst] = dep;
      mask[base + dst] = msk;
    }
    if (mv) {
      moves[base + mcarry + mpre] = n;
      moves_dst[base + mcarry + mpre] = dst;
    }
    mcarry += mtot;
    __syncthreads();
  }
  if (threadIdx.x < b_live) {
    const int l = leaf[r * TRIE_MAX_BEAMS + threadIdx.x];
    const int nl = (l >= 0 && l < N) ? (l < t ? l : nidx[l]) : -1;
    if (nl < 0) latch(status, TRIE_ST_LEAF);
    leaf[r * TRIE_MAX_BEAMS + threadIdx.x] = nl < 0 ? 0 : nl;
  }
  if (threadIdx.x == 0) {
    nn[r] = N_new;
    n_moves[r] = mcarry;
  }
}

// ---- §3.5 Compaction of the KV cache (the paper's index_select) -----------------
// One CTA per (request, layer, group of hg KV heads): the K and V rows of the moved slots
// of those heads (regions no other CTA touches), 16-byte vectors, (source, destination)
// pairs written by k_prune_scan.  hg keeps the grid near 2048 CTAs of 256 threads (r61:
// one head per CTA cut Llama's GC 40 -> 25 us per step but made Phi's 32-head launch of
// 65k CTAs slower, 44 -> 78 us).  Moves are applied in ascending
// batches (read-all, barrier, write-all) for the same in-place safety argument as above;
// a few moved rows per request (r08 ncu: ~9 on Llama) fit one batch.
struct PoolPtrs {
  void* k[TRIE_MAX_LAYERS];
  void* v[TRIE_MAX_LAYERS];
};

constexpr int COMPACT_BS = 256;
constexpr int COMPACT_VEC = 8;   // 16-byte vectors in flight per thread per batch
constexpr int COMPACT_MV = 512;  // (source, destination) pairs staged in shared memory per pass
// The request's move list is staged in shared memory once per CTA (one coalesced read per
// COMPACT_MV pairs), so a batch is ONE dependent global load deep (the K/V vectors) before
// its stores, with up to 256 x 8 x 16 B = 32 KB in flight per CTA.
__global__ void __launch_bounds__(COMPACT_BS) k_kv_compact(const __grid_constant__ PoolPtrs pp,
                                                           const int32_t* moves,
                                                           const int32_t* moves_dst,
                                                           const int32_t* n_moves, int Hkv,
                                                           int hg, int row_bytes, int cap,
                                                           const int32_t* __restrict__ pt) {
  __shared__ int sm_src[COMPACT_MV], sm_dst[COMPACT_MV];
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, layer = blockIdx.y, h0 = blockIdx.z * hg;
  const int nm = n_moves[r];
  if (nm == 0) return;
  const int nh = min(hg, Hkv - h0);
  const size_t base = (size_t)r * cap;
  const int vpr = row_bytes / 16;  // 16-byte vectors per (head, slot) row
  const size_t hoff = ((size_t)r * Hkv + h0) * cap * row_bytes;
  const size_t hstride = (size_t)cap * row_bytes;
  char* kb = (char*)pp.k[layer] + hoff;
  char* vb = (char*)pp.v[layer] + hoff;
  const int* ptr = pt ? pt + r * (cap / 64) : nullptr;
  const int per_slot = 2 * nh * vpr;
  for (int m0 = 0; m0 < nm; m0 += COMPACT_MV) {
    const int cnt = min(COMPACT_MV, nm - m0);
    __syncthreads();  // the previous pass's reads of sm_src / sm_dst are done
    for (int i = threadIdx.x; i < cnt; i += COMPACT_BS) {
      sm_src[i] = moves[base + m0 + i];
      sm_dst[i] = moves_dst[base + m0 + i];
    }
    __syncthreads();
    const int total = cnt * per_slot;
    for (int b0 = 0; b0 < total; b0 += COMPACT_BS * COMPACT_VEC) {
      int4 val[COMPACT_VEC];
      char* dstp[COMPACT_VEC];
#pragma unroll
      for (int u = 0; u < COMPACT_VEC; ++u) {
        const int e = b0 + u * COMPACT_BS + threadIdx.x;
        dstp[u] = nullptr;
        if (e < total) {
          const int mi = e / per_slot;
          int rem = e - mi * per_slot;
          const int kv = rem / (nh * vpr);
          rem -= kv * nh * vpr;
          const int hh = rem / vpr, c = rem - hh * vpr;
          const int src = sm_src[mi], dst = sm_dst[mi];
          if (ptr) {  // paged pools (NEXT-2): rows (page * Hkv + h) * 64 + slot % 64
            char* pool = (char*)(kv ? pp.v[layer] : pp.k[layer]);
            const size_t rs = ((size_t)ptr[src >> 6] * Hkv + h0 + hh) * 64 + (src & 63);
            const size_t rd = ((size_t)ptr[dst >> 6] * Hkv + h0 + hh) * 64 + (dst & 63);
            val[u] = *(const int4*)(pool + rs * row_bytes + (size_t)c * 16);
            dstp[u] = pool + rd * row_bytes + (size_t)c * 16;
            continue;
          }
          char* pool = (kv ? vb : kb) + (size_t)hh * hstride;
          val[u] = *(const int4*)(pool + (size_t)src * row_bytes + (size_t)c * 16);
          dstp[u] = pool + (size_t)dst * row_bytes + (size_t)c * 16;
        }
      }
      __syncthreads();  // in-place safety: every read of the batch before any write
#pragma unroll
      for (int u = 0; u < COMPACT_VEC; ++u)
        if (dstp[u]) *(int4*)dstp[u] = val[u];
      __syncthreads();
    }
  }
}

// Paged pools (NEXT-2): after the compaction's K/V moves, the pages above each request's
// new N go back to the free queue (a separate launch: the moves read those pages).
__global__ void k_page_release(PageArgs pg, const int32_t* nn, int R, int cap) {
  pdl_trigger();
  pdl_wait();
  const int stride = cap / 64;
  const uint32_t nfree0 = (uint32_t)(pg.n_pages - pg.prompt_pages);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const int keep = (nn[r] + 63) / 64, used = pg.used[r];
    for (int i = keep; i < used; ++i) {
      const uint32_t k = atomicAdd(&pg.ctr[1], 1u);
      pg.fq[(nfree0 + k) % (uint32_t)pg.n_pages] = pg.pt[r * stride + i];
      pg.pt[r * stride + i] = -1;
    }
    if (used > keep) pg.used[r] = keep;
  }
}

// SURVEY §8(f) NEXT-3, SWA eviction (paged pools, window W > 0): every 64-slot block of
// request r made only of prompt rows below min over the live leaves of
// (depth[leaf] - W + 1) is outside every beam's window (reading R14) for the rest of the
// job -- leaf depths only grow -- so its page goes back to the free queue.  The attention
// kernels start at the window's first slot and never read such a block; prompt rows never
// move (GC compacts generated rows only), so no later compaction touches it.
__global__ void k_swa_evict(PageArgs pg, const int32_t* depth, const int32_t* leaf,
                            const int32_t* tlen, int b_live, int window, int cap) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, lane = threadIdx.x;
  const size_t base = (size_t)r * cap;
  const int lo = lane < b_live ? depth[base + leaf[r * TRIE_MAX_BEAMS + lane]] - window + 1 : INT_MAX;
  const int lo_dep = __reduce_min_sync(0xffffffffu, lo);
  if (lane != 0) return;
  const int t = tlen[r], stride = cap / 64;
  const int nblk = min(lo_dep, t) / 64;  // prompt rows have depth == slot (Alg. 2 l.1)
  const uint32_t nfree0 = (uint32_t)(pg.n_pages - pg.prompt_pages);
  for (int i = 0; i < nblk; ++i) {
    const int pgid = pg.pt[r * stride + i];
    if (pgid < 0) continue;  // evicted by an earlier step
    const uint32_t k = atomicAdd(&pg.ctr[1], 1u);
    pg.fq[(nfree0 + k) % (uint32_t)pg.n_pages] = pgid;
    pg.pt[r * stride + i] = -1;
  }
}

int launch_swa_evict(trie_handle* h, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  launch_k(k_swa_evict, dim3(c.n_requests), dim3(32), 0, s, page_args(h), (const int32_t*)h->depth,
           (const int32_t*)h->leaf, (const int32_t*)h->tlen, h->b_live, c.window, c.capacity);
  return trie_check_launch("k_swa_evict");
}

int launch_prune(trie_handle* h, void* const* kp, void* const* vp, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  launch_k(k_prune_scan, dim3(c.n_requests), dim3(PRUNE_BS), 0, s, h->token, h->parent, h->depth,
           h->mask, h->leaf, h->n_nodes, (const int32_t*)h->n_kv, (const int32_t*)h->tlen, h->newidx,
           h->moves, h->moves_dst, h->n_moves, h->b_live, c.capacity, h->status);
  int rc = trie_check_launch("k_prune_scan");
  if (rc) return rc;
  auto release = [&]() -> int {
    if (c.n_pages <= 0) return TRIE_OK;
    launch_k(k_page_release, dim3((c.n_requests + 127) / 128), dim3(128), 0, s, page_args(h),
             (const int32_t*)h->n_nodes, c.n_requests, c.capacity);
    return trie_check_launch("k_page_release");
  };
  if (c.n_layers == 0 || kp == nullptr) return release();
  PoolPtrs pp;
  for (int l = 0; l < c.n_layers; ++l) {
    pp.k[l] = kp[l];
    pp.v[l] = vp[l];
  }
  const int esz = c.kv_dtype == TRIE_BF16 ? 2 : 4;
  const long units = (long)c.n_requests * c.n_layers * c.n_kv_heads;
  int hg = (int)((units + 2047) / 2048);
  if (hg > c.n_kv_heads) hg = c.n_kv_heads;
  if (hg < 1) hg = 1;
  dim3 grid(c.n_requests, c.n_layers, (c.n_kv_heads + hg - 1) / hg);
  launch_k(k_kv_compact, grid, dim3(COMPACT_BS), 0, s, pp, (const int32_t*)h->moves,
           (const int32_t*)h->moves_dst, (const int32_t*)h->n_moves, c.n_kv_heads, hg,
           c.head_dim * esz, c.capacity, (const int32_t*)h->page_table);
  rc = trie_check_launch("k_kv_compact");
  if (rc) return rc;
  return release();
}

// ---- Alg. 2 l.14: hypotheses = root-to-leaf token paths ---------------------------------
__global__ void k_read_hyps(const int32_t* token, const int32_t* parent, const int32_t* depth,
                            const int32_t* leaf, int b_live, int cap, int max_len,
                            int32_t* out) {
  const int r = blockIdx.x, j = threadIdx.x;
  if (j >= b_live) return;
  int32_t* o = out + ((size_t)r * b_live + j) * (max_len + 1);
  const size_t base = (size_t)r * cap;
  int n = leaf[r * TRIE_MAX_BEAMS + j];
  const int len = depth[base + n] + 1;
  o[0] = len;
  for (int i = 0; i < max_len; ++i) o[1 + i] = -1;
  int guard = 0;
  while (n >= 0 && guard++ < cap) {
    const int d = depth[base + n];
    if (d < max_len) o[1 + d] = token[base + n];
    n = parent[base + n];
  }
}

int launch_read_hyps(trie_handle* h, int32_t max_len, int32_t* out_dev, cudaStream_t s) {
  k_read_hyps<<<h->cfg.n_requests, 32, 0, s>>>(h->token, h->parent, h->depth, h->leaf,
                                                h->b_live, h->cfg.capacity, max_len, out_dev);
  return trie_check_launch("k_read_hyps");
}

// ---- Alg. 3 as per-leaf walks (used when trie_attn_decode gets beam_mask == NULL) -------
// Reading R19: the b simultaneous walkers of Alg. 3 give the same set as independent
// per-leaf walks.  Bit j of word n is set iff generated node n lies on leaf j's path.
__global__ void k_mask_walk(const int32_t* tlen, const int32_t* parent, const int32_t* leaf,
                            const int32_t* nn, int b_live, int cap, uint32_t* mask_out,
                            uint32_t* status) {
  const int r = blockIdx.x;
  const int t = tlen[r], N = nn[r];
  const size_t base = (size_t)r * cap;
  for (int n = threadIdx.x; n < N; n += blockDim.x) mask_out[base + n] = 0u;
  __syncthreads();
  const int j = threadIdx.x;
  if (j < b_live) {
    int n = leaf[r * TRIE_MAX_BEAMS + j];
    if (n < 0 || n >= N) {
      latch(status, TRIE_ST_LEAF);
      return;
    }
    int guard = 0;
    while (n >= t) {
      atomicOr(&mask_out[base + n], 1u << j);
      const int p = parent[base + n];
      if (p >= n || p < 0 || ++guard > N) {
        latch(status, TRIE_ST_PARENT);
        break;
      }
      n = p;
    }
  }
}

int launch_mask_walk(const trie_cfg* c, int32_t b_live, const int32_t* tlen,
                     const int32_t* parent, const int32_t* leaf, const int32_t* nn,
                     uint32_t* mask_out, uint32_t* status, cudaStream_t s) {
  k_mask_walk<<<c->n_requests, 256, 0, s>>>(tlen, parent, leaf, nn, b_live, c->capacity,
                                            mask_out, status);
  return trie_check_launch("k_mask_walk");
}

}  // namespace trie
