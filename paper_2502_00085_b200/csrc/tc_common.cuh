// Shared device helpers of the tensor-core trie attention kernels (sm_100a): PTX wrappers
// for mbarrier / TMA / bulk copies / ldmatrix / movmatrix / mma.sync, the 64-byte swizzle
// address map of a TMA tile, the stage ring geometry, the per-item tile range.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <float.h>
#include <limits.h>

#include "attn_common.cuh"
#include "common.cuh"

namespace trie {

constexpr int TC_TR = 64;  // slots per tile

// TMA maps of a layer's pool ([rows][D] bf16, 64-byte swizzle, 32-column boxes of box_rows
// rows), encoded once per (base, rows, D, box rows) -- attn_decode_tc.cu
int cached_tensor_map(CUtensorMap* out, const void* base, int D, long rows, int box_rows = TC_TR);
constexpr int TC_CW = 32;  // elements per swizzle box column (64 bytes, SWIZZLE_64B)

// ---- PTX helpers -------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load_1d(uint32_t dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                        uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                          uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 2^x by one MUFU.EX2 (ex2.approx.ftz: ~2 ulp, 2^-inf = +0, results below 2^-126 flushed to
// zero -- softmax weights that small are below bf16 P's resolution anyway); exp2f adds a
// denormal range fix-up (compare + two predicated multiplies) around the same MUFU
__device__ __forceinline__ float ex2_ftz(float x) {
#ifdef TRIE_EXP2_PRECISE  // A/B builds only: the libdevice exp2f
  return exp2f(x);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(uint32_t*)&v;
}

// byte offset of (row, col) inside one tile: D/32 boxes of [TR rows][32 cols], 64B swizzle
// (CUTLASS Swizzle<2,4,3>: address bits [4,5] ^= bits [7,8]; boxes are 1024-B aligned)
__device__ __forceinline__ uint32_t tile_off(int row, int col) {
  const int box = col / TC_CW;
  const uint32_t o = (uint32_t)row * 64u + (uint32_t)(col % TC_CW) * 2u;
  return (uint32_t)box * (TC_TR * 64u) + (o ^ (((o >> 7) & 3u) << 4));
}

template <int D, int STAGES_>
struct Ring {
  static constexpr int STAGES = STAGES_;
  static constexpr int TILE_BYTES = TC_TR * D * 2;
  // stage = K tile | V tile | mask words | depth words, 1024-byte aligned (swizzle atoms)
  static constexpr int STAGE_BYTES = (2 * TILE_BYTES + 2 * TC_TR * 4 + 1023) / 1024 * 1024;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
};

struct ItemInfo {
  int tile0, ntiles, lo, N, t, fast_from;
  int done;  // NEXT-3: every beam of the request finished (no tiles, no output)
};

// Whole warp 0 (lane 0 writes *info): tile range of this (r, split) and the first tile
// index from which the mask is needed (tiles below it are prompt-only and inside every
// beam's window).  Few dependent global loads: the leaves' depths in parallel (one per
// lane), then the window's first slot.  That slot is the first n with depth[n] >= lo_dep
// (depth is non-decreasing in slot order, invariant 1); on the prompt chain depth[n] = n
// (Alg. 2 l.1), so lo_dep itself is probed first and a 32-ary search only runs if the
// probe fails (lo_dep beyond the prompt or a non-standard trie).
__device__ __forceinline__ void item_setup(const AttnParams& p, int r, int split, ItemInfo* info) {
  const int lane = threadIdx.x & 31;
  const size_t mbase = (size_t)r * p.cap;
  const int N = p.nn[r], t = p.tlen[r];
  int lo = 0, lo_dep_max = INT_MIN;
  if (p.window > 0) {
    int dl = INT_MAX, dh = INT_MIN;
    if (lane < p.b_live) {
      dl = dh = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + lane]] - p.window + 1;
    }
    const int lo_dep = __reduce_min_sync(0xffffffffu, dl);
    lo_dep_max = __reduce_max_sync(0xffffffffu, dh);
    if (lo_dep > 0) {
      bool found = false;
      if (lo_dep < N) {  // probe: depth[lo_dep - 1] < lo_dep <= depth[lo_dep]
        const int pr = lane < 2 ? p.depth[mbase + lo_dep - 1 + lane] : 0;
        const int d0 = __shfl_sync(0xffffffffu, pr, 0), d1 = __shfl_sync(0xffffffffu, pr, 1);
        found = d0 < lo_dep && d1 >= lo_dep;
        lo = lo_dep;
      }
      if (!found) {  // answer in [a, b]: depth < lo_dep below a; b == N or depth[b] >= lo_dep
        int a = 0, b = N;
        while (a < b) {
          const int step = (b - a + 31) / 32;
          const int pos = a + lane * step;
          const bool ge = pos >= b || p.depth[mbase + pos] >= lo_dep;
          const int first = __ffs(__ballot_sync(0xffffffffu, ge)) - 1;
          const int nb = min(b, a + first * step);
          a = first == 0 ? a : a + (first - 1) * step + 1;
          b = nb;
        }
        lo = a;
      }
    }
  }
  const int first = lo / TC_TR;
  const int total = (N + TC_TR - 1) / TC_TR - first;
  const int per = (total + p.splits - 1) / p.splits;
  const int tb = min(total, split * per), te = min(total, (split + 1) * per);
  // NEXT-3: a request whose live beams have all finished (EOS) is done -- skip it
  const bool done = p.fin != nullptr &&
                    __all_sync(0xffffffffu, lane >= p.b_live || p.fin[r * TRIE_MAX_BEAMS + lane] != 0u);
  if (lane == 0) {
    info->done = done ? 1 : 0;
    info->tile0 = first + tb;
    info->ntiles = done ? 0 : te - tb;
    info->lo = lo;
    info->N = N;
    info->t = t;
    // unmasked tiles: every row n satisfies n < t (prompt: depth = n), n < N and
    // depth = n >= every beam's lower depth  <=>  tile in [ceil(lo_dep_max / TR), t / TR)
    info->fast_from = p.window > 0 ? (max(lo_dep_max, 0) + TC_TR - 1) / TC_TR : 0;
  }
}

// Fused a-1 (trie_attn_decode_rope): lanes 1..31 of the producer warp append the leaves
// whose slots lie in [slot_lo, slot_hi) -- K rotated at the beam's depth with the step's
// (cos, sin) table, V copied, 8-element chunks with all loads of an item issued together
// (write-before-read, §3.4 / Alg. 3 l.7) -- then fence the generic writes for the TMA
// (async proxy) reads of lane 0, which waits on app_done before the tile of the first leaf.
// The leaves are the last b_live slots (invariant 2 of the handle's trie: appends go to
// the end, compaction is stable), so leaf j's slot is first_leaf + j -- no load of leaf[].
// The append itself, by `nw` workers (worker index w): 16-byte chunks of the leaves' K (rotated)
// and V rows in [slot_lo, slot_hi).  The caller fences and signals (see below).
template <int D>
__device__ __forceinline__ void append_leaves_rope_work(const AttnParams& p, int r, int h,
                                                        int slot_lo, int slot_hi, int w, int nw,
                                                        int first_leaf) {
  constexpr int HALF = D / 2, CH = HALF / 8;
  static_assert(HALF % 8 == 0, "head_dim must be a multiple of 16");
  const __nv_bfloat16* __restrict__ kn = (const __nv_bfloat16*)p.k_new;
  const __nv_bfloat16* __restrict__ vn = (const __nv_bfloat16*)p.v_new;
  __nv_bfloat16* kpool = (__nv_bfloat16*)p.k;
  __nv_bfloat16* vpool = (__nv_bfloat16*)p.v;
  const int nk = p.b_live * CH, nv = p.b_live * (D / 8);
  for (int e = w; e < nk + nv; e += nw) {
    const int j = e < nk ? e / CH : (e - nk) / (D / 8);
    const int slot = first_leaf + j;
    if (slot < slot_lo || slot >= slot_hi) continue;
    const size_t rj = (size_t)r * p.b_live + j;
    __nv_bfloat16* dst = (e < nk ? kpool : vpool) + (size_t)attn_row(p, r, h, slot) * D;
    if (e < nk) {
      const int c = (e % CH) * 8;
      const __nv_bfloat16* src = kn + (rj * p.Hkv + h) * D;
      const int4 a = __ldg((const int4*)(src + c)), b = __ldg((const int4*)(src + HALF + c));
      const float4* tb = (const float4*)(p.rope_tab + rj * HALF + c);  // 8 (cos, sin) pairs
      float4 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = __ldg(tb + u);
      const __nv_bfloat162* a2 = (const __nv_bfloat162*)&a;
      const __nv_bfloat162* b2 = (const __nv_bfloat162*)&b;
      int4 y1, y2;
      __nv_bfloat162* o1 = (__nv_bfloat162*)&y1;
      __nv_bfloat162* o2 = (__nv_bfloat162*)&y2;
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // elements 2u, 2u + 1: table pairs t[u].(x,y), t[u].(z,w)
        const float2 x1 = __bfloat1622float2(a2[u]), x2 = __bfloat1622float2(b2[u]);
        o1[u] = __floats2bfloat162_rn(x1.x * t[u].x - x2.x * t[u].y, x1.y * t[u].z - x2.y * t[u].w);
        o2[u] = __floats2bfloat162_rn(x2.x * t[u].x + x1.x * t[u].y, x2.y * t[u].z + x1.y * t[u].w);
      }
      *(int4*)(dst + c) = y1;
      *(int4*)(dst + HALF + c) = y2;
    } else {
      const int d = ((e - nk) % (D / 8)) * 8;
      *(int4*)(dst + d) = __ldg((const int4*)(vn + (rj * p.Hkv + h) * D + d));
    }
  }
  // the generic-proxy writes must be visible to the TMA (async proxy) reads of the tile
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Lanes 1..31 of the producer warp append, then lane 1 arrives on app_done.
template <int D>
__device__ __forceinline__ void append_leaves_rope(const AttnParams& p, int r, int h, int slot_lo,
                                                   int slot_hi, int lane, uint64_t* app_done,
                                                   int first_leaf) {
  append_leaves_rope_work<D>(p, r, h, slot_lo, slot_hi, lane - 1, 31, first_leaf);
  __syncwarp(0xfffffffeu);
  if (lane == 1) mbar_arrive(app_done);
}

// Pre-wait prefetch (thread 0 = the producer lane, barriers initialised): K/V of the
// request's first n <= STAGES prompt-only tiles into ring stages 0..n-1 (no mask/depth
// words: those tiles take the unmasked path); the producer loop then starts at tile n.
template <int D, int STAGES>
__device__ __forceinline__ void prefetch_prompt_tiles(const CUtensorMap* kmap,
                                                      const CUtensorMap* vmap,
                                                      const AttnParams& p, int r, int h,
                                                      uint8_t* ring, uint64_t* full, int n) {
  using RG = Ring<D, STAGES>;
  for (int i = 0; i < n; ++i) {
    const uint32_t st = smem_u32(ring + i * RG::STAGE_BYTES);
    // prompt tiles: their pages (paged pools) are fixed at trie_create
    const int row = (int)attn_row(p, r, h, i * TC_TR);
    mbar_expect_tx(&full[i], 2 * RG::TILE_BYTES);
#pragma unroll
    for (int bx = 0; bx < D / TC_CW; ++bx) {
      tma_load_2d(st + bx * TC_TR * 64, kmap, bx * TC_CW, row, &full[i]);
      tma_load_2d(st + RG::TILE_BYTES + bx * TC_TR * 64, vmap, bx * TC_CW, row, &full[i]);
    }
  }
}

template <int D, int STAGES>
__device__ __forceinline__ void producer_loop(const CUtensorMap* kmap, const CUtensorMap* vmap,
                                              const AttnParams& p, int r, int h,
                                              const ItemInfo& it, uint8_t* ring, uint64_t* full,
                                              uint64_t* empty, uint64_t* app_done = nullptr,
                                              int first_leaf_slot = INT_MAX, int i_begin = 0,
                                              int i_end = INT_MAX, uint32_t* trc = nullptr,
                                              const CUtensorMap* kmh = nullptr,
                                              const CUtensorMap* vmh = nullptr) {
  // kmh / vmh: maps with 32-row boxes.  The request's last tile, when it holds <= 32 rows
  // below N, loads only its first 32 rows (the rest of the stage keeps the finite K/V of
  // an earlier tile -- hence only stages already used, i >= STAGES -- and those rows are
  // masked, n >= N): the 64-row tile granularity over-fetched ~half a tile per item.
  using RG = Ring<D, STAGES>;
  const size_t mbase = (size_t)r * p.cap;
  bool appended = app_done == nullptr;
  for (int i = i_begin; i < min(it.ntiles, i_end); ++i) {
    const int s = i % STAGES;
    const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
    mbar_wait(&empty[s], ph ^ 1u);
    if (trc && i < 400) trc[i * 12 + 7] = (uint32_t)clock();
    if (!appended && (it.tile0 + i + 1) * TC_TR > first_leaf_slot) {
      // fused RoPE: the consumer wrote this tile's leaf K/V rows (generic proxy) and
      // fenced them for the async proxy before arriving; TMA may read them now
      mbar_wait(app_done, 0u);
      appended = true;
    }
    const uint32_t st = smem_u32(ring + s * RG::STAGE_BYTES);
    const int n0 = (it.tile0 + i) * TC_TR;
    const int row = (int)attn_row(p, r, h, n0);
    // mask / depth words clamped to the [R][cap] arrays (cap % 4 == 0: 16-byte granules)
    const uint32_t mdb = (uint32_t)min(TC_TR, p.cap - n0) * 4u;
    const bool half = kmh != nullptr && i >= STAGES && it.N - n0 <= TC_TR / 2;
    mbar_expect_tx(&full[s], (half ? RG::TILE_BYTES : 2 * RG::TILE_BYTES) + 2 * mdb);
    const CUtensorMap* km = half ? kmh : kmap;
    const CUtensorMap* vm = half ? vmh : vmap;
#pragma unroll
    for (int bx = 0; bx < D / TC_CW; ++bx) {
      tma_load_2d(st + bx * TC_TR * 64, km, bx * TC_CW, row, &full[s]);
      tma_load_2d(st + RG::TILE_BYTES + bx * TC_TR * 64, vm, bx * TC_CW, row, &full[s]);
    }
    bulk_load_1d(st + 2 * RG::TILE_BYTES, p.mask + mbase + n0, mdb, &full[s]);
    bulk_load_1d(st + 2 * RG::TILE_BYTES + TC_TR * 4, p.depth + mbase + n0, mdb, &full[s]);
    if (trc && i < 400) trc[i * 12 + 8] = (uint32_t)clock();
  }
}

}  // namespace trie
