// K3: decode paged attention (HBM-bound), tensor-core + TMA version.
//
// Realizes the KV-read term kv_cache_bytes(model, total_kv_tokens) of
// decode_time (reference pkg/src/pdsim/costmodel.py:129-133).
//
// Cache layout (one layer): [num_blocks][2 (K,V)][Hkv][16 tokens][D=128] bf16,
// viewed by TMA as a 2D tensor of 256-byte rows; one page of one kv-head is 16
// consecutive rows. Each page half (64 dims) is fetched by one
// cp.async.bulk.tensor box {64, 16} with the 128B swizzle, so every ldmatrix
// below is bank-conflict free.
//
// Work decomposition: item = (sequence b, kv head h, chunk c of `chunk_pages`
// pages); the host picks whole sequences when B x Hkv fills the partition.
// Persistent grid; every warp owns a private STAGES-deep smem ring and streams
// the pages of its items (item = global_warp, +num_warps, ...) back to back:
// lane 0 keeps STAGES pages in flight across item boundaries.
//
// Math per page (transposed so GQA padding is free):
//   S^T[16 tok x 8 heads] = K[16 x 128] . Q^T[128 x 8]   (8 x mma.m16n8k16)
//   online softmax per head (column) over tokens
//   O^T[128 x 8] += V^T[128 x 16] . P^T[16 x 8]           (8 x mma.m16n8k16)
// P^T goes accumulator -> bf16 -> 256 B smem -> ldmatrix.trans (B operand).
// Items of multi-chunk sequences write fp32 partials (m, l, O) that a combine
// kernel merges; single-chunk sequences write the output directly.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cfloat>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

constexpr int kD = 128;
constexpr int kPage = 16;
// (warps per CTA, smem stages per warp): 8 x 3 on large partitions; 12 x 2 on <= 64-SM
// partitions, where more warps in flight per SM measured up to +35% (56 SMs, B=226)
constexpr int kStageBytes = 4 * 2048;     // K lo/hi + V lo/hi, 16 rows x 128 B each
constexpr int kPStageBytes = 256;         // P^T staging per warp
constexpr float kLazyLog2 = 8.0f;         // stale-max slack of the online softmax (P <= 2^8)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// byte offset of 16-byte chunk `ch` (0..15 over 128 dims) of token row `r` in a staged page half-pair
__device__ __forceinline__ uint32_t pg_off(int r, int ch) {
  return (uint32_t)((ch >> 3) * 2048 + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}

struct DecArgs {
  const __nv_bfloat16* q;
  long long q_tok_stride;
  const int* block_table;
  int bt_stride;
  const int* row_slot;
  const int* seq_lens;
  __nv_bfloat16* out;
  long long out_tok_stride;
  float* part_o;   // [items][G][128]
  float* part_ml;  // [items][G][2]
  int B, Hkv, G, splits, chunk_pages;
  float scale_log2;
  int* work;  // [2] self-resetting (next item, finished warps): dynamic item assignment; null = static
  int one_op;  // 1: kv_map is the 5D page map (one 8 KB TMA op per page); 0: 2D rows (four 2 KB boxes)
};

constexpr int kQueue = 8;  // per-warp ring of acquired item ids (producer lane 0 -> all lanes)

// decode an item index -> (b, h, chunk); returns pages [p0, p1) (empty if past the sequence)
__device__ __forceinline__ void item_pages(const DecArgs& a, int item, int& b, int& h, int& c, int& p0, int& p1,
                                           int& n) {
  c = item % a.splits;
  const int bh = item / a.splits;
  h = bh % a.Hkv;
  b = bh / a.Hkv;
  n = a.seq_lens[b];
  const int nb = (n + kPage - 1) / kPage;
  p0 = c * a.chunk_pages;
  p1 = min(nb, p0 + a.chunk_pages);
}

template <int kWarps, int kStages>
__global__ void __launch_bounds__(kWarps * 32, 1)
    decode_attn_tc_kernel(const __grid_constant__ CUtensorMap kv_map, const DecArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * kStages * kStageBytes;
  uint8_t* pst = smem + (size_t)kWarps * kStages * kStageBytes + warp * kPStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * kStages * kStageBytes +
                                               kWarps * kPStageBytes) + warp * kStages;
  int* queue = reinterpret_cast<int*>(reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * kStages * kStageBytes +
                                                                  kWarps * kPStageBytes) + kWarps * kStages) +
               warp * kQueue;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    tma_prefetch_desc(&kv_map);
  }
  __syncwarp();

  const int total_items = a.B * a.Hkv * a.splits;
  const int gw = blockIdx.x * kWarps + warp;
  const int nw = gridDim.x * kWarps;
  const int g = lane >> 2;  // group id (row of the fragment)
  const int t = lane & 3;

  // ---------------- producer cursor (lane 0): next page to fetch. Items come from a global
  // atomic counter when a.work is set (warps that finish early take more: no tail from the
  // items-per-warp quantization), else statically gw, gw + nw, ... The producer runs ahead of
  // the consumer across item boundaries, so each acquired item id (and a final -1) goes
  // through a per-warp smem ring in acquisition order.
  int qtail = 0;
  auto next_item = [&](int cur) { return a.work ? atomicAdd(&a.work[0], 1) : cur + nw; };
  int pi = a.work ? -1 : gw, pp = 0, pp1 = 0, pb = 0, ph = 0, pc = 0, pn = 0;
  // the block-table entry of the NEXT page to fetch is loaded one issue ahead (npage): the
  // producer lane runs inside the consumer warp, so a dependent slot -> page load at issue
  // time stalled the whole warp once per page (ncu: profiles/r02/dattn/)
  const int* bt_row = nullptr;
  int npage = 0;
  auto p_seek = [&]() {  // advance pi to an item with pages; sets pp..pp1 and enqueues it
    while (pi < total_items) {
      item_pages(a, pi, pb, ph, pc, pp, pp1, pn);
      if (pp < pp1) {
        queue[qtail++ & (kQueue - 1)] = pi;
        bt_row = a.block_table + (size_t)a.row_slot[pb] * a.bt_stride;
        npage = bt_row[pp];
        return;
      }
      pi = next_item(pi);
    }
    queue[qtail++ & (kQueue - 1)] = -1;
  };
  int issued = 0;
  auto p_issue = [&](int stage) {
    const int page = npage;
    const int rowK = ((page * 2 + 0) * a.Hkv + ph) * kPage;
    const int rowV = ((page * 2 + 1) * a.Hkv + ph) * kPage;
    uint8_t* dst = ring + (size_t)stage * kStageBytes;
    mbar_arrive_expect_tx(&bars[stage], kStageBytes);
    if (a.one_op) {
      // the page's K and V halves of this head in one op (the per-op TMA cost, not bytes in
      // flight, bounds small partitions: scripts/ingest_probe.py, profiles/r02/ingest/)
      tma_load_5d(dst, &kv_map, &bars[stage], 0, 0, 0, 0, (page * 2) * a.Hkv + ph, kEvictFirst);
    } else {
      tma_load_2d(dst, &kv_map, &bars[stage], 0, rowK, kEvictFirst);
      tma_load_2d(dst + 2048, &kv_map, &bars[stage], 64, rowK, kEvictFirst);
      tma_load_2d(dst + 4096, &kv_map, &bars[stage], 0, rowV, kEvictFirst);
      tma_load_2d(dst + 6144, &kv_map, &bars[stage], 64, rowV, kEvictFirst);
    }
    if (++pp == pp1) {
      pi = next_item(pi);
      p_seek();
    } else {
      npage = bt_row[pp];  // consumed at the next issue, a page of math later
    }
  };
  if (lane == 0) {
    if (a.work) pi = atomicAdd(&a.work[0], 1);
    p_seek();
    for (int s = 0; s < kStages && pi < total_items; ++s) {
      p_issue(s);
      ++issued;
    }
  }

  int stage = 0;
  uint32_t phase = 0;
  for (int qhead = 0;; ++qhead) {
    __syncwarp();  // lane 0's queue writes are visible to the warp
    const int item = queue[qhead & (kQueue - 1)];
    if (item < 0) break;
    int b, h, c, p0, p1, n;
    item_pages(a, item, b, h, c, p0, p1, n);
    // Q^T fragments (B operand): b0 = (dims 16kk+2t.., head g), b1 = (dims 16kk+8+2t.., head g)
    uint32_t qb[8][2];
    {
      const __nv_bfloat16* qrow = a.q + (size_t)b * a.q_tok_stride + (size_t)(h * a.G + g) * kD;
      const bool hv = g < a.G;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = hv ? *reinterpret_cast<const uint32_t*>(qrow + 16 * kk + 2 * t) : 0u;
        qb[kk][1] = hv ? *reinterpret_cast<const uint32_t*>(qrow + 16 * kk + 8 + 2 * t) : 0u;
      }
    }
    float o[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -FLT_MAX, m1 = -FLT_MAX;  // running max for heads 2t, 2t+1
    float l0 = 0.f, l1 = 0.f;            // per-thread partial sums (tokens g, g+8)

    for (int p = p0; p < p1; ++p) {
      mbar_wait(&bars[stage], phase);
      const uint32_t base = smem_u32(ring + (size_t)stage * kStageBytes);
      // ---- S^T = K Q^T: even / odd k-steps into two accumulators (halves the MMA
      // dependency chain on the critical path of every page)
      // (four accumulators over the 8 k-steps: a dependent chain of 2 MMAs, not 8)
      float sa[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c) sa[c][0] = sa[c][1] = sa[c][2] = sa[c][3] = 0.f;
      const int mi = lane >> 3;
      const int rr = (mi & 1) * 8 + (lane & 7);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(base + pg_off(rr, 2 * kk + (mi >> 1)), a0, a1, a2, a3);
        mma_bf16_16816(sa[kk & 3], a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
      }
      float s[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) s[e] = (sa[0][e] + sa[1][e]) + (sa[2][e] + sa[3][e]);
      // ---- mask + online softmax (columns = heads 2t, 2t+1; rows = tokens g, g+8)
      const int tok0 = p * kPage + g;
      float s00 = s[0] * a.scale_log2, s01 = s[1] * a.scale_log2;
      float s10 = s[2] * a.scale_log2, s11 = s[3] * a.scale_log2;
      if (tok0 >= n) { s00 = -FLT_MAX; s01 = -FLT_MAX; }
      if (tok0 + 8 >= n) { s10 = -FLT_MAX; s11 = -FLT_MAX; }
      float mx0 = fmaxf(s00, s10), mx1 = fmaxf(s01, s11);
      // lazy max: the running (per-head, warp-uniform) max moves only when some score of the
      // page exceeds it by more than 2^kLazyLog2 — otherwise P = 2^(s - m) <= 2^8 against the
      // stale max (exact after the final 1/l) and the page skips the shuffle reduction, the
      // alpha exp2 and the 32-register O rescale (the first page always takes the full path)
      if (__any_sync(0xffffffffu, mx0 > m0 + kLazyLog2 || mx1 > m1 + kLazyLog2)) {
#pragma unroll
        for (int off = 4; off <= 16; off <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);  // m0=-FLT_MAX first: exp2(-huge)=0
        m0 = mn0;
        m1 = mn1;
        l0 *= al0;
        l1 *= al1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o[i][0] *= al0;
          o[i][1] *= al1;
          o[i][2] *= al0;
          o[i][3] *= al1;
        }
      }
      const float p00 = (s00 == -FLT_MAX) ? 0.f : exp2f(s00 - m0);
      const float p01 = (s01 == -FLT_MAX) ? 0.f : exp2f(s01 - m1);
      const float p10 = (s10 == -FLT_MAX) ? 0.f : exp2f(s10 - m0);
      const float p11 = (s11 == -FLT_MAX) ? 0.f : exp2f(s11 - m1);
      l0 += p00 + p10;
      l1 += p01 + p11;
      // ---- rows past the sequence end in the last page hold stale (possibly non-finite)
      // V; P is 0 there but 0 * NaN would still poison the MMA, so zero those rows.
      const int valid = n - p * kPage;
      if (valid < kPage) {
        for (int i = lane; i < (kPage - valid) * 16; i += 32) {
          const int r = valid + (i >> 4);
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + 4096 + pg_off(r, i & 15)), "r"(0u)
                       : "memory");
        }
      }
      // ---- P^T -> smem [16 tok][8 heads] bf16 -> B fragments
      uint32_t* pw = reinterpret_cast<uint32_t*>(pst);
      pw[g * 4 + t] = pack_bf16x2(p00, p01);
      pw[(g + 8) * 4 + t] = pack_bf16x2(p10, p11);
      __syncwarp();
      uint32_t pb0, pb1;
      ldsm_x2_t(smem_u32(pst) + (lane & 15) * 16, pb0, pb1);
      // ---- O^T += V^T P^T over 8 m-tiles of 16 dims
      const int vr = (mi >> 1) * 8 + (lane & 7);
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(base + 4096 + pg_off(vr, 2 * mt + (mi & 1)), a0, a1, a2, a3);
        mma_bf16_16816(o[mt], a0, a1, a2, a3, pb0, pb1);
      }
      __syncwarp();  // every lane done with this stage and with pst
      if (lane == 0 && pi < total_items) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        p_issue(stage);
      }
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
    // ---- finalize item: reduce l over the 8 row groups
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const int nchunks = ((n + kPage - 1) / kPage + a.chunk_pages - 1) / a.chunk_pages;
    const int hd0 = 2 * t, hd1 = 2 * t + 1;
    if (nchunks == 1) {
      const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
      __nv_bfloat16* ob = a.out + (size_t)b * a.out_tok_stride + (size_t)h * a.G * kD;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int d0 = mt * 16 + g;
        if (hd0 < a.G) {
          ob[(size_t)hd0 * kD + d0] = __float2bfloat16_rn(o[mt][0] * i0);
          ob[(size_t)hd0 * kD + d0 + 8] = __float2bfloat16_rn(o[mt][2] * i0);
        }
        if (hd1 < a.G) {
          ob[(size_t)hd1 * kD + d0] = __float2bfloat16_rn(o[mt][1] * i1);
          ob[(size_t)hd1 * kD + d0 + 8] = __float2bfloat16_rn(o[mt][3] * i1);
        }
      }
    } else {
      const size_t pbase = (size_t)item * a.G;
      const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int d0 = mt * 16 + g;
        if (hd0 < a.G) {
          a.part_o[(pbase + hd0) * kD + d0] = o[mt][0] * i0;
          a.part_o[(pbase + hd0) * kD + d0 + 8] = o[mt][2] * i0;
        }
        if (hd1 < a.G) {
          a.part_o[(pbase + hd1) * kD + d0] = o[mt][1] * i1;
          a.part_o[(pbase + hd1) * kD + d0 + 8] = o[mt][3] * i1;
        }
      }
      if (g == 0) {
        if (hd0 < a.G) { a.part_ml[(pbase + hd0) * 2] = m0; a.part_ml[(pbase + hd0) * 2 + 1] = l0; }
        if (hd1 < a.G) { a.part_ml[(pbase + hd1) * 2] = m1; a.part_ml[(pbase + hd1) * 2 + 1] = l1; }
      }
    }
  }
  // re-arm the work counter for the next launch / graph replay: the last warp to finish resets it
  // (every warp has drawn its final, out-of-range ticket before it counts itself done)
  if (a.work && lane == 0) {
    if (atomicAdd(&a.work[1], 1) == nw - 1) {
      a.work[0] = 0;
      a.work[1] = 0;
      __threadfence();
    }
  }
}

// merges the chunk partials of multi-chunk sequences; grid (B, Hq), 128 threads
__global__ void decode_attn_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                           const int* __restrict__ seq_lens, __nv_bfloat16* __restrict__ out,
                                           long long out_tok_stride, int Hkv, int G, int splits,
                                           int chunk_pages) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const int hq = blockIdx.y;
  const int d = threadIdx.x;
  const int n = seq_lens[b];
  const int nchunks = ((n + kPage - 1) / kPage + chunk_pages - 1) / chunk_pages;
  if (n <= 0 || nchunks <= 1) return;
  const int h = hq / G, hd = hq % G;
  float mx = -FLT_MAX;
  for (int c = 0; c < nchunks; ++c) {
    const size_t it = ((size_t)(b * Hkv + h) * splits + c) * G + hd;
    if (part_ml[it * 2 + 1] > 0.f) mx = fmaxf(mx, part_ml[it * 2]);
  }
  float l = 0.f, o = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const size_t it = ((size_t)(b * Hkv + h) * splits + c) * G + hd;
    const float lc = part_ml[it * 2 + 1];
    if (lc <= 0.f) continue;
    const float w = exp2f(part_ml[it * 2] - mx) * lc;
    l += w;
    o += w * part_o[it * kD + d];
  }
  out[(size_t)b * out_tok_stride + (size_t)hq * kD + d] = __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
}

static int g_decode_shape = 0;     // debug: ring shape override (0 = auto)
int decode_attn_set_shape(int shape) {
  if (shape < 0 || shape > 4) return -1;
  g_decode_shape = shape;
  return 0;
}
static int g_decode_kv_one_op = 1;  // 1: one 5D TMA op per page (default), 0: four 2D boxes
int decode_attn_set_kv_ops(int one_op) {
  g_decode_kv_one_op = one_op ? 1 : 0;
  return 0;
}

int decode_attention_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* block_table,
                            int bt_stride, const int* row_slot, const int* seq_lens, void* out,
                            long long out_tok_stride, void* workspace, size_t ws_bytes, int B, int Hq, int Hkv,
                            int head_dim, int max_pages, float scale, int num_blocks, int num_sms, cudaStream_t st) {
  if (B <= 0) return 0;
  if (head_dim != kD) return set_error("decode attention: head_dim must be 128");
  if (Hkv <= 0 || Hq % Hkv != 0) return set_error("decode attention: Hq must be a multiple of Hkv");
  const int G = Hq / Hkv;
  if (G > 8) return set_error("decode attention: GQA group > 8 unsupported");
  if (max_pages < 1) max_pages = 1;
  if (num_sms <= 0) num_sms = 148;
  // Work-item size: whole sequences when (B x Hkv) already gives every warp of the
  // partition at least one item (no partials, no combine pass); otherwise cut sequences into
  // chunks so there are ~4 items per warp (load balance for long contexts / small B).
  const bool small = num_sms <= 100;
  // ring shape (warps x stages per warp): auto 12 x 2 on <= 100-SM partitions, else 8 x 3;
  // debug override g_decode_shape 1..4 = 12x2, 8x3, 6x4, 4x6
  int shape = g_decode_shape ? g_decode_shape : (small ? 1 : 2);
  static const int kShapeWarps[5] = {0, 12, 8, 6, 4};
  static const int kShapeStages[5] = {0, 2, 3, 4, 6};
  const int kWarps = kShapeWarps[shape];
  const int kStages = kShapeStages[shape];
  const long long warps = (long long)num_sms * kWarps;
  const long long seqs = (long long)B * Hkv;
  int chunk_pages = max_pages;
  // small partitions are bound per SM: fewer than ~1.5 whole sequences per warp leaves a
  // ragged last round even with dynamic assignment, so cut sequences there too
  if (seqs < warps || (small && 2 * seqs < 3 * warps)) {
    chunk_pages = (int)((max_pages * seqs + 4 * warps - 1) / (4 * warps));
    if (chunk_pages < 8) chunk_pages = 8;
    if (chunk_pages > max_pages) chunk_pages = max_pages;
  }
  // the last 64 bytes of the workspace hold the self-resetting work counters (zero before the
  // first call); the partials use the rest
  int* work = nullptr;
  if (workspace != nullptr && ws_bytes >= 64) {
    work = reinterpret_cast<int*>(static_cast<char*>(workspace) + ((ws_bytes - 64) & ~size_t(63)));
    ws_bytes = (ws_bytes - 64) & ~size_t(63);
  }
  // splitting is an optimisation: without room for the partials, keep whole sequences
  if ((size_t)B * Hq * ((max_pages + chunk_pages - 1) / chunk_pages) * (kD + 2) * sizeof(float) > ws_bytes ||
      workspace == nullptr)
    chunk_pages = max_pages;
  const int splits = (max_pages + chunk_pages - 1) / chunk_pages;  // work items per (sequence, kv head)
  DecArgs a{};
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.q_tok_stride = q_tok_stride;
  a.block_table = block_table;
  a.bt_stride = bt_stride;
  a.row_slot = row_slot;
  a.seq_lens = seq_lens;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_tok_stride = out_tok_stride;
  a.B = B;
  a.Hkv = Hkv;
  a.G = G;
  a.splits = splits;
  a.chunk_pages = chunk_pages;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.work = work;
  const size_t items = (size_t)B * Hkv * splits;
  if (splits > 1) {
    const size_t need = items * G * (kD + 2) * sizeof(float);
    if (workspace == nullptr || ws_bytes < need) return set_error("decode attention: workspace too small");
    a.part_o = reinterpret_cast<float*>(workspace);
    a.part_ml = a.part_o + items * G * kD;
  }
  CUtensorMap map;
  a.one_op = 0;
  if (g_decode_kv_one_op && make_tmap_kv5d_bf16(&map, cache_layer, (uint64_t)num_blocks, Hkv) == 0) {
    a.one_op = 1;
  } else {
    const uint64_t rows = (uint64_t)num_blocks * 2 * Hkv * kPage;
    int rc = make_tmap_2d_bf16(&map, cache_layer, kD, rows, kD, 64, kPage);
    if (rc) return rc;
  }
  const int smem = kWarps * kStages * kStageBytes + kWarps * kPStageBytes + kWarps * kStages * 8 +
                   kWarps * kQueue * 4 + 1024;
  using Fn = void (*)(const CUtensorMap, const DecArgs);
  static const Fn kerns[5] = {nullptr, decode_attn_tc_kernel<12, 2>, decode_attn_tc_kernel<8, 3>,
                              decode_attn_tc_kernel<6, 4>, decode_attn_tc_kernel<4, 6>};
  const Fn kern = kerns[shape];
  {
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(kern), 227 * 1024);
    if (e != cudaSuccess) return set_cuda_error("decode attn smem attr", e);
  }
  const size_t warps_needed = items;
  int grid = (int)((warps_needed + kWarps - 1) / kWarps);
  if (grid > num_sms) grid = num_sms;
  if (grid < 1) grid = 1;
  cudaError_t e = launch_k(kern, dim3(grid), dim3(kWarps * 32), smem, st, 1, map, a);
  if (e != cudaSuccess) return set_cuda_error("decode attn launch", e);
  if (splits > 1) {
    e = launch_k(decode_attn_combine_kernel, dim3(B, Hq), dim3(kD), 0, st, 1, a.part_o, a.part_ml, seq_lens, a.out, out_tok_stride, Hkv, G, splits, chunk_pages);
    if (e != cudaSuccess) return set_cuda_error("decode combine launch", e);
  }
  return 0;
}

}  // namespace rb
