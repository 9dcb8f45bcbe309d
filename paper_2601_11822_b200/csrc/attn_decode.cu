// K3: decode paged attention (HBM-bound).
//
// Realizes the KV-read term kv_cache_bytes(model, total_kv_tokens) of
// decode_time (reference pkg/src/pdsim/costmodel.py:129-133).
//
// Cache layout (one layer): [num_blocks][2 (K,V)][Hkv][16 tokens][D] bf16, so
// the K (or V) page of one kv-head is a contiguous 4 KB run that one
// cp.async.bulk moves into shared memory. Grid = (Hkv, B, splits); each CTA
// serves all G = Hq/Hkv query heads of one kv head (GQA) over one split of
// the sequence's pages. Each of the 4 warps owns a private STAGES-deep smem
// ring fed by bulk copies (lane 0 issues, mbarrier completes), so the warp
// keeps STAGES x 8 KB in flight without spending registers on it.
//
// Lane mapping inside a page: lane = 8*grp + c; grp (0..3) owns tokens
// 4*grp..4*grp+3, c (0..7) owns dims {8c..8c+7} U {64+8c..64+8c+7}. q.k
// partials reduce over the 8 lanes of a group (3 shuffles); every group keeps
// its own online-softmax state, merged once at the end (no per-page
// cross-group traffic).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cfloat>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

constexpr int kDecD = 128;
constexpr int kPage = 16;
constexpr int kDecWarps = 4;
constexpr int kDecStages = 3;
constexpr int kPageBytes = kPage * kDecD * 2;  // 4 KB

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(kEvictFirst)
      : "memory");
}

template <int G>
__global__ void __launch_bounds__(kDecWarps * 32)
    decode_attn_kernel(const __nv_bfloat16* __restrict__ q, long long q_tok_stride,
                       const __nv_bfloat16* __restrict__ cache, const int* __restrict__ block_table, int bt_stride,
                       const int* __restrict__ row_slot, const int* __restrict__ seq_lens,
                       __nv_bfloat16* __restrict__ out, long long out_tok_stride, float* __restrict__ part_o,
                       float* __restrict__ part_ml, int Hkv, int splits, float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;  // [warps][stages][8 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kDecWarps * kDecStages * 2 * kPageBytes);

  const int h = blockIdx.x;
  const int b = blockIdx.y;
  const int s = blockIdx.z;
  const int Hq = Hkv * G;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n = seq_lens[b];
  const int nb = (n + kPage - 1) / kPage;
  const int per = (nb + splits - 1) / max(splits, 1);
  const int j0 = s * per;
  const int j1 = min(nb, j0 + per);

  if (n <= 0 || j0 >= j1) {
    // empty split (or padded row): publish a neutral partial
    if (splits > 1 && threadIdx.x < G) {
      const size_t idx = ((size_t)b * Hq + h * G + threadIdx.x) * splits + s;
      part_ml[2 * idx] = -FLT_MAX;
      part_ml[2 * idx + 1] = 0.f;
    }
    return;
  }
  const int* bt = block_table + (size_t)row_slot[b] * bt_stride;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kDecWarps * kDecStages; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  __syncthreads();

  // blocks of this warp: j0 + warp + 4*i
  const int my_first = j0 + warp;
  const int cnt = (my_first < j1) ? (j1 - my_first + kDecWarps - 1) / kDecWarps : 0;
  uint8_t* my_ring = ring + (size_t)warp * kDecStages * 2 * kPageBytes;
  uint64_t* my_bars = bars + warp * kDecStages;
  const size_t head_off = (size_t)h * kPage * kDecD;                // within K or V half
  const size_t half_stride = (size_t)Hkv * kPage * kDecD;           // K -> V
  const size_t page_stride = 2 * half_stride;

  if (lane == 0) {
    for (int i = 0; i < kDecStages && i < cnt; ++i) {
      const int page = bt[my_first + i * kDecWarps];
      const __nv_bfloat16* kp = cache + (size_t)page * page_stride + head_off;
      mbar_arrive_expect_tx(&my_bars[i], 2 * kPageBytes);
      bulk_g2s(my_ring + (size_t)i * 2 * kPageBytes, kp, kPageBytes, &my_bars[i]);
      bulk_g2s(my_ring + (size_t)i * 2 * kPageBytes + kPageBytes, kp + half_stride, kPageBytes, &my_bars[i]);
    }
  }

  const int grp = lane >> 3;
  const int c = lane & 7;
  // q fragment: dims 8c..8c+7 and 64+8c..64+8c+7 for every head of the group
  float qf[G][16];
  const __nv_bfloat16* qb = q + (size_t)b * q_tok_stride + (size_t)h * G * kDecD;
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      uint4 u = *reinterpret_cast<const uint4*>(qb + g * kDecD + hh * 64 + 8 * c);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = unpack_bf16x2(w[j]);
        qf[g][hh * 8 + 2 * j] = f.x * scale_log2;
        qf[g][hh * 8 + 2 * j + 1] = f.y * scale_log2;
      }
    }
  }
  float m_run[G], l_run[G], acc[G][16];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m_run[g] = -FLT_MAX;
    l_run[g] = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[g][j] = 0.f;
  }

  for (int i = 0; i < cnt; ++i) {
    const int stage = i % kDecStages;
    const uint32_t parity = (uint32_t)((i / kDecStages) & 1);
    mbar_wait(&my_bars[stage], parity);
    const uint8_t* kbuf = my_ring + (size_t)stage * 2 * kPageBytes;
    const uint8_t* vbuf = kbuf + kPageBytes;
    const int jpage = my_first + i * kDecWarps;
    float sc[G][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = grp * 4 + u;
      const uint4 k0 = *reinterpret_cast<const uint4*>(kbuf + t * 256 + 16 * c);
      const uint4 k1 = *reinterpret_cast<const uint4*>(kbuf + t * 256 + 128 + 16 * c);
      const uint32_t kw[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
      float kf[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2 f = unpack_bf16x2(kw[j]);
        kf[2 * j] = f.x;
        kf[2 * j + 1] = f.y;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) a = fmaf(qf[g][j], kf[j], a);
        sc[g][u] = a;
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float a = sc[g][u];
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 4);
        const int pos = jpage * kPage + grp * 4 + u;
        sc[g][u] = (pos < n) ? a : -FLT_MAX;
      }
    }
    float vf[4][16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = grp * 4 + u;
      const uint4 v0 = *reinterpret_cast<const uint4*>(vbuf + t * 256 + 16 * c);
      const uint4 v1 = *reinterpret_cast<const uint4*>(vbuf + t * 256 + 128 + 16 * c);
      const uint32_t vw[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      const bool ok = (jpage * kPage + t) < n;  // stale cache rows may hold NaN bit patterns
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2 f = unpack_bf16x2(vw[j]);
        vf[u][2 * j] = ok ? f.x : 0.f;
        vf[u][2 * j + 1] = ok ? f.y : 0.f;
      }
    }
    // all lanes are done with this stage's smem: refill it
    __syncwarp();
    if (lane == 0 && i + kDecStages < cnt) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int page = bt[my_first + (i + kDecStages) * kDecWarps];
      const __nv_bfloat16* kp = cache + (size_t)page * page_stride + head_off;
      mbar_arrive_expect_tx(&my_bars[stage], 2 * kPageBytes);
      bulk_g2s(my_ring + (size_t)stage * 2 * kPageBytes, kp, kPageBytes, &my_bars[stage]);
      bulk_g2s(my_ring + (size_t)stage * 2 * kPageBytes + kPageBytes, kp + half_stride, kPageBytes,
               &my_bars[stage]);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mx = fmaxf(fmaxf(sc[g][0], sc[g][1]), fmaxf(sc[g][2], sc[g][3]));
      const float m_new = fmaxf(m_run[g], mx);
      if (m_new == -FLT_MAX) continue;  // nothing valid yet for this group
      const float alpha = exp2f(m_run[g] - m_new);
      float p[4];
      float ps = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        p[u] = (sc[g][u] == -FLT_MAX) ? 0.f : exp2f(sc[g][u] - m_new);
        ps += p[u];
      }
      l_run[g] = l_run[g] * alpha + ps;
      m_run[g] = m_new;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float a = acc[g][j] * alpha;
#pragma unroll
        for (int u = 0; u < 4; ++u) a = fmaf(p[u], vf[u][j], a);
        acc[g][j] = a;
      }
    }
  }

  // merge the 4 token groups of this warp (lanes c, c+8, c+16, c+24)
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, m_run[g], off);
      const float lo = __shfl_xor_sync(0xffffffffu, l_run[g], off);
      const float mn = fmaxf(m_run[g], mo);
      const float a_self = (m_run[g] == -FLT_MAX) ? 0.f : exp2f(m_run[g] - mn);
      const float a_oth = (mo == -FLT_MAX) ? 0.f : exp2f(mo - mn);
      l_run[g] = l_run[g] * a_self + lo * a_oth;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float ao = __shfl_xor_sync(0xffffffffu, acc[g][j], off);
        acc[g][j] = acc[g][j] * a_self + ao * a_oth;
      }
      m_run[g] = mn;
    }
  }
  // publish per-warp partials [g][m, l, D] into this warp's (now idle) ring:
  // every bulk copy the warp issued has been waited on inside the loop.
  const int mstride = 2 + kDecD;
  const size_t ring_floats = (size_t)kDecStages * 2 * kPageBytes / 4;
  float* merge = reinterpret_cast<float*>(ring);
  if (grp == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float* dst = merge + (size_t)warp * ring_floats + (size_t)g * mstride;
      if (c == 0) {
        dst[0] = m_run[g];
        dst[1] = l_run[g];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dst[2 + 8 * c + j] = acc[g][j];
        dst[2 + 64 + 8 * c + j] = acc[g][8 + j];
      }
    }
  }
  __syncthreads();
  // final merge across warps: thread -> (g, d) pairs
  for (int idx = threadIdx.x; idx < G * kDecD; idx += blockDim.x) {
    const int g = idx / kDecD;
    const int d = idx % kDecD;
    float mx = -FLT_MAX;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) mx = fmaxf(mx, merge[(size_t)w * ring_floats + (size_t)g * mstride]);
    float l = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) {
      const float* src = merge + (size_t)w * ring_floats + (size_t)g * mstride;
      const float a = (src[0] == -FLT_MAX) ? 0.f : exp2f(src[0] - mx);
      l += src[1] * a;
      o += src[2 + d] * a;
    }
    const int hq = h * G + g;
    if (splits == 1) {
      out[(size_t)b * out_tok_stride + (size_t)hq * kDecD + d] = __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
    } else {
      const size_t pidx = ((size_t)b * Hq + hq) * splits + s;
      part_o[pidx * kDecD + d] = (l > 0.f) ? o / l : 0.f;
      if (d == 0) {
        part_ml[2 * pidx] = mx;
        part_ml[2 * pidx + 1] = l;
      }
    }
  }
}

__global__ void decode_attn_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                           const int* __restrict__ seq_lens, __nv_bfloat16* __restrict__ out,
                                           long long out_tok_stride, int Hq, int splits) {
  const int b = blockIdx.x;
  const int hq = blockIdx.y;
  const int d = threadIdx.x;
  if (seq_lens[b] <= 0) return;
  const size_t base = ((size_t)b * Hq + hq) * splits;
  float mx = -FLT_MAX;
  for (int s = 0; s < splits; ++s)
    if (part_ml[2 * (base + s) + 1] > 0.f) mx = fmaxf(mx, part_ml[2 * (base + s)]);
  float l = 0.f, o = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float ls = part_ml[2 * (base + s) + 1];
    if (ls <= 0.f) continue;
    const float a = exp2f(part_ml[2 * (base + s)] - mx) * ls;
    l += a;
    o += a * part_o[(base + s) * kDecD + d];
  }
  out[(size_t)b * out_tok_stride + (size_t)hq * kDecD + d] = __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
}

template <int G>
static int launch_decode(const void* q, long long qs, const void* cache, const int* bt, int bt_stride,
                         const int* row_slot, const int* seq_lens, void* out, long long os, float* part_o,
                         float* part_ml, int B, int Hkv, int splits, float scale_log2, cudaStream_t st) {
  const int smem = kDecWarps * kDecStages * 2 * kPageBytes + kDecWarps * kDecStages * 8;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error("decode attn smem attr", e);
    attr = true;
  }
  dim3 grid(Hkv, B, splits);
  decode_attn_kernel<G><<<grid, kDecWarps * 32, smem, st>>>(
      (const __nv_bfloat16*)q, qs, (const __nv_bfloat16*)cache, bt, bt_stride, row_slot, seq_lens,
      (__nv_bfloat16*)out, os, part_o, part_ml, Hkv, splits, scale_log2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("decode attn launch", e);
  if (splits > 1) {
    decode_attn_combine_kernel<<<dim3(B, Hkv * G), kDecD, 0, st>>>(part_o, part_ml, seq_lens,
                                                                   (__nv_bfloat16*)out, os, Hkv * G, splits);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("decode combine launch", e);
  }
  return 0;
}

int decode_attention_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* block_table,
                            int bt_stride, const int* row_slot, const int* seq_lens, void* out,
                            long long out_tok_stride, void* workspace, size_t ws_bytes, int B, int Hq, int Hkv,
                            int head_dim, int splits, float scale, cudaStream_t st) {
  if (B <= 0) return 0;
  if (head_dim != kDecD) return set_error("decode attention: head_dim must be 128");
  if (Hkv <= 0 || Hq % Hkv != 0) return set_error("decode attention: Hq must be a multiple of Hkv");
  if (splits < 1) splits = 1;
  float* part_o = nullptr;
  float* part_ml = nullptr;
  if (splits > 1) {
    const size_t need = (size_t)B * Hq * splits * (kDecD + 2) * sizeof(float);
    if (workspace == nullptr || ws_bytes < need) return set_error("decode attention: workspace too small");
    part_o = reinterpret_cast<float*>(workspace);
    part_ml = part_o + (size_t)B * Hq * splits * kDecD;
  }
  const float sl2 = scale * 1.4426950408889634f;
  const int G = Hq / Hkv;
  switch (G) {
    case 1: return launch_decode<1>(q, q_tok_stride, cache_layer, block_table, bt_stride, row_slot, seq_lens, out, out_tok_stride, part_o, part_ml, B, Hkv, splits, sl2, st);
    case 2: return launch_decode<2>(q, q_tok_stride, cache_layer, block_table, bt_stride, row_slot, seq_lens, out, out_tok_stride, part_o, part_ml, B, Hkv, splits, sl2, st);
    case 4: return launch_decode<4>(q, q_tok_stride, cache_layer, block_table, bt_stride, row_slot, seq_lens, out, out_tok_stride, part_o, part_ml, B, Hkv, splits, sl2, st);
    case 5: return launch_decode<5>(q, q_tok_stride, cache_layer, block_table, bt_stride, row_slot, seq_lens, out, out_tok_stride, part_o, part_ml, B, Hkv, splits, sl2, st);
    case 8: return launch_decode<8>(q, q_tok_stride, cache_layer, block_table, bt_stride, row_slot, seq_lens, out, out_tok_stride, part_o, part_ml, B, Hkv, splits, sl2, st);
    default: return set_error("decode attention: unsupported GQA group size");
  }
}

}  // namespace rb
