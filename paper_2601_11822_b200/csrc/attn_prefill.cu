// K2: prefill causal flash-attention over the paged KV cache (GQA-packed).
//
// Realizes the attention part of the compute term of prefill_time (reference
// pkg/src/pdsim/costmodel.py:104) for one prefill chunk of one request
// (rapid.py:313 chunk = min(chunk_tokens, target - written)). The chunk's own
// K,V were written into the paged cache by the fused RoPE/cache-write kernel,
// so a chunk attends uniformly to [paged prefix U chunk] with the causal mask
// shifted by the chunk's start position.
//
// One CTA = one kv head x PB blocks of 16 query positions; warp (pb, g) owns
// the 16 positions of block pb for query head g of the group, so every 64-key
// K/V tile (4 pages, cp.async, XOR-swizzled, 3-stage ring) is fetched once for
// all G heads that share it. Heaviest (latest) position blocks launch first.
// Math: mma.sync m16n8k16 bf16 with the FA2 register-resident P.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cfloat>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

constexpr int kPD = 128;      // head dim
constexpr int kPBN = 64;      // keys per tile
constexpr int kPPage = 16;
constexpr int kRowBytes = kPD * 2;            // 256
constexpr int kTileBytes = kPBN * kRowBytes;  // 16 KB
constexpr int kPStages = 3;
constexpr int kPMaxWarps = 8;

// 16-byte chunk c of row r lives at chunk (c ^ (r & 7)).
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * kRowBytes + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4p(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4p_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816p(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(kPMaxWarps * 32)
    prefill_attn_kernel(const __nv_bfloat16* __restrict__ q, long long q_tok_stride,
                        const __nv_bfloat16* __restrict__ cache, const int* __restrict__ bt, int T, int start,
                        int Hq, int Hkv, int PB, __nv_bfloat16* __restrict__ out, long long out_tok_stride,
                        float scale_log2) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  const int G = Hq / Hkv;
  const int nwarps = G * PB;
  const int nblk = (T + 16 * PB - 1) / (16 * PB);
  const int blk = nblk - 1 - (int)blockIdx.x;  // heaviest (latest positions) first
  const int hk = blockIdx.y;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int pb = warp / G;
  const int gh = warp % G;
  const int hq = hk * G + gh;
  const int q0 = blk * 16 * PB + pb * 16;  // first chunk row of this warp
  const uint32_t sQ = smem_u32(smem) + (uint32_t)warp * 16 * kRowBytes;
  const uint32_t sK0 = smem_u32(smem) + (uint32_t)nwarps * 16 * kRowBytes;

  const size_t half_stride = (size_t)Hkv * kPPage * kPD;
  const size_t page_stride = 2 * half_stride;
  const size_t head_off = (size_t)hk * kPPage * kPD;

  // ---- this warp's 16 query rows
  for (int i = lane; i < 16 * 16; i += 32) {
    const int r = i >> 4, c = i & 15;
    const int row = q0 + r < T ? q0 + r : T - 1;
    cp_async16(sQ + swz(r, c), q + (size_t)row * q_tok_stride + (size_t)hq * kPD + c * 8);
  }
  cp_async_commit();

  const int cta_last = min(T, blk * 16 * PB + 16 * PB) - 1;
  const int kv_end = start + cta_last + 1;  // keys needed by the CTA's last row
  const int n_tiles = (kv_end + kPBN - 1) / kPBN;
  const int nthreads = nwarps * 32;

  auto load_kv = [&](int tile, int stage) {
    const uint32_t dk = sK0 + (uint32_t)stage * 2 * kTileBytes;
    const uint32_t dv = dk + kTileBytes;
    for (int i = tid; i < kPBN * 16; i += nthreads) {
      const int r = i >> 4, c = i & 15;
      int key = tile * kPBN + r;
      if (key >= kv_end) key = kv_end - 1;  // clamp: masked below, stays finite
      const int page = bt[key / kPPage];
      const __nv_bfloat16* base = cache + (size_t)page * page_stride + head_off + (size_t)(key % kPPage) * kPD + c * 8;
      cp_async16(dk + swz(r, c), base);
      cp_async16(dv + swz(r, c), base + half_stride);
    }
  };
#pragma unroll
  for (int s = 0; s < kPStages - 1; ++s) {
    if (s < n_tiles) load_kv(s, s);
    cp_async_commit();
  }

  const int g = lane >> 2;
  const int tq = lane & 3;
  const int qpos0 = start + q0 + g;
  const int qpos1 = qpos0 + 8;
  const int warp_kv_end = min(kv_end, start + q0 + 16);  // keys this warp can see at all

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -FLT_MAX, m1 = -FLT_MAX, l0 = 0.f, l1 = 0.f;

  uint32_t qa[8][4];
  for (int t = 0; t < n_tiles; ++t) {
    if (t + kPStages - 1 < n_tiles) load_kv(t + kPStages - 1, (t + kPStages - 1) % kPStages);
    cp_async_commit();
    cp_async_wait<kPStages - 1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int r = lane & 15;
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4p(sQ + swz(r, c), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
      }
    }
    const int kbase = t * kPBN;
    if (kbase < warp_kv_end) {  // tiles entirely past this warp's causal horizon are skipped
      const uint32_t sK = sK0 + (uint32_t)(t % kPStages) * 2 * kTileBytes;
      const uint32_t sV = sK + kTileBytes;
      float sc[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const int r = jp * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int c = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4p(sK + swz(r, c), b0, b1, b2, b3);
          mma16816p(sc[2 * jp], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
          mma16816p(sc[2 * jp + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
        }
      }
      float mx0 = -FLT_MAX, mx1 = -FLT_MAX;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kp = kbase + j * 8 + 2 * tq + e;
          float v0 = sc[j][e] * scale_log2;
          float v1 = sc[j][2 + e] * scale_log2;
          if (kp > qpos0 || kp >= kv_end) v0 = -FLT_MAX;
          if (kp > qpos1 || kp >= kv_end) v1 = -FLT_MAX;
          sc[j][e] = v0;
          sc[j][2 + e] = v1;
          mx0 = fmaxf(mx0, v0);
          mx1 = fmaxf(mx1, v1);
        }
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float a0 = (mn0 == -FLT_MAX) ? 1.f : exp2f(m0 - mn0);
      const float a1 = (mn1 == -FLT_MAX) ? 1.f : exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      float ps0 = 0.f, ps1 = 0.f;
      uint32_t pa[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float p00 = (sc[j][0] == -FLT_MAX) ? 0.f : exp2f(sc[j][0] - mn0);
        const float p01 = (sc[j][1] == -FLT_MAX) ? 0.f : exp2f(sc[j][1] - mn0);
        const float p10 = (sc[j][2] == -FLT_MAX) ? 0.f : exp2f(sc[j][2] - mn1);
        const float p11 = (sc[j][3] == -FLT_MAX) ? 0.f : exp2f(sc[j][3] - mn1);
        ps0 += p00 + p01;
        ps1 += p10 + p11;
        pa[j][0] = pack_bf16x2(p00, p01);
        pa[j][1] = pack_bf16x2(p10, p11);
      }
      l0 = l0 * a0 + ps0;
      l1 = l1 * a1 + ps1;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        o[i][0] *= a0;
        o[i][1] *= a0;
        o[i][2] *= a1;
        o[i][3] *= a1;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t A0 = pa[2 * kk][0], A1 = pa[2 * kk][1], A2 = pa[2 * kk + 1][0], A3 = pa[2 * kk + 1][1];
#pragma unroll
        for (int dp = 0; dp < 8; ++dp) {
          const int r = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int c = dp * 2 + (lane >> 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4p_t(sV + swz(r, c), b0, b1, b2, b3);
          mma16816p(o[2 * dp], A0, A1, A2, A3, b0, b1);
          mma16816p(o[2 * dp + 1], A0, A1, A2, A3, b2, b3);
        }
      }
    }
    __syncthreads();  // stage (t % kPStages) is refilled at iteration t+1
  }
  cp_async_wait<0>();
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
  const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int row0 = q0 + g;
  const int row1 = row0 + 8;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int d = i * 8 + 2 * tq;
    if (row0 < T)
      *reinterpret_cast<uint32_t*>(out + (size_t)row0 * out_tok_stride + (size_t)hq * kPD + d) =
          pack_bf16x2(o[i][0] * inv0, o[i][1] * inv0);
    if (row1 < T)
      *reinterpret_cast<uint32_t*>(out + (size_t)row1 * out_tok_stride + (size_t)hq * kPD + d) =
          pack_bf16x2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

int prefill_attention_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* bt, int T,
                             int start, int Hq, int Hkv, int head_dim, void* out, long long out_tok_stride,
                             float scale, cudaStream_t st) {
  if (T <= 0) return 0;
  if (head_dim != kPD) return set_error("prefill attention: head_dim must be 128");
  if (Hkv <= 0 || Hq % Hkv != 0) return set_error("prefill attention: bad head counts");
  const int G = Hq / Hkv;
  if (G > kPMaxWarps) return set_error("prefill attention: GQA group > 8 unsupported");
  int PB = kPMaxWarps / G;  // 16-position blocks per CTA
  if (PB < 1) PB = 1;
  const int nwarps = G * PB;
  const int smem = nwarps * 16 * kRowBytes + kPStages * 2 * kTileBytes;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kPMaxWarps * 16 * kRowBytes + kPStages * 2 * kTileBytes);
    if (e != cudaSuccess) return set_cuda_error("prefill attn smem attr", e);
    attr = true;
  }
  dim3 grid((T + 16 * PB - 1) / (16 * PB), Hkv);
  cudaError_t e = launch_k(prefill_attn_kernel, dim3(grid), dim3(nwarps * 32), smem, st, 1, (const __nv_bfloat16*)q, q_tok_stride, (const __nv_bfloat16*)cache_layer, bt, T, start, Hq, Hkv, PB, (__nv_bfloat16*)out, out_tok_stride, scale * 1.4426950408889634f);
  if (e != cudaSuccess) return set_cuda_error("prefill attn launch", e);
  return 0;
}

}  // namespace rb
