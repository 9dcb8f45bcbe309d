// K5: the small fused ops around the GEMMs and attention. Together they are
// the device-side part of `fixed_iteration_overhead_us` ("sampling,
// bookkeeping kernels", reference pkg/src/pdsim/costmodel.py:44,53,83) plus
// the KV write term kv_cache_bytes(model, tokens) of prefill_time
// (costmodel.py:105) / kv_cache_bytes(model, batch) of decode_time (:132).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cfloat>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

// ------------------------------------------------------------------ RMSNorm
// y = x * rsqrt(mean(x^2) + eps) * w   (fp32 math, bf16 io), one CTA per row.
__global__ void rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, long long ldx, const __nv_bfloat16* __restrict__ w,
                               __nv_bfloat16* __restrict__ y, long long ldy, int H, float eps) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const __nv_bfloat16* xr = x + (size_t)row * ldx;
  __nv_bfloat16* yr = y + (size_t)row * ldy;
  float ss = 0.f;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    uint4 u = *reinterpret_cast<const uint4*>(xr + i);
    const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(wv[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)H + eps);
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    uint4 u = *reinterpret_cast<const uint4*>(xr + i);
    uint4 wu = *reinterpret_cast<const uint4*>(w + i);
    const uint32_t xv[4] = {u.x, u.y, u.z, u.w};
    const uint32_t ww[4] = {wu.x, wu.y, wu.z, wu.w};
    uint32_t ov[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(xv[j]);
      float2 g = unpack_bf16x2(ww[j]);
      ov[j] = pack_bf16x2(f.x * inv * g.x, f.y * inv * g.y);
    }
    *reinterpret_cast<uint4*>(yr + i) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
  }
}

int rmsnorm_launch(const void* x, long long ldx, const void* w, void* y, long long ldy, int T, int H, float eps,
                   cudaStream_t st) {
  if (T <= 0) return 0;
  if (H % 8) return set_error("rmsnorm: H must be a multiple of 8");
  int threads = H / 8;
  if (threads > 1024) threads = 1024;
  threads = ((threads + 31) / 32) * 32;
  cudaError_t e = launch_k(rmsnorm_kernel, dim3(T), dim3(threads), 0, st, 1, (const __nv_bfloat16*)x, ldx, (const __nv_bfloat16*)w, (__nv_bfloat16*)y, ldy, H, eps);
  return e == cudaSuccess ? 0 : set_cuda_error("rmsnorm launch", e);
}

// Consumer of a K-sliced decode GEMM (O / down projection, gemm mode bit 16): the residual
// stream row x[t] += sum over slices s (in order) of the fp32 partial P[s][t][:], rounded to
// bf16 and written back, then y[t] = rmsnorm(x[t]) * w — the split-K reduction rides on the
// RMSNorm that follows anyway (no finisher SM in the GEMM). The sum of squares is taken over
// the rounded row, as rmsnorm_kernel reads it.
__global__ void add_partials_rmsnorm_kernel(const float* __restrict__ part, int ks, long long slice,
                                            __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                                            __nv_bfloat16* __restrict__ y, int H, float eps) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) uint8_t rowbuf[];  // the updated row, bf16
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(rowbuf);
  const int row = blockIdx.x;
  __nv_bfloat16* xr = x + (size_t)row * H;
  float ss = 0.f;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(xr + i);
    const uint32_t xv[4] = {u.x, u.y, u.z, u.w};
    float a[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(xv[j]);
      a[2 * j] = f.x;
      a[2 * j + 1] = f.y;
    }
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int sl = 0; sl < ks; ++sl) {
      const float4* pp = reinterpret_cast<const float4*>(part + sl * slice + (size_t)row * H + i);
      const float4 p0 = __ldcg(pp), p1 = __ldcg(pp + 1);
      acc[0] += p0.x; acc[1] += p0.y; acc[2] += p0.z; acc[3] += p0.w;
      acc[4] += p1.x; acc[5] += p1.y; acc[6] += p1.z; acc[7] += p1.w;
    }
    uint32_t ov[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ov[j] = pack_bf16x2(a[2 * j] + acc[2 * j], a[2 * j + 1] + acc[2 * j + 1]);
      const float2 r = unpack_bf16x2(ov[j]);
      ss += r.x * r.x + r.y * r.y;
    }
    const uint4 o4 = make_uint4(ov[0], ov[1], ov[2], ov[3]);
    *reinterpret_cast<uint4*>(xr + i) = o4;
    *reinterpret_cast<uint4*>(xs + i) = o4;
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)H + eps);
  __nv_bfloat16* yr = y + (size_t)row * H;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(xs + i);
    const uint4 wu = *reinterpret_cast<const uint4*>(w + i);
    const uint32_t xv[4] = {u.x, u.y, u.z, u.w};
    const uint32_t ww[4] = {wu.x, wu.y, wu.z, wu.w};
    uint32_t ov[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(xv[j]);
      const float2 g = unpack_bf16x2(ww[j]);
      ov[j] = pack_bf16x2(f.x * inv * g.x, f.y * inv * g.y);
    }
    *reinterpret_cast<uint4*>(yr + i) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
  }
}

int add_partials_rmsnorm_launch(const float* part, int ks, long long slice, void* x, const void* w, void* y, int T,
                                int H, float eps, cudaStream_t st) {
  if (T <= 0) return 0;
  if (H % 8 || ks < 1) return set_error("add_partials_rmsnorm: H % 8 == 0, ks >= 1");
  int threads = H / 8;
  if (threads > 1024) threads = 1024;
  threads = ((threads + 31) / 32) * 32;
  cudaError_t e = launch_k(add_partials_rmsnorm_kernel, dim3(T), dim3(threads), (size_t)H * 2, st, 1, part, ks, slice,
                           (__nv_bfloat16*)x, (const __nv_bfloat16*)w, (__nv_bfloat16*)y, H, eps);
  return e == cudaSuccess ? 0 : set_cuda_error("add_partials_rmsnorm launch", e);
}

// ------------------------------------------------------------------ RoPE + paged KV write
// qkv row layout: [Hq*D | Hkv*D | Hkv*D]. Rotates q and k (neox / rotate_half
// pairing i <-> i+D/2) at position pos[t], writes q to q_out and k, v into the
// paged cache page bt[slot][pos/16], row pos%16. Rows with pos < 0 are skipped.
// cos_sin: [max_pos][D] fp32 = [cos(0..D/2) | sin(0..D/2)].
__global__ void rope_cache_kernel(const __nv_bfloat16* __restrict__ qkv, long long ld_qkv,
                                  const int* __restrict__ pos, const int* __restrict__ tok_slot,
                                  const int* __restrict__ block_table, int bt_stride,
                                  const float* __restrict__ cos_sin, __nv_bfloat16* __restrict__ q_out,
                                  long long ld_q, __nv_bfloat16* __restrict__ cache, int Hq, int Hkv, int D) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const int p = pos[t];
  if (p < 0) return;
  const int half = D / 2;
  const __nv_bfloat16* row = qkv + (size_t)t * ld_qkv;
  const float* cs = cos_sin + (size_t)p * D;
  const int* bt = block_table + (size_t)tok_slot[t] * bt_stride;
  const int page = bt[p >> 4];
  const int off = p & 15;
  const size_t half_stride = (size_t)Hkv * 16 * D;
  __nv_bfloat16* kdst = cache + (size_t)page * 2 * half_stride + (size_t)off * D;
  // q and k heads: each thread handles one rotation pair (i, i+half)
  const int pairs = (Hq + Hkv) * half;
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int h = i / half;
    const int j = i % half;
    const float c = cs[j], s = cs[half + j];
    const __nv_bfloat16* src = row + (size_t)h * D;
    const float x0 = __bfloat162float(src[j]);
    const float x1 = __bfloat162float(src[j + half]);
    const __nv_bfloat16 r0 = __float2bfloat16_rn(x0 * c - x1 * s);
    const __nv_bfloat16 r1 = __float2bfloat16_rn(x1 * c + x0 * s);
    if (h < Hq) {
      __nv_bfloat16* qd = q_out + (size_t)t * ld_q + (size_t)h * D;
      qd[j] = r0;
      qd[j + half] = r1;
    } else {
      __nv_bfloat16* kd = kdst + (size_t)(h - Hq) * 16 * D;
      kd[j] = r0;
      kd[j + half] = r1;
    }
  }
  // v: straight copy, 16 bytes per thread
  const __nv_bfloat16* vsrc = row + (size_t)(Hq + Hkv) * D;
  const int vchunks = Hkv * D / 8;
  for (int i = threadIdx.x; i < vchunks; i += blockDim.x) {
    const int h = (i * 8) / D;
    const int d = (i * 8) % D;
    *reinterpret_cast<uint4*>(kdst + half_stride + (size_t)h * 16 * D + d) =
        *reinterpret_cast<const uint4*>(vsrc + (size_t)i * 8);
  }
}

int rope_cache_launch(const void* qkv, long long ld_qkv, const int* pos, const int* tok_slot, const int* bt,
                      int bt_stride, const float* cos_sin, void* q_out, long long ld_q, void* cache_layer, int T,
                      int Hq, int Hkv, int D, cudaStream_t st) {
  if (T <= 0) return 0;
  if (D % 8) return set_error("rope: head dim must be a multiple of 8");
  cudaError_t e = launch_k(rope_cache_kernel, dim3(T), dim3(256), 0, st, 1, (const __nv_bfloat16*)qkv, ld_qkv, pos, tok_slot, bt, bt_stride, cos_sin, (__nv_bfloat16*)q_out, ld_q, (__nv_bfloat16*)cache_layer, Hq, Hkv, D);
  return e == cudaSuccess ? 0 : set_cuda_error("rope launch", e);
}

// ------------------------------------------------------------------ SiLU(gate) * up
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, long long ld_gu, __nv_bfloat16* __restrict__ y,
                                long long ldy, int I) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i >= I) return;
  const __nv_bfloat16* g = gu + (size_t)t * ld_gu;
  uint4 a = *reinterpret_cast<const uint4*>(g + i);
  uint4 b = *reinterpret_cast<const uint4*>(g + I + i);
  const uint32_t av[4] = {a.x, a.y, a.z, a.w};
  const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
  uint32_t ov[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 x = unpack_bf16x2(av[j]);
    float2 u = unpack_bf16x2(bv[j]);
    const float s0 = x.x / (1.f + __expf(-x.x));
    const float s1 = x.y / (1.f + __expf(-x.y));
    ov[j] = pack_bf16x2(s0 * u.x, s1 * u.y);
  }
  *reinterpret_cast<uint4*>(y + (size_t)t * ldy + i) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
}

int silu_mul_launch(const void* gu, long long ld_gu, void* y, long long ldy, int T, int I, cudaStream_t st) {
  if (T <= 0) return 0;
  if (I % 8) return set_error("silu_mul: I must be a multiple of 8");
  dim3 grid((I / 8 + 255) / 256, T);
  cudaError_t e = launch_k(silu_mul_kernel, dim3(grid), dim3(256), 0, st, 1, (const __nv_bfloat16*)gu, ld_gu, (__nv_bfloat16*)y, ldy, I);
  return e == cudaSuccess ? 0 : set_cuda_error("silu_mul launch", e);
}

// Same for gate|up columns interleaved in 16-blocks [g x16 | u x16] (the layout the
// fused-SwiGLU GEMM epilogue expects); used where the GEMM runs unfused (decode).
__global__ void silu_mul_il_kernel(const __nv_bfloat16* __restrict__ gu, long long ld_gu,
                                   __nv_bfloat16* __restrict__ y, long long ldy, int I) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) * 8;  // 8 features, inside one 16-block
  if (f >= I) return;
  const __nv_bfloat16* g = gu + (size_t)t * ld_gu + (size_t)(f >> 4) * 32 + (f & 15);
  uint4 a = *reinterpret_cast<const uint4*>(g);
  uint4 b = *reinterpret_cast<const uint4*>(g + 16);
  const uint32_t av[4] = {a.x, a.y, a.z, a.w};
  const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
  uint32_t ov[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 x = unpack_bf16x2(av[j]);
    float2 u = unpack_bf16x2(bv[j]);
    ov[j] = pack_bf16x2(x.x / (1.f + __expf(-x.x)) * u.x, x.y / (1.f + __expf(-x.y)) * u.y);
  }
  *reinterpret_cast<uint4*>(y + (size_t)t * ldy + f) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
}

int silu_mul_interleaved_launch(const void* gu, long long ld_gu, void* y, long long ldy, int T, int I,
                                cudaStream_t st) {
  if (T <= 0) return 0;
  if (I % 16) return set_error("silu_mul_interleaved: I must be a multiple of 16");
  dim3 grid((I / 8 + 255) / 256, T);
  cudaError_t e = launch_k(silu_mul_il_kernel, dim3(grid), dim3(256), 0, st, 1, (const __nv_bfloat16*)gu, ld_gu, (__nv_bfloat16*)y, ldy, I);
  return e == cudaSuccess ? 0 : set_cuda_error("silu_mul_interleaved launch", e);
}

// ------------------------------------------------------------------ embedding gather
// ids come either from `ids` directly or, when `slot_of_row` is given, from
// the per-slot device state last_tok[slot] (decode: the previous step's
// sampled token never leaves the device).
__global__ void embed_kernel(const int* __restrict__ ids, const int* __restrict__ slot_of_row,
                             const int* __restrict__ last_tok, const __nv_bfloat16* __restrict__ table,
                             __nv_bfloat16* __restrict__ y, int H, int* __restrict__ ids_out) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const int id = slot_of_row ? last_tok[slot_of_row[t]] : ids[t];
  if (threadIdx.x == 0 && ids_out) ids_out[t] = id;
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)id * H);
  uint4* dst = reinterpret_cast<uint4*>(y + (size_t)t * H);
  for (int i = threadIdx.x; i < H / 8; i += blockDim.x) dst[i] = src[i];
}

int embed_launch(const int* ids, const int* slot_of_row, const int* last_tok, const void* table, void* y, int T, int H,
                 int* ids_out, cudaStream_t st) {
  if (T <= 0) return 0;
  cudaError_t e = launch_k(embed_kernel, dim3(T), dim3(128), 0, st, 1, ids, slot_of_row, last_tok, (const __nv_bfloat16*)table, (__nv_bfloat16*)y, H, ids_out);
  return e == cudaSuccess ? 0 : set_cuda_error("embed launch", e);
}

// ------------------------------------------------------------------ argmax (greedy sampling)
// One CTA per row; ties resolve to the lowest index (torch.argmax semantics).
// Optionally scatters the winner into last_tok[slot_of_row[row]].
__global__ void argmax_kernel(const __nv_bfloat16* __restrict__ logits, long long ld, int V, int* __restrict__ out,
                              const int* __restrict__ slot_of_row, int* __restrict__ last_tok,
                              const int* __restrict__ row_valid) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  if (row_valid && row_valid[row] <= 0) return;
  const __nv_bfloat16* x = logits + (size_t)row * ld;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x * 8; i < V; i += blockDim.x * 8) {
    if (i + 8 <= V) {
      uint4 u = *reinterpret_cast<const uint4*>(x + i);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = unpack_bf16x2(w[j]);
        if (f.x > best) { best = f.x; bi = i + 2 * j; }
        if (f.y > best) { best = f.y; bi = i + 2 * j + 1; }
      }
    } else {
      for (int j = i; j < V; ++j) {
        float f = __bfloat162float(x[j]);
        if (f > best) { best = f; bi = j; }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) { sb[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = threadIdx.x < nw ? sb[threadIdx.x] : -FLT_MAX;
    bi = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (threadIdx.x == 0) {
      out[row] = bi;
      if (slot_of_row && last_tok) last_tok[slot_of_row[row]] = bi;
    }
  }
}

int argmax_launch(const void* logits, long long ld, int T, int V, int* out, const int* slot_of_row, int* last_tok,
                  const int* row_valid, cudaStream_t st) {
  if (T <= 0) return 0;
  if (V % 8 || ld % 8) return set_error("argmax: V and ld must be multiples of 8");
  cudaError_t e = launch_k(argmax_kernel, dim3(T), dim3(512), 0, st, 1, (const __nv_bfloat16*)logits, ld, V, out, slot_of_row, last_tok, row_valid);
  return e == cudaSuccess ? 0 : set_cuda_error("argmax launch", e);
}

// ------------------------------------------------------------------ block-table / slot-state updates
// upd = [count, (slot, index, block) x count]; applied on device so a decode
// graph replay only needs a small H2D copy of the step's new pages.
__global__ void bt_update_kernel(const int* __restrict__ upd, int* __restrict__ block_table, int bt_stride) {
  pdl_trigger();
  pdl_wait();
  const int n = upd[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int slot = upd[1 + 3 * i];
    const int idx = upd[2 + 3 * i];
    const int blk = upd[3 + 3 * i];
    block_table[(size_t)slot * bt_stride + idx] = blk;
  }
}

int bt_update_launch(const int* upd, int* block_table, int bt_stride, int max_updates, cudaStream_t st) {
  int threads = 256;
  int blocks = (max_updates + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  cudaError_t e = launch_k(bt_update_kernel, dim3(blocks), dim3(threads), 0, st, 1, upd, block_table, bt_stride);
  return e == cudaSuccess ? 0 : set_cuda_error("bt_update launch", e);
}

// set last_tok[slot] = value (prefill completion hands the next input token to decode)
__global__ void set_last_tok_kernel(int* last_tok, int slot, const int* value_ptr, int value) {
  pdl_trigger();
  pdl_wait();
  last_tok[slot] = value_ptr ? *value_ptr : value;
}

int set_last_tok_launch(int* last_tok, int slot, const int* value_ptr, int value, cudaStream_t st) {
  cudaError_t e = launch_k(set_last_tok_kernel, dim3(1), dim3(1), 0, st, 1, last_tok, slot, value_ptr, value);
  return e == cudaSuccess ? 0 : set_cuda_error("set_last_tok launch", e);
}

}  // namespace rb
