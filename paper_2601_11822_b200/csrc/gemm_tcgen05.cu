// K1 / K4: bf16 "linear" GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   Y[t, o] = sum_k X[t, k] * W[o, k]  (+ bias[o]) (+ R[t, o])
//
// Realizes the compute term of prefill_time / the weight term of decode_time
// (reference pkg/src/pdsim/costmodel.py:104 and :130).
//
// Two operand mappings onto the UMMA tile (M rows x N=BN columns):
//   normal  (prefill, many tokens): MMA-M = tokens t, MMA-N = features o.
//   swap-AB (decode, M=B <= 256):   MMA-M = features o, MMA-N = tokens t,
//            so the tiny batch becomes the UMMA N dimension and the weight
//            matrix streams through the A operand (HBM-bound path).
// Both operands are K-major; TMA loads 64-element (128 B) K slabs with the
// 128B swizzle straight into the UMMA smem layout.
//
// kPair = 2 (default): a cluster of two CTAs on an SM pair computes a 256-row
// tile with tcgen05.mma.cta_group::2 — each CTA stages 128 rows of A and BN/2
// rows of B (32 KB per 64-wide k-block instead of 48 KB for a 1-CTA 128x256
// tile), the leader issues the MMAs, both CTAs hold half the accumulator in
// their TMEM. kPair = 1 keeps the single-CTA M=128 kernel.
//
// Warp roles (192 threads/CTA): w0 = TMA producer, w1 = TMEM owner + MMA issuer
// (leader CTA), w2..w5 = epilogue. Persistent grid, static stride schedule over
// work units (tile x K-split), 2 TMEM accumulators so the epilogue of unit i
// overlaps the MMAs of unit i+1. Epilogue: TMEM -> registers -> per-warp smem
// tile in OUTPUT orientation -> 16-byte coalesced stores with bias / residual
// fused. Split-K (decode only): fp32 partials in lane-major order, the last
// arriving split sums all splits in fixed order (deterministic).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

constexpr int kBM = 128;                // rows of A per CTA
constexpr int kBK = 64;                 // bf16 elements per 128-byte swizzle row
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
// Epilogue warp sets (template kSets): each TMEM quadrant is drained by kSets warps taking
// alternate 32-column chunks. Decode (swap-AB) GEMMs are short and their split-tile epilogue
// is on the critical path: 2 sets; prefill GEMMs overlap the epilogue with the next tile's
// MMAs: 1 set (192 threads: producer, MMA, 4 epilogue warps; no register cap).
// The 2-set kernel runs 384 threads as three warpgroups: WG0 = producer, MMA issuer and two
// idle warps, which give their registers back (setmaxnreg.dec 56) so the epilogue warpgroups
// WG1/WG2 run at 224 registers instead of the 168 a flat 384-thread launch allows (the flat
// 320-thread layout spilled ~210 bytes per thread in the split-tile accumulate).
constexpr int threads_for(int sets) { return sets == 2 ? 384 : 64 + 128 * sets; }
constexpr int epi_first_warp(int sets) { return sets == 2 ? 4 : 2; }
constexpr int kMaxEpiWarps = 8;
constexpr int kStgStride = 40;          // bf16 per staging row (32 + 8 pad, 80 B)
constexpr int kStgBytes = 32 * kStgStride * 2;  // per epilogue warp

struct GemmArgs {
  int m_tiles, n_tiles, num_kb, total_tiles;
  int streamk;     // 1: stream-K — each cluster owns an equal run of the (tile, k-block) iterations
  int total_iters; // total_tiles * num_kb
  int mt;          // A sub-tiles of kBM*kPair rows per tile, sharing one B stage
  int nacc;        // TMEM accumulator buffers (2: epilogue of segment i overlaps MMAs of i+1)
  int kacc;        // independent K-interleaved accumulators per buffer (MMA kk -> kk % kacc), summed
                   // in the epilogue: breaks the serial dependence of skinny (small-N) MMAs
  int BN, stages;
  int a_blocked;   // A (swap: the weight) stored as [rows/128][num_kb][128][64] contiguous 16 KB blocks
  int pf_dist;     // k-blocks of A to warm in L2 ahead of the smem ring (0 = off)
  int dbg;         // debug (kPair 1 only): 1 = skip the MMAs, 2 = skip the TMA loads
  int M_valid, N_valid;  // extents in MMA space
  int swap;              // 1: MMA-M = features (output columns), MMA-N = tokens (output rows)
  int glu;               // 1: W rows are [gate x16 | up x16] blocks; Y = silu(gate) * up, width O/2
  long long ldy;
  __nv_bfloat16* out;
  const __nv_bfloat16* residual;
  const __nv_bfloat16* bias;
  uint64_t hint_a, hint_b;
  float* ws;      // stream-K partials [cluster][rank][mt][BN/32][4 warps][8][32 lanes] float4
  int* counters;  // per (tile, rank), self-resetting
  GemmRope rp;    // rp.q_out != nullptr: fused RoPE + paged K/V write epilogue (QKV projection)
  GemmPush push;  // push.world > 0: tiles go to every TP rank's receive slot (tp.cu mode 3)
  unsigned long long* trace;  // debug timeline: [cta][8] globaltimer stamps of this launch, or null
  int ksplit;        // > 1 (decode): units = tiles x ksplit K-slices, each writes an fp32 partial slice
  float* part;       // ksplit partials [ksplit][N_valid tokens][M_valid features] (swap orientation)
  long long part_slice;  // floats per slice
};

// Work schedule shared by the producer, MMA and epilogue roles. Data-parallel: whole
// tiles, strided over clusters. Stream-K: cluster c owns iterations
// [c*I/G, (c+1)*I/G) of the flattened (tile, k-block) space and walks them from the
// end, so a tile split between clusters c_first..c_last is reached FIRST by c_first..
// c_last-1 (their runs end in it: they publish fp32 partials early) and LAST by c_last
// (its run starts in it): c_last is the finisher. It waits only on lower-numbered
// clusters, which are dispatched first, so the spin cannot deadlock even when the grid
// is not fully co-resident; the sum order is fixed (deterministic for a partition size).
__device__ __forceinline__ int sk_start(const GemmArgs& g, int c, int ncl) {
  return (int)(((long long)c * g.total_iters) / ncl);
}
// first cluster whose run contains iteration x
__device__ __forceinline__ int sk_owner(const GemmArgs& g, int x, int ncl) {
  return (int)((((long long)x + 1) * ncl - 1) / g.total_iters);
}
struct SegIter {
  int lo, it;   // stream-K: this cluster's run [lo, it), walked from the END (descending)
  int t, step;  // data-parallel cursor (units = tiles x ksplit)
  int slice;    // K-slice of the current unit (ksplit > 1)
  __device__ __forceinline__ SegIter(const GemmArgs& g, int cid, int ncl) {
    lo = sk_start(g, cid, ncl);
    it = sk_start(g, cid + 1, ncl);
    t = cid;
    step = ncl;
    slice = 0;
  }
  __device__ __forceinline__ bool next(const GemmArgs& g, int& tile, int& kb0, int& kb1) {
    if (g.streamk) {
      if (it <= lo) return false;
      tile = (it - 1) / g.num_kb;
      const int base = tile * g.num_kb;
      const int seg_lo = max(lo, base);
      kb0 = seg_lo - base;
      kb1 = it - base;
      it = seg_lo;
      return true;
    }
    if (t >= g.total_tiles * g.ksplit) return false;
    tile = t % g.total_tiles;
    slice = t / g.total_tiles;
    kb0 = (int)(((long long)slice * g.num_kb) / g.ksplit);
    kb1 = (int)(((long long)(slice + 1) * g.num_kb) / g.ksplit);
    t += step;
    return true;
  }
};

// Optional timeline trace (debug): per CTA 16 globaltimer stamps; consecutive launches
// after rb_debug_gemm_trace(buf) go to buf + (i % 16) * 148 * 16 (absolute times, so a
// chain of PDL-overlapped launches can be laid side by side).
static unsigned long long* g_trace_host = nullptr;
static unsigned g_trace_launch = 0;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// `trace` is a kernel-local copy of g_gemm_trace, read once: a global read inside the
// pipelined loops would be re-issued every k-block (the barrier asm clobbers memory).
#define TRACE(slot)                                           \
  do {                                                        \
    if (trace) trace[blockIdx.x * 16 + (slot)] = gtime();    \
  } while (0)

// Fused QKV epilogue readback: this lane's 8 columns [col, col+8) of 4 token rows.
// q|k heads arrive with their RoPE pairs adjacent (pair-interleaved weight rows, see
// model.interleave_rope_pairs: column 2j <-> rotate-half dim j, 2j+1 <-> dim j+64), so
// the rotation is local to the 8 values; q goes to q_out, k/v straight into the token's
// paged cache slot [page][K|V][kv-head][pos & 15][128]. Rows with pos < 0 (padding) skip.
__device__ __forceinline__ void rope_readback(const GemmArgs& g, const __nv_bfloat16* stg, int lane, int row0,
                                              int col, int rows_valid) {
  const GemmRope& r = g.rp;
  const int head = col >> 7;  // uniform over the 4 rows this lane handles
  const int d = col & 127;
  const bool rot = head < r.hq + r.hkv;
  const bool is_q = head < r.hq;
  const int is_v = head >= r.hq + r.hkv ? 1 : 0;
  const int hk = head - r.hq - is_v * r.hkv;
  // dependent loads batched over the 4 rows: pos/slot -> cos,sin / block-table page
  int p[4], sl[4], page[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = row0 + i * 8 + (lane >> 2);
    p[i] = row < rows_valid ? __ldg(r.pos + row) : -1;
    sl[i] = is_q ? 0 : __ldg(r.tok_slot + min(row, rows_valid - 1));
  }
  float4 c[4], sn[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pp = max(p[i], 0);
    if (rot) {
      const float* t = r.cos_sin + (size_t)pp * 128 + (d >> 1);
      c[i] = __ldg(reinterpret_cast<const float4*>(t));
      sn[i] = __ldg(reinterpret_cast<const float4*>(t + 64));
    }
    page[i] = is_q ? 0 : __ldg(r.block_table + (size_t)sl[i] * r.bt_stride + (pp >> 4));
  }
  float bv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) bv[j] = 0.f;
  if (g.bias) {
    const uint4 b = *reinterpret_cast<const uint4*>(g.bias + col);
    const uint32_t w[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(w[j]);
      bv[2 * j] = f.x;
      bv[2 * j + 1] = f.y;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (p[i] < 0) continue;
    const int rl = i * 8 + (lane >> 2);
    const uint4 sv = *reinterpret_cast<const uint4*>(stg + rl * kStgStride + (lane & 3) * 8);
    const uint32_t w[4] = {sv.x, sv.y, sv.z, sv.w};
    float x[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16x2(w[j]);
      x[2 * j] = f.x + bv[2 * j];
      x[2 * j + 1] = f.y + bv[2 * j + 1];
    }
    if (rot) {
      const float cc[4] = {c[i].x, c[i].y, c[i].z, c[i].w};
      const float ss[4] = {sn[i].x, sn[i].y, sn[i].z, sn[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x0 = x[2 * j], x1 = x[2 * j + 1];
        x[2 * j] = x0 * cc[j] - x1 * ss[j];
        x[2 * j + 1] = x1 * cc[j] + x0 * ss[j];
      }
    }
    const int row = row0 + rl;
    __nv_bfloat16* dst =
        is_q ? static_cast<__nv_bfloat16*>(r.q_out) + (long long)row * r.ld_q + col
             : static_cast<__nv_bfloat16*>(r.cache) + (((size_t)page[i] * 2 + is_v) * r.hkv + hk) * (16 * 128) +
                   (size_t)(p[i] & 15) * 128 + d;
    *reinterpret_cast<uint4*>(dst) = make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]),
                                                pack_bf16x2(x[4], x[5]), pack_bf16x2(x[6], x[7]));
  }
}

// One warp's 32 (MMA rows) x 32 (MMA cols) accumulator block -> Y.
// The residual / bias vectors this lane adds come preloaded (epi_preload), all four rows
// at once and one 32-column chunk ahead: R may alias Y (in-place residual), so loads
// interleaved with the stores would serialize into dependent L2 round trips.
struct EpiPre {
  uint4 rr[4];  // residual, rows i*8 + lane/4
  uint4 bb;     // bias
};

__device__ __forceinline__ void epi_preload(const GemmArgs& g, int lane, int m0, int n0, EpiPre& pre) {
  const int row0 = g.swap ? n0 : m0;
  const int col = (g.swap ? m0 : n0) + (lane & 3) * 8;
  const int rows_valid = g.swap ? g.N_valid : g.M_valid;
  const int cols_valid = g.swap ? g.M_valid : g.N_valid;
#pragma unroll
  for (int i = 0; i < 4; ++i) pre.rr[i] = make_uint4(0, 0, 0, 0);
  pre.bb = make_uint4(0, 0, 0, 0);
  if (g.rp.q_out || g.glu || col + 8 > cols_valid) return;
  if (g.bias) pre.bb = *reinterpret_cast<const uint4*>(g.bias + col);
  if (g.residual) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = row0 + i * 8 + (lane >> 2);
      if (row < rows_valid) pre.rr[i] = *reinterpret_cast<const uint4*>(g.residual + (long long)row * g.ldy + col);
    }
  }
}

__device__ __forceinline__ void epi_block(const GemmArgs& g, __nv_bfloat16* stg, int lane, int m0, int n0,
                                          const uint32_t (&v)[32], const EpiPre& pre, bool tstamp = false) {
  const int row0 = g.swap ? n0 : m0;  // output row (token) base
  const int col0 = g.swap ? m0 : n0;  // output col (feature) base
  const int rows_valid = g.swap ? g.N_valid : g.M_valid;
  const int cols_valid = g.swap ? g.M_valid : g.N_valid;
  const int cs = (lane & 3) * 8;
  const int col = col0 + cs;
  const bool vec = col + 8 <= cols_valid;
  const uint4* rr = pre.rr;
  const uint4 bb = pre.bb;
  if (!g.swap) {
    uint4* dst = reinterpret_cast<uint4*>(stg + lane * kStgStride);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      dst[k] = make_uint4(pack_bf16x2(__uint_as_float(v[8 * k + 0]), __uint_as_float(v[8 * k + 1])),
                          pack_bf16x2(__uint_as_float(v[8 * k + 2]), __uint_as_float(v[8 * k + 3])),
                          pack_bf16x2(__uint_as_float(v[8 * k + 4]), __uint_as_float(v[8 * k + 5])),
                          pack_bf16x2(__uint_as_float(v[8 * k + 6]), __uint_as_float(v[8 * k + 7])));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[j * kStgStride + lane] = __float2bfloat16_rn(__uint_as_float(v[j]));
  }
  __syncwarp();
  if (tstamp && lane == 0 && g.trace) g.trace[blockIdx.x * 16 + 15] = gtime();
  if (g.rp.q_out) {
    rope_readback(g, stg, lane, row0, col, rows_valid);
    __syncwarp();
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i * 8 + (lane >> 2);
    const int row = row0 + r;
    if (row >= rows_valid || col >= cols_valid) continue;
    const uint4 sv = *reinterpret_cast<const uint4*>(stg + r * kStgStride + cs);
    float x[8];
    {
      const uint32_t w[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = unpack_bf16x2(w[j]);
        x[2 * j] = f.x;
        x[2 * j + 1] = f.y;
      }
    }
    __nv_bfloat16* dst = g.out + (long long)row * g.ldy + col;
    if (g.dbg & 4) {
      if (x[0] == 12345.f) dst[0] = __float2bfloat16_rn(x[1]);  // keep the math alive
      continue;
    }
    if (vec) {
      if (g.bias) {
        const uint32_t w[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = unpack_bf16x2(w[j]);
          x[2 * j] += f.x;
          x[2 * j + 1] += f.y;
        }
      }
      if (g.residual) {
        const uint32_t w[4] = {rr[i].x, rr[i].y, rr[i].z, rr[i].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = unpack_bf16x2(w[j]);
          x[2 * j] += f.x;
          x[2 * j + 1] += f.y;
        }
      }
      const uint4 o4 = make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                                  pack_bf16x2(x[6], x[7]));
      if (g.push.world) {  // TP push: this tile into every rank's receive slot (NVLink P2P stores)
        for (int pj = 0; pj < g.push.world; ++pj)
          *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(g.push.dst[pj]) + (long long)row * g.ldy + col) =
              o4;
      } else {
        *reinterpret_cast<uint4*>(dst) = o4;
      }
    } else {
      for (int j = 0; j < 8 && col + j < cols_valid; ++j) {
        float y = x[j];
        if (g.bias) y += __bfloat162float(g.bias[col + j]);
        if (g.residual) y += __bfloat162float(g.residual[(long long)row * g.ldy + col + j]);
        dst[j] = __float2bfloat16_rn(y);
      }
    }
  }
  __syncwarp();
}

// SwiGLU epilogue: the 32 accumulator columns (normal) / rows (swap) of a block are
// [gate f..f+15 | up f..f+15] for 16 output features f = (block start) / 2.
__device__ __forceinline__ float silu_mul_f(float gt, float up) {
  return __fdividef(gt, 1.f + __expf(-gt)) * up;  // MUFU ex2 + rcp, no IEEE-division slow path
}

__device__ __forceinline__ void epi_block_glu(const GemmArgs& g, __nv_bfloat16* stg, int lane, int m0, int n0,
                                              const uint32_t (&v)[32]) {
  if (!g.swap) {
    // row m0+lane; features n0/2 .. n0/2+15
    const int row = m0 + lane;
    const int f0 = n0 >> 1;
    const int fv = g.N_valid >> 1;
    if (row < g.M_valid && f0 < fv) {
      float a[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) a[j] = silu_mul_f(__uint_as_float(v[j]), __uint_as_float(v[16 + j]));
      __nv_bfloat16* dst = g.out + (long long)row * g.ldy + f0;
      if (f0 + 16 <= fv) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]),
                                                      pack_bf16x2(a[4], a[5]), pack_bf16x2(a[6], a[7]));
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(pack_bf16x2(a[8], a[9]), pack_bf16x2(a[10], a[11]),
                                                      pack_bf16x2(a[12], a[13]), pack_bf16x2(a[14], a[15]));
      } else {
        for (int j = 0; j < 16 && f0 + j < fv; ++j) dst[j] = __float2bfloat16_rn(a[j]);
      }
    }
    return;
  }
  // swap: lane l < 16 holds gate of feature m0/2 + l, lane l + 16 its up; columns = tokens n0..n0+31
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float up = __shfl_down_sync(0xffffffffu, __uint_as_float(v[j]), 16);
    if (lane < 16) stg[j * kStgStride + lane] = __float2bfloat16_rn(silu_mul_f(__uint_as_float(v[j]), up));
  }
  __syncwarp();
  const int f0 = m0 >> 1;
  const int fv = g.M_valid >> 1;
  // 32 token rows x 16 features: lane -> (row lane, 2 x 16 B)
  const int row = n0 + lane;
  if (row < g.N_valid && f0 < fv) {
    __nv_bfloat16* dst = g.out + (long long)row * g.ldy + f0;
    const uint4* src = reinterpret_cast<const uint4*>(stg + lane * kStgStride);
    if (f0 + 16 <= fv) {
      reinterpret_cast<uint4*>(dst)[0] = src[0];
      reinterpret_cast<uint4*>(dst)[1] = src[1];
    } else {
      for (int j = 0; j < 16 && f0 + j < fv; ++j) dst[j] = stg[lane * kStgStride + j];
    }
  }
  __syncwarp();
}

// 32 accumulator columns at taddr, summed over the K-interleaved accumulators (fixed order).
__device__ __forceinline__ void tmem_ld_sum(uint32_t taddr, int ka, uint32_t stride, uint32_t (&v)[32]) {
  tmem_ld_32x32b_x32(taddr, v);
  tmem_ld_wait();
  for (int j = 1; j < ka; ++j) {
    uint32_t w[32];
    tmem_ld_32x32b_x32(taddr + (uint32_t)j * stride, w);
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) + __uint_as_float(w[e]));
  }
}

template <int kPair, int kMT, int kSets>
__global__ void __launch_bounds__(threads_for(kSets), 1)
    gemm_bf16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_a,
                             const __grid_constant__ CUtensorMap tmap_b, const GemmArgs g) {
  constexpr int kEpiSets = kSets;
  constexpr int kEpiWarps = 4 * kSets;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (an integer round
  // trip would drop the address space: every staging access would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int BN = g.BN;
  const int stages = g.stages;
  constexpr int MT = kMT;
  const int bn_cta = BN / kPair;                       // B rows staged by this CTA
  const uint32_t a_bytes = (uint32_t)MT * kABytes;     // A bytes per stage
  const uint32_t b_bytes = (uint32_t)bn_cta * kBK * 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)stages * a_bytes;
  __nv_bfloat16* stg_all = reinterpret_cast<__nv_bfloat16*>(sB + (size_t)stages * b_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg_all) + kEpiWarps * kStgBytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;  // 2
  uint64_t* tempty = tfull + 2;      // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  unsigned long long* const trace = g.trace;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (kPair == 2) ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int cid = blockIdx.x / kPair;   // cluster (pair) id
  const int ncl = gridDim.x / kPair;
  const int KA = g.kacc;
  const uint32_t sub_stride = (uint32_t)(MT * BN);          // one K-interleaved accumulator
  const uint32_t acc_stride = (uint32_t)KA * sub_stride;    // TMEM columns per accumulator buffer
  const int tile_rows = kBM * kPair * MT;           // MMA-space rows per tile
  uint32_t tmem_cols = 32;
  while (tmem_cols < (uint32_t)g.nacc * acc_stride) tmem_cols <<= 1;

  if (threadIdx.x == 0) TRACE(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * kPair);  // one arrive per epilogue warp of every CTA of the pair
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (kPair == 2) tmem_alloc_pair(tmem_slot, tmem_cols);
    else tmem_alloc(tmem_slot, tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  if (kPair == 2) cluster_sync();  // peers' barriers/TMEM exist before any remote op
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  if (threadIdx.x == 0) TRACE(1);
  pdl_trigger();  // the next kernel may start its prologue as our CTAs drain
  // setmaxnreg sits at the top of each warpgroup's branch: ptxas allocates the code below it
  // with that budget (code reachable from both would get the smaller one)
  if (warp < epi_first_warp(kSets)) {
    if constexpr (kSets == 2) {
      // 384 x 168 at launch; WG0 hands 128 x 112 registers to the two epilogue warpgroups
      asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    }
    if (warp == 0) {
      // Weights do not depend on the preceding kernel: warm L2 with this CTA's first
      // k-blocks of them while that kernel finishes, then wait for its outputs.
      SegIter s0(g, cid, ncl);
      int t, kb0, kb1;
      if (s0.next(g, t, kb0, kb1)) {
        const int mt = t % g.m_tiles;
        const int nt = t / g.m_tiles;
        const int kend = min(kb1, kb0 + stages);
        for (int kb = kb0; kb < kend; ++kb) {
          if (g.swap) {
            const int r0 = mt * tile_rows + (int)rank * kBM;
#pragma unroll
            for (int i = 0; i < kMT; ++i) {
              const int r = r0 + i * kBM * kPair;
              if (g.a_blocked) tma_prefetch_l2_2d_w(&tmap_a, 0, ((r / kBM) * g.num_kb + kb) * kBM);
              else tma_prefetch_l2_2d_w(&tmap_a, kb * kBK, r);
            }
          } else {
            tma_prefetch_l2_2d_w(&tmap_b, kb * kBK, nt * BN + (int)rank * bn_cta);
          }
        }
      }
    }
    pdl_wait();

    if (warp == 0) {
      // ================= TMA producer (both CTAs; whole warp, one elected lane issues) =================
      const uint32_t full_leader0 = (kPair == 2) ? mapa_shared(&full[0], 0) : 0u;
      int stage = 0;
      uint32_t phase = 0;
      SegIter seg(g, cid, ncl);
      int t, kb0, kb1;
      while (seg.next(g, t, kb0, kb1)) {
        const int mt = t % g.m_tiles;
        const int nt = t / g.m_tiles;
        const int arow = mt * tile_rows + (int)rank * kBM;
        const int brow = nt * BN + (int)rank * bn_cta;
        // blocked A: 128-row block r, k-block kb lives at rows (r * num_kb + kb) * 128, column 0
        auto a_x = [&](int kb) { return g.a_blocked ? 0 : kb * kBK; };
        auto a_y = [&](int kb, int i) {
          const int r = arow + i * kBM * kPair;
          return g.a_blocked ? ((r / kBM) * g.num_kb + kb) * kBM : r;
        };
        if (g.pf_dist > 0) {
          for (int kb = kb0; kb < min(kb1, kb0 + g.pf_dist); ++kb)
#pragma unroll
            for (int i = 0; i < kMT; ++i) tma_prefetch_l2_2d_w(&tmap_a, a_x(kb), a_y(kb, i));
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          if (g.pf_dist > 0 && kb + g.pf_dist < kb1) {
#pragma unroll
            for (int i = 0; i < kMT; ++i) tma_prefetch_l2_2d_w(&tmap_a, a_x(kb + g.pf_dist), a_y(kb + g.pf_dist, i));
          }
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a_dst = sA + (size_t)stage * a_bytes;
          if (kPair == 1 && (g.dbg & 2)) {
            mbar_arrive_w(&full[stage]);
          } else if (kPair == 2) {
            const uint32_t lbar = full_leader0 + (uint32_t)stage * 8u;
            if (leader) mbar_arrive_expect_tx_w(&full[stage], kPair * (a_bytes + b_bytes));
#pragma unroll
            for (int i = 0; i < kMT; ++i)
              tma_load_2d_pair_w(a_dst + (size_t)i * kABytes, &tmap_a, lbar, a_x(kb), a_y(kb, i), g.hint_a);
            tma_load_2d_pair_w(sB + (size_t)stage * b_bytes, &tmap_b, lbar, kb * kBK, brow, g.hint_b);
          } else {
            mbar_arrive_expect_tx_w(&full[stage], a_bytes + b_bytes);
#pragma unroll
            for (int i = 0; i < kMT; ++i)
              tma_load_2d_w(a_dst + (size_t)i * kABytes, &tmap_a, &full[stage], a_x(kb), a_y(kb, i), g.hint_a);
            tma_load_2d_w(sB + (size_t)stage * b_bytes, &tmap_b, &full[stage], kb * kBK, brow, g.hint_b);
          }
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
    } else if (warp == 1) {
      if (leader) {
        // ================= MMA issuer (leader CTA; whole warp, one elected lane issues) =================
        const uint32_t idesc = make_idesc_bf16(kBM * kPair, BN);
        const uint32_t ka_mask = (uint32_t)KA - 1u;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        bool first = true;
        SegIter seg(g, cid, ncl);
        int t, kb0, kb1;
        while (seg.next(g, t, kb0, kb1)) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)acc * acc_stride;
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full[stage], phase);
            if (lane == 0 && first && kb == kb0) TRACE(2);
            if (lane == 0 && first && kb == kb1 - 1) TRACE(3);
            tc_fence_after();
            if (kPair == 1 && (g.dbg & 1)) {
              mbar_arrive_w(&empty[stage]);
            } else {
              const uint64_t bdesc = make_sdesc_sw128(sB + (size_t)stage * b_bytes);
              const uint64_t adesc0 = make_sdesc_sw128(sA + (size_t)stage * a_bytes);
              // kk outer, sub-tile inner: consecutive MMAs hit different accumulators
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk) {
                // advance 16 elements (32 bytes) inside the swizzle atom: +2 in 16-byte units
                const uint32_t j = (uint32_t)kk & ka_mask;
                const uint32_t accum = (kb > kb0 || (uint32_t)kk > ka_mask) ? 1u : 0u;
#pragma unroll
                for (int i = 0; i < kMT; ++i) {
                  const uint64_t adesc = adesc0 + (uint64_t)((i * kABytes) >> 4) + (uint64_t)(kk * 2);
                  const uint32_t d = d_tmem + j * sub_stride + (uint32_t)(i * BN);
                  if (kPair == 2) umma_bf16_pair_w(d, adesc, bdesc + (uint64_t)(kk * 2), idesc, accum);
                  else umma_bf16_w(d, adesc, bdesc + (uint64_t)(kk * 2), idesc, accum);
                }
              }
              if (kPair == 2) umma_commit_pair_mc_w(&empty[stage], 0x3);
              else umma_commit_w(&empty[stage]);
            }
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
          if (kPair == 2) umma_commit_pair_mc_w(&tfull[acc], 0x3);
          else if (g.dbg & 1) mbar_arrive_w(&tfull[acc]);
          else umma_commit_w(&tfull[acc]);
          if (++acc == g.nacc) { acc = 0; acc_phase ^= 1; }
          first = false;
        }
      }
    }
  } else {
    if constexpr (kSets == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    pdl_wait();
    // ================= epilogue warps (both CTAs) =================
    // warp w may only read TMEM lane quadrant w % 4; the kEpiSets warps of a quadrant take
    // alternate 32-column chunks of every accumulator (the epilogue is latency-bound per warp)
    const int q = warp & 3;
    const int ew = warp - epi_first_warp(kSets);
    const int set = ew >> 2;
    const bool lead = lane == 0 && q == 0 && set == 0;  // one thread of the CTA's epilogue
    __nv_bfloat16* stg = stg_all + (size_t)ew * (kStgBytes / 2);
    const uint32_t tempty_leader0 = (kPair == 2) ? mapa_shared(&tempty[0], 0) : 0u;
    const int nchunk = BN / 32;
    const size_t part_floats = (size_t)kBM * BN;  // one CTA's partial of one sub-tile
    int acc = 0;
    uint32_t acc_phase = 0;
    bool first = true;
    SegIter seg(g, cid, ncl);
    int t, kb0, kb1;
    while (seg.next(g, t, kb0, kb1)) {
      const int mtile = t % g.m_tiles;
      const int nt = t / g.m_tiles;
      const int mbase = mtile * tile_rows + (int)rank * kBM + q * 32;  // + i * kBM * kPair per sub-tile
      mbar_wait(&tfull[acc], acc_phase);
      if (lead && first) TRACE(4);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)acc * acc_stride;
      auto release_acc = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kPair == 2) mbar_arrive_remote(tempty_leader0 + (uint32_t)acc * 8u);
          else mbar_arrive(&tempty[acc]);
        }
      };
      if (kSets == 2 && g.ksplit > 1) {  // (decode kernels only: compiled out of the prefill ones)
        // K-slice unit (decode): the fp32 partial of this slice goes to its own slot, row-major
        // in the output orientation [token][feature]; the consumer kernel (RoPE / residual +
        // RMSNorm) sums the slices in order — no finisher SM, no wait (deterministic)
        float* slot = g.part + (size_t)seg.slice * g.part_slice;
        for (int i = 0; i < MT; ++i) {
          const int m0 = mbase + i * kBM * kPair;
          const int f = m0 + lane;  // this lane's feature (MMA row)
          for (int c = set; c < nchunk; c += kEpiSets) {
            uint32_t v[32];
            tmem_ld_sum(tbase + (uint32_t)(i * BN + c * 32), KA, sub_stride, v);
            const int n0 = nt * BN + c * 32;
            if (f < g.M_valid) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < g.N_valid) __stcg(slot + (size_t)(n0 + j) * g.M_valid + f, __uint_as_float(v[j]));
            }
          }
        }
        release_acc();
      } else if (kb0 == 0 && kb1 == g.num_kb) {
        // whole tile in this segment: straight to Y
        for (int i = 0; i < MT; ++i) {
          const int m0 = mbase + i * kBM * kPair;
          if (m0 >= g.M_valid) continue;
          for (int c = set * 32; c < BN; c += 32 * kEpiSets) {
            EpiPre pre;
            epi_preload(g, lane, m0, nt * BN + c, pre);
            uint32_t v[32];
            if (lead && first && i == 0 && c < 64) TRACE(11 + (c >> 5));
            tmem_ld_sum(tbase + (uint32_t)(i * BN + c), KA, sub_stride, v);
            if (lead && first && i == 0 && c == 32) TRACE(13);
            if (nt * BN + c < g.N_valid) {
              if (g.glu) epi_block_glu(g, stg, lane, m0, nt * BN + c, v);
              else epi_block(g, stg, lane, m0, nt * BN + c, v, pre, lead && first && i == 0 && c == 32);
            }
            if (lead && first && i == 0 && c == 32) TRACE(14);
          }
        }
        release_acc();
      } else {
        // ---- stream-K split tile (see SegIter): c_first..c_last-1 publish fp32 partials
        // and signal; the finisher c_last adds them, in cluster order, to its own TMEM
        // accumulator — no partial of its own, no reload.
        const int x0 = t * g.num_kb;
        const int c_first = sk_owner(g, x0, ncl);
        const int c_last = sk_owner(g, x0 + g.num_kb - 1, ncl);
        const int region = t * kPair + (int)rank;
        if (cid != c_last) {
          float* mine = g.ws + (((size_t)cid * kPair + rank) * MT) * part_floats;
          for (int i = 0; i < MT; ++i) {
            for (int c = set; c < nchunk; c += kEpiSets) {
              uint32_t v[32];
              tmem_ld_sum(tbase + (uint32_t)(i * BN + c * 32), KA, sub_stride, v);
              // lane-major layout: float4 j of lane l at (j*32 + l) -> 512 contiguous bytes per store
              float4* dst = reinterpret_cast<float4*>(mine + i * part_floats + ((size_t)c * 4 + q) * 1024) + lane;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                __stcg(dst + j * 32, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                 __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
            }
          }
          if (lead && first) TRACE(7);  // partials stored
          release_acc();
          __threadfence();
          named_bar_sync(1, 32 * kEpiWarps);
          if (lead) red_release_gpu_add(&g.counters[region], 1);
          if (lead && first) TRACE(8);  // published
        } else {
          if (lead) {
            const int need = c_last - c_first;
            while (ld_acquire_gpu(&g.counters[region]) < need) {
            }
            g.counters[region] = 0;  // re-arm for the next launch / graph replay
          }
          named_bar_sync(1, 32 * kEpiWarps);
          if (lead) TRACE(9);  // finisher: contributors in
          __threadfence();
          // The first contributor's partial and the residual of a chunk are requested together,
          // before the TMEM load, so the chunk costs one L2 round trip.
          auto part_ptr = [&](int c2, int i, int c) {
            return reinterpret_cast<const float4*>(g.ws + (((size_t)c2 * kPair + rank) * MT + i) * part_floats +
                                                   ((size_t)c * 4 + q) * 1024) + lane;
          };
          for (int i = 0; i < MT; ++i) {
            const int m0 = mbase + i * kBM * kPair;
            if (m0 >= g.M_valid) continue;
            for (int c = set; c < nchunk; c += kEpiSets) {
              float4 pf[8];
              EpiPre pre;
              {
                const float4* s0 = part_ptr(c_first, i, c);
#pragma unroll
                for (int j = 0; j < 8; ++j) pf[j] = __ldcg(s0 + j * 32);
                epi_preload(g, lane, m0, nt * BN + c * 32, pre);
              }
              uint32_t v[32];
              tmem_ld_sum(tbase + (uint32_t)(i * BN + c * 32), KA, sub_stride, v);
              auto add4 = [&](const float4 (&f)[8]) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  v[4 * j] = __float_as_uint(__uint_as_float(v[4 * j]) + f[j].x);
                  v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + f[j].y);
                  v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + f[j].z);
                  v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + f[j].w);
                }
              };
              add4(pf);
              for (int c2 = c_first + 1; c2 < c_last; ++c2) {  // further contributors, in cluster order
                const float4* s0 = part_ptr(c2, i, c);
#pragma unroll
                for (int j = 0; j < 8; ++j) pf[j] = __ldcg(s0 + j * 32);
                add4(pf);
              }
              if (nt * BN + c * 32 < g.N_valid) {
                if (g.glu) epi_block_glu(g, stg, lane, m0, nt * BN + c * 32, v);
                else epi_block(g, stg, lane, m0, nt * BN + c * 32, v, pre);
              }
            }
          }
          release_acc();
          if (lead) TRACE(10);  // finisher: tile stored
        }
      }
      if (lead && first) TRACE(5);
      if (++acc == g.nacc) { acc = 0; acc_phase ^= 1; }
      first = false;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (g.push.world && threadIdx.x == 0) {
    // every output tile of this CTA is stored (bar.sync above); make them visible system-wide,
    // and the last CTA of the grid tells every rank this GEMM's slot is complete
    __threadfence_system();
    if (atomicAdd(g.push.done_local, 1u) == gridDim.x - 1) {
      *g.push.done_local = 0u;  // re-arm (next launch is stream-ordered after this one)
      __threadfence_system();
      for (int pj = 0; pj < g.push.world; ++pj) atomicAdd_system(g.push.arrive[pj], 1u);
    }
  }
  if (kPair == 2) cluster_sync();  // the leader's MMAs into the peer's TMEM are done
  if (threadIdx.x == 0) TRACE(6);
  if (warp == 1) {
    __syncwarp();
    if (kPair == 2) tmem_dealloc_pair(tmem_base, tmem_cols);
    else tmem_dealloc(tmem_base, tmem_cols);
  }
}

// ------------------------------------------------------------------ host side

int gemm_set_trace(unsigned long long* buf) {
  g_trace_host = buf;
  g_trace_launch = 0;
  return 0;
}

static int gemm_smem_bytes(int a_bytes, int b_rows_per_cta, int stages) {
  return stages * (a_bytes + b_rows_per_cta * kBK * 2) + kMaxEpiWarps * kStgBytes + 1024 /*align*/ +
         (2 * stages + 4) * 8 + 32;
}

static int g_force_pair = -1;  // debug override: -1 auto, 0 single-CTA, 1 CTA pair
int gemm_set_pair_mode(int mode) {
  g_force_pair = mode;
  return 0;
}
// debug override of the decode (swap-AB) schedule: -1 auto; else bit0 = 2 A sub-tiles
// per tile, bit1 = stream-K (without it: data-parallel whole tiles)
static int g_force_variant = -1;
static int g_mt2_sets = 1;  // debug: epilogue sets of the two-sub-tile (MT=2) decode kernel
static int g_prefill_bn = 0;  // token-major tile width: 0 = wave-aware choice, else forced (debug)
int gemm_set_prefill_bn(int bn) {
  if (bn != 0 && (bn < 32 || bn > 256 || bn % 32 != 0)) return -1;
  g_prefill_bn = bn;
  return 0;
}
// Decode (swap-AB) K-slice count for a GEMM whose consumer sums fp32 partials (O / down ->
// add_partials_rmsnorm): 1 = keep the stream-K schedule with the residual epilogue. Whole
// K-slice units run with no finisher; used where two slices fit one wave of clusters (8B:
// partitions >= 64 SMs), measured on 72 SMs: O 28.4 -> 19.7 us, down 49.3 -> 42.7 us (B=256),
// whole decode step 8.91 -> 8.54 ms (B=128) / 13.18 -> 12.75 ms (B=256) alone
// (profiles/r02/gemm/).
int gemm_pick_ksplit(int O, int T, int K, int num_sms, size_t ws_bytes) {
  if (T < 96 || T > 256 || K % kBK != 0 || num_sms < 2) return 1;  // MT = 1 swap-AB tiles only
  const int BN = ((T + 31) / 32) * 32;
  const int pair = (O > kBM && (BN > 128 || (BN == 128 && num_sms < 100))) ? 2 : 1;
  const int clusters = num_sms / pair;
  const int tiles = (O + kBM * pair - 1) / (kBM * pair);
  const int nkb = K / kBK;
  const double sk = (double)tiles * nkb / clusters;  // stream-K k-blocks per cluster
  int best = 1;
  double best_cost = 1e30;
  // two slices at most: every slice is T x O fp32 the consumer re-reads (3 slices on 48 SMs won
  // 10 us per layer in the GEMMs and lost it in the consumer: decode step unchanged)
  for (int ks = 2; ks <= 2; ++ks) {
    if (nkb < 2 * ks || (size_t)ks * T * O * sizeof(float) > ws_bytes) continue;
    const double cost = (double)((tiles * ks + clusters - 1) / clusters) * ((nkb + ks - 1) / ks);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = ks;
    }
  }
  // stream-K's even share pays a finisher (one SM sums 96 KB partials per contributor): K-slices
  // win up to ~20% more k-blocks per unit (72 SMs, O: 32 vs 28.4 k-blocks, 19.7 vs 28.4 us)
  return (best > 1 && best_cost <= 1.2 * sk + 4) ? best : 1;
}

static int g_ksplit = 0;  // debug (decode, swap-AB): > 1 = data-parallel K-slices with fp32 partial output
int gemm_set_ksplit(int s) {
  if (s < 0 || s > 16) return -1;
  g_ksplit = s;
  return 0;
}
static int g_prefill_streamk = 0;          // stream-K for badly wave-quantized token-major GEMMs
static double g_prefill_streamk_frac = 0.6;
int gemm_set_prefill_streamk(int on, double max_frac) {
  g_prefill_streamk = on;
  g_prefill_streamk_frac = max_frac;
  return 0;
}
static int g_gemm_pf = -1;  // decode (swap-AB) weight k-blocks warmed into L2 ahead of the ring: -1 auto, 0 off
int gemm_set_prefetch(int kblocks) {
  if (kblocks < -1 || kblocks > 64) return -1;
  g_gemm_pf = kblocks;
  return 0;
}
int gemm_set_variant(int v) {
  g_force_variant = v;
  g_mt2_sets = (v >= 0 && (v & (1 << 14))) ? 2 : 1;
  return 0;
}

int gemm_bf16_launch(const void* X, const void* W, void* Y, const void* bias, const void* residual, int T,
                     int O, int K, long long ldx, long long ldw, long long ldy, int mode, int num_sms,
                     void* workspace, size_t ws_bytes, int* counters, int counters_len, cudaStream_t stream,
                     const GemmRope* rope, const GemmPush* push) {
  if (T <= 0 || O <= 0) return 0;
  if (rope && (rope->q_out == nullptr || rope->hd != 128 || O != (rope->hq + 2 * rope->hkv) * 128 ||
               residual != nullptr || (mode & 4) || rope->ld_q % 8 ||
               reinterpret_cast<uintptr_t>(rope->q_out) % 16 || reinterpret_cast<uintptr_t>(rope->cache) % 16 ||
               reinterpret_cast<uintptr_t>(rope->cos_sin) % 16))
    return set_error("gemm: fused RoPE epilogue needs head_dim 128, O = (Hq + 2 Hkv) * 128, no residual / SwiGLU, "
                     "16-byte aligned q_out / cache / cos_sin");
  if (K % kBK != 0) return set_error("gemm: K must be a multiple of 64");
  if ((ldx * 2) % 16 || (ldw * 2) % 16) return set_error("gemm: row strides must be 16-byte multiples");
  if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(W) % 16)
    return set_error("gemm: operands must be 16-byte aligned");
  if (ldy % 8 || reinterpret_cast<uintptr_t>(Y) % 16 || (residual && reinterpret_cast<uintptr_t>(residual) % 16) ||
      (bias && reinterpret_cast<uintptr_t>(bias) % 16))
    return set_error("gemm: Y/residual/bias must be 16-byte aligned with ldy % 8 == 0");
  const int glu = (mode & 4) ? 1 : 0;      // flag bit: fused SwiGLU epilogue
  const int blocked = (mode & 8) ? 1 : 0;  // flag bit: W is block-packed (see rb_pack_weight)
  const int ks_req = (mode >> 8) & 15;     // bits 8..11: decode K-slices with fp32 partial output (no Y)
  mode &= 3;
  if (ks_req > 1 && (bias != nullptr || residual != nullptr || glu || rope != nullptr || push != nullptr))
    return set_error("gemm: K-sliced partial output takes no bias / residual / SwiGLU / RoPE / push");
  if (glu && (O % 32 != 0 || bias != nullptr || residual != nullptr))
    return set_error("gemm: SwiGLU epilogue needs O % 32 == 0 and no bias / residual");
  if (mode == 0) mode = (T <= 256) ? 2 : 1;
  const bool swap = (mode == 2);
  if (blocked && (!swap || O % kBM != 0 || ldw != K))
    return set_error("gemm: block-packed weights need swap-AB mode, O % 128 == 0 and a dense [O, K] buffer");
  if (num_sms <= 0) num_sms = 148;
  GemmArgs g{};
  const int M = swap ? O : T;  // MMA-space rows
  const int N = swap ? T : O;  // MMA-space cols
  int BN;
  if (swap) {
    BN = ((N + 31) / 32) * 32;
    if (BN > 256) BN = 256;
  } else {
    // Token-major (prefill) tiles are 256 x BN on CTA pairs. Whole-tile waves quantize: the
    // O / down projections of a 1K-token chunk are 4 x 16 tiles of 256 columns, 1.5 waves on a
    // 42-pair partition, run as 2. Pick the width (multiple of 32, >= 128) that minimises
    // waves x (BN + per-tile overhead): 224 there (2 waves of narrower tiles).
    BN = 256;
    if (g_prefill_bn) {
      BN = g_prefill_bn;
    } else if (T > kBM) {
      const long long slots = num_sms >= 2 ? num_sms / 2 : 1;
      const long long mt = (T + 2 * kBM - 1) / (2 * kBM);
      long long best = -1;
      for (int bn = 256; bn >= 128; bn -= 32) {
        const long long tiles = mt * ((N + bn - 1) / bn);
        const long long cost = ((tiles + slots - 1) / slots) * (bn + 32);
        if (best < 0 || cost < best) {
          best = cost;
          BN = bn;
        }
      }
    }
  }
  // CTA pairs halve the per-SM operand stream: prefill tiles always; decode (swap-AB)
  // tiles when the batch tile is wide (each CTA of the pair stages BN/2 activation rows,
  // halving the activation re-read that otherwise matches the weight bytes per k-block).
  int pair = (num_sms >= 2 && M > kBM && (!swap || BN > 128 || (BN == 128 && num_sms < 100))) ? 2 : 1;
  if (g_force_pair == 0) pair = 1;
  if (g_force_pair == 1 && num_sms >= 2 && BN >= 32) pair = 2;
  // Decode (swap-AB): stream-K balances the tiles x k-blocks over the partition (no wave
  // quantization, small weight matrices spread over every SM). Two A sub-tiles per B stage
  // (variant bit 0) measured slower once the MMA issue loop was lean: off by default.
  int variant = swap ? 2 : 0;
  if (g_force_variant >= 0) variant = swap ? g_force_variant : (g_force_variant & ~1);
  int MT = ((variant & 1) && 2 * BN <= 512 && M > kBM * pair) ? 2 : 1;
  // Small decode batches: two A sub-tiles per stage (36 KB stages, half the stages and
  // barrier round trips per weight byte) measured 9-26% faster at B <= 32 and on the large
  // projections at B <= 64 on decode partitions up to ~88 SMs (per-SM ingest bound; see
  // scripts/gemm_chain.py); on the whole GPU (HBM bound) the extra split-tile fixups of the
  // halved tile count cost 2-15%, and the wider epilogue loses above B = 64.
  if (swap && g_force_variant < 0 && M > kBM * pair && num_sms <= 88 &&
      (BN <= 32 || (BN <= 64 && (long long)M * K >= (32ll << 20))))
    MT = 2;
  const int bn_cta = BN / pair;
  const int a_bytes = MT * kABytes;
  const int stage_bytes = a_bytes + bn_cta * kBK * 2;
  int stages = (200 * 1024 - kMaxEpiWarps * kStgBytes) / stage_bytes;
  if (stages > 8) stages = 8;
  if (stages < 2) stages = 2;
  if (variant > 0 && ((variant >> 5) & 15) >= 2 && ((variant >> 5) & 15) <= stages) stages = (variant >> 5) & 15;
  g.BN = BN;
  g.stages = stages;
  g.mt = MT;
  g.a_blocked = blocked;
  g.pf_dist = (variant & 4) ? 8 : 0;
  if (swap && g_gemm_pf >= 0) g.pf_dist = g_gemm_pf;
  g.dbg = (pair == 1 && variant > 0) ? (variant >> 3) & 3 : 0;
  if (variant > 0 && (variant & (1 << 12))) g.dbg |= 4;  // debug: epilogue skips its global stores
  int KA = 1;
  if (variant > 0 && ((variant >> 9) & 3)) KA = 1 << ((variant >> 9) & 3);
  while (KA > 1 && KA * MT * BN > 512) KA >>= 1;
  g.kacc = KA;
  g.nacc = (2 * KA * MT * BN <= 512) ? 2 : 1;
  g.m_tiles = (M + kBM * pair * MT - 1) / (kBM * pair * MT);
  g.n_tiles = (N + BN - 1) / BN;
  g.num_kb = K / kBK;
  g.total_tiles = g.m_tiles * g.n_tiles;
  g.total_iters = g.total_tiles * g.num_kb;
  const int slots = num_sms / pair;  // concurrent clusters
  int clusters = g.total_tiles < slots ? g.total_tiles : slots;
  g.streamk = 0;
  if (!swap && g_force_variant < 0 && g_prefill_streamk) {
    // token-major (prefill) tiles (off by default: measured slower, the split-tile fixup costs
    // more than the quantization it removes): stream-K only where whole-tile waves quantize badly
    // (a few waves with a small last one, e.g. the O / down projections of a 1K-token
    // chunk: 64 tiles on 42 clusters = 1.5 waves run as 2); long GEMMs stay data-parallel
    const double waves = (double)g.total_tiles / slots;
    const double frac = waves - (int)waves;
    if (waves < 4.0 && frac > 0.0 && frac <= g_prefill_streamk_frac) variant |= 2;
  }
  if ((variant & 2) && workspace != nullptr && counters != nullptr && g.total_tiles * pair <= counters_len &&
      g.total_tiles % slots != 0) {
    // every cluster gets >= 8 k-blocks; one partial slot per cluster: [cluster][pair][MT][128 x BN] fp32
    int ncl = slots;
    if (g.total_iters / ncl < 8) ncl = g.total_iters / 8 > 0 ? g.total_iters / 8 : 1;
    const size_t need = (size_t)ncl * pair * MT * kBM * BN * sizeof(float);
    if (need <= ws_bytes && ncl > 0) {
      g.streamk = 1;
      clusters = ncl;
    }
  }
  g.ksplit = 1;
  const int ks_use = ks_req > 1 ? ks_req : g_ksplit;
  if (ks_req > 1 && !(swap && MT == 1 && workspace != nullptr && (size_t)ks_req * N * M * sizeof(float) <= ws_bytes &&
                      g.num_kb >= 2 * ks_req))
    return set_error("gemm: K-sliced partial output needs the swap-AB single-sub-tile schedule and workspace room "
                     "(use gemm_pick_ksplit)");
  if (swap && MT == 1 && ks_use > 1 && workspace != nullptr && !glu && rope == nullptr && push == nullptr &&
      (size_t)ks_use * N * M * sizeof(float) <= ws_bytes && g.num_kb >= 2 * ks_use) {
    g.ksplit = ks_use;
    g.streamk = 0;
    g.part = reinterpret_cast<float*>(workspace);
    g.part_slice = (long long)N * M;
    const int units = g.total_tiles * g.ksplit;
    clusters = units < slots ? units : slots;
  }
  if (clusters < 1) clusters = 1;
  g.ws = reinterpret_cast<float*>(workspace);
  g.counters = counters;
  g.M_valid = M;
  g.N_valid = N;
  g.swap = swap ? 1 : 0;
  g.glu = glu;
  g.ldy = ldy;
  g.out = reinterpret_cast<__nv_bfloat16*>(Y);
  g.residual = reinterpret_cast<const __nv_bfloat16*>(residual);
  g.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
  if (rope) g.rp = *rope;
  if (push) {
    if (glu || residual != nullptr || rope != nullptr)
      return set_error("gemm: the TP push epilogue takes a plain output (no SwiGLU / residual / RoPE)");
    g.push = *push;
  }
  if (g_trace_host) g.trace = g_trace_host + (size_t)(g_trace_launch++ % 16) * 148 * 16;
  if (swap) {
    g.hint_a = kEvictFirst;  // weights stream once
    g.hint_b = kEvictLast;   // activations reused by every weight tile
  } else {
    g.hint_a = kEvictLast;
    g.hint_b = kEvictNormal;
  }

  CUtensorMap ta, tb;
  const void* a_ptr = swap ? W : X;
  const void* b_ptr = swap ? X : W;
  const long long lda = swap ? ldw : ldx;
  const long long ldb = swap ? ldx : ldw;
  int rc = blocked ? make_tmap_2d_bf16(&ta, a_ptr, (uint64_t)kBK, (uint64_t)M * (K / kBK), (uint64_t)kBK, kBK, kBM)
                   : make_tmap_2d_bf16(&ta, a_ptr, (uint64_t)K, (uint64_t)M, (uint64_t)lda, kBK, kBM);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tb, b_ptr, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, kBK, bn_cta);
  if (rc) return rc;

  const int smem = gemm_smem_bytes(a_bytes, bn_cta, stages);
  using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const GemmArgs);
  // [pair][MT][sets]: decode (swap-AB) with single A sub-tiles uses 2 epilogue sets
  static const KernelFn kernels[2][2][2] = {
      {{gemm_bf16_tcgen05_kernel<1, 1, 1>, gemm_bf16_tcgen05_kernel<1, 1, 2>},
       {gemm_bf16_tcgen05_kernel<1, 2, 1>, gemm_bf16_tcgen05_kernel<1, 2, 2>}},
      {{gemm_bf16_tcgen05_kernel<2, 1, 1>, gemm_bf16_tcgen05_kernel<2, 1, 2>},
       {gemm_bf16_tcgen05_kernel<2, 2, 1>, gemm_bf16_tcgen05_kernel<2, 2, 2>}}};
  // decode epilogue sets: 2 (three warpgroups, setmaxnreg) except the MT=2 kernel at B <= 32
  const int sets = (swap && (MT == 1 || g_mt2_sets == 2 || (g_force_variant < 0 && BN > 32))) ? 2 : 1;
  const KernelFn kern = kernels[pair - 1][MT - 1][sets - 1];
  {
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(kern), 227 * 1024);
    if (e != cudaSuccess) return set_cuda_error("gemm: set smem attr", e);
  }
  cudaError_t e = launch_k(kern, dim3(pair * clusters), dim3(threads_for(sets)), smem, stream, pair, ta, tb, g);
  if (e != cudaSuccess) return set_cuda_error("gemm launch", e);
  return 0;
}

}  // namespace rb
