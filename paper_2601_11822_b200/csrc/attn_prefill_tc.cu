// K2 (tcgen05): prefill causal flash-attention over the paged KV cache on
// 5th-gen tensor cores, TMA-fed.
//
// Realizes the attention share of prefill_time's compute term (reference
// pkg/src/pdsim/costmodel.py:104) for one prefill chunk (rapid.py:313): queries
// at positions start..start+T-1 of one request attend to keys [0, start+T) of its
// paged cache (prefix U chunk; the chunk's K,V were written by the RoPE/cache
// kernel that precedes this one), causal mask shifted by `start`.
//
// CTA = 128 query positions x 1 query head, 192 threads:
//   w0      TMA producer: Q once (3D map over [T][Hq][128]), then 64-key K/V
//           tiles = 4 pages x {K lo, K hi, V lo, V hi} boxes {64 x 16} (2D map
//           over the cache layer) into a 3-stage ring, 128B swizzle.
//   w1      TMEM owner + single-thread MMA issuer:
//             S_j = Q K_j^T   (M=128, N=64,  K=128; A,B K-major)     -> TMEM S[j%2]
//             O_j = P_j V_j   (M=128, N=128, K=64;  B = V MN-major)  -> TMEM O[j%2]
//           S_{j+1} is issued before O_j so QK^T overlaps the softmax.
//   w2..w5  softmax (thread = query row = TMEM lane): S row -> mask, running
//           max/sum (exp2) -> P row (bf16) into smem in the UMMA K-major layout.
// O accumulates in TMEM across all key tiles (PV_j with accumulate). The softmax
// keeps a stale row max and rescales the TMEM O row (ld, scale, st) only when the
// max grows by more than kRescaleLog2 (P <= 2^8 otherwise): no per-tile O fold.
// Output row = O / l, read from TMEM once at the end (256 B per row).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cfloat>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

namespace fa {
constexpr int kD = 128;
constexpr int kBMq = 128;                  // query rows per CTA
constexpr int kBN = 64;                    // keys per tile
constexpr int kPage = 16;
constexpr int kStages = 4;
constexpr int kQBytes = 2 * kBMq * 128;    // two 64-dim halves, 16 KB each
constexpr int kKVHalf = kBN * 128;         // 8 KB: 64 keys x 64 dims
constexpr int kKVStage = 4 * kKVHalf;      // K lo, K hi, V lo, V hi = 32 KB
constexpr int kThreads = 192;
constexpr int kTmemCols = 256;             // S[2] x 64 + O x 128
constexpr uint32_t kSCol = 0, kOCol = 128;
constexpr float kRescaleLog2 = 8.0f;       // rescale O only when the row max grows by > 2^8
}  // namespace fa

// K-major SW128 descriptor with explicit SBO (atoms of 8 rows x 128 B)
__device__ __forceinline__ uint64_t sdesc_kmajor(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// MN-major SW128 descriptor: 64-element MN blocks LBO apart, 8-row K groups SBO=1024 apart
__device__ __forceinline__ uint64_t sdesc_mnmajor(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_3d(void* dst_smem, const void* tmap, uint64_t* bar, int32_t x, int32_t y,
                                            int32_t z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2; ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld_32x32b_x32(taddr, r);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// kTiles query tiles per CTA (same head, one softmax warpgroup each; two = the mirrored
// causal pair g, nqb-1-g): every K/V tile is loaded once for both, and two warpgroups run
// softmax while the tensor cores work on the other tile. The short tile of a pair needs
// fewer key tiles (causal); its MMAs simply stop there.
constexpr int pattn_threads(int tiles) { return 32 * (1 + tiles) + 128 * tiles; }

template <int kTiles>
__global__ void __launch_bounds__(pattn_threads(kTiles), 1)
    prefill_attn_tc_kernel(const __grid_constant__ CUtensorMap q_map, const __grid_constant__ CUtensorMap kv_map,
                           const int* __restrict__ bt, int T, int start, int Hq, int Hkv,
                           __nv_bfloat16* __restrict__ out, long long out_tok_stride, float scale_log2) {
  pdl_trigger();
  pdl_wait();
  using namespace fa;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                                   // [kTiles][32 KB]
  uint8_t* sKV = sQ + kTiles * kQBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kKVStage);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + kStages;
  uint64_t* s_full = kv_empty + kStages;  // [kTiles][2]
  uint64_t* s_free = s_full + 2 * kTiles;
  uint64_t* p_full = s_free + 2 * kTiles;
  uint64_t* p_free = p_full + 2 * kTiles;
  uint64_t* o_full = p_free + 2 * kTiles;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2 * kTiles);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nqb = (T + kBMq - 1) / kBMq;
  const int ngroups = (nqb + kTiles - 1) / kTiles;
  const int hq = blockIdx.y;
  const int hk = hq / (Hq / Hkv);
  const int chunk_end = start + T;
  const int last_page = (chunk_end - 1) / kPage;  // highest page index this chunk may touch
  // Query tiles of this CTA. One tile: latest (heaviest) first. Two: mirrored pairs
  // (g, nqb-1-g), so every CTA of a causal chunk carries the same number of key tiles
  // (the short tile's keys are a prefix of the long one's: its MMAs stop early).
  int qtile[kTiles];
  int ntile[kTiles];  // key tiles of each query tile (0: no such tile)
  if (kTiles == 1) {
    qtile[0] = ngroups - 1 - (int)blockIdx.x;
  } else {
    const int gsel = (int)blockIdx.x;
    qtile[0] = nqb - 1 - gsel;               // the long tile first (warpgroup 0)
    qtile[kTiles - 1] = gsel < nqb - 1 - gsel ? gsel : nqb;  // middle of an odd count: alone
  }
#pragma unroll
  for (int w = 0; w < kTiles; ++w) {
    const int qb = qtile[w];
    const int kv_end = start + min(T, qb * kBMq + kBMq);
    ntile[w] = qb < nqb ? (kv_end + kBN - 1) / kBN : 0;
  }
  int n_max = 0;
#pragma unroll
  for (int w = 0; w < kTiles; ++w) n_max = max(n_max, ntile[w]);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&kv_full[st], 1);
      mbar_init(&kv_empty[st], kTiles);  // one commit / arrive per tile's MMA issuer
    }
    for (int i = 0; i < 2 * kTiles; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 1);  // PV of the P aliased onto this S buffer has completed
      mbar_init(&p_full[i], 4);
      mbar_init(&p_free[i], 1);
      mbar_init(&o_full[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256 * kTiles);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: tile w -> S[2] at w*256 + {0, 64}, O at w*256 + 128
  auto s_col = [](int w, int b) { return (uint32_t)(w * 256 + b * kBN); };
  auto o_col = [](int w) { return (uint32_t)(w * 256 + 128); };

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer =================
      tma_prefetch_desc(&q_map);
      tma_prefetch_desc(&kv_map);
      int nq = 0;
#pragma unroll
      for (int w = 0; w < kTiles; ++w) nq += ntile[w] > 0 ? 1 : 0;
      mbar_arrive_expect_tx(q_full, (uint32_t)(nq * kQBytes));
#pragma unroll
      for (int w = 0; w < kTiles; ++w) {
        if (ntile[w] == 0) continue;
        const int q0 = qtile[w] * kBMq;
        tma_load_3d(sQ + w * kQBytes, &q_map, q_full, 0, hq, q0);
        tma_load_3d(sQ + w * kQBytes + kQBytes / 2, &q_map, q_full, 64, hq, q0);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int j = 0; j < n_max; ++j) {
        mbar_wait(&kv_empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&kv_full[stage], kKVStage);
        uint8_t* dst = sKV + (size_t)stage * kKVStage;
        for (int pg = 0; pg < kBN / kPage; ++pg) {
          int pidx = j * (kBN / kPage) + pg;
          if (pidx > last_page) pidx = last_page;  // past the chunk: finite data, masked in softmax
          const int page = bt[pidx];
          const int rowK = ((page * 2 + 0) * Hkv + hk) * kPage;
          const int rowV = ((page * 2 + 1) * Hkv + hk) * kPage;
          tma_load_2d(dst + 0 * kKVHalf + pg * 2048, &kv_map, &kv_full[stage], 0, rowK, kEvictNormal);
          tma_load_2d(dst + 1 * kKVHalf + pg * 2048, &kv_map, &kv_full[stage], 64, rowK, kEvictNormal);
          tma_load_2d(dst + 2 * kKVHalf + pg * 2048, &kv_map, &kv_full[stage], 0, rowV, kEvictNormal);
          tma_load_2d(dst + 3 * kKVHalf + pg * 2048, &kv_map, &kv_full[stage], 64, rowV, kEvictNormal);
        }
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp <= kTiles) {
    if (lane == 0) {
      // ================= MMA issuers: warp 1 + w drives query tile w =================
      // One issuer per tile decouples the tiles' S -> softmax -> P -> PV chains: S_{j+1}(w)
      // is issued as soon as tile w's PV_{j-1} is, not after the other tile's softmax too
      // (with one issuer the softmax warps waited on S ~40% of their time: profiles/r02/pattn/).
      const int w = warp - 1;
      const int nt = ntile[w];
      const uint32_t idesc_s = make_idesc_bf16(kBMq, kBN);
      const uint32_t idesc_o = make_idesc_bf16(kBMq, kD) | (1u << 16);  // B (V) MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      const uint32_t qa = smem_u32(sQ + w * kQBytes);
      auto issue_s = [&](int j) {
        const int st = j % kStages;
        const int b = j & 1;
        mbar_wait(&kv_full[st], (uint32_t)((j / kStages) & 1));
        mbar_wait(&s_free[2 * w + b], (uint32_t)(((j >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t kb = smem_u32(sKV + (size_t)st * kKVStage);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (uint32_t)((kk & 3) * 32);
          const uint64_t ad = sdesc_kmajor(qa + (kk >> 2) * (kQBytes / 2) + off);
          const uint64_t bd = sdesc_kmajor(kb + (kk >> 2) * kKVHalf + off);
          umma_bf16(tmem + s_col(w, b), ad, bd, idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[2 * w + b]);
      };
      if (nt > 0) issue_s(0);
      for (int j = 0; j < nt; ++j) {
        if (j + 1 < nt) issue_s(j + 1);
        const int st = j % kStages;
        const int b = j & 1;
        const uint32_t vb = smem_u32(sKV + (size_t)st * kKVStage + 2 * kKVHalf);
        mbar_wait(&p_full[2 * w + b], (uint32_t)((j >> 1) & 1));  // also orders any O rescale
        tc_fence_after();
        // P_j (bf16, K-major) sits in the first 32 columns of S buffer b: A operand from TMEM,
        // 16 keys = 8 columns per MMA
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t bd = sdesc_mnmajor(vb + kk * 2048, kKVHalf);
          umma_bf16_ts(tmem + o_col(w), tmem + s_col(w, b) + (uint32_t)(kk * 8), bd, idesc_o,
                       (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&o_full[2 * w + b]);
        umma_commit(&s_free[2 * w + b]);  // S buffer b (and the P in it) free for S_{j+2}
        umma_commit(&kv_empty[st]);
      }
      // key tiles past this query tile's diagonal (the short tile of a mirrored pair): release
      // each stage once it has landed, so the producer's refill needs only the long tile
      for (int j = nt; j < n_max; ++j) {
        const int st = j % kStages;
        mbar_wait(&kv_full[st], (uint32_t)((j / kStages) & 1));
        mbar_arrive(&kv_empty[st]);
      }
    }
  } else {
    // ================= softmax warpgroups: thread = query row of tile w =================
    const int w = (warp - 1 - kTiles) >> 2;
    const int qd = warp & 3;
    const int row = qd * 32 + lane;
    const int q0 = qtile[w] * kBMq;
    const int qpos = start + q0 + row;
    const int kv_end = start + min(T, q0 + kBMq);
    const int nt = ntile[w];
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const uint32_t o_taddr = tmem + lane_off + o_col(w);
    float m = -INFINITY, l = 0.f;  // m: the (stale) max P is taken against
    for (int j = 0; j < nt; ++j) {
      const int b = j & 1;
      const uint32_t ph2 = (uint32_t)((j >> 1) & 1);
      mbar_wait(&s_full[2 * w + b], ph2);
      tc_fence_after();
      float s[kBN];
      {
        uint32_t t0[32], t1[32];
        tmem_ld_32x32b_x32(tmem + lane_off + s_col(w, b), t0);
        tmem_ld_32x32b_x32(tmem + lane_off + s_col(w, b) + 32, t1);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(t0[i]);
          s[32 + i] = __uint_as_float(t1[i]);
        }
      }
      const int kbase = j * kBN;
      // masked scores are -inf (exp2 -> 0 with no select); tile 0 always holds key 0 <= qpos,
      // so the max is finite from the first tile on. Only tiles crossing this row's diagonal
      // or the chunk end need the per-key mask. The max runs on the raw scores (scale > 0)
      // with four independent chains; the scale folds into the exponent's FFMA below.
      float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if (kbase + kBN - 1 <= qpos && kbase + kBN <= kv_end) {
#pragma unroll
        for (int i = 0; i < kBN; ++i) mq[i & 3] = fmaxf(mq[i & 3], s[i]);
      } else {
#pragma unroll
        for (int i = 0; i < kBN; ++i) {
          const int kp = kbase + i;
          const float v = (kp > qpos || kp >= kv_end) ? -INFINITY : s[i];
          s[i] = v;
          mq[i & 3] = fmaxf(mq[i & 3], v);
        }
      }
      const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * scale_log2;
      // warp-uniform decision (tcgen05.ld/st below are warp-collective): when any row's stale
      // max is too far behind, every row of the warp moves its max up and rescales l and O
      if (__any_sync(0xffffffffu, mx > m + kRescaleLog2)) {
        const float mn = fmaxf(m, mx);
        const float alpha = ex2_approx(m - mn);  // tile 0: m = -inf -> 0 (l and O still empty)
        l *= alpha;
        if (j > 0) {
          // O holds PV_0..PV_{j-1}: wait for the last of them, then O_row *= alpha in TMEM.
          // (PV_{j+1} cannot run before this warp's p_full(j+1), so the barrier is at most one
          // phase past the one waited for.)
          mbar_wait(&o_full[2 * w + ((j - 1) & 1)], (uint32_t)(((j - 1) >> 1) & 1));
          tc_fence_after();
#pragma unroll
          for (int cc = 0; cc < kD / 32; cc += 2) {
            uint32_t t0[32], t1[32];
            tmem_ld_32x32b_x32(o_taddr + cc * 32, t0);
            tmem_ld_32x32b_x32(o_taddr + (cc + 1) * 32, t1);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              t0[i] = __float_as_uint(__uint_as_float(t0[i]) * alpha);
              t1[i] = __float_as_uint(__uint_as_float(t1[i]) * alpha);
            }
            tmem_st_32x32b_x32(o_taddr + cc * 32, t0);
            tmem_st_32x32b_x32(o_taddr + (cc + 1) * 32, t1);
          }
          tmem_st_wait();
          tc_fence_before();
        }
        m = mn;
      }
      float pq[4] = {0.f, 0.f, 0.f, 0.f};
      const float neg_m = -m;
#pragma unroll
      for (int i = 0; i < kBN; ++i) {
        const float p = ex2_approx(fmaf(s[i], scale_log2, neg_m));
        s[i] = p;
        pq[i & 3] += p;
      }
      l += (pq[0] + pq[1]) + (pq[2] + pq[3]);
      // P row -> TMEM over this row's S (already in registers): bf16 pairs, K-major
      // (four 8-column stores: the packed row is never live at once next to s[], which keeps
      // the 11-warp kernel within its 168 registers)
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t pk[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) pk[c] = pack_bf16x2(s[16 * q4 + 2 * c], s[16 * q4 + 2 * c + 1]);
        tmem_st_32x32b_x8(tmem + lane_off + s_col(w, b) + (uint32_t)(8 * q4), pk);
      }
      if (kbase + kBN > chunk_end) {
        // keys past the chunk in its last page may never have been written (non-finite bit
        // patterns); P is 0 there but 0 * NaN would poison the PV MMA -> zero those V rows.
        // (Keys in [kv_end, chunk_end) are real data another tile of the CTA may use.) Both
        // warpgroups may zero the same rows: identical values, each before its own p_full.
        const int st = j % kStages;
        uint8_t* vbase = sKV + (size_t)st * kKVStage + 2 * kKVHalf;
        const int first = max(0, chunk_end - kbase);
        for (int i = row; i < (kBN - first) * 16; i += kBMq) {  // 16 chunks of 16 B per key (2 halves)
          const int key = first + (i >> 4);
          const int ch = i & 15;
          uint8_t* p = vbase + (ch >> 3) * kKVHalf + (key >> 3) * 1024 + (key & 7) * 128 + (ch & 7) * 16;
          *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the zeroed V rows (generic -> async)
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * w + b]);
    }
    if (nt > 0) {
      mbar_wait(&o_full[2 * w + ((nt - 1) & 1)], (uint32_t)(((nt - 1) >> 1) & 1));
      tc_fence_after();
      const int trow = q0 + row;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* dst = out + (size_t)trow * out_tok_stride + (size_t)hq * kD;
#pragma unroll
      for (int cc = 0; cc < kD / 32; ++cc) {
        uint32_t t[32];
        tmem_ld_32x32b_x32(o_taddr + cc * 32, t);  // warp-collective: every lane loads, valid rows store
        tmem_ld_wait();
        if (trow < T) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            reinterpret_cast<uint4*>(dst + cc * 32)[c] = make_uint4(
                pack_bf16x2(__uint_as_float(t[8 * c]) * inv, __uint_as_float(t[8 * c + 1]) * inv),
                pack_bf16x2(__uint_as_float(t[8 * c + 2]) * inv, __uint_as_float(t[8 * c + 3]) * inv),
                pack_bf16x2(__uint_as_float(t[8 * c + 4]) * inv, __uint_as_float(t[8 * c + 5]) * inv),
                pack_bf16x2(__uint_as_float(t[8 * c + 6]) * inv, __uint_as_float(t[8 * c + 7]) * inv));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem, 256 * kTiles);
  }
}

typedef CUresult (*PFN_encodeTiled3)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int g_pattn_tiles = 0;  // debug override: 0 auto, 1 or 2 query tiles per CTA
int prefill_attn_set_tiles(int tiles) {
  if (tiles < 0 || tiles > 2) return -1;
  g_pattn_tiles = tiles;
  return 0;
}

int prefill_attention_tc_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* bt, int T,
                                int start, int Hq, int Hkv, int head_dim, void* out, long long out_tok_stride,
                                float scale, int num_blocks, cudaStream_t st) {
  using namespace fa;
  if (T <= 0) return 0;
  if (head_dim != kD) return set_error("prefill attention (tc): head_dim must be 128");
  if (Hkv <= 0 || Hq % Hkv != 0) return set_error("prefill attention (tc): bad head counts");
  if ((q_tok_stride * 2) % 16) return set_error("prefill attention (tc): q token stride must be 16-byte aligned");
  static PFN_encodeTiled3 enc = nullptr;
  if (!enc) {
    enc = reinterpret_cast<PFN_encodeTiled3>(driver_symbol("cuTensorMapEncodeTiled"));
    if (!enc) return set_error("cuTensorMapEncodeTiled unavailable");
  }
  CUtensorMap qmap;
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)Hq, (cuuint64_t)T};
    cuuint64_t strides[2] = {(cuuint64_t)kD * 2, (cuuint64_t)q_tok_stride * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kBMq};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_cu_error("cuTensorMapEncodeTiled(q)", r);
  }
  CUtensorMap kvmap;
  int rc = make_tmap_2d_bf16(&kvmap, cache_layer, kD, (uint64_t)num_blocks * 2 * Hkv * kPage, kD, 64, kPage);
  if (rc) return rc;
  // two query tiles per CTA (mirrored causal pairs sharing every K/V tile, two softmax
  // warpgroups) unless that leaves too few CTAs to fill the GPU. Measured on 148 SMs
  // (Llama-8B heads, profiles/r02/pattn/): T=1023 from 0 23.6 us (1 tile: 33.3), T=2048 from
  // 0 71.2 (82.8), 2048 after 6144 363 (394), 1023 after 1024 48.3 (60.2); T=512 (64 pair
  // CTAs) 15.5 vs 13.3 with one tile per CTA.
  const int nqb = (T + kBMq - 1) / kBMq;
  int tiles = (nqb >= 2 && ((nqb + 1) / 2) * Hq >= 96) ? 2 : 1;
  if (g_pattn_tiles == 1 || (g_pattn_tiles == 2 && nqb >= 2)) tiles = g_pattn_tiles;
  const int smem = tiles * kQBytes + kStages * kKVStage + (2 * kStages + 1 + 10 * tiles) * 8 + 16 +
                   1024;
  using Fn = void (*)(const CUtensorMap, const CUtensorMap, const int*, int, int, int, int, __nv_bfloat16*, long long,
                      float);
  static const Fn fns[2] = {prefill_attn_tc_kernel<1>, prefill_attn_tc_kernel<2>};
  {
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(fns[tiles - 1]), 227 * 1024);
    if (e != cudaSuccess) return set_cuda_error("prefill attn tc smem attr", e);
  }
  if (smem > 227 * 1024) return set_error("prefill attn tc: shared memory budget exceeded");
  dim3 grid((nqb + tiles - 1) / tiles, Hq);
  cudaError_t e = launch_k(fns[tiles - 1], dim3(grid), dim3(tiles == 2 ? pattn_threads(2) : pattn_threads(1)), smem, st, 1, qmap, kvmap, bt, T, start,
                           Hq, Hkv, reinterpret_cast<__nv_bfloat16*>(out), out_tok_stride, scale * 1.4426950408889634f);
  if (e != cudaSuccess) return set_cuda_error("prefill attn tc launch", e);
  return 0;
}

}  // namespace rb
