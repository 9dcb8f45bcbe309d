// Tensor parallelism for the decoder forward (cfg 4: Llama-3.1-70B, TP=8 over NVLink).
//
// The reference prices one GPU (tp folded into GpuSpec.aggregate, core.py:147-165) and
// models no collective at all; this is the physical TP of SURVEY.md §8(e): QKV and
// gate|up column-parallel, O and down row-parallel (one all-reduce after each), lm_head
// vocab-parallel with a max-reduce of packed (logit, -index) keys.
//
// Two collective back-ends per phase (prefill and decode each own one, so the phase
// streams never share a communicator or a flag):
//   mode 1 (NCCL): the row-parallel GEMM writes x + partial on rank 0 and the bare
//          partial elsewhere, then ncclAllReduce(sum) in place. NCCL is reached through
//          dlopen of the libnccl.so.2 the process already has (torch's), no link-time
//          dependency.
//   mode 2 (peer): one-shot all-reduce over peer memory for decode-size messages with
//          the residual add fused: every rank's GEMM writes its partial into its own
//          staging buffer; the AR kernel raises a per-CTA flag in every peer, waits for
//          all peers' flags, then computes x += P_0 + ... + P_{w-1} (fp32, fixed rank
//          order: bit-identical on all ranks) over its slice, reading peers' staging
//          buffers directly (NVLink P2P; cudaIpc handles on a real node, plain pointers
//          when several ranks share one device, as in the single-GPU tests). Staging is
//          double-buffered by call parity, so a rank never overwrites a buffer a peer may
//          still be reading (two flag rounds separate the reuse).
//   mode 3 (push, GEMM and collective fused): the row-parallel GEMM's epilogue stores every
//          output tile straight into each rank's receive slot for this sender (NVLink P2P
//          stores overlapping the remaining tiles' MMAs) and its last CTA raises one arrival
//          per rank; the reduce kernel waits for `world` arrivals and sums its own receive
//          slots + the residual — all reads local. Receive buffers and arrival counters are
//          double-buffered by call parity; the reducer's last CTA re-arms its counter.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cfloat>
#include <cstdio>
#include <cstring>
#include "ptx.cuh"
#include "rb_common.h"
#include "../../include/rapid_b200.h"

namespace rb {

constexpr int kMaxRanks = 8;
constexpr int kMaxArBlocks = 128;  // flag slots per rank per phase

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string;
    }
  }
  return api;
}

static int nccl_error(const char* where, ncclResult_t r) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", where, nccl().error_string ? nccl().error_string(r) : "nccl error");
  return set_error(buf);
}

// ------------------------------------------------------------------ TP context
struct TpPeers {                        // passed by value to the peer kernels
  int world, rank;
  __nv_bfloat16* part[2][kMaxRanks];    // staging buffer of every rank, per parity
  unsigned long long* keys[kMaxRanks];  // argmax keys of every rank
  unsigned* flags[kMaxRanks];           // rank j's flag array [kMaxRanks][kMaxArBlocks]
  unsigned* epoch;                      // this rank's per-CTA round counters [kMaxArBlocks]
  int nowait;                           // debug: skip the flag wait
};

struct TpCtx {
  int world, rank, mode;
  ncclComm_t comm;
  TpPeers peers;
  size_t part_elems;
  int parity;  // next staging parity; reset at the start of every forward (see tp_begin)
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Flag round of CTA `b`: announce this rank's data, wait for every peer's.
__device__ __forceinline__ void peer_round(const TpPeers& p, int b) {
  const unsigned e = p.epoch[b] + 1;
  p.epoch[b] = e;
  __threadfence_system();
  for (int j = 0; j < p.world; ++j) st_release_sys(p.flags[j] + p.rank * kMaxArBlocks + b, e);
  if (p.nowait) return;
  for (int j = 0; j < p.world; ++j)
    while (ld_acquire_sys(p.flags[p.rank] + j * kMaxArBlocks + b) < e) {
    }
}

// x[i] += sum_j part[par][j][i] over this CTA's slice (n % 8 == 0)
__global__ void __launch_bounds__(256) tp_ar_add_kernel(const TpPeers p, __nv_bfloat16* __restrict__ x,
                                                        long long n, int par) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  if (threadIdx.x == 0) peer_round(p, b);
  __syncthreads();
  const long long per = ((n / 8 + gridDim.x - 1) / gridDim.x) * 8;
  const long long lo = (long long)b * per;
  const long long hi = lo + per < n ? lo + per : n;
  for (long long i = lo + threadIdx.x * 8; i < hi; i += blockDim.x * 8) {
    float acc[8];
    {
      const uint4 u = *reinterpret_cast<const uint4*>(x + i);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        acc[2 * k] = f.x;
        acc[2 * k + 1] = f.y;
      }
    }
    for (int j = 0; j < p.world; ++j) {
      const uint4 u = __ldcv(reinterpret_cast<const uint4*>(p.part[par][j] + i));
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
    *reinterpret_cast<uint4*>(x + i) = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  }
}

// mode 3: x[i] += sum_j recv[j][i] once all `world` senders have arrived; flags[par] counts
// arrivals, flags[2 + par] this kernel's finished CTAs (the last re-arms both)
__global__ void __launch_bounds__(256) tp_push_reduce_kernel(const __nv_bfloat16* __restrict__ recv, long long slot,
                                                             int world, unsigned* flags, __nv_bfloat16* __restrict__ x,
                                                             long long n, int par) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0)
    while (ld_acquire_sys(flags + par) < (unsigned)world) {
    }
  __syncthreads();
  const long long per = ((n / 8 + gridDim.x - 1) / gridDim.x) * 8;
  const long long lo = (long long)blockIdx.x * per;
  const long long hi = lo + per < n ? lo + per : n;
  for (long long i = lo + threadIdx.x * 8; i < hi; i += blockDim.x * 8) {
    float acc[8];
    {
      const uint4 u = *reinterpret_cast<const uint4*>(x + i);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        acc[2 * k] = f.x;
        acc[2 * k + 1] = f.y;
      }
    }
    for (int j = 0; j < world; ++j) {  // fixed sender order: bit-identical on every rank
      const uint4 u = __ldcv(reinterpret_cast<const uint4*>(recv + j * slot + i));
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
    *reinterpret_cast<uint4*>(x + i) = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(flags + 2 + par, 1u) == gridDim.x - 1) {
    flags[par] = 0u;
    flags[2 + par] = 0u;
    __threadfence_system();
  }
}

// ------------------------------------------------------------------ vocab-parallel argmax
// key = (order-preserving bits of the logit) << 32 | (0xffffffff - global index):
// max over keys = max logit, lowest index among ties (torch.argmax semantics).
__device__ __forceinline__ unsigned long long argmax_key(float v, unsigned idx) {
  unsigned u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (0xffffffffu - idx);
}

__global__ void argmax_key_kernel(const __nv_bfloat16* __restrict__ logits, long long ld, int V, int offset,
                                  unsigned long long* __restrict__ keys) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const __nv_bfloat16* x = logits + (size_t)row * ld;
  unsigned long long best = 0ull;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const unsigned long long k = argmax_key(__bfloat162float(x[i]), (unsigned)(offset + i));
    best = k > best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
    best = k > best ? k : best;
  }
  __shared__ unsigned long long sk[32];
  if ((threadIdx.x & 31) == 0) sk[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = sk[w] > best ? sk[w] : best;
    keys[row] = best;
  }
}

// merge: keys of every rank (peer mode: read from peers after a flag round; NCCL mode:
// already max-reduced in keys_mine) -> token ids, scattered into last_tok like rb_argmax
__global__ void argmax_merge_kernel(const TpPeers p, int use_peers, const unsigned long long* __restrict__ keys_mine,
                                    int T, int* __restrict__ out, const int* __restrict__ slot_of_row,
                                    int* __restrict__ last_tok, const int* __restrict__ row_valid) {
  pdl_trigger();
  pdl_wait();
  if (use_peers) {
    if (threadIdx.x == 0) peer_round(p, kMaxArBlocks - 1);
    __syncthreads();
  }
  for (int row = threadIdx.x; row < T; row += blockDim.x) {
    unsigned long long best = keys_mine[row];
    if (use_peers)
      for (int j = 0; j < p.world; ++j) {
        const unsigned long long k = __ldcv(p.keys[j] + row);
        best = k > best ? k : best;
      }
    if (row_valid && row_valid[row] <= 0) continue;
    const int id = (int)(0xffffffffu - (unsigned)(best & 0xffffffffull));
    out[row] = id;
    if (slot_of_row && last_tok) last_tok[slot_of_row[row]] = id;
  }
}

// ------------------------------------------------------------------ forward hooks
// Row-parallel GEMM output target: peer mode -> this rank's staging buffer (no
// residual); NCCL mode -> x itself, residual added on rank 0 only.
// mode 3: the row-parallel GEMM's push arguments for the current call parity (nullptr otherwise)
bool tp_gemm_push(void* tp_, GemmPush* out) {
  TpCtx* tp = static_cast<TpCtx*>(tp_);
  if (!tp || tp->mode != 3 || tp->world <= 1) return false;
  out->world = tp->world;
  for (int j = 0; j < tp->world; ++j) {
    out->dst[j] = tp->peers.part[tp->parity][j] + (size_t)tp->rank * tp->part_elems;
    out->arrive[j] = tp->peers.flags[j] + tp->parity;
  }
  out->done_local = tp->peers.flags[tp->rank] + 4 + tp->parity;
  return true;
}

void* tp_gemm_out(void* tp_, void* x, const void** residual) {
  TpCtx* tp = static_cast<TpCtx*>(tp_);
  if (!tp) return x;
  if (tp->mode == 3 && tp->world > 1) {
    *residual = nullptr;  // the reduce kernel adds it
    return x;             // (unused: the push epilogue writes the receive slots)
  }
  if (tp->mode == 2 && tp->world > 1) {
    *residual = nullptr;
    return tp->peers.part[tp->parity][tp->rank];
  }
  if (tp->rank != 0) *residual = nullptr;
  return x;
}

void tp_begin(void* tp_) {
  if (tp_) static_cast<TpCtx*>(tp_)->parity = 0;
}

int tp_reduce(void* tp_, void* x, long long n, cudaStream_t st) {
  TpCtx* tp = static_cast<TpCtx*>(tp_);
  if (!tp) return 0;
  if (tp->mode == 1) {  // NCCL at any world size (world 1: an in-place identity)
    ncclResult_t r = nccl().all_reduce(x, x, (size_t)n, ncclBfloat16, ncclSum, tp->comm, st);
    return r == ncclSuccess ? 0 : nccl_error("ncclAllReduce", r);
  }
  if (tp->world <= 1) return 0;
  if ((size_t)n > tp->part_elems || n % 8) return set_error("tp: all-reduce exceeds the staging buffers");
  if (tp->mode == 3) {
    int blocks = (int)((n + 256 * 8 * 4 - 1) / (256 * 8 * 4));
    if (blocks > 120) blocks = 120;
    if (blocks < 1) blocks = 1;
    cudaError_t e = launch_k(tp_push_reduce_kernel, dim3(blocks), dim3(256), 0, st, 1,
                             (const __nv_bfloat16*)tp->peers.part[tp->parity][tp->rank], (long long)tp->part_elems,
                             tp->world, tp->peers.flags[tp->rank], static_cast<__nv_bfloat16*>(x), n, tp->parity);
    tp->parity ^= 1;
    return e == cudaSuccess ? 0 : set_cuda_error("tp push reduce launch", e);
  }
  int blocks = (int)((n + 256 * 8 * 4 - 1) / (256 * 8 * 4));
  if (blocks > kMaxArBlocks - 1) blocks = kMaxArBlocks - 1;  // the last flag slot belongs to the argmax merge
  if (blocks < 1) blocks = 1;
  cudaError_t e = launch_k(tp_ar_add_kernel, dim3(blocks), dim3(256), 0, st, 1, tp->peers,
                           static_cast<__nv_bfloat16*>(x), n, tp->parity);
  tp->parity ^= 1;
  return e == cudaSuccess ? 0 : set_cuda_error("tp all-reduce launch", e);
}

int tp_argmax(void* tp_, const void* logits, long long ld, int T, int V_local, int offset, int* out,
              const int* slot_of_row, int* last_tok, const int* row_valid, cudaStream_t st) {
  TpCtx* tp = static_cast<TpCtx*>(tp_);
  unsigned long long* keys = tp->peers.keys[tp->rank];
  cudaError_t e = launch_k(argmax_key_kernel, dim3(T), dim3(512), 0, st, 1,
                           static_cast<const __nv_bfloat16*>(logits), ld, V_local, offset, keys);
  if (e != cudaSuccess) return set_cuda_error("tp argmax launch", e);
  int use_peers = 0;
  if (tp->mode == 1) {
    ncclResult_t r = nccl().all_reduce(keys, keys, (size_t)T, ncclUint64, ncclMax, tp->comm, st);
    if (r != ncclSuccess) return nccl_error("ncclAllReduce(max)", r);
  } else if (tp->world > 1) {
    use_peers = 1;
  }
  e = launch_k(argmax_merge_kernel, dim3(1), dim3(256), 0, st, 1, tp->peers, use_peers,
               (const unsigned long long*)keys, T, out, slot_of_row, last_tok, row_valid);
  return e == cudaSuccess ? 0 : set_cuda_error("tp argmax merge launch", e);
}

}  // namespace rb

// ------------------------------------------------------------------ C ABI
extern "C" {

int rb_tp_nccl_available(void) { return rb::nccl().ok ? 1 : 0; }

int rb_tp_nccl_unique_id(void* id_out) {
  if (!rb::nccl().ok) return rb::set_error("tp: libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = rb::nccl().get_unique_id(&id);
  if (r != ncclSuccess) return rb::nccl_error("ncclGetUniqueId", r);
  memcpy(id_out, &id, sizeof id);
  return 0;
}

int rb_tp_nccl_comm_init(const void* id_in, int nranks, int rank, void** comm_out) {
  if (!rb::nccl().ok) return rb::set_error("tp: libnccl.so.2 not loadable");
  ncclUniqueId id;
  memcpy(&id, id_in, sizeof id);
  ncclComm_t comm;
  ncclResult_t r = rb::nccl().comm_init_rank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return rb::nccl_error("ncclCommInitRank", r);
  *comm_out = comm;
  return 0;
}

int rb_tp_nccl_comm_destroy(void* comm) {
  if (!comm) return 0;
  ncclResult_t r = rb::nccl().comm_destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? 0 : rb::nccl_error("ncclCommDestroy", r);
}

int rb_tp_create(int world, int rank, int mode, void* nccl_comm, void* const* part0, void* const* part1,
                 void* const* keys, void* const* flags, void* epoch, size_t part_elems, void** tp_out) {
  if (world < 1 || world > rb::kMaxRanks || rank < 0 || rank >= world)
    return rb::set_error("tp: world must be 1..8 and 0 <= rank < world");
  if (mode < 1 || mode > 3) return rb::set_error("tp: mode 1 (NCCL), 2 (peer memory) or 3 (GEMM push)");
  if (mode == 1 && world > 1 && !nccl_comm) return rb::set_error("tp: NCCL mode needs a communicator");
  if (!keys || !keys[rank]) return rb::set_error("tp: every rank needs an argmax key buffer");
  if (mode >= 2 && world > 1 && (!part0 || !part1 || !flags || !epoch))
    return rb::set_error("tp: peer mode needs staging, flag and epoch buffers of every rank");
  rb::TpCtx* tp = new rb::TpCtx{};
  tp->world = world;
  tp->rank = rank;
  tp->mode = mode;
  tp->comm = static_cast<ncclComm_t>(nccl_comm);
  tp->part_elems = part_elems;
  tp->peers.world = world;
  tp->peers.rank = rank;
  for (int j = 0; j < world; ++j) {
    tp->peers.keys[j] = static_cast<unsigned long long*>(keys[j]);
    if (mode >= 2 && world > 1) {
      tp->peers.part[0][j] = static_cast<__nv_bfloat16*>(part0[j]);
      tp->peers.part[1][j] = static_cast<__nv_bfloat16*>(part1[j]);
      tp->peers.flags[j] = static_cast<unsigned*>(flags[j]);
    }
  }
  tp->peers.epoch = static_cast<unsigned*>(epoch);
  *tp_out = tp;
  return 0;
}

int rb_tp_destroy(void* tp) {
  delete static_cast<rb::TpCtx*>(tp);
  return 0;
}

size_t rb_tp_flag_words(void) { return (size_t)rb::kMaxRanks * rb::kMaxArBlocks; }

int rb_tp_debug_nowait(void* tp, int on) {
  static_cast<rb::TpCtx*>(tp)->peers.nowait = on;
  return 0;
}

/* x += sum over ranks of the partials (peer mode: this rank's partial must already be in
 * its staging buffer of the current parity; NCCL mode: x holds this rank's contribution). */
int rb_tp_allreduce(void* tp, void* x, long long n, void* stream) {
  rb::TpCtx* t = static_cast<rb::TpCtx*>(tp);
  if (t && t->mode == 3 && t->world > 1)  // its inputs arrive only from a row-parallel GEMM's push epilogue
    return rb::set_error("tp: mode 3 reduces only behind a pushing GEMM (rb_decoder_forward)");
  if (t && t->mode == 2 && t->world > 1) {
    // standalone use: stage x as this rank's partial and reduce into x (x = sum of partials)
    void* stage = t->peers.part[t->parity][t->rank];
    cudaError_t e = cudaMemcpyAsync(stage, x, (size_t)n * 2, cudaMemcpyDeviceToDevice,
                                    reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return rb::set_cuda_error("tp stage copy", e);
    e = cudaMemsetAsync(x, 0, (size_t)n * 2, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return rb::set_cuda_error("tp zero", e);
  }
  return rb::tp_reduce(tp, x, n, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
