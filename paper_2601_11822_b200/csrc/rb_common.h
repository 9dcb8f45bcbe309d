// Shared host-side plumbing for the C-ABI library: error slot, driver entry
// points (resolved at runtime so the .so has no link-time libcuda dependency),
// and TMA tensor-map encoding.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace rb {

int set_error(const char* msg);
int set_cuda_error(const char* where, cudaError_t e);
int set_cu_error(const char* where, CUresult r);
const char* last_error();

// Resolve a driver API symbol (e.g. "cuTensorMapEncodeTiled") via the runtime.
void* driver_symbol(const char* name);

// Encode a 2D bf16 tensor map: inner dim `inner` elements (contiguous), outer
// dim `outer` rows with row stride `ld` elements; box = box_inner x box_outer,
// 128-byte swizzle. Returns 0 or an error code.
cudaError_t set_smem_attr_once(const void* fn, int bytes);
int make_tmap_kv5d_bf16(CUtensorMap* map, const void* cache_layer, uint64_t num_blocks, int hkv);
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer);

// Programmatic dependent launch (PDL): kernels of the forward are launched with
// programmaticStreamSerialization so kernel N+1's CTAs start (prologue, weight
// prefetch) while kernel N drains; every such kernel calls griddepcontrol.wait before
// touching its predecessors' outputs (pdl_wait in ptx.cuh). rb_set_pdl(0) disables it.
bool pdl_enabled();
void set_pdl(bool on);

template <typename... Exp, typename... Act>
cudaError_t launch_k(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                     Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Act&&>(args)...);
}

// Fused QKV-projection epilogue (see rope_store in gemm_tcgen05.cu): RoPE on q/k and the
// paged K/V write of every token row, straight from the GEMM accumulators.
struct GemmRope {
  const int* pos;          // [T] position of each row, < 0 = padding (skipped)
  const int* tok_slot;     // [T] block-table row of each token
  const int* block_table;  // [slots][bt_stride]
  int bt_stride;
  const float* cos_sin;    // fp32 [max_pos][128] = [cos | sin]
  void* q_out;             // bf16 [T][ld_q]: rotated q heads
  long long ld_q;
  void* cache;             // one layer: [num_blocks][2][hkv][16][128] bf16
  int hq, hkv, hd;
};

// TP push epilogue (tp.cu mode 3): the GEMM writes its output tile straight into every
// rank's receive slot for this rank (peer memory, tile by tile while the GEMM runs); the last
// CTA to finish raises one arrival in every rank's counter.
struct GemmPush {
  int world;        // 0: off
  void* dst[8];     // rank j's receive slot for this sender (bf16 [rows][ldy])
  unsigned* arrive[8];
  unsigned* done_local;  // this GEMM's CTA completion counter (self-resetting)
};

int gemm_pick_ksplit(int O, int T, int K, int num_sms, size_t ws_bytes);
int add_partials_rmsnorm_launch(const float* part, int ks, long long slice, void* x, const void* w, void* y, int T,
                                int H, float eps, cudaStream_t st);
int gemm_bf16_launch(const void* X, const void* W, void* Y, const void* bias, const void* residual, int T,
                     int O, int K, long long ldx, long long ldw, long long ldy, int mode, int num_sms,
                     void* workspace, size_t ws_bytes, int* counters, int counters_len, cudaStream_t stream,
                     const GemmRope* rope = nullptr, const GemmPush* push = nullptr);

}  // namespace rb

#define RB_ERR_ARG 1
#define RB_ERR_CUDA 2
#define RB_ERR_DRIVER 3
