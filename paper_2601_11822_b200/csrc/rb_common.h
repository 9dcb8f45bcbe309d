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
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer);

int gemm_bf16_launch(const void* X, const void* W, void* Y, const void* bias, const void* residual, int T,
                     int O, int K, long long ldx, long long ldw, long long ldy, int mode, int num_sms,
                     void* workspace, size_t ws_bytes, int* counters, int counters_len, cudaStream_t stream);

}  // namespace rb

#define RB_ERR_ARG 1
#define RB_ERR_CUDA 2
#define RB_ERR_DRIVER 3
