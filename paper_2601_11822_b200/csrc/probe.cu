// Diagnostic (not on the serving path): per-SM ingest ceiling of a partition.
//
// rb_debug_stream_read streams `bytes` of global memory into shared memory with 1D bulk
// copies (cp.async.bulk, mbarrier completion) and no compute: one CTA per SM of the
// launch's partition, a ring of `stages` x `chunk` bytes kept full by one elected thread.
// The achieved GB/s / SMs is the most an SM-resident consumer (decode attention K3, the
// decode GEMMs' operand stream) can pull through the SM's L2 port at this ring depth.
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "rb_common.h"

namespace rb {

__global__ void __launch_bounds__(32, 1)
    stream_read_kernel(const uint8_t* __restrict__ src, long long bytes, int chunk, int stages, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  const long long nchunks = bytes / chunk;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
  fence_barrier_init();
  // chunks c = blockIdx.x + k * gridDim.x
  long long issued = blockIdx.x, done = blockIdx.x;
  int st_issue = 0, st_done = 0;
  uint32_t ph = 0;
  for (int s = 0; s < stages && issued < nchunks; ++s, issued += gridDim.x) {
    mbar_arrive_expect_tx(&full[st_issue], (uint32_t)chunk);
    bulk_g2s(smem + (size_t)st_issue * chunk, src + issued * chunk, (uint32_t)chunk, &full[st_issue]);
    st_issue = st_issue + 1 == stages ? 0 : st_issue + 1;
  }
  uint32_t acc = 0;
  for (; done < nchunks; done += gridDim.x) {
    mbar_wait(&full[st_done], ph);
    acc += smem[(size_t)st_done * chunk];
    if (issued < nchunks) {  // refill the slot just drained
      mbar_arrive_expect_tx(&full[st_done], (uint32_t)chunk);
      bulk_g2s(smem + (size_t)st_done * chunk, src + issued * chunk, (uint32_t)chunk, &full[st_done]);
      issued += gridDim.x;
    }
    if (++st_done == stages) {
      st_done = 0;
      ph ^= 1;
    }
  }
  if (acc == 0x12345678u) *sink = (int)acc;
}

// Same ring, filled with 2D tensor-TMA boxes {64 bf16, box_rows} (128B swizzle, the decode
// attention's box shape at box_rows = 16): `per_stage` boxes per stage, so the op size and the
// bytes in flight can be varied independently.
__global__ void __launch_bounds__(32, 1)
    stream_read_tma_kernel(const __grid_constant__ CUtensorMap map, long long nrows, int box_rows, int per_stage,
                           int stages, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int box_bytes = box_rows * 128;
  const int stage_bytes = box_bytes * per_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  const long long nchunks = nrows / ((long long)box_rows * per_stage);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
  fence_barrier_init();
  auto issue = [&](int slot, long long c) {
    mbar_arrive_expect_tx(&full[slot], (uint32_t)stage_bytes);
    for (int b = 0; b < per_stage; ++b)
      tma_load_2d(smem + (size_t)slot * stage_bytes + b * box_bytes, &map, &full[slot], 0,
                  (int32_t)((c * per_stage + b) * box_rows), kEvictNormal);
  };
  long long issued = blockIdx.x, done = blockIdx.x;
  int st_issue = 0, st_done = 0;
  uint32_t ph = 0;
  for (int s = 0; s < stages && issued < nchunks; ++s, issued += gridDim.x) {
    issue(st_issue, issued);
    st_issue = st_issue + 1 == stages ? 0 : st_issue + 1;
  }
  uint32_t acc = 0;
  for (; done < nchunks; done += gridDim.x) {
    mbar_wait(&full[st_done], ph);
    acc += smem[(size_t)st_done * stage_bytes];
    if (issued < nchunks) {
      issue(st_done, issued);
      issued += gridDim.x;
    }
    if (++st_done == stages) {
      st_done = 0;
      ph ^= 1;
    }
  }
  if (acc == 0x12345678u) *sink = (int)acc;
}

int stream_read_tma_launch(const void* src, long long bytes, int box_rows, int per_stage, int stages, int num_sms,
                           int* sink, cudaStream_t st) {
  if (box_rows < 1 || box_rows > 256 || per_stage < 1 || stages < 1)
    return set_error("stream_read_tma: box_rows in [1, 256], per_stage >= 1, stages >= 1");
  const long long nrows = bytes / 128;
  CUtensorMap map;
  int rc = make_tmap_2d_bf16(&map, src, 64, (uint64_t)nrows, 64, 64, (uint32_t)box_rows);
  if (rc) return rc;
  const int smem = stages * per_stage * box_rows * 128 + stages * 8 + 1024;
  if (smem > 227 * 1024) return set_error("stream_read_tma: ring exceeds shared memory");
  cudaError_t e =
      cudaFuncSetAttribute(stream_read_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return set_cuda_error("stream_read_tma attr", e);
  stream_read_tma_kernel<<<num_sms, 32, smem, st>>>(map, nrows, box_rows, per_stage, stages, sink);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("stream_read_tma launch", e);
  return 0;
}

int stream_read_launch(const void* src, long long bytes, int chunk, int stages, int num_sms, int* sink,
                       cudaStream_t st) {
  if (chunk % 16 || chunk <= 0 || stages < 1) return set_error("stream_read: chunk % 16 == 0, stages >= 1");
  const int smem = stages * chunk + stages * 8;
  if (smem > 227 * 1024) return set_error("stream_read: ring exceeds shared memory");
  cudaError_t e = cudaFuncSetAttribute(stream_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return set_cuda_error("stream_read attr", e);
  stream_read_kernel<<<num_sms, 32, smem, st>>>(static_cast<const uint8_t*>(src), bytes, chunk, stages, sink);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("stream_read launch", e);
  return 0;
}

}  // namespace rb
