// extern "C" entry points declared in include/rapid_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include "rb_common.h"
#include "../../include/rapid_b200.h"

namespace rb {
int decode_attention_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* block_table,
                            int bt_stride, const int* row_slot, const int* seq_lens, void* out,
                            long long out_tok_stride, void* workspace, size_t ws_bytes, int B, int Hq, int Hkv,
                            int head_dim, int max_pages, float scale, int num_blocks, int num_sms, cudaStream_t st);
int rmsnorm_launch(const void* x, long long ldx, const void* w, void* y, long long ldy, int T, int H, float eps,
                   cudaStream_t st);
int rope_cache_launch(const void* qkv, long long ld_qkv, const int* pos, const int* tok_slot, const int* bt,
                      int bt_stride, const float* cos_sin, void* q_out, long long ld_q, void* cache_layer, int T,
                      int Hq, int Hkv, int D, cudaStream_t st);
int silu_mul_launch(const void* gu, long long ld_gu, void* y, long long ldy, int T, int I, cudaStream_t st);
int embed_launch(const int* ids, const int* slot_of_row, const int* last_tok, const void* table, void* y, int T, int H,
                 int* ids_out, cudaStream_t st);
int argmax_launch(const void* logits, long long ld, int T, int V, int* out, const int* slot_of_row, int* last_tok,
                  const int* row_valid, cudaStream_t st);
int bt_update_launch(const int* upd, int* block_table, int bt_stride, int max_updates, cudaStream_t st);
int set_last_tok_launch(int* last_tok, int slot, const int* value_ptr, int value, cudaStream_t st);
int prefill_attention_tc_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* bt, int T,
                                int start, int Hq, int Hkv, int head_dim, void* out, long long out_tok_stride,
                                float scale, int num_blocks, cudaStream_t st);
int gemm_set_trace(unsigned long long* buf);
int gemm_set_pair_mode(int mode);
int gemm_set_variant(int v);
int gemm_set_prefetch(int kblocks);
int gemm_set_prefill_streamk(int on, double max_frac);
int gemm_set_prefill_bn(int bn);
int prefill_attn_set_tiles(int tiles);
int decode_attn_set_kv_ops(int one_op);
int decode_attn_set_shape(int shape);
int gemm_set_ksplit(int s);
int stream_read_launch(const void* src, long long bytes, int chunk, int stages, int num_sms, int* sink,
                       cudaStream_t st);
int stream_read_tma_launch(const void* src, long long bytes, int box_rows, int per_stage, int stages, int num_sms,
                           int* sink, cudaStream_t st);
}  // namespace rb

#define ST(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

const char* rb_version(void) { return "rapid_b200 0.1 sm_100a"; }
const char* rb_last_error(void) { return rb::last_error(); }

int rb_debug_gemm_trace(unsigned long long* buf) { return rb::gemm_set_trace(buf); }
int rb_debug_gemm_pair_mode(int mode) { return rb::gemm_set_pair_mode(mode); }
int rb_debug_gemm_variant(int v) { return rb::gemm_set_variant(v); }
int rb_debug_gemm_prefetch(int kblocks) { return rb::gemm_set_prefetch(kblocks); }
int rb_debug_gemm_prefill_streamk(int on, double max_frac) { return rb::gemm_set_prefill_streamk(on, max_frac); }
int rb_debug_gemm_prefill_bn(int bn) { return rb::gemm_set_prefill_bn(bn); }
int rb_debug_pattn_tiles(int tiles) { return rb::prefill_attn_set_tiles(tiles); }
int rb_debug_decode_kv_one_op(int on) { return rb::decode_attn_set_kv_ops(on); }
int rb_debug_decode_attn_shape(int shape) { return rb::decode_attn_set_shape(shape); }
int rb_debug_gemm_ksplit(int s) { return rb::gemm_set_ksplit(s); }
int rb_debug_stream_read(const void* src, long long bytes, int chunk, int stages, int num_sms, int* sink,
                         void* stream) {
  return rb::stream_read_launch(src, bytes, chunk, stages, num_sms, sink, static_cast<cudaStream_t>(stream));
}
int rb_debug_stream_read_tma(const void* src, long long bytes, int box_rows, int per_stage, int stages, int num_sms,
                             int* sink, void* stream) {
  return rb::stream_read_tma_launch(src, bytes, box_rows, per_stage, stages, num_sms, sink,
                                    static_cast<cudaStream_t>(stream));
}
int rb_set_pdl(int on) {
  rb::set_pdl(on != 0);
  return 0;
}

int rb_device_sm_count(int device, int* out) {
  cudaError_t e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device);
  return e == cudaSuccess ? 0 : rb::set_cuda_error("sm count", e);
}

int rb_gemm_bf16(const void* X, const void* W, void* Y, const void* bias, const void* R, int T, int O, int K,
                 long long ldx, long long ldw, long long ldy, int mode, int num_sms, void* workspace,
                 size_t ws_bytes, int* counters, int counters_len, void* stream) {
  return rb::gemm_bf16_launch(X, W, Y, bias, R, T, O, K, ldx, ldw, ldy, mode, num_sms, workspace, ws_bytes, counters,
                              counters_len, ST(stream));
}

int rb_gemm_qkv_rope(const void* X, const void* W, const void* bias, int T, int K, long long ldx, int Hq, int Hkv,
                     int head_dim, const int* pos, const int* tok_slot, const int* block_table, int bt_stride,
                     const float* cos_sin, void* q_out, long long ld_q, void* cache_layer, int mode, int num_sms,
                     void* workspace, size_t ws_bytes, int* counters, int counters_len, void* stream) {
  const int nq = (Hq + 2 * Hkv) * head_dim;
  const rb::GemmRope rp{pos, tok_slot, block_table, bt_stride, cos_sin, q_out, ld_q, cache_layer, Hq, Hkv, head_dim};
  return rb::gemm_bf16_launch(X, W, q_out, bias, nullptr, T, nq, K, ldx, K, ld_q, mode, num_sms, workspace, ws_bytes,
                              counters, counters_len, ST(stream), &rp);
}

int rb_decode_attention(const void* q, long long q_tok_stride, const void* cache_layer, const int* block_table,
                        int bt_stride, const int* row_slot, const int* seq_lens, void* out,
                        long long out_tok_stride, void* workspace, size_t ws_bytes, int B, int Hq, int Hkv,
                        int head_dim, int max_pages, float scale, int num_blocks, int num_sms, void* stream) {
  return rb::decode_attention_launch(q, q_tok_stride, cache_layer, block_table, bt_stride, row_slot, seq_lens, out,
                                     out_tok_stride, workspace, ws_bytes, B, Hq, Hkv, head_dim, max_pages, scale,
                                     num_blocks, num_sms, ST(stream));
}

int rb_prefill_attention(const void* q, long long q_tok_stride, const void* cache_layer,
                            const int* block_table_row, int T, int start, int Hq, int Hkv, int head_dim, void* out,
                            long long out_tok_stride, float scale, int num_blocks, void* stream) {
  return rb::prefill_attention_tc_launch(q, q_tok_stride, cache_layer, block_table_row, T, start, Hq, Hkv, head_dim,
                                         out, out_tok_stride, scale, num_blocks, ST(stream));
}

int rb_rope_cache_write(const void* qkv, long long ld_qkv, const int* pos, const int* tok_slot,
                        const int* block_table, int bt_stride, const float* cos_sin, void* q_out, long long ld_q,
                        void* cache_layer, int T, int Hq, int Hkv, int head_dim, void* stream) {
  return rb::rope_cache_launch(qkv, ld_qkv, pos, tok_slot, block_table, bt_stride, cos_sin, q_out, ld_q, cache_layer,
                               T, Hq, Hkv, head_dim, ST(stream));
}

int rb_rmsnorm(const void* x, long long ldx, const void* w, void* y, long long ldy, int T, int H, float eps,
               void* stream) {
  return rb::rmsnorm_launch(x, ldx, w, y, ldy, T, H, eps, ST(stream));
}

int rb_silu_mul(const void* gate_up, long long ld_gu, void* y, long long ldy, int T, int I, void* stream) {
  return rb::silu_mul_launch(gate_up, ld_gu, y, ldy, T, I, ST(stream));
}

int rb_embed(const int* ids, const int* slot_of_row, const int* last_tok, const void* table, void* y, int T, int H,
             int* ids_out, void* stream) {
  return rb::embed_launch(ids, slot_of_row, last_tok, table, y, T, H, ids_out, ST(stream));
}

int rb_argmax(const void* logits, long long ld, int T, int V, int* out, const int* slot_of_row, int* last_tok,
              const int* row_valid, void* stream) {
  return rb::argmax_launch(logits, ld, T, V, out, slot_of_row, last_tok, row_valid, ST(stream));
}

int rb_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : rb::set_cuda_error("rb_memcpy_async", e);
}

int rb_graph_launch(void* graph_exec, void* stream) {
  cudaError_t e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : rb::set_cuda_error("rb_graph_launch", e);
}

int rb_block_table_update(const int* upd, int* block_table, int bt_stride, int max_updates, void* stream) {
  return rb::bt_update_launch(upd, block_table, bt_stride, max_updates, ST(stream));
}

int rb_set_last_token(int* last_tok, int slot, const int* value_ptr, int value, void* stream) {
  return rb::set_last_tok_launch(last_tok, slot, value_ptr, value, ST(stream));
}

// ------------------------------------------------------------------ green contexts
struct GreenSplit {
  CUgreenCtx ctx[2];
  CUstream stream[2];
};

typedef CUresult (*PFN_cuDeviceGet)(CUdevice*, int);
typedef CUresult (*PFN_cuDeviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType);
typedef CUresult (*PFN_cuDevSmResourceSplitByCount)(CUdevResource*, unsigned int*, const CUdevResource*,
                                                    CUdevResource*, unsigned int, unsigned int);
typedef CUresult (*PFN_cuDevResourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int);
typedef CUresult (*PFN_cuGreenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
typedef CUresult (*PFN_cuGreenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned int, int);
typedef CUresult (*PFN_cuGreenCtxDestroy)(CUgreenCtx);
typedef CUresult (*PFN_cuStreamDestroy)(CUstream);

#define RB_SYM(T, name)                                                  \
  T name = reinterpret_cast<T>(rb::driver_symbol(#name));                \
  if (!name) return rb::set_error("driver symbol " #name " unavailable");

int rb_green_split(int device, int first_sms, void** handle, void** stream_first, void** stream_second,
                   int* sms_first, int* sms_second) {
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) return rb::set_cuda_error("cudaSetDevice", ce);
  cudaFree(0);  // make sure the primary context exists
  RB_SYM(PFN_cuDeviceGet, cuDeviceGet);
  RB_SYM(PFN_cuDeviceGetDevResource, cuDeviceGetDevResource);
  RB_SYM(PFN_cuDevSmResourceSplitByCount, cuDevSmResourceSplitByCount);
  RB_SYM(PFN_cuDevResourceGenerateDesc, cuDevResourceGenerateDesc);
  RB_SYM(PFN_cuGreenCtxCreate, cuGreenCtxCreate);
  RB_SYM(PFN_cuGreenCtxStreamCreate, cuGreenCtxStreamCreate);
  CUdevice dev;
  CUresult r = cuDeviceGet(&dev, device);
  if (r != CUDA_SUCCESS) return rb::set_cu_error("cuDeviceGet", r);
  CUdevResource all;
  r = cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  if (r != CUDA_SUCCESS) return rb::set_cu_error("cuDeviceGetDevResource", r);
  CUdevResource group, rest;
  unsigned int ng = 1;
  r = cuDevSmResourceSplitByCount(&group, &ng, &all, &rest, 0, (unsigned)first_sms);
  if (r != CUDA_SUCCESS || ng != 1) return rb::set_cu_error("cuDevSmResourceSplitByCount", r);
  GreenSplit* gs = new GreenSplit();
  CUdevResource parts[2] = {group, rest};
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc desc;
    r = cuDevResourceGenerateDesc(&desc, &parts[i], 1);
    if (r != CUDA_SUCCESS) { delete gs; return rb::set_cu_error("cuDevResourceGenerateDesc", r); }
    r = cuGreenCtxCreate(&gs->ctx[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r != CUDA_SUCCESS) { delete gs; return rb::set_cu_error("cuGreenCtxCreate", r); }
    r = cuGreenCtxStreamCreate(&gs->stream[i], gs->ctx[i], CU_STREAM_NON_BLOCKING, 0);
    if (r != CUDA_SUCCESS) { delete gs; return rb::set_cu_error("cuGreenCtxStreamCreate", r); }
  }
  *handle = gs;
  *stream_first = gs->stream[0];
  *stream_second = gs->stream[1];
  *sms_first = (int)group.sm.smCount;
  *sms_second = (int)rest.sm.smCount;
  return 0;
}

int rb_green_destroy(void* handle) {
  if (!handle) return 0;
  RB_SYM(PFN_cuStreamDestroy, cuStreamDestroy);
  RB_SYM(PFN_cuGreenCtxDestroy, cuGreenCtxDestroy);
  GreenSplit* gs = reinterpret_cast<GreenSplit*>(handle);
  for (int i = 0; i < 2; ++i) {
    cuStreamDestroy(gs->stream[i]);
    cuGreenCtxDestroy(gs->ctx[i]);
  }
  delete gs;
  return 0;
}

}  // extern "C"

// Profiling probe: make the (regular) context of green partition i current on this thread,
// so launches can be issued with the green context current instead of through a green
// stream from the primary context.
typedef CUresult (*PFN_cuCtxFromGreenCtx)(CUcontext*, CUgreenCtx);
typedef CUresult (*PFN_cuCtxPushCurrent)(CUcontext);
typedef CUresult (*PFN_cuCtxPopCurrent)(CUcontext*);
extern "C" {
int rb_debug_green_ctx_push(void* handle, int i) {
  RB_SYM(PFN_cuCtxFromGreenCtx, cuCtxFromGreenCtx);
  RB_SYM(PFN_cuCtxPushCurrent, cuCtxPushCurrent);
  GreenSplit* gs = reinterpret_cast<GreenSplit*>(handle);
  CUcontext c;
  CUresult r = cuCtxFromGreenCtx(&c, gs->ctx[i]);
  if (r != CUDA_SUCCESS) return rb::set_cu_error("cuCtxFromGreenCtx", r);
  r = cuCtxPushCurrent(c);
  if (r != CUDA_SUCCESS) return rb::set_cu_error("cuCtxPushCurrent", r);
  return 0;
}

int rb_debug_ctx_pop(void) {
  RB_SYM(PFN_cuCtxPopCurrent, cuCtxPopCurrent);
  CUcontext c;
  CUresult r = cuCtxPopCurrent(&c);
  if (r != CUDA_SUCCESS) return rb::set_cu_error("cuCtxPopCurrent", r);
  return 0;
}
}  // extern "C"
