// Native decoder-forward driver: one C call launches a whole forward pass.
//
// The reference prices a prefill chunk / decode step / fused hybrid iteration
// as one number (costmodel.py:89-163). Here one rb_decoder_forward() call
// launches every kernel of that iteration on one stream — the host-side cost
// of a 32-layer chunk drops from ~300 Python->C calls to one — and the same
// entry serves all three shapes:
//   rows [0, n_decode)           one token per sequence, paged decode attention
//   rows [n_decode, rows)        one chunk of one sequence (causal over its paged prefix)
// Decode graphs capture this call; hybrid (chunked-prefill) iterations call it
// with both segments non-empty (K9).
#include <cuda_runtime.h>
#include "rb_common.h"
#include "../../include/rapid_b200.h"

namespace rb {
int decode_attention_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* block_table,
                            int bt_stride, const int* row_slot, const int* seq_lens, void* out,
                            long long out_tok_stride, void* workspace, size_t ws_bytes, int B, int Hq, int Hkv,
                            int head_dim, int max_pages, float scale, int num_blocks, int num_sms, cudaStream_t st);
int prefill_attention_tc_launch(const void* q, long long q_tok_stride, const void* cache_layer, const int* bt, int T,
                                int start, int Hq, int Hkv, int head_dim, void* out, long long out_tok_stride,
                                float scale, int num_blocks, cudaStream_t st);
int rmsnorm_launch(const void* x, long long ldx, const void* w, void* y, long long ldy, int T, int H, float eps,
                   cudaStream_t st);
int rope_cache_launch(const void* qkv, long long ld_qkv, const int* pos, const int* tok_slot, const int* bt,
                      int bt_stride, const float* cos_sin, void* q_out, long long ld_q, void* cache_layer, int T,
                      int Hq, int Hkv, int D, cudaStream_t st);
int silu_mul_interleaved_launch(const void* gu, long long ld_gu, void* y, long long ldy, int T, int I,
                                cudaStream_t st);
int embed_launch(const int* ids, const int* slot_of_row, const int* last_tok, const void* table, void* y, int T, int H,
                 int* ids_out, cudaStream_t st);
int argmax_launch(const void* logits, long long ld, int T, int V, int* out, const int* slot_of_row, int* last_tok,
                  const int* row_valid, cudaStream_t st);
void* tp_gemm_out(void* tp, void* x, const void** residual);
bool tp_gemm_push(void* tp, GemmPush* out);
void tp_begin(void* tp);
int tp_reduce(void* tp, void* x, long long n, cudaStream_t st);
int tp_argmax(void* tp, const void* logits, long long ld, int T, int V_local, int offset, int* out,
              const int* slot_of_row, int* last_tok, const int* row_valid, cudaStream_t st);
}  // namespace rb

// swap-AB (decode) gate|up: 1 = SwiGLU fused into the GEMM epilogue, 0 = separate kernel
static int g_decode_ksplit = 1;  // decode O / down as K-slice partials summed in the following RMSNorm
extern "C" int rb_set_decode_ksplit(int on) {
  g_decode_ksplit = on ? 1 : 0;
  return 0;
}
static int g_decode_glu = 0;
extern "C" int rb_set_decode_glu(int on) {
  g_decode_glu = on;
  return 0;
}

// An event record that survives stream capture: inside a capture it must be an external
// event-record node (a plain record would become a graph-internal dependency).
static int record_event(void* ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return rb::set_error("probe: cudaStreamIsCapturing failed");
  const unsigned flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (cudaEventRecordWithFlags(reinterpret_cast<cudaEvent_t>(ev), st, flags) != cudaSuccess)
    return rb::set_error("probe: cudaEventRecordWithFlags failed");
  return 0;
}

#define RB_TRY(x)          \
  do {                     \
    int _rc = (x);         \
    if (_rc) return _rc;   \
  } while (0)

extern "C" int rb_decoder_forward(const rb_model_t* m, const rb_workspace_t* w, const rb_batch_t* b, void* stream) {
  using namespace rb;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int T = b->rows;
  if (T <= 0) return 0;
  if (T > w->rows_cap) return set_error("decoder_forward: rows exceed workspace");
  const int nd = b->n_decode, np = b->n_prefill;
  if (nd < 0 || np < 0 || nd + np != T) return set_error("decoder_forward: rows != n_decode + n_prefill");
  const int H = m->hidden, D = m->head_dim, Hq = m->q_heads, Hkv = m->kv_heads, I = m->intermediate;
  const int nq = (Hq + 2 * Hkv) * D;
  const size_t e = 2;  // bf16 bytes
  char* x = static_cast<char*>(w->x);
  char* h = static_cast<char*>(w->h);
  char* qkv = static_cast<char*>(w->qkv);
  char* q = static_cast<char*>(w->q);
  char* attn = static_cast<char*>(w->attn);
  char* act = static_cast<char*>(w->act);
  const int sms = b->num_sms;
  void* tp = w->tp;  // tensor-parallel context of this phase (NULL: single GPU)
  tp_begin(tp);
  // ---- embedding: decode rows from device slot state, prefill rows from ids[]
  if (nd > 0) {
    if (b->ids_from_slots)
      RB_TRY(embed_launch(nullptr, w->slot, m->last_tok, m->embed, x, nd, H, w->ids, st));
    else
      RB_TRY(embed_launch(w->ids, nullptr, nullptr, m->embed, x, nd, H, nullptr, st));
  }
  if (np > 0) RB_TRY(embed_launch(w->ids + nd, nullptr, nullptr, m->embed, x + (size_t)nd * H * e, np, H, nullptr, st));
  // Decode-only iterations on a single GPU: the O and down projections run as K-slice units
  // writing fp32 partials (gemm mode bits 8..11) and the RMSNorm that follows each adds them to
  // the residual stream (add_partials_rmsnorm) — the split-K reduction without a finisher SM.
  const bool ksplit_ok = g_decode_ksplit && np == 0 && tp == nullptr && w->gemm_ws != nullptr;
  const int ks_o = ksplit_ok ? gemm_pick_ksplit(H, T, Hq * D, sms, w->gemm_ws_bytes) : 1;
  const int ks_d = ksplit_ok ? gemm_pick_ksplit(H, T, I, sms, w->gemm_ws_bytes) : 1;
  const float* part = static_cast<const float*>(w->gemm_ws);
  bool h_ready = false;  // h already holds ln1(x) of this layer (fused into the previous down's consumer)
  for (int l = 0; l < m->layers; ++l) {
    char* cache = static_cast<char*>(m->kv_cache) + (size_t)l * m->kv_layer_stride_bytes;
    if (!h_ready) RB_TRY(rmsnorm_launch(x, H, m->ln1[l], h, H, T, H, m->rms_eps, st));
    h_ready = false;
    if (m->qk_layout == 1) {
      // q|k rows pair-interleaved: RoPE and the paged K/V write run in the QKV GEMM's
      // epilogue (no qkv round trip through HBM, no separate RoPE kernel)
      const GemmRope rp{w->pos, w->slot, m->block_table, m->bt_stride, m->cos_sin, q, (long long)Hq * D, cache,
                        Hq, Hkv, D};
      RB_TRY(gemm_bf16_launch(h, m->wqkv[l], qkv, m->bqkv ? m->bqkv[l] : nullptr, nullptr, T, nq, H, H, H, nq, 0,
                              sms, w->gemm_ws, w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st, &rp));
    } else {
      RB_TRY(gemm_bf16_launch(h, m->wqkv[l], qkv, m->bqkv ? m->bqkv[l] : nullptr, nullptr, T, nq, H, H, H, nq, 0,
                              sms, w->gemm_ws, w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st));
      RB_TRY(rope_cache_launch(qkv, nq, w->pos, w->slot, m->block_table, m->bt_stride, m->cos_sin, q, Hq * D, cache,
                               T, Hq, Hkv, D, st));
    }
    if (nd > 0) {
      const bool probe = w->probe_ev0 && w->probe_ev1 && l == w->probe_layer;
      if (probe) RB_TRY(record_event(w->probe_ev0, st));
      RB_TRY(decode_attention_launch(q, (long long)Hq * D, cache, m->block_table, m->bt_stride, w->slot, w->seq, attn,
                                     (long long)Hq * D, w->attn_ws, w->attn_ws_bytes, nd, Hq, Hkv, D, b->max_pages,
                                     m->attn_scale, m->num_blocks, sms, st));
      if (probe) RB_TRY(record_event(w->probe_ev1, st));
    }
    if (np > 0)
      RB_TRY(prefill_attention_tc_launch(q + (size_t)nd * Hq * D * e, (long long)Hq * D, cache,
                                         m->block_table + (size_t)b->prefill_slot * m->bt_stride, np,
                                         b->prefill_start, Hq, Hkv, D, attn + (size_t)nd * Hq * D * e,
                                         (long long)Hq * D, m->attn_scale, m->num_blocks, st));
    if (ks_o > 1) {
      RB_TRY(gemm_bf16_launch(attn, m->wo[l], nullptr, nullptr, nullptr, T, H, Hq * D, Hq * D, Hq * D, H,
                              2 | (ks_o << 8), sms, w->gemm_ws, w->gemm_ws_bytes, w->gemm_counters,
                              w->gemm_counters_len, st));
      RB_TRY(add_partials_rmsnorm_launch(part, ks_o, (long long)T * H, x, m->ln2[l], h, T, H, m->rms_eps, st));
    } else {
      {  // row-parallel under TP: partial -> all-reduce with the residual add
        const void* res = x;
        void* y = tp_gemm_out(tp, x, &res);
        GemmPush push{};
        const bool pushed = tp_gemm_push(tp, &push);  // mode 3: the epilogue stores into every rank
        RB_TRY(gemm_bf16_launch(attn, m->wo[l], y, nullptr, res, T, H, Hq * D, Hq * D, Hq * D, H, 0, sms, w->gemm_ws,
                                w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st, nullptr,
                                pushed ? &push : nullptr));
        RB_TRY(tp_reduce(tp, x, (long long)T * H, st));
      }
      RB_TRY(rmsnorm_launch(x, H, m->ln2[l], h, H, T, H, m->rms_eps, st));
    }
    // gate|up (rows interleaved in 16-blocks): token-major tiles fuse the SwiGLU into the
    // GEMM epilogue; swap-AB (decode) tiles measured faster with the separate kernel.
    if (T > 256 || g_decode_glu) {
      RB_TRY(gemm_bf16_launch(h, m->wgu[l], act, nullptr, nullptr, T, 2 * I, H, H, H, I, 4, sms, w->gemm_ws,
                              w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st));
    } else {
      char* gu = static_cast<char*>(w->gu);
      RB_TRY(gemm_bf16_launch(h, m->wgu[l], gu, nullptr, nullptr, T, 2 * I, H, H, H, 2 * I, 0, sms, w->gemm_ws,
                              w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st));
      RB_TRY(silu_mul_interleaved_launch(gu, 2 * I, act, I, T, I, st));
    }
    if (ks_d > 1) {
      RB_TRY(gemm_bf16_launch(act, m->wd[l], nullptr, nullptr, nullptr, T, H, I, I, I, H, 2 | (ks_d << 8), sms,
                              w->gemm_ws, w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st));
      // the residual add rides on the next layer's ln1 (or, after the last layer, on the final
      // norm, which the sampling rows below then skip)
      const void* wn = l + 1 < m->layers ? m->ln1[l + 1] : m->final_norm;
      RB_TRY(add_partials_rmsnorm_launch(part, ks_d, (long long)T * H, x, wn, h, T, H, m->rms_eps, st));
      h_ready = true;
    } else {
      const void* res = x;
      void* y = tp_gemm_out(tp, x, &res);
      GemmPush push{};
      const bool pushed = tp_gemm_push(tp, &push);
      RB_TRY(gemm_bf16_launch(act, m->wd[l], y, nullptr, res, T, H, I, I, I, H, 0, sms, w->gemm_ws, w->gemm_ws_bytes,
                              w->gemm_counters, w->gemm_counters_len, st, nullptr, pushed ? &push : nullptr));
      RB_TRY(tp_reduce(tp, x, (long long)T * H, st));
    }
  }
  const bool final_normed = h_ready;  // h = final_norm(x) for every (decode) row already
  // ---- sampling rows: decode rows, plus the chunk's last row when it finishes a prompt
  int nl = 0;
  if (b->logits_decode && nd > 0) {
    if (!final_normed) RB_TRY(rmsnorm_launch(x, H, m->final_norm, h, H, nd, H, m->rms_eps, st));
    nl = nd;
  }
  if (b->emit_prefill && np > 0) {
    RB_TRY(rmsnorm_launch(x + (size_t)(T - 1) * H * e, H, m->final_norm, h + (size_t)nl * H * e, H, 1, H, m->rms_eps,
                          st));
    nl += 1;
  }
  if (nl > 0) {
    RB_TRY(gemm_bf16_launch(h, m->lm_head, w->logits, nullptr, nullptr, nl, m->vocab, H, H, H, m->vocab, 0, sms,
                            w->gemm_ws, w->gemm_ws_bytes, w->gemm_counters, w->gemm_counters_len, st));
    if (b->sample) {
      // row_valid = seq (padding rows have seq 0); the emitted prefill row uses the slot of row nd
      const int* valid = b->emit_prefill && np > 0 ? nullptr : w->seq;
      if (tp)  // vocab-parallel lm_head: max-reduce of (logit, -index) keys over the ranks
        RB_TRY(tp_argmax(tp, w->logits, m->vocab, nl, m->vocab, m->vocab_offset, w->out_ids, w->slot, m->last_tok,
                         valid, st));
      else
        RB_TRY(argmax_launch(w->logits, m->vocab, nl, m->vocab, w->out_ids, w->slot, m->last_tok, valid, st));
    }
  }
  return 0;
}
