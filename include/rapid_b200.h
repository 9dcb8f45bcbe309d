/*
 * rapid_b200.h — C ABI of the B200-native RAPID-Serve hot path
 * (librapid_b200.so, built from paper_2601_11822_b200/csrc/).
 *
 * The reference (arxiv/paper_2601_11822, a pure-Python simulator) has no
 * native code; its GPU work is a price returned by pure functions. Each entry
 * point below is the physical realization of one of those prices and cites the
 * reference interface it replaces (paths relative to /root/reference/).
 *
 * Conventions
 *  - Plain pointers are device pointers unless stated; sizes are element counts.
 *  - `stream` is a cudaStream_t (CUstream) — e.g. torch.cuda.current_stream()
 *    .cuda_stream or a green-context stream from rb_green_split().
 *  - Every call is asynchronous and stream-ordered; nothing synchronizes.
 *  - Return value: 0 on success, non-zero on error; rb_last_error() returns a
 *    thread-local message. Argument errors never launch anything.
 *  - bf16 tensors are row-major; `ld*` are row strides in elements.
 *  - Paged KV cache, one layer: [num_blocks][2 (K,V)][Hkv][16][head_dim] bf16.
 *  - Block table: int32 [num_slots][bt_stride]; a request occupies one slot.
 */
#ifndef RAPID_B200_H
#define RAPID_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Host path: stream-ordered copy (pinned host <-> device, cudaMemcpyDefault) and the launch of an
 * instantiated CUDA graph (the decode step's captured forward) on a stream — one C call each on the
 * per-step issue path instead of the framework's tensor copy / graph-replay dispatch. */
int rb_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
int rb_graph_launch(void* graph_exec, void* stream);

/* Library identity / diagnostics. */
const char* rb_version(void);
const char* rb_last_error(void);
int rb_device_sm_count(int device, int* out);
/* Debug: when buf != NULL, every GEMM CTA writes 8 globaltimer stamps to buf[8*cta..]. */
int rb_debug_gemm_trace(unsigned long long* buf);
/* Debug (profiling probe): push the regular context of green partition i of a
 * rb_green_split handle onto this thread / pop it again. */
int rb_debug_green_ctx_push(void* handle, int i);
int rb_debug_ctx_pop(void);
/* Debug: GEMM CTA-pair policy, -1 auto (default), 0 force single-CTA, 1 force 2-CTA pairs. */
int rb_debug_gemm_pair_mode(int mode);
/* Debug: decode (swap-AB) GEMM schedule, -1 auto (default); else bit0 = two 128-row weight
 * sub-tiles per activation stage, bit1 = stream-K (else data-parallel whole tiles). */
int rb_debug_gemm_variant(int v);
/* Debug: decode (swap-AB) GEMMs, weight k-blocks warmed into L2 ahead of the smem ring
 * (cp.async.bulk.prefetch.tensor); -1 = auto (default), 0 = off, 1..64 = forced. */
int rb_debug_gemm_prefetch(int kblocks);
/* Debug: stream-K for token-major (prefill) GEMMs whose whole-tile waves quantize badly
 * (fewer than 4 waves, last wave at most max_frac full); default off (measured slower). */
int rb_debug_gemm_prefill_streamk(int on, double max_frac);
/* Debug: token-major (prefill) GEMM tile width; 0 = wave-aware choice (default), else a forced
 * multiple of 32 in [32, 256]. Returns -1 for an invalid width. */
int rb_debug_gemm_prefill_bn(int bn);
/* Debug: query tiles per prefill-attention CTA; 0 = auto (default), 1, or 2 (mirrored causal
 * pairs). Returns -1 for an invalid count. */
int rb_debug_pattn_tiles(int tiles);
/* Debug: decode attention page loads, 1 = one 5D TMA op per page and kv-head (default), 0 = four
 * 2D {64, 16} boxes. */
int rb_debug_decode_kv_one_op(int on);
/* Debug: decode attention ring shape, 0 = auto (default), 1..4 = 12x2, 8x3, 6x4, 4x6
 * (warps per CTA x smem stages per warp). Returns -1 for an invalid shape. */
int rb_debug_decode_attn_shape(int shape);
/* Debug: decode (swap-AB) GEMMs as data-parallel K-slice units writing fp32 partials
 * [s][token][feature] into the workspace (no output written; timing experiments), 0 = off. */
int rb_debug_gemm_ksplit(int s);
/* Debug (diagnostic, csrc/probe.cu): stream `bytes` of global memory into shared memory with
 * 1D bulk copies over a ring of `stages` x `chunk` bytes, one CTA per SM, no compute — the
 * per-SM ingest ceiling of a partition. `sink` is a device int the kernel may write. */
int rb_debug_stream_read(const void* src, long long bytes, int chunk, int stages, int num_sms, int* sink,
                         void* stream);
/* Debug: the same with 2D tensor-TMA boxes {64 bf16, box_rows} (128B swizzle), per_stage boxes
 * per ring stage. */
int rb_debug_stream_read_tma(const void* src, long long bytes, int box_rows, int per_stage, int stages, int num_sms,
                             int* sink, void* stream);
/* Programmatic dependent launch for the forward's kernels (default on): each kernel may
 * start its prologue while its predecessor in the stream drains. 0 = plain serialization. */
int rb_set_pdl(int on);
/* Decode (swap-AB) gate|up GEMM: 1 = SwiGLU fused into its epilogue, 0 = separate kernel. */
int rb_set_decode_glu(int on);
/* Decode-only single-GPU iterations: O / down projections as K-slice units whose fp32 partials
 * the following RMSNorm adds to the residual stream (default 1); 0 = stream-K + residual epilogue. */
int rb_set_decode_ksplit(int on);

/* K1/K4 — bf16 linear layer on tcgen05 tensor cores:
 *   Y[t,o] = sum_k X[t,k] W[o,k] (+bias[o]) (+R[t,o])
 * Replaces the compute term of prefill_time (pkg/src/pdsim/costmodel.py:104)
 * and the weight-streaming term of decode_time (costmodel.py:130).
 * mode: 0 auto, 1 token-major tiles (prefill), 2 swap-AB (decode, T<=256);
 * | 4 = fused SwiGLU epilogue: W rows in [gate x16 | up x16] blocks,
 * Y[t, f] = silu(gate_f) * up_f with O/2 output columns (no bias / R).
 * num_sms: SMs of the partition the stream runs on (persistent grid size).
 * workspace/counters: split-K scratch (fp32) and zeroed int32 tile counters;
 * may be NULL (no split-K). R may alias Y (in-place residual add). */
int rb_gemm_bf16(const void* X, const void* W, void* Y, const void* bias, const void* R, int T, int O, int K,
                 long long ldx, long long ldw, long long ldy, int mode, int num_sms, void* workspace,
                 size_t ws_bytes, int* counters, int counters_len, void* stream);

/* K3 — decode paged attention, one query token per row:
 *   out[b,h,:] = softmax(scale * q[b,h,:] . K[slot_b, :seq_lens[b]]) V
 * Replaces the KV-read term kv_cache_bytes(model, total_kv_tokens) of
 * decode_time (costmodel.py:131). row_slot[b] selects the block-table row;
 * rows with seq_lens[b] <= 0 are skipped (graph padding). max_pages bounds
 * ceil(seq_lens[b]/16) over the launch (sequences are cut into 16-page work
 * items, whole sequences when B*Hkv fills the partition); when sequences are
 * split the workspace must hold B*Hq*splits*(head_dim+2)*4 bytes of partials
 * (splits <= ceil(max_pages/8)). The last 64 bytes of a non-NULL workspace hold
 * self-resetting work counters (items are handed to warps dynamically) and must be
 * zero before the first call. num_blocks = pages in the
 * cache layer (TMA extent); num_sms = SMs of the launching partition. */
int rb_decode_attention(const void* q, long long q_tok_stride, const void* cache_layer, const int* block_table,
                        int bt_stride, const int* row_slot, const int* seq_lens, void* out,
                        long long out_tok_stride, void* workspace, size_t ws_bytes, int B, int Hq, int Hkv,
                        int head_dim, int max_pages, float scale, int num_blocks, int num_sms, void* stream);

/* K2 — causal prefill attention of one chunk (positions start..start+T-1)
 * against the paged cache [0, start+T), on tcgen05 (S = QK^T and O = PV
 * accumulate in TMEM, Q and paged K/V fed by TMA). Replaces the attention share
 * of prefill_time's compute term (costmodel.py:104) for the chunk priced at
 * pkg/src/pdsim/engines/rapid.py:313. num_blocks = pages in the cache layer
 * (TMA extent). */
int rb_prefill_attention(const void* q, long long q_tok_stride, const void* cache_layer,
                            const int* block_table_row, int T, int start, int Hq, int Hkv, int head_dim, void* out,
                            long long out_tok_stride, float scale, int num_blocks, void* stream);

/* K5 — RoPE on q,k + paged KV write of k,v for T rows (pos[t] < 0 skips).
 * Replaces the KV-write term kv_cache_bytes(model, tokens) of prefill_time
 * (costmodel.py:105) and kv_cache_bytes(model, batch) of decode_time (:132).
 * cos_sin: fp32 [max_pos][head_dim] = [cos | sin]. */
int rb_rope_cache_write(const void* qkv, long long ld_qkv, const int* pos, const int* tok_slot,
                        const int* block_table, int bt_stride, const float* cos_sin, void* q_out, long long ld_q,
                        void* cache_layer, int T, int Hq, int Hkv, int head_dim, void* stream);

/* K1 + K5 fused — QKV projection whose epilogue applies RoPE and writes the paged KV:
 *   qkv = X W^T (+bias); q heads rotated -> q_out[t]; k heads rotated and v heads
 *   -> cache_layer[block_table[tok_slot[t]][pos[t]/16]][K|V][h][pos[t]%16]; pos[t] < 0 skips.
 * W: [(Hq+2Hkv)*128, K] with the q and k rows of every head pair-interleaved (row 2j holds
 * rotate-half dim j, row 2j+1 dim j+64; v rows unchanged), so attention scores are
 * unchanged and each RoPE pair is adjacent in the accumulator.
 * Replaces, in one launch, the compute term of prefill_time (costmodel.py:104) / weight
 * term of decode_time (:130) for the QKV projection and the KV-write terms (:105, :132).
 * mode / num_sms / workspace / counters as rb_gemm_bf16; head_dim must be 128. */
int rb_gemm_qkv_rope(const void* X, const void* W, const void* bias, int T, int K, long long ldx, int Hq, int Hkv,
                     int head_dim, const int* pos, const int* tok_slot, const int* block_table, int bt_stride,
                     const float* cos_sin, void* q_out, long long ld_q, void* cache_layer, int mode, int num_sms,
                     void* workspace, size_t ws_bytes, int* counters, int counters_len, void* stream);

/* K5 — small fused ops (part of fixed_iteration_overhead_us, costmodel.py:53). */
int rb_rmsnorm(const void* x, long long ldx, const void* w, void* y, long long ldy, int T, int H, float eps,
               void* stream);
int rb_silu_mul(const void* gate_up, long long ld_gu, void* y, long long ldy, int T, int I, void* stream);
int rb_embed(const int* ids, const int* slot_of_row, const int* last_tok, const void* table, void* y, int T, int H,
             int* ids_out, void* stream);
int rb_argmax(const void* logits, long long ld, int T, int V, int* out, const int* slot_of_row, int* last_tok,
              const int* row_valid, void* stream);

/* Device-side block-table maintenance (BlockPool physical IDs,
 * pkg/src/pdsim/kvcache.py:85-127): upd = [count, (slot, idx, block)*count]. */
int rb_block_table_update(const int* upd, int* block_table, int bt_stride, int max_updates, void* stream);
int rb_set_last_token(int* last_tok, int slot, const int* value_ptr, int value, void* stream);

/* Whole-iteration decoder forward (Llama-3.x / Qwen2 family), launched from
 * native code: replaces one priced iteration of the reference —
 * prefill_time (costmodel.py:89-106), decode_time (:109-134) or hybrid_time
 * (:137-163) — with every kernel of that iteration on `stream`.
 * Rows [0, n_decode) are single-token decode rows (paged decode attention);
 * rows [n_decode, rows) are one prefill chunk of slot `prefill_slot` at
 * positions prefill_start.. (causal over its paged prefix). Host arrays in
 * rb_model_t hold one device pointer per layer. Graph-capturable. */
typedef struct {
  int hidden, layers, q_heads, kv_heads, head_dim, intermediate, vocab;
  float rms_eps, attn_scale;
  const void* embed;
  const void* final_norm;
  const void* lm_head;
  const void* const* ln1;   /* [layers] */
  const void* const* wqkv;  /* [layers] fused q|k|v, [(Hq+2Hkv)*D, H] */
  const void* const* bqkv;  /* [layers] or NULL (Qwen2 bias) */
  const void* const* wo;
  const void* const* ln2;
  const void* const* wgu;   /* [layers] gate|up rows interleaved in 16-row blocks, [2I, H] */
  const void* const* wd;
  void* kv_cache;           /* layer 0 of [L][num_blocks][2][Hkv][16][D] */
  size_t kv_layer_stride_bytes;
  int num_blocks;
  int* block_table;
  int bt_stride;
  const float* cos_sin;
  int* last_tok;
  /* 0: q/k weight rows in the standard rotate-half order (separate RoPE + cache-write
   * kernel); 1: q/k rows pair-interleaved within each head (row 2j = dim j, 2j+1 = dim
   * j+64), RoPE and the paged K/V write fused into the QKV GEMM epilogue. */
  int qk_layout;
  /* tensor parallel: this rank's q/kv heads, intermediate and vocab above are its shard;
   * global token id of local lm_head row v is vocab_offset + v (0 on a single GPU). */
  int vocab_offset;
} rb_model_t;

typedef struct {
  void *x, *h, *qkv, *q, *attn, *gu, *act, *logits; /* bf16 activations, rows_cap rows */
  int rows_cap;
  int *ids, *pos, *slot, *seq, *out_ids;            /* int32 [rows_cap] */
  void* gemm_ws;
  size_t gemm_ws_bytes;
  int* gemm_counters;
  int gemm_counters_len;
  void* attn_ws;
  size_t attn_ws_bytes;
  void* tp;  /* this phase's TP context from rb_tp_create (NULL: single GPU) */
  /* in-situ roofline probe (bench.py): when both are non-NULL, cudaEvent_t handles (timing
   * enabled) recorded on the stream right before and after layer probe_layer's decode
   * attention launch; captured as event-record nodes when the call is graph-captured. */
  void* probe_ev0;
  void* probe_ev1;
  int probe_layer;
} rb_workspace_t;

typedef struct {
  int rows, n_decode, n_prefill;
  int max_pages;       /* bound on decode rows' ceil(seq/16) */
  int prefill_slot, prefill_start;
  int ids_from_slots;  /* decode rows read their input id from last_tok[slot] */
  int logits_decode;   /* lm_head over the decode rows */
  int emit_prefill;    /* lm_head over the chunk's last row (appended after the decode rows) */
  int sample;          /* greedy argmax -> out_ids, scattered into last_tok[slot] */
  int num_sms;         /* SMs of the partition `stream` runs on */
} rb_batch_t;

int rb_decoder_forward(const rb_model_t* model, const rb_workspace_t* ws, const rb_batch_t* batch, void* stream);

/* Tensor parallelism (cfg 4, 70B TP=8). The reference models no
 * collective (tp folds into GpuSpec.aggregate, pkg/src/pdsim/core.py:147-165); these
 * realize the one all-reduce after each row-parallel GEMM (O, down) and the
 * vocab-parallel greedy argmax. Each phase (prefill, decode) owns one context.
 * mode 1: NCCL (dlopen'ed libnccl.so.2; comm from rb_tp_nccl_comm_init).
 * mode 2: one-shot all-reduce over peer memory with the residual add fused: part0/part1
 *   [world] = every rank's two staging buffers (part_elems bf16 each), flags[world] =
 *   every rank's zeroed uint32 flag array (rb_tp_flag_words() words), epoch = this rank's
 *   zeroed uint32 [128]; keys[world] = uint64 argmax key buffers (rows_cap each).
 * Pointers are device pointers valid in this process (cudaIpc-opened on a multi-GPU
 * node; plain pointers when ranks share one device). */
int rb_tp_nccl_available(void);
int rb_tp_nccl_unique_id(void* id_out /* 128 bytes */);
int rb_tp_nccl_comm_init(const void* id /* 128 bytes */, int nranks, int rank, void** comm_out);
int rb_tp_nccl_comm_destroy(void* comm);
int rb_tp_create(int world, int rank, int mode, void* nccl_comm, void* const* part0, void* const* part1,
                 void* const* keys, void* const* flags, void* epoch, size_t part_elems, void** tp_out);
int rb_tp_destroy(void* tp);
size_t rb_tp_flag_words(void);
/* debug: skip the peer flag wait (results are then undefined) */
int rb_tp_debug_nowait(void* tp, int on);
/* standalone sum all-reduce of a bf16 vector (tests / benchmarks) */
int rb_tp_allreduce(void* tp, void* x, long long n, void* stream);

/* K7 — SM partitioning with CUDA green contexts (replaces the CU-fraction
 * scalars of AllocationDecision, pkg/src/pdsim/core.py:215-245, and the
 * cu_fraction argument of effective_bandwidth/_roofline_us,
 * costmodel.py:62-86). Splits the device into a group of >= first_sms SMs and
 * the remainder; returns one non-blocking stream bound to each partition and
 * the actual SM counts. handle is released by rb_green_destroy. */
int rb_green_split(int device, int first_sms, void** handle, void** stream_first, void** stream_second,
                   int* sms_first, int* sms_second);
int rb_green_destroy(void* handle);

#ifdef __cplusplus
}
#endif
#endif /* RAPID_B200_H */
