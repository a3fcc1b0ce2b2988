/*
 * spmoe.h — C ABI of the B200-native SP-MoE verification-time expert path.
 *
 * The reference (arxiv 2510.10302, package `moesim`) is pure Python with no
 * FFI; every entry point below realises one reference function on sm_100a
 * and is called from the Python drop-in layer (paper_2510_10302_b200) via
 * ctypes.  Each declaration cites the reference symbol it replaces.
 *
 * ABI conventions
 *   - plain pointers and sizes only; all device memory is caller-owned, no
 *     allocation happens inside a compute entry point;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - every function returns an int status: 0 (cudaSuccess) or a
 *     cudaError_t value (cudaErrorInvalidValue = 1 for bad arguments);
 *   - no C++ exception crosses the ABI; everything is stream-ordered and
 *     re-entrant per stream;
 *   - bf16 tensors are passed as uint16_t* (raw bfloat16 bits).
 *
 * Determinism contract (what makes CPU-oracle parity bit-exact):
 *   - every dot product multiplies bf16 x bf16 (exact in fp32) and adds in a
 *     documented fixed order: lane j of a warp sums the 8-element chunks
 *     c = j, j+32, j+64, ... in ascending order, elements 0..7 in order,
 *     then a xor-butterfly over offsets 16,8,4,2,1;
 *   - exp is spmoe's own range-reduced polynomial built from IEEE mul/add
 *     (no FMA contraction, no SFU approximation), so softmax weights and
 *     SiLU are reproducible on the CPU;
 *   - top-k orders by (logit desc, expert index asc), the tie-break of
 *     moesim.trace.top_k_indices (trace.py:28-37).
 */
#ifndef SPMOE_H
#define SPMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --------------------------------------------------------------------- */
/* library                                                                */
/* --------------------------------------------------------------------- */

/* ABI version (major*100 + minor). */
int spmoe_abi_version(void);

/* Last CUDA error string for a status code (static storage). */
const char* spmoe_status_string(int status);

/* --------------------------------------------------------------------- */
/* K1  router_topk                                                        */
/*   replaces predictor.predict_scores + select_critical                  */
/*   (predictor.py:79-106), trace.top_k_indices (trace.py:28-37), and     */
/*   Algorithm 1 lines 2-3 Gates[l](s) / TopK_Index.   */
/* --------------------------------------------------------------------- */
/*
 * x        [T, H]  bf16   layer MLP input (post-attention RMSNorm)
 * w_gate   [E, H]  bf16   router weight of the target layer
 * renorm   1: weights = softmax over the k selected logits (Mixtral);
 *          0: weights = softmax over all E logits, picked at the top-k
 *             (DeepSeek-V2 / Qwen1.5-MoE, norm_topk_prob = False)
 * weights  [T, k]  f32    out
 * idx      [T, k]  i32    out, descending logit, ties -> lowest index
 * logits   [T, E]  f32    out, nullable
 * host_idx [T, k]  i32    nullable; mapped pinned host memory also receiving
 *                          idx (the predictor's zero-copy hand-off to the
 *                          prefetch worker)
 * shared_gate_w [H] bf16  nullable; when set, shared_gate[T] f32 receives
 *                          sigmoid(x . shared_gate_w) (Qwen1.5-MoE)
 * Constraints: H % 8 == 0, 1 <= k <= E <= 256, T >= 0.
 */
int spmoe_router_topk(const uint16_t* x, const uint16_t* w_gate, int T, int H, int E,
                      int k, int renorm, float* weights, int32_t* idx, float* logits,
                      int32_t* host_idx, const uint16_t* shared_gate_w, float* shared_gate,
                      void* stream);

/* --------------------------------------------------------------------- */
/* K2  moe_permute                                                        */
/*   replaces the union-of-required loop of Simulation._verify_stage      */
/*   (simcore.py:365-372) with a device-side grouping of verify tokens.   */
/* --------------------------------------------------------------------- */
/*
 * idx             [T, k] i32  routed experts per token
 * expert_offsets  [E+1]  i32  out: exclusive prefix of per-expert counts
 * perm_token      [T*k]  i32  out: token of each permuted row (grouped by
 *                              expert ascending, then token ascending)
 * inv_pos         [T*k]  i32  out: permuted row of (token t, choice i)
 */
int spmoe_moe_permute(const int32_t* idx, int T, int k, int E, int32_t* expert_offsets,
                      int32_t* perm_token, int32_t* inv_pos, void* stream);

/* --------------------------------------------------------------------- */
/* K3  expert_ffn (grouped SwiGLU over the HBM slot pool)                 */
/*   realises Eq. 1's E_i(x) for every routed expert,  */
/*   charged as t_comp_target in Simulation._verify_stage (simcore.py:397)*/
/* --------------------------------------------------------------------- */
/*
 * Expert blob layout (one slot, bf16, contiguous, 3*F*H elements):
 *     W1 [F, H] (gate) | W3 [F, H] (up) | W2 [H, F] (down)
 * pool            base of the slot pool [S, 3*F*H] bf16
 * slot_of_expert  HOST array [E] of slot indices (copied into the kernel
 *                 parameters; only experts in `expert_mask` are read)
 * expert_mask     bit e set => process expert e in this launch (E <= 64);
 *                 lets the caller run cache-resident experts first and the
 *                 demand-loaded ones as their copies land
 * x               [T, H] bf16 layer MLP input (unpermuted)
 * expert_offsets, perm_token   from spmoe_moe_permute
 * h_scratch       [T*k, F] bf16 scratch (SwiGLU activations, permuted rows)
 * y               [T*k, H] f32  out: per-(token, choice) expert outputs
 * max_tokens_per_expert  hint selecting the register tile (any value is
 *                 correct; <=0 means unknown)
 * Dense mode: E = 1, k = 1, expert_offsets = {0, T}, perm_token = identity
 * runs a dense SwiGLU MLP (draft FFN, shared experts).
 */
int spmoe_expert_ffn(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                     uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E,
                     int k, const int32_t* expert_offsets, const int32_t* perm_token,
                     uint16_t* h_scratch, float* y, int max_tokens_per_expert, void* stream);

/* Phase entry points (exposed for profiling and the tcgen05 comparison). */
int spmoe_expert_ffn_up(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                        uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E,
                        int k, const int32_t* expert_offsets, const int32_t* perm_token,
                        uint16_t* h_scratch, int max_tokens_per_expert, void* stream);
int spmoe_expert_ffn_down(const uint16_t* pool, int64_t slot_elems,
                          const int32_t* slot_of_expert, uint64_t expert_mask, int T, int H,
                          int F, int E, int k, const int32_t* expert_offsets,
                          const uint16_t* h_scratch, float* y, int max_tokens_per_expert,
                          void* stream);

/*
 * tcgen05/TMEM/TMA variant of spmoe_expert_ffn (same inputs, same h / y
 * outputs): weight rows as the UMMA M=128 operand, routed tokens as N
 * (<= 64 per tile), TMA over a 3-D tensor map of the slot pool, fp32
 * accumulators in TMEM.  Needs H % 128 == 0 and F % 128 == 0.  Workspaces:
 * x_perm [T*k, H] bf16 (routed rows gathered by perm_token) and workspace
 * f32 of max(2*split_up*T*k*F, split_dn*T*k*H) elements holding split-K
 * partials (up: gate then up sums, reduced with SiLU; down: y partials),
 * always reduced in split order, so results are deterministic; unused
 * when both splits are 1.  split_up <= H/64, split_dn <= F/64: the host
 * picks them so that (tiles x split) fills the SMs (kernels.tc_plan).
 * Results equal the CUDA-core path within fp32 rounding of the tensor
 * core's accumulation order.
 */
int spmoe_expert_ffn_tc(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                        uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E, int k,
                        const int32_t* expert_offsets, const int32_t* perm_token, uint16_t* x_perm,
                        uint16_t* h_scratch, float* y, float* workspace, int split_up, int split_dn,
                        void* stream);

/*
 * Single-launch variant: up phase, grid-wide barrier, down phase in one
 * persistent cooperative kernel (one CTA per SM); the TMA producer streams
 * the first W2 stages before the barrier.  grid_sync: caller-owned device
 * uint32 (reset by the call).  Up phase unsplit; workspace holds the
 * split_dn down partials (split_dn * T*k * H floats) when split_dn > 1.
 */
int spmoe_expert_ffn_tc_fused(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                              uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E, int k,
                              const int32_t* expert_offsets, const int32_t* perm_token, uint16_t* x_perm,
                              uint16_t* h_scratch, float* y, float* workspace, int split_dn,
                              uint32_t* grid_sync, void* stream);

/*
 * Unit-fused variant for verify-sized calls (<= 16 routed tokens per
 * expert): each work unit (expert, 128-feature block m) runs
 * W1/W3 rows of block m -> h block in shared memory -> the matching W2
 * column block -> partial y_m; a PDL-chained second launch sums the F/128
 * partials per element in a fixed order into y.  The kernel loads each
 * unit's token rows straight from x (TMA gather4 over perm_token), so no
 * row-gather launch precedes it; x_perm is unused (nullable, kept for the
 * ABI).  workspace:
 * spmoe_expert_ffn_tc_units_workspace_floats(T*k, H, F) floats.
 * h_scratch (nullable) receives h.  Same
 * tolerance contract as spmoe_expert_ffn_tc; an expert's result never
 * depends on which experts share the launch.  Returns
 * cudaErrorInvalidValue when max_tokens_per_expert > 16.
 */
int spmoe_expert_ffn_tc_units(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                              uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E, int k,
                              const int32_t* expert_offsets, const int32_t* perm_token,
                              int max_tokens_per_expert, uint16_t* x_perm, uint16_t* h_scratch, float* y,
                              float* workspace, void* stream);
int64_t spmoe_expert_ffn_tc_units_workspace_floats(int rows, int H, int F);

/* Profiling hook: CUDA events (cudaEvent_t, timing-enabled) recorded on the
 * stream right before the first kernel and after the last kernel of the
 * NEXT spmoe_expert_ffn / _tc / _tc_fused call made by this host thread, so
 * the measured span excludes host-side launch preparation.  NULLs clear. */
int spmoe_k3_timing(void* start, void* end);
/* Device-clock variant for the NEXT spmoe_expert_ffn_tc / _tc_units call on
 * this host thread: span points at a zeroed device {uint64 t0, t1}; t0 =
 * globaltimer (ns) when the call's first kernel starts its first CTA, t1 =
 * when its last kernel ends its last CTA.  Unlike events it is not skewed
 * by a saturated host link (tools/probes/tma_stream.cu h2d).  NULL clears. */
int spmoe_k3_devtiming(void* span);

/* --------------------------------------------------------------------- */
/* K4  moe_combine                                                        */
/*   Eq. 1 weighted sum Output = sum_i G(x)_i E_i(x)  */
/* --------------------------------------------------------------------- */
/*
 * out[t] = bf16( residual[t] + sum_{i<k} weights[t,i] * y[inv_pos[t,i]]
 *                + shared_gate[t] * y_shared[t] )
 * fp32, fixed order: i ascending with separate mul and add, then the
 * shared term, then the residual.  residual, weights (NULL => 1.0),
 * y_shared and shared_gate (NULL => 1.0) are nullable.  out may alias
 * residual.
 */
int spmoe_moe_combine(const float* y, const int32_t* inv_pos, const float* weights, int T,
                      int H, int k, const float* y_shared, const float* shared_gate,
                      const uint16_t* residual, uint16_t* out, void* stream);

/* --------------------------------------------------------------------- */
/* gather_rows  (expert-parallel exchange, SURVEY §8 e)                   */
/*   dst[j] = src[idx[j] / div] for j < n, rows of row_bytes (multiple of */
/*   4).  Packs routed rows in K2's expert order before the dispatch     */
/*   all-to-all (div = 1, idx = perm_token, the token of each permuted   */
/*   row) and restores receive order before the combine all-to-all      */
/*   (div = 1, idx = inv_pos).  No                                       */
/*   reference counterpart: the reference has no expert parallelism.     */
/* --------------------------------------------------------------------- */
int spmoe_gather_rows(const void* src, const int32_t* idx, int n, int div, int64_t row_bytes,
                      void* dst, void* stream);

/* --------------------------------------------------------------------- */
/* K6  greedy_accept                                                      */
/*   replaces the Bernoulli acceptance of Simulation.run                  */
/*   (simcore.py:440-446) with the SD greedy rule:      */
/*   longest prefix where draft[i] == argmax(target_logits[i]), plus one  */
/*   correction / bonus token.                                           */
/* --------------------------------------------------------------------- */
/*
 * logits  [B, N+1, V] f32 (row stride ld >= V)
 * draft   [B, N]      i32
 * argmax_out [B, N+1] i32 out (ties -> lowest index)
 * result  [B, 2]      i32 out: {accepted, next_token}
 */
int spmoe_greedy_accept(const float* logits, int64_t ld, const int32_t* draft, int B, int N,
                        int V, int32_t* argmax_out, int32_t* result, void* stream);

/* Row argmax over bf16/f32 rows (draft-token selection). */
int spmoe_argmax_rows(const float* logits, int64_t ld, int rows, int V, int32_t* out,
                      void* stream);

/* --------------------------------------------------------------------- */
/* Layer block around the MoE (the draft forward    */
/* and the target verify pass outside the MoE; simcore.py:323-359).       */
/* Latency-bound helpers that replace ~30 framework kernels per layer.    */
/* --------------------------------------------------------------------- */
/* out[r] = bf16((x[r] * s) * w), s = 1 / sqrt(dot_fixed(x[r], x[r]) / H + eps)
 * (IEEE division and square root), rows of H (H % 8 == 0). */
int spmoe_rms_norm(const uint16_t* x, const uint16_t* w, int rows, int H, float eps, uint16_t* out,
                   void* stream);
/*
 * qkv     [B*T, (nh + 2*nkv)*hd] bf16  fused projection output
 * cos/sin [max_pos, hd] f32 rotate-half RoPE tables (host-computed, shared
 *         bit for bit with the oracle)
 * start   [B] i64 device: position of each sequence's first new token
 * q_out   [B, nh, T, hd] bf16 out (rotated queries)
 * k_cache, v_cache [B, nkv, S, hd] bf16: rotated keys / values appended
 *         at positions start[b] .. start[b] + T - 1
 * y = bf16(x*cos + rot*sin), each product and the sum IEEE-rounded.
 * Rows whose position is >= S or >= max_pos write nothing (callers check
 * lengths first; the guard keeps a bad position from corrupting memory).
 */
int spmoe_rope_kv(const uint16_t* qkv, const float* cos_t, const float* sin_t, const int64_t* start,
                  int B, int T, int nh, int nkv, int hd, int S, int max_pos, uint16_t* q_out,
                  uint16_t* k_cache, uint16_t* v_cache, void* stream);
/* Causal GQA attention of the T new queries over keys 0 .. start[b] + t;
 * out [B, T, nh*hd] bf16; hd in {64, 128}; S * 32 + 33 KB of shared memory
 * must fit 200 KB.  Fixed order: scores by lane-blocked dims + butterfly,
 * det_exp(s - max), 8 key streams (key mod 8) summed ascending and merged in
 * stream order, IEEE division (restated in oracle/forward_oracle.c). */
int spmoe_attention(const uint16_t* q, const uint16_t* k_cache, const uint16_t* v_cache,
                    const int64_t* start, int B, int T, int nh, int nkv, int hd, int S, float scale,
                    uint16_t* out, void* stream);

/* --------------------------------------------------------------------- */
/* K9  linear: the projections around the MoE (fused qkv, W_o, lm_head)   */
/*   of the draft and target forwards (SURVEY §8(f) rows 1-2,            */
/*   simcore.py:323-359 compute slots; PAPER.md:352 draft model).         */
/* --------------------------------------------------------------------- */
/*
 * y[t][n] = dot_fixed(w[n, 0:K], xin[t, 0:K]) with the determinism
 * contract's order (K % 8 == 0).  xin = x, or RMSNorm(x; norm_w, eps) when
 * norm_w != NULL (spmoe_rms_norm's arithmetic, fused into the staging).
 *   y_f32  != NULL: y_f32[t*ldy + n] = y (fp32, e.g. lm_head logits)
 *   y_bf16 != NULL: y_bf16[t*N + n] = bf16(y), or with resid != NULL
 *                   bf16(resid[t*N + n] + bf16(y)) (resid may alias y_bf16)
 * Weight-streaming (one warp per weight row pair, pipelined rounds),
 * activations staged in shared memory as fp32, up to 8 token rows per
 * register tile (16 beyond).  Launched with programmatic dependent launch:
 * x and resid are read only after the previous kernel on `stream` has
 * completed, but the first rounds of w are requested into L2 before that --
 * w must not be written by the immediately preceding kernel on `stream`
 * (weights are static in the engine; SPMOE_NO_PDL=1 launches without it).
 */
int spmoe_linear(const uint16_t* w, const uint16_t* x, int64_t ldx, int T, int K, int N,
                 const uint16_t* norm_w, float eps, float* y_f32, int64_t ldy, uint16_t* y_bf16,
                 const uint16_t* resid, void* stream);

/* --------------------------------------------------------------------- */
/* K5  h2d_batch                                                          */
/*   IoChannel.transfer / worker_step batched copy (prefetch.py:60-74,    */
/*   191-214); Algorithm 2 line 12 copy_non_blocking.     */
/* --------------------------------------------------------------------- */
int spmoe_h2d_batch(void* const* dst, const void* const* src, const size_t* bytes, int n,
                    void* stream);

/* --------------------------------------------------------------------- */
/* Deterministic init: counter-hash N(0, std^2) bf16, identical on CPU.   */
/* --------------------------------------------------------------------- */
int spmoe_fill_normal_bf16(uint16_t* dst, int64_t n, uint64_t seed, uint64_t offset,
                           float std, void* stream);

/* --------------------------------------------------------------------- */
/* XC: lossless exponent coding of expert blobs on the host link          */
/*   The offload tier moves every routed expert over PCIe               */
/*   (IoChannel.transfer prefetch.py:45-74; t_io = size/bw + overhead,   */
/*   config.py:229-231), so the bytes per expert set TPOT.  A bf16       */
/*   weight is sign(1) | exponent(8) | mantissa(7); the exponent of      */
/*   trained or N(0, s^2) weights has ~2.5 bits of entropy.  XC stores   */
/*   each value as one sign|mantissa byte                                */
/*   and the exponent as a 4-bit symbol (its offset from the segment's   */
/*   base exponent, 15 = escape) in a per-segment canonical Huffman code */
/*   (<= 12 bits, 32 independent lane substreams per 4096-value block so */
/*   a warp decodes a block in parallel); escaped exponents travel in a  */
/*   per-block exception list.  Decoding is exact: decode(encode(x)) ==  */
/*   x bit for bit.  Per-value coding only: no cross-value or            */
/*   cross-expert modelling.                                             */
/* --------------------------------------------------------------------- */
#define SPMOE_XC_MAGIC 0x35435853u /* "SXC5" */
#define SPMOE_XC_BLOCK 4096        /* values per coding block */
#define SPMOE_XC_LANES 32          /* exponent substreams per block */
#define SPMOE_XC_LMAX 12           /* longest symbol code, bits */
#define SPMOE_XC_NSYM 16           /* 15 in-window offsets + escape */
#define SPMOE_XC_MAX_SEG 4

/*
 * One segment = one weight matrix of n bf16 values (n % SPMOE_XC_BLOCK == 0),
 * nb = n / SPMOE_XC_BLOCK blocks.  base = the lowest exponent b <= 240 whose
 * window [b, b + 14] holds the most values (ties: lowest b); exponent e
 * codes as symbol e - base inside the window, else as the escape symbol 15.
 * Symbols are coded with the segment's canonical Huffman code, lengths
 * len[16] (1..SPMOE_XC_LMAX, 0 = symbol absent) built deterministically from
 * the symbol histogram (two-queue Huffman, ties to leaves and lower ids;
 * lengths over LMAX capped and the Kraft excess repaid by lengthening the
 * longest codes under LMAX, rarest then highest id first; codes assigned in
 * (length, symbol) order).
 * Streams (byte offsets from the blob start, each 256-byte aligned, in this
 * order, so a segment's bytes are contiguous from its off_lut):
 *   lut   [4096]    u32  multi-symbol decode table: entry p (the next 12
 *                        code bits, LSB first) = up to five whole codes,
 *                        sym_i << 4 i (i < 5) | 4 count << 20 |
 *                        bits << 25 (count >= 1: an unused pattern of an
 *                        incomplete code advances one bit as symbol 0);
 *                        derived from len[] at encode time, so a decoder
 *                        loads it
 *   sm    [n]       u8   (v >> 8 & 0x80) | (v & 0x7f)
 *   ex    [ex_words] u32 per block, SPMOE_XC_LANES lane substreams back to
 *                        back; lane l holds the bit-reversed codes of values
 *                        128 l .. 128 l + 127 of the block, LSB first; in
 *                        bit mode the substreams are bit-contiguous and only
 *                        the block's run is padded to a whole word, in word
 *                        mode each substream is padded to a whole word (8
 *                        readable slack bytes after the stream)
 *   bofs  [nb+1]    u32  first ex word of each block (exclusive prefix)
 *   lanes [nb*32]   u8   per lane: bit mode, its code bits - the block's
 *                        lbase; word mode, its word count
 *   lbase [nb]      u16  bit 15 = word mode (a block whose lane lengths
 *                        spread over more than 255 bits); bits 0-14 = the
 *                        shortest lane's code bits (bit mode)
 *   xofs  [nb+1]    u32  first exception of each block (exclusive prefix)
 *   xrec  [n_exc]   u32  escaped values in value order: index in block << 8
 *                        | exponent
 * Every bf16 bit pattern round-trips (zeros, denormals, inf, NaN).
 */
typedef struct spmoe_xc_segment {
  uint64_t n;
  uint64_t off_lut, off_sm, off_ex, off_bofs, off_lanes, off_lbase, off_xofs, off_xrec;
  uint32_t ex_words, n_exc;
  uint32_t base, pad;
  uint8_t len[SPMOE_XC_NSYM];
} spmoe_xc_segment; /* 104 bytes */

typedef struct spmoe_xc_header {
  uint32_t magic; /* SPMOE_XC_MAGIC */
  uint32_t nseg;  /* 1..SPMOE_XC_MAX_SEG; segments decode back to back */
  uint64_t blob_bytes; /* header + streams (what crosses the host link) */
  uint64_t raw_bytes;  /* 2 * sum(n) */
  spmoe_xc_segment seg[SPMOE_XC_MAX_SEG];
} spmoe_xc_header; /* 440 bytes; the first stream starts at 512 */

/* Device workspace bytes spmoe_xc_plan needs for these segments. */
size_t spmoe_xc_work_bytes(int nseg, const int64_t* seg_n);
/*
 * Encoder step 1 (synchronous on `stream`): histogram each segment's
 * exponents, choose its base and code, count each block's code words and
 * exceptions, and fill *hdr (host) with the blob layout.  src: the nseg
 * segments back to back on the device.  work: device, spmoe_xc_work_bytes.
 * Returns 1 (invalid value) if a segment size is not a multiple of
 * SPMOE_XC_BLOCK.
 */
int spmoe_xc_plan(const uint16_t* src, int nseg, const int64_t* seg_n, void* work,
                  spmoe_xc_header* hdr, void* stream);
/* Encoder step 2: write the blob (hdr->blob_bytes bytes, device) for the
 * plan in hdr / work (synchronous). */
int spmoe_xc_encode(const uint16_t* src, const spmoe_xc_header* hdr, const void* work,
                    uint8_t* blob, void* stream);
/* Decode a device-resident blob whose header (host copy) is hdr into dst
 * (hdr->raw_bytes bytes, device).  Stream-ordered; no host sync. */
int spmoe_xc_decode(const uint8_t* blob, const spmoe_xc_header* hdr, uint16_t* dst,
                    void* stream);
/* Decode only segments [first, first + count) of the blob; dst is the base
 * of the WHOLE decoded blob (each segment lands at its own offset).  Lets a
 * copy path decode a segment as soon as its bytes have landed. */
int spmoe_xc_decode_segments(const uint8_t* blob, const spmoe_xc_header* hdr, int first, int count,
                             uint16_t* dst, void* stream);
/* Same, with device-clock timing: span (nullable) points at a zeroed device
 * {uint64 t0, t1}; the launch sets t0 = globaltimer (ns) when its first CTA
 * starts and t1 = when its last CTA ends. */
int spmoe_xc_decode_segments_timed(const uint8_t* blob, const spmoe_xc_header* hdr, int first, int count,
                                   uint16_t* dst, void* stream, void* span);

/* --------------------------------------------------------------------- */
/* Native runtime: LRU slot cache + prefetch worker (prefetch.py,        */
/* cache.py, Algorithm 2)                                */
/* --------------------------------------------------------------------- */
typedef struct spmoe_rt spmoe_rt;

/*
 * Create the expert-cache runtime.
 *   capacity        HBM slots (cache_capacity_slots, config.py:234-242)
 *   num_layers, num_experts   expert id space (layer, expert)
 *   dev_pool        device slot pool base; slot s lives at
 *                   dev_pool + s * slot_bytes
 *   host_pool       pinned host pool; expert (l, e) lives at
 *                   host_pool + host_index[l*E+e] * slot_bytes
 *   host_index      [L*E] host-pool index of each expert (lets a bounded
 *                   host pool alias experts; identity when NULL)
 *   copy_stream     dedicated copy stream (cudaStream_t)
 *   batched_io      PolicySpec.batched_io (config.py:190-221)
 */
spmoe_rt* spmoe_rt_create(int capacity, int num_layers, int num_experts, void* dev_pool,
                          const void* host_pool, const int32_t* host_index, size_t slot_bytes,
                          void* copy_stream, int batched_io);
void spmoe_rt_destroy(spmoe_rt* rt);

/* ExpertCache.lookup (cache.py:62-77).  Returns 1 hit / 0 miss. */
int spmoe_rt_lookup(spmoe_rt* rt, int layer, int expert, int touch);
/* Slot of a resident expert, -1 if absent. */
int spmoe_rt_slot_of(spmoe_rt* rt, int layer, int expert);
/* ExpertCache.insert_batch metadata only (cache.py:79-122), no copy.
 * kind: 0 prefetch, 1 demand.  victims_out [2*n] receives (layer, expert)
 * pairs; returns the number of victims, or -1 on CacheError. */
int spmoe_rt_insert_batch(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n,
                          int kind, int32_t* victims_out);
/* ExpertCache.pin / unpin (cache.py:124-133).  pin returns -1 if any id
 * is not resident. */
int spmoe_rt_pin(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n);
void spmoe_rt_unpin(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n);
/* LRU order, head (least recent) first; returns count written (<= cap). */
int spmoe_rt_lru_order(spmoe_rt* rt, int32_t* layers, int32_t* experts, int cap);
/* counters: hits, misses, evictions, prefetch_evictions,
 * prefetch_insertions, demand_insertions, tasks_completed, tasks_aborted,
 * prefetch_bytes, demand_bytes, n_resident, evictions_of_queued_targets,
 * handoff_timeouts (tasks dropped after the bounded 5 s index hand-off wait,
 * prefetch.py:353-355) */
void spmoe_rt_counters(spmoe_rt* rt, int64_t* out13);
void spmoe_rt_reset_stats(spmoe_rt* rt);

/*
 * Demand load (prefetch.on_demand_load, prefetch.py:276-301): insert the
 * non-resident ids as one DEMAND batch, copy them on the copy stream behind
 * whatever is queued there, and record each slot's ready event.  Slots are
 * written to slots_out[n] (resident ids keep their slot).  Returns 0 or a
 * status (-1: CacheError).
 */
int spmoe_rt_demand_load(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n,
                         int32_t* slots_out);

/* Make `stream` wait until slot's pending copy (if any) has landed. */
int spmoe_rt_wait_slot(spmoe_rt* rt, int slot, void* stream);
/* Record that kernels on `stream` read `slot` (the copy stream waits on it
 * before the slot is overwritten: slot-reuse hazard, SURVEY hard part 5). */
int spmoe_rt_mark_read(spmoe_rt* rt, int slot, void* stream);
/* 1 if slot's last copy has completed (cudaEventQuery), else 0. */
int spmoe_rt_slot_ready(spmoe_rt* rt, int slot);

/*
 * Prefetch worker (Algorithm 1 enqueue + Algorithm 2 worker thread).
 * push: one task = the top-k predicted experts of `layer`, whose indices
 * the predictor kernel writes to mapped pinned memory `host_idx` [k];
 * `ready_event` (cudaEvent_t) is recorded after that kernel.  The worker
 * waits on the event, drops resident ids (non-touch probe,
 * enqueue_critical prefetch.py:118-145 + pop-time re-check
 * prefetch.py:186-189), picks LRU victims, issues the batched copy on the
 * copy stream and installs the batch (move-to-end).  Tasks run FIFO.
 */
int spmoe_rt_worker_start(spmoe_rt* rt);
int spmoe_rt_push_task(spmoe_rt* rt, int layer, const int32_t* host_idx, int k,
                       void* ready_event, int issue_token);
/* Same, with a graph-safe hand-off: the worker waits until the int32
 * counter *flag (mapped pinned memory, bumped on the device by
 * spmoe_signal_bump after the predictor kernel) reaches `expected`, then
 * reads host_idx.  Used for predictor kernels replayed inside CUDA graphs. */
int spmoe_rt_push_task_flag(spmoe_rt* rt, int layer, const int32_t* host_idx, int k,
                            const int32_t* flag, int32_t expected, int issue_token);
/* Device-side increment of a host-visible counter in mapped memory
 * (stream-ordered; system-scope fenced). */
int spmoe_signal_bump(int32_t* flag, void* stream);
/* Block until every pushed task has been popped and its copies issued.
 * Returns (and clears) the first error since the last drain: a failed H2D
 * copy / event record (the experts whose copies were not issued are
 * uninstalled, never left resident over stale bytes), a failed ready-event
 * wait, or cudaErrorTimeout when a task's indices were not published within
 * 5 s (the task is dropped and counted in handoff_timeouts). */
int spmoe_rt_drain(spmoe_rt* rt);
/* Fault injection for tests: the next n expert copies fail with
 * cudaErrorInvalidValue before anything is enqueued. */
int spmoe_rt_debug_fail_copies(spmoe_rt* rt, int n);
/* Drop queued-but-unpopped tasks (end of inference); returns count. */
int spmoe_rt_abort_pending(spmoe_rt* rt);
int spmoe_rt_worker_stop(spmoe_rt* rt);

/* Copy log: one record per issued copy batch. rec = {layer, n_experts,
 * kind(0 prefetch / 1 demand), issue_seq}; t = {start_ms, end_ms} from CUDA
 * events relative to the runtime epoch (valid after the copies complete).
 * Returns number of records written. */
int spmoe_rt_transfer_log(spmoe_rt* rt, int32_t* rec4, double* t2, int cap);
/* Experts of record i (expert ids, up to cap). */
int spmoe_rt_transfer_experts(spmoe_rt* rt, int i, int32_t* experts, int cap);
/* Milliseconds from the runtime epoch (a timing event recorded on the copy
 * stream at creation) to `event` (a timing cudaEvent_t on any stream), so
 * compute slots and transfers share one clock.  -1 if not measurable. */
double spmoe_rt_since_epoch_ms(spmoe_rt* rt, void* event);
/* Bytes of transfer record i that crossed the host link (XC blob bytes
 * with a codec, raw expert bytes without); -1 if out of range. */
int64_t spmoe_rt_transfer_wire_bytes(spmoe_rt* rt, int i);
/* ms from the runtime epoch to the end of record i's last H2D copy (the
 * link is free from then on; with the XC tier the record's end_ms follows
 * after the last decode); -1 if not complete. */
double spmoe_rt_transfer_copy_end_ms(spmoe_rt* rt, int i);

/*
 * XC host tier (see "XC" above): from now on expert (l, e)'s host row at
 * host_pool + host_index[l*E+e] * row_stride holds an XC blob of the
 * slot's raw bytes.  Each copy goes to one of n_staging device buffers of
 * staging_bytes (round robin, reused once the decode that read it is done)
 * on the copy stream; decode_stream waits for it (and for the slot's
 * readers), decodes into the slot and records the slot's ready event, so
 * wait_slot / slot_ready keep their meaning.  Call once, before any copy.
 * Returns cudaErrorInvalidValue if a row is not a valid blob of slot_bytes
 * raw bytes or does not fit a staging buffer.
 */
int spmoe_rt_set_codec(spmoe_rt* rt, size_t row_stride, void* staging, size_t staging_bytes,
                       int n_staging, void* decode_stream);
/* Profiling hook for every XC segment decode issued from now on:
 * enable = 1 brackets each launch with timing events on the decode stream,
 * enable = 2 records its device-clock span (globaltimer, first CTA start ->
 * last CTA end), 0 stops. */
int spmoe_rt_decode_timing(spmoe_rt* rt, int enable);
/* Sum of the timed decode durations (ms), the bytes they read (blob) plus
 * wrote (raw), and their count since the last call; clears the record
 * (synchronizes on the decode stream). */
int spmoe_rt_decode_stats(spmoe_rt* rt, double* ms, int64_t* bytes, int64_t* launches);
/* Host-link bytes since the last reset: {prefetch, demand}. */
void spmoe_rt_wire_bytes(spmoe_rt* rt, int64_t* out2);

/* Drop the transfer log (waits for logged copies to finish). */
void spmoe_rt_clear_log(spmoe_rt* rt);

/* --------------------------------------------------------------------- */
/* Host memory helpers                                                    */
/* --------------------------------------------------------------------- */
/* Page-locked, portable, mapped host allocation; *dev receives the device
 * alias (what a kernel writes to for zero-copy hand-off). */
int spmoe_host_alloc_mapped(size_t bytes, void** host, void** dev);
int spmoe_host_free(void* host);
/* Pin an existing host range (e.g. a /dev/shm expert pool shared by the
 * per-GPU processes of one box), portable + mapped. */
int spmoe_host_register(void* host, size_t bytes);
int spmoe_host_unregister(void* host);

/* --------------------------------------------------------------------- */
/* Events usable across CUDA-graph replays: record_external inside stream */
/* capture creates an external event-record node (cudaEventRecordExternal)*/
/* so the prefetch worker can wait on a predictor kernel that runs inside */
/* a replayed draft-step graph; outside capture it is cudaEventRecord.    */
/* --------------------------------------------------------------------- */
int spmoe_event_create(void** ev);
int spmoe_event_destroy(void* ev);
int spmoe_event_record_external(void* ev, void* stream);
int spmoe_event_synchronize(void* ev);

#ifdef __cplusplus
}
#endif
#endif /* SPMOE_H */
