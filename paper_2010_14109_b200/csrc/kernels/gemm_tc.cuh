// Batched tcgen05 GEMM for the attention products of the GAN step and the
// bf16 dense layers (ops_gan.cu, ops_dense.cu): C[b] = A[b] · B[b], fp32
// accumulation in TMEM.
//
//   A(m, k) at A + b·a_b + m·a_m + k·a_k   (bf16, or fp32 split into bf16 hi + lo)
//   B(k, n) at B + b·b_b + k·b_k + n·b_n   (bf16)
//   C(m, n) at C + b·c_b + m·ldc + n       (fp32, or bf16 rounded to nearest even)
//
// Each operand must be contiguous along one of its two indices (a_m or a_k
// equal to 1, b_k or b_n equal to 1); the shared-memory tile takes the matching
// UMMA layout (K-major or MN-major, SWIZZLE_128B), so no operand is transposed
// in memory.  An fp32 A (the softmax gradient dS) is split exactly into
// hi = rnd_bf16(a), lo = rnd_bf16(a − hi) and both halves are multiplied:
// |a − hi − lo| ≤ 2^-16 |a|, i.e. fp32-grade products on the bf16 tensor cores.
//
// Optional fused epilogue (fp32 C only): the softmax backward
// C(m, n) = P(m, n) · (acc(m, n) − rs[m]) with P bf16 (b·p_b + m·ldp + n) and
// rs fp32 (b·rs_b + m) — dS straight from the dP product.
//
// When the output tiles are too few to fill the GPU the K range is split;
// the splits' fp32 partials go to `ws` and a second kernel sums them in split
// order (deterministic).  ws_bytes(g) is the workspace a call needs.
#pragma once
#include "common.cuh"

namespace oc {
namespace tcg {

struct Gemm {
  int M, N, K, batch;
  const void* A;
  int64_t a_m, a_k, a_b;
  bool a_f32;
  const void* B;
  int64_t b_k, b_n, b_b;
  void* C;
  int64_t ldc, c_b;
  bool c_f32;
  // fused softmax-backward epilogue (null: plain store)
  const __nv_bfloat16* ep_p = nullptr;
  int64_t ldp = 0, p_b = 0;
  const float* ep_rs = nullptr;
  int64_t rs_b = 0;
  // dense layers: B fp32 (a master weight) rounded to bf16 as staged; bias[n]
  // added and ReLU applied in the epilogue; no K split (no workspace)
  bool b_f32 = false;
  const float* bias = nullptr;
  bool relu = false;
  bool no_split = false;
};

// K splits the call will use (1 = none)
int splits_of(const Gemm& g);
// workspace bytes for the split partials (0 when unsplit)
size_t ws_bytes(const Gemm& g);
// OC_E_UNSUPPORTED when neither stride of an operand is 1; OC_E_INVARIANT when
// ws is smaller than ws_bytes(g)
Status gemm(OpArgs& a, const Gemm& g, void* ws = nullptr, size_t ws_size = 0);

// Attention probabilities without the fp32 score map: P[b] = rnd(softmax_rows(
// q[b] k[b]ᵀ)) for q, k [nb, L, dq] bf16 (dq ≤ 64), P [nb, L, L] bf16.  Two
// launches over (query block, key range): the first recomputes the scores on
// the tensor cores and keeps per-row running (max, Σexp) for its key range;
// the second merges the ranges' statistics in fixed order, recomputes the
// scores and writes P = exp(s − max) / Σ.  Scores are never stored: HBM
// traffic is P's write alone.  ws: attn_softmax_ws() bytes.
size_t attn_softmax_ws(int nb, int L);
Status attn_softmax(OpArgs& a, const __nv_bfloat16* q, const __nv_bfloat16* k, __nv_bfloat16* P, int nb, int L,
                    int dq, void* ws, size_t ws_size);

}  // namespace tcg
}  // namespace oc
