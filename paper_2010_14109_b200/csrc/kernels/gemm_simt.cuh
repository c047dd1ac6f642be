// SIMT FFMA GEMM (fp32 accumulation), generic strides and an optional batch
// dimension: the dense layers (ops_dense.cu) and the attention products of the
// GAN step (ops_gan.cu).  No TF32: the fp32 parity mode needs exact FFMA.
#pragma once
#include "common.cuh"

namespace oc {
namespace simt {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;

// C[m,n] (+)= Σ_k A(m,k)·B(k,n), generic strides; blockIdx.z = batch index
// (A, B, C advanced by sab, sbb, scb elements per batch entry).
//   maskA: A(m,k) is used only where mask(m,k) > 0 (ReLU'(·), same strides as A)
//   RB:    round B to bf16 on load (bf16 copy of an fp32 master weight)
//   bias:  per-n bias; relu: max(·,0); accumulate: C = rnd(C + acc)
template <typename TA, typename TB, typename TC, bool RB>
__global__ void __launch_bounds__(256) gemm_simt(int M, int N, int K, const TA* __restrict__ A, int64_t sam,
                                                 int64_t sak, const TA* __restrict__ maskA, const TB* __restrict__ B,
                                                 int64_t sbk, int64_t sbn, TC* C, int64_t scm, int64_t scn,
                                                 const float* __restrict__ bias, int relu, int accumulate,
                                                 int64_t sab = 0, int64_t sbb = 0, int64_t scb = 0) {
  A += blockIdx.z * sab;
  if (maskA) maskA += blockIdx.z * sab;
  B += blockIdx.z * sbb;
  C += blockIdx.z * scb;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = tid % 16, ty = tid / 16;
  float acc[TM][TN] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + r * 256;  // 0..1023
      int mm = e % BM, kk = e / BM;
      int gm = m0 + mm, gk = k0 + kk;
      float va = 0.f;
      if (gm < M && gk < K) {
        int64_t off = (int64_t)gm * sam + (int64_t)gk * sak;
        va = ld_f(A + off);
        if (maskA && !(ld_f(maskA + off) > 0.f)) va = 0.f;
      }
      As[kk][mm] = va;
      int nn = e % BN, kb = e / BN;
      int gn = n0 + nn, gk2 = k0 + kb;
      float vb = 0.f;
      if (gn < N && gk2 < K) {
        vb = ld_f(B + (int64_t)gk2 * sbk + (int64_t)gn * sbn);
        if (RB) vb = rnd<__nv_bfloat16>(vb);
      }
      Bs[kb][nn] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gn = n0 + tx * TN + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (bias) v += bias[gn];
      if (relu) v = fmaxf(v, 0.f);
      TC* p = C + (int64_t)gm * scm + (int64_t)gn * scn;
      if (accumulate) v = v + ld_f(p);
      st_f(p, v);
    }
  }
}

template <typename TA, typename TB, typename TC, bool RB>
Status gemm(OpArgs& a, int M, int N, int K, const TA* A, int64_t sam, int64_t sak, const TA* mask, const TB* B,
            int64_t sbk, int64_t sbn, TC* C, int64_t scm, int64_t scn, const float* bias, bool relu, bool acc,
            int batch = 1, int64_t sab = 0, int64_t sbb = 0, int64_t scb = 0) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  gemm_simt<TA, TB, TC, RB><<<grid, 256, 0, a.stream>>>(M, N, K, A, sam, sak, mask, B, sbk, sbn, C, scm, scn, bias,
                                                        relu ? 1 : 0, acc ? 1 : 0, sab, sbb, scb);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

}  // namespace simt
}  // namespace oc
