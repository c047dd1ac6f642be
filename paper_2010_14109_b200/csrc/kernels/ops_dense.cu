// Dense-layer kernels of the training step:
// linear forward/backward, softmax cross-entropy, SGD with momentum and the
// data-parallel gradient all-reduce.  All reductions run in a fixed order so
// a step is bitwise reproducible whatever the swap schedule (swap
// transparency).
//
// bf16 layers run their products on the tensor cores (gemm_tc.cuh: the fp32
// master weight rounded to bf16 as it is staged, an fp32 logits gradient as an
// exact bf16 hi + lo pair, bias / ReLU in the epilogue); the fp32 parity mode
// and ReLU-masked gradients keep the SIMT FFMA kernel (no TF32).
#include "common.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"

namespace oc {

namespace {

using simt::gemm;

// db[n] = Σ_m dz[m,n] (masked), sequential over m per column: deterministic
template <typename T>
__global__ void colsum(int M, int N, const T* __restrict__ dy, const T* __restrict__ mask, float* __restrict__ out) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int m = 0; m < M; ++m) {
    int64_t o = (int64_t)m * N + n;
    float v = ld_f(dy + o);
    if (mask && !(ld_f(mask + o) > 0.f)) v = 0.f;
    s += v;
  }
  out[n] = s;
}

// ---------------------------------------------------------------- linear
enum { L_X, L_W, L_B, L_Y };
Status linear_fwd(OpArgs& a) {
  const int M = (int)A(a, "M"), N = (int)A(a, "N"), K = (int)A(a, "K");
  const bool relu = Ab(a, "relu");
  const std::string dt = As(a, "dtype", "f32");
  const float* w = (const float*)a.p(L_W);
  const float* b = (const float*)a.p(L_B);
  if (dt == "f32")
    return gemm<float, float, float, false>(a, M, N, K, (const float*)a.p(L_X), K, 1, nullptr, w, 1, K,
                                            (float*)a.p(L_Y), N, 1, b, relu, false);
  {
    // y = x Wᵀ + b: A = x (K-major), B(k, n) = W[n][k] (fp32, rounded, K-major)
    tcg::Gemm g{M, N, K, 1, a.p(L_X), K, 1, 0, false, w, 1, K, 0, a.p(L_Y), N, 0, Ab(a, "out_f32")};
    g.b_f32 = true;
    g.bias = b;
    g.relu = relu;
    g.no_split = true;
    return tcg::gemm(a, g);
  }
}

// roles: dy, y (ReLU mask source), x, w, dw, db, dx
enum { LB_DY, LB_Y, LB_X, LB_W, LB_DW, LB_DB, LB_DX };
Status linear_bwd(OpArgs& a) {
  const int M = (int)A(a, "M"), N = (int)A(a, "N"), K = (int)A(a, "K");
  const bool relu = Ab(a, "relu");
  const std::string dt = As(a, "dtype", "f32");
  const bool dy_f32 = dt == "f32" || Ab(a, "dy_f32");
  float* dw = (float*)a.p(LB_DW);
  float* db = (float*)a.p(LB_DB);
  if (dt == "f32" || dy_f32) {
    // dy fp32 [M,N]; mask (if any) has dy's layout and type
    const float* dy = (const float*)a.p(LB_DY);
    const float* mask = relu ? (const float*)a.p(LB_Y) : nullptr;
    if (dt != "f32" && !mask) {
      // tensor cores: dW[n,k] = Σ_m dy[m,n] x[m,k] (A = dyᵀ, MN-major fp32 split; B = x, MN-major)
      if (dw) {
        tcg::Gemm g{N, K, M, 1, dy, 1, N, 0, true, a.p(LB_X), K, 1, 0, dw, K, 0, true};
        g.no_split = true;
        OC_TRY(tcg::gemm(a, g));
      }
      if (db) {
        colsum<float><<<(N + 255) / 256, 256, 0, a.stream>>>(M, N, dy, nullptr, db);
        OC_LAUNCH_CHECK(a);
      }
      if (a.p(LB_DX)) {   // dx = dy W: A = dy (K-major fp32 split), B(k, n) = W[k][n] (fp32 rounded, MN-major)
        tcg::Gemm g{M, K, N, 1, dy, N, 1, 0, true, a.p(LB_W), K, 1, 0, a.p(LB_DX), K, 0, false};
        g.b_f32 = true;
        g.no_split = true;
        OC_TRY(tcg::gemm(a, g));
      }
      return Status::ok();
    }
    // dW[n,k] = Σ_m dz[m,n] x[m,k]  (dw / db null: data gradient only)
    if (dw && dt == "f32") {
      OC_TRY((gemm<float, float, float, false>(a, N, K, M, dy, 1, N, mask, (const float*)a.p(LB_X), K, 1, dw, K, 1,
                                               nullptr, false, false)));
    } else if (dw) {
      // x is bf16: A = dz (fp32), B = x (bf16 exact)
      OC_TRY((gemm<float, __nv_bfloat16, float, false>(a, N, K, M, dy, 1, N, mask,
                                                       (const __nv_bfloat16*)a.p(LB_X), K, 1, dw, K, 1, nullptr,
                                                       false, false)));
    }
    if (db) {
      colsum<float><<<(N + 255) / 256, 256, 0, a.stream>>>(M, N, dy, mask, db);
      OC_LAUNCH_CHECK(a);
    }
    if (a.p(LB_DX)) {
      if (dt == "f32")
        return gemm<float, float, float, false>(a, M, K, N, dy, N, 1, mask, (const float*)a.p(LB_W), K, 1,
                                                (float*)a.p(LB_DX), K, 1, nullptr, false, false);
      return gemm<float, float, __nv_bfloat16, true>(a, M, K, N, dy, N, 1, mask, (const float*)a.p(LB_W), K, 1,
                                                     (__nv_bfloat16*)a.p(LB_DX), K, 1, nullptr, false, false);
    }
    return Status::ok();
  }
  // bf16 dy (hidden bf16 linear layers)
  const __nv_bfloat16* dy = (const __nv_bfloat16*)a.p(LB_DY);
  const __nv_bfloat16* mask = relu ? (const __nv_bfloat16*)a.p(LB_Y) : nullptr;
  if (!mask) {
    if (dw) {   // A = dyᵀ (MN-major bf16), B = x (MN-major)
      tcg::Gemm g{N, K, M, 1, dy, 1, N, 0, false, a.p(LB_X), K, 1, 0, dw, K, 0, true};
      g.no_split = true;
      OC_TRY(tcg::gemm(a, g));
    }
    if (db) {
      colsum<__nv_bfloat16><<<(N + 255) / 256, 256, 0, a.stream>>>(M, N, dy, nullptr, db);
      OC_LAUNCH_CHECK(a);
    }
    if (a.p(LB_DX)) {
      tcg::Gemm g{M, K, N, 1, dy, N, 1, 0, false, a.p(LB_W), K, 1, 0, a.p(LB_DX), K, 0, false};
      g.b_f32 = true;
      g.no_split = true;
      OC_TRY(tcg::gemm(a, g));
    }
    return Status::ok();
  }
  if (dw)
    OC_TRY((gemm<__nv_bfloat16, __nv_bfloat16, float, false>(a, N, K, M, dy, 1, N, mask,
                                                             (const __nv_bfloat16*)a.p(LB_X), K, 1, dw, K, 1,
                                                             nullptr, false, false)));
  if (db) {
    colsum<__nv_bfloat16><<<(N + 255) / 256, 256, 0, a.stream>>>(M, N, dy, mask, db);
    OC_LAUNCH_CHECK(a);
  }
  if (a.p(LB_DX))
    return gemm<__nv_bfloat16, float, __nv_bfloat16, true>(a, M, K, N, dy, N, 1, mask, (const float*)a.p(LB_W), K,
                                                           1, (__nv_bfloat16*)a.p(LB_DX), K, 1, nullptr, false,
                                                           false);
  return Status::ok();
}

// ---------------------------------------------------------------- softmax CE
// per row: loss_m = logsumexp(z_m) − z_m[y_m]; dz = (softmax(z) − onehot)/M
__global__ void softmax_ce_rows(int M, int N, const float* __restrict__ z, const int* __restrict__ y,
                                float* __restrict__ row_loss, float* __restrict__ dz) {
  const int m = blockIdx.x;
  const float* zr = z + (int64_t)m * N;
  __shared__ float red[32];
  __shared__ float bcast;
  float mx = -INFINITY;
  for (int n = threadIdx.x; n < N; n += blockDim.x) mx = fmaxf(mx, zr[n]);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) bcast = v;
  }
  __syncthreads();
  mx = bcast;
  __syncthreads();
  float s = 0.f;
  for (int n = threadIdx.x; n < N; n += blockDim.x) s += expf(zr[n] - mx);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) bcast = v;
  }
  __syncthreads();
  s = bcast;
  const int lab = y[m];
  const float inv = 1.f / (float)M;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    float p = expf(zr[n] - mx) / s;
    dz[(int64_t)m * N + n] = (p - (n == lab ? 1.f : 0.f)) * inv;
  }
  if (threadIdx.x == 0) row_loss[m] = (logf(s) + mx) - zr[lab];
}

__global__ void mean_fixed_order(int M, const float* __restrict__ v, float* __restrict__ out) {
  double s = 0;
  for (int m = threadIdx.x; m < M; m += 32) s += v[m];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[0] = (float)(s / M);
}

enum { S_LOGITS, S_LABELS, S_LOSS, S_DLOGITS };
Status softmax_ce(OpArgs& a) {
  const int M = (int)A(a, "M"), N = (int)A(a, "N");
  if (a.ws_bytes < (size_t)M * 4) return Status::make(OC_E_INVARIANT, "softmax_ce: workspace too small");
  softmax_ce_rows<<<M, 256, 0, a.stream>>>(M, N, (const float*)a.p(S_LOGITS), (const int*)a.p(S_LABELS),
                                           (float*)a.ws, (float*)a.p(S_DLOGITS));
  OC_LAUNCH_CHECK(a);
  mean_fixed_order<<<1, 32, 0, a.stream>>>(M, (const float*)a.ws, (float*)a.p(S_LOSS));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
size_t softmax_ce_ws(const JVal& at) { return (size_t)at.geti("M") * 4; }

// ---------------------------------------------------------------- SGD
// v ← μ v + g ; w ← w − lr v  (fp32 state).  Multi-tensor: one launch updates
// up to kSgdMax tensors of a function; the tensor table travels
// by value in the kernel parameters (addresses are fixed per step, so a CUDA
// graph replays it), each block takes chunks of 16 KB of one tensor.
constexpr int kSgdMax = 48;
constexpr int64_t kSgdChunk = 4096;   // elements per block-chunk
struct SgdTab {
  float* w[kSgdMax];
  const float* g[kSgdMax];
  float* v[kSgdMax];
  int64_t n[kSgdMax];
  int32_t first_chunk[kSgdMax + 1];   // prefix sums of chunks per tensor
  int count;
};

__global__ void __launch_bounds__(256) sgd_multi(const __grid_constant__ SgdTab T, float lr, float mu) {
  for (int c = blockIdx.x; c < T.first_chunk[T.count]; c += gridDim.x) {
    int t = 0;
    while (T.first_chunk[t + 1] <= c) ++t;
    const int64_t base = (int64_t)(c - T.first_chunk[t]) * kSgdChunk;
    const int64_t end = min(T.n[t], base + kSgdChunk);
    float* __restrict__ w = T.w[t];
    const float* __restrict__ g = T.g[t];
    float* __restrict__ v = T.v[t];
    if (((((uintptr_t)w | (uintptr_t)g | (uintptr_t)v) & 15) == 0) && ((end - base) & 3) == 0) {
      for (int64_t k = base + 4 * threadIdx.x; k < end; k += 4 * blockDim.x) {
        float4 gw = *reinterpret_cast<const float4*>(g + k);
        float4 vv = *reinterpret_cast<float4*>(v + k);
        float4 ww = *reinterpret_cast<float4*>(w + k);
        vv.x = fmaf(mu, vv.x, gw.x); vv.y = fmaf(mu, vv.y, gw.y);
        vv.z = fmaf(mu, vv.z, gw.z); vv.w = fmaf(mu, vv.w, gw.w);
        ww.x = fmaf(-lr, vv.x, ww.x); ww.y = fmaf(-lr, vv.y, ww.y);
        ww.z = fmaf(-lr, vv.z, ww.z); ww.w = fmaf(-lr, vv.w, ww.w);
        *reinterpret_cast<float4*>(v + k) = vv;
        *reinterpret_cast<float4*>(w + k) = ww;
      }
    } else {
      for (int64_t k = base + threadIdx.x; k < end; k += blockDim.x) {
        const float vk = fmaf(mu, v[k], g[k]);
        v[k] = vk;
        w[k] = fmaf(-lr, vk, w[k]);
      }
    }
  }
}

enum { G_W, G_G, G_M };
Status sgd(OpArgs& a) {
  const float lr = (float)Ad(a, "lr"), mu = (float)Ad(a, "momentum");
  const size_t cnt = a.ptr[G_W].size();
  if (a.ptr[G_G].size() != cnt || a.ptr[G_M].size() != cnt) return Status::make(OC_E_INVALID, "sgd: role lengths differ");
  for (size_t t0 = 0; t0 < cnt; t0 += kSgdMax) {
    SgdTab T{};
    T.count = (int)std::min<size_t>(kSgdMax, cnt - t0);
    T.first_chunk[0] = 0;
    for (int t = 0; t < T.count; ++t) {
      T.w[t] = (float*)a.ptr[G_W][t0 + t];
      T.g[t] = (const float*)a.ptr[G_G][t0 + t];
      T.v[t] = (float*)a.ptr[G_M][t0 + t];
      T.n[t] = (int64_t)(a.bytes[G_W][t0 + t] / 4);
      T.first_chunk[t + 1] = T.first_chunk[t] + (int32_t)((T.n[t] + kSgdChunk - 1) / kSgdChunk);
    }
    if (T.first_chunk[T.count] == 0) continue;
    const int grid = std::min(T.first_chunk[T.count], 4 * kNumSMs);
    sgd_multi<<<grid, 256, 0, a.stream>>>(T, lr, mu);
    OC_LAUNCH_CHECK(a);
  }
  return Status::ok();
}

// ---------------------------------------------------------------- all-reduce
// Mean of the replicas' gradients: NCCL (ncclAvg; one
// ncclGroup per bucket — the tensors of one allreduce function), or the
// attached custom communicator, one call per tensor.  The executor launches
// it on its communication stream (a.stream) when a communicator is attached.
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_t)();
Status allreduce(OpArgs& a) {
  if (a.comm_fn) {
    for (size_t t = 0; t < a.ptr[0].size(); ++t)
      if (a.comm_fn(a.comm_user, a.ptr[0][t], a.bytes[0][t] / 4, (void*)a.stream))
        return Status::make(OC_E_NCCL, "custom allreduce failed");
    return Status::ok();
  }
  if (!a.nccl_comm) return Status::ok();  // single replica
  auto f = (nccl_allreduce_t)a.nccl_allreduce;
  const bool grp = a.nccl_group_start && a.nccl_group_end && a.ptr[0].size() > 1;
  if (grp) ((nccl_group_t)a.nccl_group_start)();
  for (size_t t = 0; t < a.ptr[0].size(); ++t) {
    // ncclFloat32 = 7, ncclAvg = 4
    int r = f(a.ptr[0][t], a.ptr[0][t], a.bytes[0][t] / 4, 7, 4, a.nccl_comm, a.stream);
    if (r) {
      if (grp) ((nccl_group_t)a.nccl_group_end)();
      Status s = Status::make(OC_E_NCCL, "ncclAllReduce failed");
      s.cuda = r;
      return s;
    }
  }
  if (grp) {
    int r = ((nccl_group_t)a.nccl_group_end)();
    if (r) { Status s = Status::make(OC_E_NCCL, "ncclGroupEnd failed"); s.cuda = r; return s; }
  }
  return Status::ok();
}

// no compute (placeholder functions in planner-only graphs)
Status nop(OpArgs&) { return Status::ok(); }

}  // namespace

extern const OpDesc kLinearFwd{"linear_fwd", {"x", "w", "b", "y"}, linear_fwd, nullptr};
extern const OpDesc kLinearBwd{"linear_bwd", {"dy", "y", "x", "w", "dw", "db", "dx"}, linear_bwd, nullptr};
extern const OpDesc kSoftmaxCE{"softmax_ce", {"logits", "labels", "loss", "dlogits"}, softmax_ce, softmax_ce_ws};
extern const OpDesc kSGD{"sgd", {"w", "g", "m"}, sgd, nullptr};
extern const OpDesc kAllreduce{"allreduce", {"bufs"}, allreduce, nullptr};
extern const OpDesc kNop{"nop", {}, nop, nullptr};

}  // namespace oc
