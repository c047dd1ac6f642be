// Batched tcgen05 GEMM (gemm_tc.cuh): the attention products of the GAN step.
//
// One CTA = 128 threads computes one 128 × BN tile of one batch entry (and one
// K split).  All threads stage the operands global → registers → shared memory
// in the UMMA SWIZZLE_128B layout that matches the operand's contiguous index
// (K-major: rows of 64 K-elements, 16-byte chunk c of row r at r·128 +
// (c ^ r%8)·16; MN-major: 64-wide MN atoms of 8 KB, K-row r at r·128 with the
// same chunk swizzle), zero-filling past M, N, K — so any stride pattern, the
// attention's 12- or 24-wide queries, and the fp32 → bf16 hi/lo split need no
// extra pass over memory.  The loads of K-block i+1 are issued into registers
// before K-block i is handed to the tensor cores (thread 0 issues kind::f16
// MMAs, M = 128, fp32 accumulator in BN TMEM columns, and commits them to the
// stage's mbarrier), so global latency overlaps the barrier and the MMAs.
// Epilogue: each warp reads its 32 TMEM lanes (rows); fp32 results go through
// a swizzled 32 × 32 staging tile so every warp store writes whole 128-byte
// row segments.  The products are HBM-bound (an L × L fp32 map written or read
// per sample), not tensor-bound: the goal is moving bytes at line rate.
#include <algorithm>
#include <type_traits>

#include "gemm_tc.cuh"
#include "tc_util.cuh"

namespace oc {
namespace tcg {
namespace {

using namespace tcu;

constexpr int BM = 128, BK = 64, NT = 128, NS = 2, STG = 4 * 4096;

struct KP {
  int M, N, K, batch, splits, kps, ns;
  const void* A;
  int64_t a_m, a_k, a_b;
  int a_mn, a_vec;
  const void* B;
  int64_t b_k, b_n, b_b;
  int b_mn, b_vec;
  void* C;
  int64_t ldc, c_b;
  int c_vec;
  float* part;                 // splits > 1: fp32 partials [split][batch][M][N]
  const uint16_t* ep_p;        // fused softmax backward: P (bf16) and rs
  int64_t ldp, p_b;
  const float* ep_rs;
  int64_t rs_b;
  int ep_vec;
  const float* bias;           // + bias[n], then ReLU if relu (unsplit calls)
  int relu;
};

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// shared-memory offset of 16-byte chunk c (along the contiguous index) of row r
__device__ __forceinline__ uint32_t chunk_off(bool mn_major, int r, int c) {
  return mn_major ? (uint32_t)((c >> 3) * 8192 + r * 128 + (((c & 7) ^ (r & 7)) << 4))
                  : (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4));
}
// global address and in-range element count of chunk (r, c)
template <typename T>
__device__ __forceinline__ const T* chunk_src(const T* X, int64_t s_mn, int64_t s_k, bool mn_major, int r, int c,
                                              int mn0, int MN, int k0, int K, int& valid) {
  if (!mn_major) {
    const int mn = mn0 + r, k = k0 + c * 8;
    valid = (mn < MN && k < K) ? K - k : 0;
    return X + (int64_t)mn * s_mn + k;
  }
  const int k = k0 + r, mn = mn0 + c * 8;
  valid = (k < K && mn < MN) ? MN - mn : 0;
  return X + (int64_t)k * s_k + mn;
}

// Per-thread view of one operand tile (ROWS MN indices × BK K indices): the
// thread's chunk i is row r0 + i·rstep along the non-contiguous index and
// 16-byte chunk c along the contiguous one (constant per thread, as NT is a
// multiple of the chunks per row), so its address advances by a fixed di per i
// and dk per K-block, and which chunks are wholly in range (vector load) or
// wholly outside (zero) is known once.  Only chunks cut by the M, N or K edge,
// or an operand whose rows are not 16-byte aligned, take the element-wise path.
// KIND 0: bf16; 1: fp32 split into bf16 hi + lo tiles; 2: fp32 rounded to bf16
template <int ROWS, int KIND>
struct Loader {
  static constexpr bool F32 = KIND != 0;
  using T = typename std::conditional<F32, float, uint16_t>::type;
  static constexpr int IT = ROWS * BK / 8 / NT;
  const T* X;
  int64_t s_mn, s_k, di, dk;
  const T* p0;
  int mn0, MN, K, r0, rstep, c;
  uint32_t vmask, zmask;
  bool mn_major;
  uint4 h[IT];        // bf16 chunks
  float4 f[F32 ? IT : 1][2];   // fp32 chunks

  __device__ __forceinline__ void init(const T* X_, int64_t s_mn_, int64_t s_k_, bool mnm, bool vec, int mn0_, int MN_,
                                       int K_) {
    X = X_;
    s_mn = s_mn_;
    s_k = s_k_;
    mn_major = mnm;
    mn0 = mn0_;
    MN = MN_;
    K = K_;
    const int t = threadIdx.x;
    if (!mnm) {
      r0 = t >> 3;
      c = t & 7;
      rstep = NT / 8;
      p0 = X + (int64_t)(mn0 + r0) * s_mn + c * 8;
      di = (int64_t)rstep * s_mn;
      dk = BK;
    } else {
      constexpr int CPR = ROWS / 8;
      r0 = t / CPR;
      c = t % CPR;
      rstep = NT / CPR;
      p0 = X + (int64_t)r0 * s_k + mn0 + c * 8;
      di = (int64_t)rstep * s_k;
      dk = (int64_t)BK * s_k;
    }
    vmask = zmask = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (!mnm) {
        if (mn0 + r0 + i * rstep >= MN) zmask |= 1u << i;
        else if (vec) vmask |= 1u << i;
      } else {
        const int v = MN - (mn0 + c * 8);
        if (v <= 0) zmask |= 1u << i;
        else if (v >= 8 && vec) vmask |= 1u << i;
      }
    }
  }
  __device__ __forceinline__ void slow(int i, int kb) {
    int valid;
    const T* p = chunk_src(X, s_mn, s_k, mn_major, r0 + i * rstep, c, mn0, MN, kb * BK, K, valid);
    if (valid >= 8 && ((vmask >> i) & 1u)) {   // this chunk is whole although the block is not
      if constexpr (F32) {
        f[i][0] = __ldg(reinterpret_cast<const float4*>(p));
        f[i][1] = __ldg(reinterpret_cast<const float4*>(p) + 1);
      } else {
        h[i] = __ldg(reinterpret_cast<const uint4*>(p));
      }
      return;
    }
    if constexpr (F32) {
      float e8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) e8[e] = e < valid ? p[e] : 0.f;
      f[i][0] = make_float4(e8[0], e8[1], e8[2], e8[3]);
      f[i][1] = make_float4(e8[4], e8[5], e8[6], e8[7]);
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < valid) w[e >> 1] |= (uint32_t)p[e] << ((e & 1) * 16);
      h[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  // K-block kb; `full`: no chunk of this block crosses K
  __device__ __forceinline__ void load(int kb, bool full) {
    const T* p = p0 + kb * dk;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (full && ((vmask >> i) & 1u)) {
        if constexpr (F32) {
          f[i][0] = __ldg(reinterpret_cast<const float4*>(p + i * di));
          f[i][1] = __ldg(reinterpret_cast<const float4*>(p + i * di) + 1);
        } else {
          h[i] = __ldg(reinterpret_cast<const uint4*>(p + i * di));
        }
      } else if ((zmask >> i) & 1u) {
        if constexpr (F32) f[i][0] = f[i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        else h[i] = make_uint4(0, 0, 0, 0);
      } else {
        slow(i, kb);
      }
    }
  }
  // bf16 / rounded fp32: one tile; split fp32: hi tile at `tile`, lo tile at `lo`
  __device__ __forceinline__ void store(uint32_t tile, uint32_t lo) const {
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const uint32_t off = chunk_off(mn_major, r0 + i * rstep, c);
      if constexpr (KIND == 2) {
        sts128(tile + off, make_uint4(pack2(f[i][0].x, f[i][0].y), pack2(f[i][0].z, f[i][0].w),
                                      pack2(f[i][1].x, f[i][1].y), pack2(f[i][1].z, f[i][1].w)));
      } else if constexpr (KIND == 1) {
        const float e8[8] = {f[i][0].x, f[i][0].y, f[i][0].z, f[i][0].w, f[i][1].x, f[i][1].y, f[i][1].z, f[i][1].w};
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __nv_bfloat162 hh = __floats2bfloat162_rn(e8[2 * e], e8[2 * e + 1]);
          const float2 hf = __bfloat1622float2(hh);
          hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
          lw[e] = pack2(e8[2 * e] - hf.x, e8[2 * e + 1] - hf.y);   // exact differences
        }
        sts128(tile + off, make_uint4(hw[0], hw[1], hw[2], hw[3]));
        sts128(lo + off, make_uint4(lw[0], lw[1], lw[2], lw[3]));
      } else {
        sts128(tile + off, h[i]);
      }
    }
  }
};

template <int BN, bool AF32, bool CF32, bool BF32>
__global__ void __launch_bounds__(NT) gemm_tc_kernel(const __grid_constant__ KP P) {
  constexpr int A_T = BM * BK * 2, B_T = BN * BK * 2;
  constexpr int STAGE = A_T * (AF32 ? 2 : 1) + B_T;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int ns = P.ns;
  uint8_t* stg = smem;   // epilogue staging: the operand stages, free once the MMAs are done
  uint64_t* empty = (uint64_t*)(smem + max(ns * STAGE, STG));
  uint64_t* done = empty + NS;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int sp = (int)blockIdx.z % P.splits, bz = (int)blockIdx.z / P.splits;
  const bool a_mn = P.a_mn, b_mn = P.b_mn;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&empty[s], 1);
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const uint32_t id = idesc_m(BM, BN, a_mn, b_mn);
  const int nkb = (P.K + BK - 1) / BK, nfull = P.K / BK;
  const int kb0 = sp * P.kps, kb1 = min(nkb, kb0 + P.kps);
  Loader<BM, AF32 ? 1 : 0> la;
  Loader<BN, BF32 ? 2 : 0> lb;
  la.init((const typename Loader<BM, AF32 ? 1 : 0>::T*)P.A + bz * P.a_b, P.a_m, P.a_k, a_mn, P.a_vec, m0, P.M, P.K);
  lb.init((const typename Loader<BN, BF32 ? 2 : 0>::T*)P.B + bz * P.b_b, P.b_n, P.b_k, b_mn, P.b_vec, n0, P.N, P.K);
  if (kb0 < kb1) {
    la.load(kb0, kb0 < nfull);
    lb.load(kb0, kb0 < nfull);
  }
  for (int kb = kb0; kb < kb1; ++kb) {
    const int i = kb - kb0, s = i % ns;
    if (i >= ns) mbar_wait(&empty[s], ((i / ns) - 1) & 1);   // the MMAs that read this stage are done
    const uint32_t a = smem_u32(smem + s * STAGE), a_lo = a + A_T, b = a + A_T * (AF32 ? 2 : 1);
    la.store(a, a_lo);
    lb.store(b, 0);
    if (kb + 1 < kb1) {   // the next K-block's loads are in flight during the barrier and the MMAs
      la.load(kb + 1, kb + 1 < nfull);
      lb.load(kb + 1, kb + 1 < nfull);
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int j = 0; j < BK / 16; ++j) {
        const uint64_t db = b_mn ? sdesc(b + j * 2048, 8192, 1024) : sdesc(b + j * 32, 16, 1024);
        const uint64_t da = a_mn ? sdesc(a + j * 2048, 8192, 1024) : sdesc(a + j * 32, 16, 1024);
        mma_bf16(tmem, da, db, id, (i > 0 || j > 0) ? 1u : 0u);
        if (AF32) {
          const uint64_t dl = a_mn ? sdesc(a_lo + j * 2048, 8192, 1024) : sdesc(a_lo + j * 32, 16, 1024);
          mma_bf16(tmem, dl, db, id, 1u);
        }
      }
      mma_commit(&empty[s]);
    }
  }
  const bool has_k = kb0 < kb1;
  if (has_k) {
    if (threadIdx.x == 0) mma_commit(done);
    mbar_wait(done, 0);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---------------------------------------------------------------- epilogue
  // warp w owns TMEM lanes (rows) 32w .. 32w + 31
  const bool split = P.splits > 1;
  if (CF32 || split) {
    // fp32 rows through the warp's 32 × 32 staging tile: lane = row on the way
    // in, 8 lanes per row segment (4 rows per instruction) on the way out
    const uint32_t st = smem_u32(stg) + warp * 4096;
    float* dst;
    int64_t ld;
    if (split) {
      dst = P.part + ((int64_t)sp * P.batch + bz) * P.M * P.N;
      ld = P.N;
    } else {
      dst = (float*)P.C + bz * P.c_b;
      ld = P.ldc;
    }
    const bool vec = split ? (P.N % 4 == 0) : P.c_vec;
    const bool ep = !split && P.ep_p;
    const int cc = lane & 7;
    // fused softmax backward: rs of the lane's 8 rows, and P of the next
    // 32-column chunk loaded ahead of its use
    float rsv[8];
    uint2 pv[8];
    auto load_p = [&](int j0) {
      const int col = n0 + j0 + cc * 4;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = m0 + warp * 32 + i * 4 + (lane >> 3);
        pv[i] = make_uint2(0, 0);
        if (row >= P.M || col >= P.N) continue;
        const uint16_t* pp = P.ep_p + bz * P.p_b + (int64_t)row * P.ldp + col;
        if (P.N - col >= 4 && P.ep_vec) {
          pv[i] = __ldg(reinterpret_cast<const uint2*>(pp));
        } else {
          uint32_t w[2] = {0, 0};
          for (int e = 0; e < 4 && e < P.N - col; ++e) w[e >> 1] |= (uint32_t)pp[e] << ((e & 1) * 16);
          pv[i] = make_uint2(w[0], w[1]);
        }
      }
    };
    if (ep) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = m0 + warp * 32 + i * 4 + (lane >> 3);
        rsv[i] = row < P.M ? P.ep_rs[bz * P.rs_b + row] : 0.f;
      }
      load_p(0);
    }
#pragma unroll 1
    for (int j0 = 0; j0 < BN && n0 + j0 < P.N; j0 += 32) {
      uint32_t v[32];
      TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16) + j0, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 8; ++c)
        sts128(st + lane * 128 + ((c ^ (lane & 7)) << 4),
               has_k ? make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]) : make_uint4(0, 0, 0, 0));
      __syncwarp();
      uint2 pc[8];
      if (ep) {
#pragma unroll
        for (int i = 0; i < 8; ++i) pc[i] = pv[i];
        if (j0 + 32 < BN && n0 + j0 + 32 < P.N) load_p(j0 + 32);
      }
      const int col = n0 + j0 + cc * 4;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = i * 4 + (lane >> 3), row = m0 + warp * 32 + rr;
        const uint4 u = lds128(st + rr * 128 + ((cc ^ (rr & 7)) << 4));
        float f[4] = {__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w)};
        if (row >= P.M || col >= P.N) continue;
        const int nv = P.N - col;
        if (!split && P.bias) {
#pragma unroll
          for (int e = 0; e < 4; ++e) f[e] += e < nv ? P.bias[col + e] : 0.f;
        }
        if (!split && P.relu) {
#pragma unroll
          for (int e = 0; e < 4; ++e) f[e] = fmaxf(f[e], 0.f);
        }
        if (ep) {   // dS = P ⊙ (dP − rs)
          f[0] = __uint_as_float(pc[i].x << 16) * (f[0] - rsv[i]);
          f[1] = __uint_as_float(pc[i].x & 0xffff0000u) * (f[1] - rsv[i]);
          f[2] = __uint_as_float(pc[i].y << 16) * (f[2] - rsv[i]);
          f[3] = __uint_as_float(pc[i].y & 0xffff0000u) * (f[3] - rsv[i]);
        }
        float* cp = dst + (int64_t)row * ld + col;
        if (nv >= 4 && vec) {
          *reinterpret_cast<float4*>(cp) = make_float4(f[0], f[1], f[2], f[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < nv) cp[e] = f[e];
        }
      }
      __syncwarp();
    }
  } else {
    const int row = m0 + warp * 32 + lane;
    const bool rin = row < P.M;
#pragma unroll 1
    for (int j0 = 0; j0 < BN && n0 + j0 < P.N; j0 += 32) {
      uint32_t v[32];
      TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16) + j0, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (!rin) continue;
      const int nv = P.N - (n0 + j0);
      __nv_bfloat16* cp = (__nv_bfloat16*)P.C + bz * P.c_b + (int64_t)row * P.ldc + n0 + j0;
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          f[e] = has_k ? __uint_as_float(v[c + e]) : 0.f;
          if (P.bias && c + e < nv) f[e] += P.bias[n0 + j0 + c + e];
          if (P.relu) f[e] = fmaxf(f[e], 0.f);
        }
        if (c + 8 <= nv && P.c_vec) {
          *reinterpret_cast<uint4*>(cp + c) =
              make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (c + e < nv) cp[c + e] = __float2bfloat16_rn(f[e]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

// C = Σ_split partials, in split order
template <typename TC>
__global__ void split_reduce_k(int64_t n, int M, int N, int splits, const float* __restrict__ part, TC* C,
                               int64_t ldc, int64_t c_b) {
  const int64_t MN = (int64_t)M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * n + i];
    const int64_t b = i / MN, r = i - b * MN;
    const int m = (int)(r / N), c = (int)(r - (int64_t)m * N);
    st_f(C + b * c_b + (int64_t)m * ldc + c, s);
  }
}

// fp32 outputs (the L × L maps) take 128-column tiles: 128 TMEM columns per
// CTA, so four CTAs share an SM and one's epilogue overlaps the others' loads
int bn_of(const Gemm& g) {
  if (g.b_f32 || (g.a_f32 && g.c_f32)) return 128;   // the dense layers: one tile width
  return g.N <= 64 ? 64 : (g.N <= 128 || g.c_f32) ? 128 : 256;
}

void plan_split(const Gemm& g, int& splits, int& kps) {
  const int nkb = (g.K + BK - 1) / BK;
  const int bn = bn_of(g);
  const int64_t tiles = (int64_t)((g.N + bn - 1) / bn) * ((g.M + BM - 1) / BM) * g.batch;
  const int64_t target = 2 * 148;
  splits = 1;
  if (!g.ep_p && !g.no_split && !g.bias && !g.relu && tiles < target && nkb >= 8) {
    // whole waves: at most two CTAs per SM fit (shared memory), so rounding the
    // split count up would start a second, mostly idle wave (384 CTAs for 296
    // slots, ncu: a 1.3-wave dS product at 0.28 of HBM); rounding down keeps one
    int64_t s = std::max<int64_t>(1, target / tiles);
    s = std::min<int64_t>(s, nkb / 4);
    s = std::min<int64_t>(s, 65535 / std::max(1, g.batch));
    splits = (int)std::max<int64_t>(1, s);
  }
  kps = std::max(1, (nkb + splits - 1) / splits);
  splits = std::max(1, (nkb + kps - 1) / kps);
}

template <int BN, bool AF32, bool CF32, bool BF32 = false>
Status launch(OpArgs& a, const KP& p) {
  constexpr int STAGE = BM * BK * 2 * (AF32 ? 2 : 1) + BN * BK * 2;
  const int smem = std::max(p.ns * STAGE, STG) + 1024 + 64;
  auto k = gemm_tc_kernel<BN, AF32, CF32, BF32>;
  static bool attr = false;
  if (!attr) {
    OC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * STAGE + 1024 + 64));
    attr = true;
  }
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.batch * p.splits);
  k<<<grid, NT, smem, a.stream>>>(p);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

bool aligned(const void* p, int64_t bytes) { return ((uintptr_t)p % bytes) == 0; }


// ---------------------------------------------------------------- fused attention probabilities
struct AP {
  int L, dq, js, jper;
  const uint16_t* q;
  const uint16_t* k;
  int64_t sb;          // q / k batch stride (L·dq)
  uint16_t* P;
  float* pm;           // per-range row statistics [nb][js][L]
  float* pl;
  int vec;
  int async_k;         // k rows 8-byte aligned (dq % 4 == 0): cp.async key tiles
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;
constexpr int AT_N = 64;    // key columns per score tile (two TMEM buffers of 64 columns)
constexpr int AT_NT = 256;
constexpr int AT_KS = 4;    // key-tile ring slots (cp.async path)
constexpr int AT_JS = 16;   // most key ranges per row (fixed-size statistics merge)  // 8 warps: warp w reads TMEM lanes 32·(w % 4).., columns 32·(w / 4).. of a tile

// one 128-query block × one key range of one sample; pass 0 (WRITE = false):
// running (max, Σexp) per row; pass 1: merge the ranges, write P.  Each thread
// owns one query row (its TMEM lane) and one 32-column half of every tile;
// exp(s − m) = 2^(s·log2e − m·log2e).  Warps 0-3 stage the operands.
template <bool WRITE>
__global__ void __launch_bounds__(AT_NT) attn_p_kernel(const __grid_constant__ AP p) {
  constexpr int T_A = BM * BK * 2, T_B = AT_N * BK * 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int T_P = BM * AT_N * 2;   // pass 1: a bf16 P tile staged for coalesced stores (two buffers)
  uint8_t* pst = smem + T_A + AT_KS * T_B;
  uint64_t* tfull = (uint64_t*)(pst + (WRITE ? 2 * T_P : 0));
  uint32_t* tmem_slot = (uint32_t*)(tfull + 2);
  float* xch = (float*)(tmem_slot + 2);   // pass 0: the second halves' (max, Σ) per row
  const int warp = threadIdx.x >> 5, half = warp >> 2, lane = threadIdx.x & 31;
  const bool stager = threadIdx.x < NT;
  const int jr = blockIdx.x, i0 = blockIdx.y * BM, b = blockIdx.z, L = p.L;
  const int rl = (warp & 3) * 32 + lane, row = i0 + rl;   // this thread's TMEM lane = query row
  const int jbeg = jr * p.jper, jend = min(L, jbeg + p.jper);
  const int T = jend > jbeg ? (jend - jbeg + AT_N - 1) / AT_N : 0;

  if (threadIdx.x == 0) {
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * AT_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint16_t* qb = p.q + b * p.sb;
  const uint16_t* kb_ = p.k + b * p.sb;
  if (stager) {
    Loader<BM, 0> la;
    la.init(qb, p.dq, 1, false, p.vec, i0, L, p.dq);
    la.load(0, p.dq >= BK);
    la.store(smem_u32(smem), 0);
  }
  // this row's statistics: running (pass 0) or merged over the ranges (pass 1)
  float m = -INFINITY, l = 0.f;
  if (WRITE && row < L) {
    const float* pm = p.pm + (int64_t)b * p.js * L + row;
    const float* pl = p.pl + (int64_t)b * p.js * L + row;
    float zm[AT_JS], zl[AT_JS];
#pragma unroll
    for (int z = 0; z < AT_JS; ++z) {
      zm[z] = z < p.js ? pm[(int64_t)z * L] : -INFINITY;
      zl[z] = z < p.js ? pl[(int64_t)z * L] : 0.f;
    }
#pragma unroll
    for (int z = 0; z < AT_JS; ++z) m = fmaxf(m, zm[z]);
#pragma unroll
    for (int z = 0; z < AT_JS; ++z)
      if (zm[z] != -INFINITY) l += zl[z] * ex2((zm[z] - m) * kLog2e);
  }
  const float inv = 1.f / l;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t id = idesc_m(BM, AT_N, false, false);
  const uint32_t a_s = smem_u32(smem);

  Loader<AT_N, 0> lb;
  auto load_k = [&](int t) {
    lb.init(kb_, p.dq, 1, false, p.vec, jbeg + t * AT_N, jend, p.dq);
    lb.load(0, p.dq >= BK);
  };
  auto epilogue = [&](int u) {
    mbar_wait(&tfull[u & 1], (u >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int j0 = jbeg + u * AT_N;
    {
      const int c4 = half;
      uint32_t v[32];
      TMEM_LD32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (u & 1) * AT_N + c4 * 32, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int jc = j0 + c4 * 32;
      const int nv = min(32, jend - jc);
      if (!WRITE) {
        if (row < L && nv > 0) {
          float x[32];
          if (nv == 32) {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = fmaxf(__uint_as_float(v[e]), __uint_as_float(v[e + 16]));
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              x[e] = fmaxf(e < nv ? __uint_as_float(v[e]) : -INFINITY, e + 16 < nv ? __uint_as_float(v[e + 16]) : -INFINITY);
          }
#pragma unroll
          for (int w = 8; w > 0; w >>= 1)
#pragma unroll
            for (int e = 0; e < w; ++e) x[e] = fmaxf(x[e], x[e + w]);
          const float mn = fmaxf(m, x[0]), mL = mn * kLog2e;
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
          if (nv == 32) {
#pragma unroll
            for (int e = 0; e < 32; ++e) s4[e & 3] += ex2(fmaf(__uint_as_float(v[e]), kLog2e, -mL));
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e < nv) s4[e & 3] += ex2(fmaf(__uint_as_float(v[e]), kLog2e, -mL));
          }
          l = (m == -INFINITY ? 0.f : l * ex2((m - mn) * kLog2e)) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
          m = mn;
        }
      } else {
        // P for this row's 32 columns into the staging tile (row rl, 16-byte
        // chunks 4·half .. 4·half + 3, swizzled by rl % 8), then the CTA stores
        // the tile as whole 128-byte row segments
        const uint32_t sb = smem_u32(pst) + (u & 1) * T_P;
        if (row < L && nv > 0) {
          const float mL = m * kLog2e;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float e8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) e8[e] = ex2(fmaf(__uint_as_float(v[c * 8 + e]), kLog2e, -mL)) * inv;
            const int ch = half * 4 + c;
            sts128(sb + rl * 128 + ((ch ^ (rl & 7)) << 4),
                   make_uint4(pack2(e8[0], e8[1]), pack2(e8[2], e8[3]), pack2(e8[4], e8[5]), pack2(e8[6], e8[7])));
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(AT_NT) : "memory");
        const int ch = threadIdx.x & 7, col = j0 + ch * 8;
#pragma unroll
        for (int i = 0; i < BM * 8 / AT_NT; ++i) {
          const int r = (threadIdx.x >> 3) + i * (AT_NT / 8), grow = i0 + r;
          if (grow >= L || col >= jend) continue;
          const uint4 w = lds128(sb + r * 128 + ((ch ^ (r & 7)) << 4));
          uint16_t* pp = p.P + (int64_t)b * L * L + (int64_t)grow * L + col;
          if (col + 8 <= jend && p.vec) {
            *reinterpret_cast<uint4*>(pp) = w;
          } else {
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (col + e < jend) pp[e] = (uint16_t)(ww[e >> 1] >> ((e & 1) * 16));
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  };

  if (p.async_k) {
    // key tiles through a ring of AT_KS shared-memory slots filled by cp.async
    // (8-byte pieces, zero-filled past the range and past dq), AT_KS − 1 tiles ahead
    auto issue_k = [&](int t) {
      if (t < T) {
        const uint32_t slot = a_s + T_A + (t % AT_KS) * T_B;
        const int c = threadIdx.x & 7;
#pragma unroll
        for (int i = 0; i < AT_N * 8 / AT_NT; ++i) {
          const int r = (threadIdx.x >> 3) + i * (AT_NT / 8), j = jbeg + t * AT_N + r;
          const uint32_t dst = slot + r * 128 + ((c ^ (r & 7)) << 4);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int e0 = c * 8 + h * 4;
            const bool ok = j < jend && e0 < p.dq;
            const uint16_t* src = ok ? kb_ + (int64_t)j * p.dq + e0 : kb_;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + h * 8), "l"(src), "r"(ok ? 8 : 0)
                         : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int t = 0; t < AT_KS - 1; ++t) issue_k(t);
    for (int t = 0; t < T; ++t) {
      asm volatile("cp.async.wait_group %0;" ::"n"(AT_KS - 2) : "memory");
      fence_async_smem();
      __syncthreads();
      const uint32_t bsm = a_s + T_A + (t % AT_KS) * T_B;
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < BK / 16; ++j)
          mma_bf16(tmem + (t & 1) * AT_N, sdesc(a_s + j * 32, 16, 1024), sdesc(bsm + j * 32, 16, 1024), id,
                   j > 0 ? 1u : 0u);
        mma_commit(&tfull[t & 1]);
      }
      if (t >= 1) epilogue(t - 1);   // waits for MMA t − 1: its slot may be refilled
      issue_k(t + AT_KS - 1);
    }
    if (T > 0) epilogue(T - 1);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
  if (T > 0 && stager) load_k(0);
  for (int t = 0; t < T; ++t) {
    const uint32_t bsm = a_s + T_A + (t & 1) * T_B;
    if (stager) lb.store(bsm, 0);   // the MMA that last read this buffer (t − 2) was waited for by epilogue(t − 2)
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int j = 0; j < BK / 16; ++j)
        mma_bf16(tmem + (t & 1) * AT_N, sdesc(a_s + j * 32, 16, 1024), sdesc(bsm + j * 32, 16, 1024), id,
                 j > 0 ? 1u : 0u);
      mma_commit(&tfull[t & 1]);
    }
    if (t + 1 < T && stager) load_k(t + 1);
    if (t >= 1) epilogue(t - 1);
  }
  if (T > 0) epilogue(T - 1);
  }
  if (!WRITE) {   // merge the two column halves of each row, in fixed order
    if (half) {
      xch[rl] = m;
      xch[BM + rl] = l;
    }
    __syncthreads();
    if (!half && row < L) {
      const float m1 = xch[rl], l1 = xch[BM + rl], mm = fmaxf(m, m1);
      const float lm = (m == -INFINITY ? 0.f : l * ex2((m - mm) * kLog2e)) +
                       (m1 == -INFINITY ? 0.f : l1 * ex2((m1 - mm) * kLog2e));
      p.pm[((int64_t)b * p.js + jr) * L + row] = mm;
      p.pl[((int64_t)b * p.js + jr) * L + row] = lm;
    }
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * AT_N));
  }
}

int attn_js(int nb, int L) {
  const int rb = (L + BM - 1) / BM, tiles = (L + AT_N - 1) / AT_N;
  const int64_t ctas = (int64_t)rb * nb;
  // two CTAs fit per SM: at most two whole waves (rounding the range count up
  // had left a 0.27-full third wave, ncu: 2.27 waves per SM)
  int js = (int)std::min<int64_t>(std::min(tiles, AT_JS), std::max<int64_t>(1, (4 * 148) / ctas));
  return std::max(1, js);
}
}  // namespace

int splits_of(const Gemm& g) {
  int s, k;
  plan_split(g, s, k);
  return s;
}

size_t ws_bytes(const Gemm& g) {
  const int s = splits_of(g);
  return s > 1 ? (size_t)s * g.batch * g.M * g.N * 4 : 0;
}

Status gemm(OpArgs& a, const Gemm& g, void* ws, size_t ws_size) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return Status::ok();
  if ((g.a_m != 1 && g.a_k != 1) || (g.b_k != 1 && g.b_n != 1))
    return Status::make(OC_E_UNSUPPORTED, "gemm_tc: an operand without a unit stride");
  if (g.ep_p && !g.c_f32) return Status::make(OC_E_UNSUPPORTED, "gemm_tc: fused epilogue needs fp32 C");
  KP p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.batch = g.batch;
  plan_split(g, p.splits, p.kps);
  if ((int64_t)p.batch * p.splits > 65535) return Status::make(OC_E_UNSUPPORTED, "gemm_tc: batch × splits > 65535");
  p.ns = std::min(NS, p.kps);
  p.A = g.A;
  p.a_m = g.a_m;
  p.a_k = g.a_k;
  p.a_b = g.a_b;
  p.a_mn = g.a_k != 1;   // contiguous along M (MN-major) unless K is the unit stride
  const int ev = g.a_f32 ? 4 : 8;
  p.a_vec = aligned(g.A, 16) && (p.a_mn ? g.a_k : g.a_m) % ev == 0 && g.a_b % ev == 0;
  p.B = g.B;
  p.b_k = g.b_k;
  p.b_n = g.b_n;
  p.b_b = g.b_b;
  p.b_mn = g.b_k != 1;
  p.b_vec = aligned(g.B, 16) && (p.b_mn ? g.b_k : g.b_n) % 8 == 0 && g.b_b % 8 == 0;
  p.C = g.C;
  p.ldc = g.ldc;
  p.c_b = g.c_b;
  const int ec = g.c_f32 ? 4 : 8;
  p.c_vec = aligned(g.C, 16) && g.ldc % ec == 0 && g.c_b % ec == 0;
  p.ep_p = (const uint16_t*)g.ep_p;
  p.ldp = g.ldp;
  p.p_b = g.p_b;
  p.ep_rs = g.ep_rs;
  p.rs_b = g.rs_b;
  p.ep_vec = g.ep_p && aligned(g.ep_p, 8) && g.ldp % 4 == 0 && g.p_b % 4 == 0;
  p.bias = g.bias;
  p.relu = g.relu ? 1 : 0;
  if (g.b_f32) p.b_vec = aligned(g.B, 16) && (p.b_mn ? g.b_k : g.b_n) % 4 == 0 && g.b_b % 4 == 0;
  if (p.splits > 1) {
    const size_t need = (size_t)p.splits * g.batch * g.M * g.N * 4;
    if (!ws || ws_size < need) return Status::make(OC_E_INVARIANT, "gemm_tc: split workspace");
    if (!aligned(ws, 16)) return Status::make(OC_E_INVARIANT, "gemm_tc: workspace alignment");
    p.part = (float*)ws;
  }
  const int BN = bn_of(g);
  Status st = Status::make(OC_E_UNSUPPORTED, "gemm_tc: no instantiation");
#define OC_TCG(bn, af, cf) \
  if (BN == bn && g.a_f32 == af && g.c_f32 == cf && !g.b_f32) st = launch<bn, af, cf>(a, p);
  OC_TCG(64, false, false)
  OC_TCG(128, false, false)
  OC_TCG(256, false, false)
  OC_TCG(64, false, true)
  OC_TCG(128, false, true)
  OC_TCG(256, false, true)
  OC_TCG(64, true, false)
  OC_TCG(128, true, false)
  OC_TCG(256, true, false)
  OC_TCG(128, true, true)
#undef OC_TCG
  // dense layers: fp32 master weights rounded to bf16 as they are staged
  if (g.b_f32 && !g.a_f32 && g.c_f32) st = launch<128, false, true, true>(a, p);
  if (g.b_f32 && !g.a_f32 && !g.c_f32) st = launch<128, false, false, true>(a, p);
  if (g.b_f32 && g.a_f32 && !g.c_f32) st = launch<128, true, false, true>(a, p);
  OC_TRY(st);
  if (p.splits > 1) {
    const int64_t n = (int64_t)g.batch * g.M * g.N;
    if (g.c_f32)
      split_reduce_k<float><<<grid_for(n, 256, 4), 256, 0, a.stream>>>(n, g.M, g.N, p.splits, p.part, (float*)g.C,
                                                                        g.ldc, g.c_b);
    else
      split_reduce_k<__nv_bfloat16><<<grid_for(n, 256, 4), 256, 0, a.stream>>>(n, g.M, g.N, p.splits, p.part,
                                                                                (__nv_bfloat16*)g.C, g.ldc, g.c_b);
    OC_LAUNCH_CHECK(a);
  }
  return Status::ok();
}

}  // namespace tcg
}  // namespace oc

namespace oc {
namespace tcg {

size_t attn_softmax_ws(int nb, int L) { return (size_t)2 * nb * attn_js(nb, L) * L * 4; }

Status attn_softmax(OpArgs& a, const __nv_bfloat16* q, const __nv_bfloat16* k, __nv_bfloat16* P, int nb, int L,
                    int dq, void* ws, size_t ws_size) {
  if (nb <= 0 || L <= 0) return Status::ok();
  if (dq > BK) return Status::make(OC_E_UNSUPPORTED, "attn_softmax: dq > 64");
  if (nb > 65535) return Status::make(OC_E_UNSUPPORTED, "attn_softmax: batch > 65535");
  if (!ws || ws_size < attn_softmax_ws(nb, L)) return Status::make(OC_E_INVARIANT, "attn_softmax: workspace");
  AP p{};
  p.L = L;
  p.dq = dq;
  p.js = attn_js(nb, L);
  p.jper = ((L + AT_N - 1) / AT_N + p.js - 1) / p.js * AT_N;
  p.q = (const uint16_t*)q;
  p.k = (const uint16_t*)k;
  p.sb = (int64_t)L * dq;
  p.P = (uint16_t*)P;
  p.pm = (float*)ws;
  p.pl = p.pm + (size_t)nb * p.js * L;
  p.vec = aligned(q, 16) && aligned(k, 16) && aligned(P, 16) && dq % 8 == 0 && L % 8 == 0;
  p.async_k = aligned(k, 8) && dq % 4 == 0;
  constexpr int SMEM0 = BM * BK * 2 + AT_KS * AT_N * BK * 2 + 1024 + 64 + 2 * BM * 4;
  constexpr int SMEM1 = SMEM0 + 2 * BM * AT_N * 2;
  static bool attr = false;
  if (!attr) {
    OC_CUDA(cudaFuncSetAttribute(attn_p_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM0));
    OC_CUDA(cudaFuncSetAttribute(attn_p_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM1));
    attr = true;
  }
  dim3 grid(p.js, (L + BM - 1) / BM, nb);
  attn_p_kernel<false><<<grid, AT_NT, SMEM0, a.stream>>>(p);
  OC_LAUNCH_CHECK(a);
  attn_p_kernel<true><<<grid, AT_NT, SMEM1, a.stream>>>(p);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

}  // namespace tcg
}  // namespace oc
