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
template <int ROWS, bool F32>
struct Loader {
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
  // bf16: one tile; fp32: hi tile at `tile`, lo tile at `lo`
  __device__ __forceinline__ void store(uint32_t tile, uint32_t lo) const {
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const uint32_t off = chunk_off(mn_major, r0 + i * rstep, c);
      if constexpr (F32) {
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

template <int BN, bool AF32, bool CF32>
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
  Loader<BM, AF32> la;
  Loader<BN, false> lb;
  la.init((const typename Loader<BM, AF32>::T*)P.A + bz * P.a_b, P.a_m, P.a_k, a_mn, P.a_vec, m0, P.M, P.K);
  lb.init((const uint16_t*)P.B + bz * P.b_b, P.b_n, P.b_k, b_mn, P.b_vec, n0, P.N, P.K);
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
        for (int e = 0; e < 8; ++e) f[e] = has_k ? __uint_as_float(v[c + e]) : 0.f;
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
int bn_of(const Gemm& g) { return g.N <= 64 ? 64 : (g.N <= 128 || g.c_f32) ? 128 : 256; }

void plan_split(const Gemm& g, int& splits, int& kps) {
  const int nkb = (g.K + BK - 1) / BK;
  const int bn = bn_of(g);
  const int64_t tiles = (int64_t)((g.N + bn - 1) / bn) * ((g.M + BM - 1) / BM) * g.batch;
  const int64_t target = 2 * 148;
  splits = 1;
  if (!g.ep_p && tiles < target && nkb >= 8) {
    int64_t s = (target + tiles - 1) / tiles;
    s = std::min<int64_t>(s, nkb / 4);
    s = std::min<int64_t>(s, 65535 / std::max(1, g.batch));
    splits = (int)std::max<int64_t>(1, s);
  }
  kps = std::max(1, (nkb + splits - 1) / splits);
  splits = std::max(1, (nkb + kps - 1) / kps);
}

template <int BN, bool AF32, bool CF32>
Status launch(OpArgs& a, const KP& p) {
  constexpr int STAGE = BM * BK * 2 * (AF32 ? 2 : 1) + BN * BK * 2;
  const int smem = std::max(p.ns * STAGE, STG) + 1024 + 64;
  auto k = gemm_tc_kernel<BN, AF32, CF32>;
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
  if (g.a_f32 && g.c_f32) return Status::make(OC_E_UNSUPPORTED, "gemm_tc: fp32 A with fp32 C");
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
  if (p.splits > 1) {
    const size_t need = (size_t)p.splits * g.batch * g.M * g.N * 4;
    if (!ws || ws_size < need) return Status::make(OC_E_INVARIANT, "gemm_tc: split workspace");
    if (!aligned(ws, 16)) return Status::make(OC_E_INVARIANT, "gemm_tc: workspace alignment");
    p.part = (float*)ws;
  }
  const int BN = bn_of(g);
  Status st = Status::make(OC_E_UNSUPPORTED, "gemm_tc: no instantiation");
#define OC_TCG(bn, af, cf) \
  if (BN == bn && g.a_f32 == af && g.c_f32 == cf) st = launch<bn, af, cf>(a, p);
  OC_TCG(64, false, false)
  OC_TCG(128, false, false)
  OC_TCG(256, false, false)
  OC_TCG(64, false, true)
  OC_TCG(128, false, true)
  OC_TCG(256, false, true)
  OC_TCG(64, true, false)
  OC_TCG(128, true, false)
  OC_TCG(256, true, false)
#undef OC_TCG
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
