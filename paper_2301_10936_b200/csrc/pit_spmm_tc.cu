// PIT sparse matmul on the 5th-gen tensor cores (tcgen05 + TMEM + TMA gather4), bf16/fp16 in,
// fp32 accumulate, bf16/fp16 out.
//
// Two persistent, warp-specialised kernels (warp 0 = TMA producer, warp 1 = MMA issuer,
// warp 2 = TMEM allocator, warps 4..7 = epilogue):
//
//  * spmm_gk ("gathered K", PIT axis k; reference executor.py:386-423 `_matmul_pit_k`).
//    A group is an M-block of GW rows (micro-tile (GW,1)); its live k coordinates index rows of
//    A^T (A is column-major, executor.py:318-325) and rows of B. Both operands are fetched with
//    TMA tile::gather4 (four k rows per instruction) into MN-major swizzled shared memory and fed
//    to tcgen05.mma in the transposed orientation D[n, m] += B^T[n, k] * A^T[k, m]:
//    M_mma = 128 output columns (n), N_mma = GW output rows (m). That keeps the group width as
//    the MMA's N, so 16..256-row micro-tiles all run as dense MMAs with no union waste.
//    Each (group, n-tile) C block is owned by exactly one CTA and accumulated in TMEM.
//
//  * spmm_gm ("gathered M", PIT axis m and the dense plan; executor.py:352-383 / :426-461).
//    Output row tiles are 128 rows of the union of live rows (rows named by any K-block group).
//    Per K-block stage the producer gathers those rows of A with gather4; a row that is not live
//    in that K-block is pointed out of bounds, so TMA fills it with zeros. B K-blocks are plain 2-D
//    TMA tiles. The C tile stays resident in TMEM across all K-blocks and is scattered to its rows
//    once (SWrite fused in the epilogue). Rows outside the union are never written (C is zeroed
//    up front), which keeps the reference's exact-zero guarantee (executor.py:8-9).
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "pit_internal.h"
#include "pit_ptx.cuh"

namespace pit {

namespace {

constexpr int kThreads = 256;  // 8 warps
constexpr int kEpiWarp0 = 4;

template <bool kBF16>
struct OutT;
template <>
struct OutT<true> {
  using T = __nv_bfloat16;
  __device__ static T cvt(float x) { return __float2bfloat16_rn(x); }
};
template <>
struct OutT<false> {
  using T = __half;
  __device__ static T cvt(float x) { return __float2half_rn(x); }
};

__device__ __forceinline__ uint32_t pack2(float a, float b, bool bf16) {
  if (bf16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int N>
__host__ __device__ constexpr uint32_t tmem_cols_pow2() {
  return N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
}

// =============================================================================================
// spmm_gk: PIT axis k.
// =============================================================================================
template <int GW, int NACC>
struct GkCfg {
  static constexpr int KS = 64;                                   // gathered k per stage
  static constexpr int A_ROW_BYTES = GW * 2 < 128 ? GW * 2 : 128; // bytes per smem row of A^T strip
  static constexpr int A_ATOMS = GW * 2 <= 128 ? 1 : GW * 2 / 128;
  static constexpr int B_BYTES = NACC * 2 * KS * 128;             // NACC halves x 2 atoms x KS rows
  static constexpr int A_BYTES = A_ATOMS * KS * A_ROW_BYTES;
  static constexpr int STAGE_BYTES = ((B_BYTES + A_BYTES + 1023) / 1024) * 1024;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = tmem_cols_pow2<2 * NACC * GW>();
  static constexpr int N_TILE = 128 * NACC;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t A_SW = sw_layout_for_row(A_ROW_BYTES);
};

template <int GW, int NACC, bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
    spmm_gk_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmAt,
                   const int32_t* __restrict__ counts, const int32_t* __restrict__ slots, int64_t slot_stride,
                   int n_groups, int n_tiles, int M, int N, int K, void* __restrict__ Cv, int64_t ldc) {
  using Cfg = GkCfg<GW, NACC>;
  using OT = OutT<kBF16>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmAt);
  }
  if (warp == 2) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int units = n_groups * n_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int g = u / n_tiles;
      const int n0 = (u % n_tiles) * Cfg::N_TILE;
      const int m0 = g * GW;
      const int cnt = counts[g];
      const int32_t* gs = slots + static_cast<int64_t>(g) * slot_stride;
      for (int kb = 0; kb < cnt; kb += Cfg::KS) {
        const int kvalid = min(Cfg::KS, cnt - kb);
        const int kpad = (kvalid + 15) & ~15;
        // lane l holds coordinates kb+l and kb+32+l (K => out of range => zero-filled rows)
        const int c0 = (lane < kvalid) ? gs[kb + lane] : K;
        const int c1 = (32 + lane < kvalid) ? gs[kb + 32 + lane] : K;
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sB = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sA = sB + Cfg::B_BYTES;
        if (lane == 0) mbar_expect_tx(&full_bar[stage], kpad * (NACC * 256 + GW * 2));
        for (int q = 0; q < kpad / 4; ++q) {
          const int src = (4 * q) & 31;
          const bool hi = 4 * q >= 32;
          const int r0 = __shfl_sync(0xffffffffu, hi ? c1 : c0, src + 0);
          const int r1 = __shfl_sync(0xffffffffu, hi ? c1 : c0, src + 1);
          const int r2 = __shfl_sync(0xffffffffu, hi ? c1 : c0, src + 2);
          const int r3 = __shfl_sync(0xffffffffu, hi ? c1 : c0, src + 3);
          if (lane == 0) {
#pragma unroll
            for (int a = 0; a < 2 * NACC; ++a)
              tma_gather4(sB + a * Cfg::KS * 128 + q * 512, &tmB, &full_bar[stage], n0 + a * 64, r0, r1, r2, r3);
#pragma unroll
            for (int a = 0; a < Cfg::A_ATOMS; ++a)
              tma_gather4(sA + a * Cfg::KS * Cfg::A_ROW_BYTES + q * 4 * Cfg::A_ROW_BYTES, &tmAt, &full_bar[stage],
                          m0 + a * 64, r0, r1, r2, r3);
          }
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_f16(128, GW, kBF16, true, true);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int g = u / n_tiles;
      const int cnt = counts[g];
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < cnt; kb += Cfg::KS) {
        const int kvalid = min(Cfg::KS, cnt - kb);
        const int ksteps = (kvalid + 15) >> 4;
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sB = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sA = sB + Cfg::B_BYTES;
          for (int ks = 0; ks < ksteps; ++ks) {
            const uint64_t bdesc = smem_desc(sA + ks * 16 * Cfg::A_ROW_BYTES, Cfg::KS * Cfg::A_ROW_BYTES,
                                             8 * Cfg::A_ROW_BYTES, Cfg::A_SW);
#pragma unroll
            for (int a = 0; a < NACC; ++a) {
              const uint64_t adesc = smem_desc(sB + a * 2 * Cfg::KS * 128 + ks * 2048, Cfg::KS * 128, 1024, kSw128);
              const uint32_t d = tmem_base + static_cast<uint32_t>((acc * NACC + a) * GW);
              umma_f16(d, adesc, bdesc, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(&tfull_bar[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue
    using T = typename OT::T;
    T* C = static_cast<T*>(Cv);
    const int q = warp & 3;  // TMEM lane quarter
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int g = u / n_tiles;
      const int n0 = (u % n_tiles) * Cfg::N_TILE;
      const int m0 = g * GW;
      const int cnt = counts[g];
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#pragma unroll
      for (int a = 0; a < NACC; ++a) {
        const int n = n0 + a * 128 + q * 32 + lane;
#pragma unroll
        for (int c = 0; c < GW; c += 16) {
          uint32_t v[16];
          if (cnt > 0) {
            tmem_ld16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                          static_cast<uint32_t>((acc * NACC + a) * GW + c),
                      v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0u;
          }
          if (n < N) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int m = m0 + c + i;
              if (m < M) C[static_cast<int64_t>(m) * ldc + n] = OT::cvt(__uint_as_float(v[i]));
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// =============================================================================================
// spmm_gm: PIT axis m (union-row tiles) and the dense plan.
// =============================================================================================
template <int KS>
struct GmCfg {
  static constexpr int BM = 128;
  static constexpr int BN = 256;
  static constexpr int A_ROW_BYTES = KS * 2;  // K-major rows
  static constexpr int A_BYTES = BM * A_ROW_BYTES;
  static constexpr int B_BYTES = (BN / 64) * KS * 128;  // MN-major, 4 atoms of 64 n
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + 1023) / 1024) * 1024;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 512;  // 2 accumulators x 256 columns
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE_BYTES + 1024 + 512;
  static constexpr uint32_t A_SW = sw_layout_for_row(A_ROW_BYTES);
};

template <int KS, bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
    spmm_gm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const int32_t* __restrict__ rows, const int32_t* __restrict__ n_rows_dev, int dense,
                   const uint32_t* __restrict__ occ, int64_t WG, int t1, int row_tiles, int n_tiles, int M, int N,
                   int K, void* __restrict__ Cv, int64_t ldc) {
  using Cfg = GmCfg<KS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int32_t* stage_live = reinterpret_cast<int32_t*>(tmem_slot + 4);  // per stage: 1 = MMA, 0 = skipped

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_rows = dense ? M : *n_rows_dev;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 2) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int live_tiles = (n_rows + Cfg::BM - 1) / Cfg::BM;
  const int units = min(row_tiles, live_tiles) * n_tiles;
  const int kblocks = (K + KS - 1) / KS;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int rt = u / n_tiles;
      const int n0 = (u % n_tiles) * Cfg::BN;
      // lane l owns tile rows 4l..4l+3
      int rid[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = rt * Cfg::BM + 4 * lane + j;
        rid[j] = (i < n_rows) ? (dense ? i : rows[i]) : -1;
      }
      for (int kb = 0; kb < kblocks; ++kb) {
        const int k0 = kb * KS;
        const int grp = dense ? 0 : k0 / t1;
        int r[4];
        bool any = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          bool live = rid[j] >= 0;
          if (live && !dense) live = (occ[static_cast<int64_t>(grp) * WG + (rid[j] >> 5)] >> (rid[j] & 31)) & 1u;
          r[j] = live ? rid[j] : M;  // M => out of range => zero row
          any |= live;
        }
        const bool stage_any = __any_sync(0xffffffffu, any);
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sB = sA + Cfg::A_BYTES;
        if (lane == 0) stage_live[stage] = stage_any ? 1 : 0;
        if (stage_any) {
          if (lane == 0) {
            mbar_expect_tx(&full_bar[stage], Cfg::A_BYTES + Cfg::B_BYTES);
#pragma unroll
            for (int a = 0; a < Cfg::BN / 64; ++a)
              tma_load_2d(sB + a * KS * 128, &tmB, &full_bar[stage], n0 + a * 64, k0);
          }
          __syncwarp();
          // every lane issues the gather for its own four rows
          tma_gather4(sA + lane * 4 * Cfg::A_ROW_BYTES, &tmA, &full_bar[stage], k0, r[0], r[1], r[2], r[3]);
        } else if (lane == 0) {
          mbar_arrive(&full_bar[stage]);
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_f16(Cfg::BM, Cfg::BN, kBF16, false, true);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      bool first = true;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const bool live = stage_live[stage] != 0;
        if (lane == 0) {
          if (live) {
            const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sB = sA + Cfg::A_BYTES;
#pragma unroll
            for (int ks = 0; ks < KS / 16; ++ks) {
              const uint64_t adesc = smem_desc(sA + ks * 32, 16, 8 * Cfg::A_ROW_BYTES, Cfg::A_SW);
              const uint64_t bdesc = smem_desc(sB + ks * 2048, KS * 128, 1024, kSw128);
              umma_f16(tmem_base + static_cast<uint32_t>(acc * Cfg::BN), adesc, bdesc, idesc,
                       (!first || ks > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty_bar[stage]);
        }
        first = first && !live;
        __syncwarp();
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(&tfull_bar[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue: row scatter
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int rt = u / n_tiles;
      const int n0 = (u % n_tiles) * Cfg::BN;
      const int i = rt * Cfg::BM + q * 32 + lane;
      const int row = (i < n_rows) ? (dense ? i : rows[i]) : -1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      uint8_t* crow = row >= 0 ? static_cast<uint8_t*>(Cv) + (static_cast<int64_t>(row) * ldc) * 2 : nullptr;
#pragma unroll 1
      for (int c = 0; c < Cfg::BN; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN + c), v);
        tmem_wait_ld();
        if (row >= 0) {
          const int nb = n0 + c;
          if (nb + 32 <= N && (ldc % 8) == 0) {
            uint4* dst = reinterpret_cast<uint4*>(crow + static_cast<int64_t>(nb) * 2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 w;
              w.x = pack2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]), kBF16);
              w.y = pack2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]), kBF16);
              w.z = pack2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]), kBF16);
              w.w = pack2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]), kBF16);
              dst[j] = w;
            }
          } else {
            using T = typename OutT<kBF16>::T;
            T* dst = reinterpret_cast<T*>(crow);
            for (int j = 0; j < 32; ++j)
              if (nb + j < N) dst[nb + j] = OutT<kBF16>::cvt(__uint_as_float(v[j]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

CUtensorMapSwizzle swizzle_enum(int row_bytes) {
  return row_bytes >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
         : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                           : CU_TENSOR_MAP_SWIZZLE_NONE;
}

template <int GW, int NACC, bool kBF16>
int run_gk(const SpmmArgs& a, cudaStream_t s) {
  using Cfg = GkCfg<GW, NACC>;
  const CUtensorMapDataType dt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmB, tmAt;
  // B: row-major [K, N]
  if (encode_tensor_map_2d(&tmB, dt, a.B, a.N, a.K, a.ldb * 2, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  // A^T: row-major [K, M] (A column-major, pitch sak)
  const int box = GW < 64 ? GW : 64;
  if (encode_tensor_map_2d(&tmAt, dt, a.A, a.M, a.K, a.sak * 2, box, 1, swizzle_enum(box * 2)) != CUDA_SUCCESS)
    return kErrCuda;
  const int n_tiles = static_cast<int>(ceil_div(a.N, Cfg::N_TILE));
  const int64_t units = a.n_groups * n_tiles;
  if (units == 0) return kOk;
  auto kern = spmm_gk_kernel<GW, NACC, kBF16>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  kern<<<grid, kThreads, Cfg::SMEM, s>>>(tmB, tmAt, a.counts, a.slots, a.slot_stride, static_cast<int>(a.n_groups),
                                         n_tiles, static_cast<int>(a.M), static_cast<int>(a.N),
                                         static_cast<int>(a.K), a.C, a.ldc);
  return cuda_status();
}

template <int KS, bool kBF16>
int run_gm(const SpmmArgs& a, cudaStream_t s) {
  using Cfg = GmCfg<KS>;
  const CUtensorMapDataType dt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmA, tmB;
  // A: row-major [M, K], gather rows, box KS columns
  if (encode_tensor_map_2d(&tmA, dt, a.A, a.K, a.M, a.sam * 2, KS, 1, swizzle_enum(KS * 2)) != CUDA_SUCCESS)
    return kErrCuda;
  // B: row-major [K, N], tile box {64 n, KS k}
  if (encode_tensor_map_2d(&tmB, dt, a.B, a.N, a.K, a.ldb * 2, 64, KS, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  const int dense = a.plan == kPlanDense ? 1 : 0;
  if (!dense) {
    // rows named by no group stay exactly zero
    if (cudaMemset2DAsync(a.C, a.ldc * 2, 0, a.N * 2, a.M, s) != cudaSuccess) return cuda_status();
  }
  const int64_t rows_bound = dense ? a.M : a.n_rows_host;
  const int row_tiles = static_cast<int>(ceil_div(rows_bound, Cfg::BM));
  const int n_tiles = static_cast<int>(ceil_div(a.N, Cfg::BN));
  const int64_t units = static_cast<int64_t>(row_tiles) * n_tiles;
  if (units == 0) return kOk;
  auto kern = spmm_gm_kernel<KS, kBF16>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  kern<<<grid, kThreads, Cfg::SMEM, s>>>(tmA, tmB, a.rows, a.n_rows, dense, a.occ, a.WG, a.t1, row_tiles, n_tiles,
                                         static_cast<int>(a.M), static_cast<int>(a.N), static_cast<int>(a.K), a.C,
                                         a.ldc);
  return cuda_status();
}

template <bool kBF16>
int dispatch_tc(const SpmmArgs& a, cudaStream_t s) {
  if (a.plan == kPlanPitK) {
    switch (a.t0) {
      case 16:
        return run_gk<16, 2, kBF16>(a, s);
      case 32:
        return run_gk<32, 2, kBF16>(a, s);
      case 64:
        return run_gk<64, 2, kBF16>(a, s);
      case 128:
        return run_gk<128, 2, kBF16>(a, s);
      case 256:
        return run_gk<256, 1, kBF16>(a, s);
      default:
        return kErrUnsupported;
    }
  }
  const int t1 = a.plan == kPlanDense ? 64 : a.t1;
  if (t1 % 64 == 0) return run_gm<64, kBF16>(a, s);
  if (t1 == 32) return run_gm<32, kBF16>(a, s);
  if (t1 == 16) return run_gm<16, kBF16>(a, s);
  return kErrUnsupported;
}

}  // namespace

bool spmm_tc_supported(const SpmmArgs& a) {
  if (a.dtype != kDtypeBF16 && a.dtype != kDtypeF16) return false;
  // TMA: 16-byte aligned bases and pitches, int32 coordinates
  if (a.M >= (1ll << 31) || a.N >= (1ll << 31) || a.K >= (1ll << 31)) return false;
  if (reinterpret_cast<uintptr_t>(a.A) % 16 || reinterpret_cast<uintptr_t>(a.B) % 16) return false;
  if ((a.ldb * 2) % 16) return false;
  if (a.plan == kPlanPitK) {
    if (a.sam != 1 || (a.sak * 2) % 16) return false;  // A column-major
    return a.t0 == 16 || a.t0 == 32 || a.t0 == 64 || a.t0 == 128 || a.t0 == 256;
  }
  if (a.sak != 1 || (a.sam * 2) % 16) return false;  // A row-major
  if (a.plan == kPlanDense) return true;
  return a.t1 % 64 == 0 || a.t1 == 32 || a.t1 == 16;
}

int launch_spmm_tc(const SpmmArgs& a, cudaStream_t s) {
  if (!spmm_tc_supported(a)) return kErrUnsupported;
  return a.dtype == kDtypeBF16 ? dispatch_tc<true>(a, s) : dispatch_tc<false>(a, s);
}

}  // namespace pit
