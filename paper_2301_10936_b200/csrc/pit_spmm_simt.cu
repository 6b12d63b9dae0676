// PIT sparse matmul on the CUDA cores (FFMA / DFMA): the fp32 and f64 parity path
// (north_star: fp32 within 1e-5 with TF32 disabled) and the fallback for micro-tiles the
// tensor-core kernels do not tile (odd widths, unaligned pitches).
//
// Same plan semantics as pit_spmm_tc.cu:
//   pit:k  (executor.py:386-423)  CTA = (group g, 64-row chunk of the group, 64-column tile);
//          K runs over the group's live coordinates in stored order.
//   pit:m  (executor.py:352-383)  CTA = (64 union rows, 64 columns); K runs ascending, an
//          (row, K-block) pair that is not live contributes 0.
//   dense  (executor.py:426-461)  union rows = all rows.
// Accumulation is fp32 (f64 for f64 operands) in ascending stored order.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "pit_internal.h"

#include <cstdlib>

namespace pit {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, TPB = 256;

int getenv_int(const char* name, int dflt) {  // A/B knobs (PIT_SIMT_GK=0: the generic K7 kernel)
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <typename T>
__device__ __forceinline__ float to_acc(T v);
template <>
__device__ __forceinline__ float to_acc<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_acc<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_acc<__half>(__half v) { return __half2float(v); }

template <typename T, typename Acc>
__device__ __forceinline__ Acc load_as(const T* p) {
  return static_cast<Acc>(to_acc<T>(*p));
}
template <>
__device__ __forceinline__ double load_as<double, double>(const double* p) {
  return *p;
}

template <typename T, typename Acc>
__device__ __forceinline__ T from_acc(Acc v);
template <>
__device__ __forceinline__ float from_acc<float, float>(float v) { return v; }
template <>
__device__ __forceinline__ double from_acc<double, double>(double v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16, float>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ __half from_acc<__half, float>(float v) { return __float2half_rn(v); }

template <typename T, typename Acc>
__global__ void __launch_bounds__(TPB) spmm_simt_kernel(SpmmArgs a) {
  __shared__ Acc As[BK][BM + 1];
  __shared__ Acc Bs[BK][BN + 1];
  __shared__ int32_t rowmap[BM];
  __shared__ int32_t kmap[BK];

  const T* A = static_cast<const T*>(a.A);
  const T* B = static_cast<const T*>(a.B);
  T* C = static_cast<T*>(a.C);
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;

  // ---- rows of this tile
  int64_t g = 0, k_count = a.K;
  const int32_t* klist = nullptr;
  if (a.plan == kPlanPitK) {
    const int64_t chunks = (a.t0 + BM - 1) / BM;
    g = blockIdx.y / chunks;
    const int64_t rc = blockIdx.y % chunks;
    if (tid < BM) {
      const int64_t lr = rc * BM + tid;  // row within the group
      const int64_t m = g * a.t0 + lr;
      rowmap[tid] = (lr < a.t0 && m < a.M) ? static_cast<int32_t>(m) : -1;
    }
    k_count = a.counts[g];
    klist = a.slots + g * a.slot_stride;
  } else {
    const int n_rows = a.plan == kPlanDense ? static_cast<int>(a.M) : *a.n_rows;
    if (tid < BM) {
      const int64_t i = static_cast<int64_t>(blockIdx.y) * BM + tid;
      rowmap[tid] = i < n_rows ? (a.plan == kPlanDense ? static_cast<int32_t>(i) : a.rows[i]) : -1;
    }
  }
  __syncthreads();

  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = Acc(0);

  for (int64_t kb = 0; kb < k_count; kb += BK) {
    if (tid < BK) {
      const int64_t kk = kb + tid;
      kmap[tid] = kk < k_count ? (klist ? klist[kk] : static_cast<int32_t>(kk)) : -1;
    }
    __syncthreads();
    // A tile: BM x BK
    for (int e = tid; e < BM * BK; e += TPB) {
      int r, kk;
      if (a.sak == 1) {
        kk = e % BK;
        r = e / BK;
      } else {
        r = e % BM;
        kk = e / BM;
      }
      const int32_t m = rowmap[r];
      const int32_t k = kmap[kk];
      Acc v = Acc(0);
      if (m >= 0 && k >= 0) {
        bool live = true;
        if (a.plan == kPlanPitM) {
          const int64_t grp = k / a.t1;
          live = (a.occ[grp * a.WG + (m >> 5)] >> (m & 31)) & 1u;
        }
        if (live) v = load_as<T, Acc>(A + m * a.sam + static_cast<int64_t>(k) * a.sak);
      }
      As[kk][r] = v;
    }
    // B tile: BK x BN
    for (int e = tid; e < BK * BN; e += TPB) {
      const int c = e % BN, kk = e / BN;
      const int32_t k = kmap[kk];
      const int64_t n = n0 + c;
      Bs[kk][c] = (k >= 0 && n < a.N) ? load_as<T, Acc>(B + static_cast<int64_t>(k) * a.ldb + n) : Acc(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      Acc av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int32_t m = rowmap[ty * 4 + i];
    if (m < 0) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n < a.N) C[m * a.ldc + n] = from_acc<T, Acc>(acc[i][j]);
    }
  }
}

// ------------------------------------------------------------------ SRead / SWrite
// Tile buffer is row-major [TR, TC]; the tensor is logical [R, C] with element strides (st0, st1).
// d is the logical axis the gather runs along. Slot s, micro offset i covers tensor
// index coord*t_d + i along d and off_o + jo along the other axis (executor.py:170-264).
template <typename T>
__global__ void sread_kernel(GatherArgs a, int zero_fill) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= a.TR * a.TC) return;
  const int64_t tr = e / a.TC, tc = e % a.TC;
  const int64_t td = a.d == 0 ? tr : tc;  // index along the gather axis in the tile
  const int64_t to = a.d == 0 ? tc : tr;
  const int64_t s = td / a.t_d, i = td % a.t_d;
  const int64_t ext_d = a.d == 0 ? a.R : a.C;
  const int64_t ext_o = a.d == 0 ? a.C : a.R;
  T* tile = static_cast<T*>(a.tile);
  const T* src = static_cast<const T*>(a.src_or_dst);
  bool copied = false;
  if (s < a.n_coords && to < a.t_o) {
    const int64_t gd = static_cast<int64_t>(a.coords[s]) * a.t_d + i;
    const int64_t go = a.off_o + to;
    if (gd < ext_d && go < ext_o) {
      const int64_t r = a.d == 0 ? gd : go, c = a.d == 0 ? go : gd;
  const int64_t off = r * a.st0 + c * a.st1;
      tile[e] = src[off];
      copied = true;
    }
  }
  if (!copied && zero_fill) tile[e] = T(0);
}

template <typename T>
__global__ void swrite_kernel(GatherArgs a) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= a.TR * a.TC) return;
  const int64_t tr = e / a.TC, tc = e % a.TC;
  const int64_t td = a.d == 0 ? tr : tc;
  const int64_t to = a.d == 0 ? tc : tr;
  const int64_t s = td / a.t_d, i = td % a.t_d;
  const int64_t ext_d = a.d == 0 ? a.R : a.C;
  const int64_t ext_o = a.d == 0 ? a.C : a.R;
  if (s >= a.n_coords || to >= a.t_o) return;
  const int64_t gd = static_cast<int64_t>(a.coords[s]) * a.t_d + i;
  const int64_t go = a.off_o + to;
  if (gd >= ext_d || go >= ext_o) return;
  const int64_t r = a.d == 0 ? gd : go, c = a.d == 0 ? go : gd;
  const int64_t off = r * a.st0 + c * a.st1;
  T* dst = static_cast<T*>(a.src_or_dst);
  const T* tile = static_cast<const T*>(a.tile);
  if (a.accumulate)
    dst[off] = from_acc<T, float>(load_as<T, float>(dst + off) + load_as<T, float>(tile + e));
  else
    dst[off] = tile[e];
}

template <>
__global__ void swrite_kernel<double>(GatherArgs a) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= a.TR * a.TC) return;
  const int64_t tr = e / a.TC, tc = e % a.TC;
  const int64_t td = a.d == 0 ? tr : tc;
  const int64_t to = a.d == 0 ? tc : tr;
  const int64_t s = td / a.t_d, i = td % a.t_d;
  const int64_t ext_d = a.d == 0 ? a.R : a.C;
  const int64_t ext_o = a.d == 0 ? a.C : a.R;
  if (s >= a.n_coords || to >= a.t_o) return;
  const int64_t gd = static_cast<int64_t>(a.coords[s]) * a.t_d + i;
  const int64_t go = a.off_o + to;
  if (gd >= ext_d || go >= ext_o) return;
  const int64_t r = a.d == 0 ? gd : go, c = a.d == 0 ? go : gd;
  const int64_t off = r * a.st0 + c * a.st1;
  double* dst = static_cast<double*>(a.src_or_dst);
  const double* tile = static_cast<const double*>(a.tile);
  dst[off] = a.accumulate ? dst[off] + tile[e] : tile[e];
}

// f64 oracle: multiply then add (no FMA contraction), reduction ascending -- the exact operation
// sequence of the reference's scalar triple loop (executor.py:267-283, test_executor.py:68-71).
__global__ void dense_ref_f64_kernel(const double* __restrict__ A, int64_t s0, int64_t s1,
                                     const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t M,
                                     int64_t N, int64_t K) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t i = e / N, j = e % N;
  double acc = 0.0;
  for (int64_t k = 0; k < K; ++k) acc = __dadd_rn(acc, __dmul_rn(A[i * s0 + k * s1], B[k * ldb + j]));
  C[e] = acc;
}

// Row reduction over live micro-tiles (executor.py:540-613): one warp per row,
// C[r] = sum of A[r, l] over l whose micro-tile is live; dead elements are selected out (never
// multiplied), so NaN in a dead position cannot leak and rows with no survivor are exactly 0.
//   mode 0: dense; mode 1 (pit:l): groups = rows, occ[r][l/32] bit l%32 (micro (1,1));
//   mode 2 (pit:p): groups = l-blocks of block_l, occ[l/block_l][r/32] bit r%32.
template <typename T, typename Acc>
__global__ void reduce_rows_kernel(const T* __restrict__ A, int64_t P, int64_t L, int64_t lda,
                                   const uint32_t* __restrict__ occ, int64_t WG, int mode, int block_l,
                                   T* __restrict__ out) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= P) return;
  const T* row = A + r * lda;
  Acc acc = Acc(0);
  for (int64_t l = lane; l < L; l += 32) {
    bool live = true;
    if (mode == 1) live = (__ldg(occ + r * WG + (l >> 5)) >> (l & 31)) & 1u;
    if (mode == 2) live = (__ldg(occ + (l / block_l) * WG + (r >> 5)) >> (r & 31)) & 1u;
    if (live) acc += load_as<T, Acc>(row + l);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[r] = from_acc<T, Acc>(acc);
}

// ---------------------------------------------------------------- pit:k fp32, pipelined (K7b)
// The reference's own configuration (C1: 1024^3 fp32, 32x1 micro-tiles) on the CUDA cores with TF32
// never used: CTA = (group g, 32-row chunk of it, 128-column tile); per stage 32 live k of the
// group (stored order): the A^T strips (32 rows, 128 contiguous bytes of column-major A) and the 32
// B rows (512 bytes each) by 16-byte cp.async into a 3-stage ring, then 16 FFMA per thread per k
// (4 rows x 4 columns, float4 shared loads: A broadcast within the warp, B conflict-free). The
// accumulation order per output is the stored k order, exactly as in spmm_simt_kernel (bitwise the
// same results).
constexpr int kGkBM = 32, kGkBN = 128, kGkBK = 32, kGkStages = 3, kGkThreads = 256;

__device__ __forceinline__ void cp16(void* smem, const void* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

__global__ void __launch_bounds__(kGkThreads) gk_simt_f32_kernel(SpmmArgs a) {
  extern __shared__ float4 gk_smem[];
  float* As = reinterpret_cast<float*>(gk_smem);           // [stages][BK][BM]
  float* Bs = As + kGkStages * kGkBK * kGkBM;               // [stages][BK][BN]
  const float* A = static_cast<const float*>(a.A);
  const float* B = static_cast<const float*>(a.B);
  float* C = static_cast<float*>(a.C);
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * kGkBN;
  const int64_t chunks = (a.t0 + kGkBM - 1) / kGkBM;
  const int64_t g = blockIdx.y / chunks;
  const int64_t lr0 = (blockIdx.y % chunks) * kGkBM;  // first row of the chunk within the group
  const int64_t m0 = g * a.t0 + lr0;
  const int rows = static_cast<int>(min(static_cast<int64_t>(kGkBM), min(static_cast<int64_t>(a.t0) - lr0, a.M - m0)));
  const int count = a.counts[g];
  const int32_t* klist = a.slots + g * a.slot_stride;
  const int nsteps = (count + kGkBK - 1) / kGkBK;

  auto load_stage = [&](int step, int buf) {
    const int kb = step * kGkBK;
    {  // A: 32 k x 8 chunks (rows 4 at a time)
      const int kk = tid >> 3, part = tid & 7;
      const bool ok = kb + kk < count && part * 4 < rows;
      const int k = ok ? __ldg(klist + kb + kk) : 0;
      cp16(As + (buf * kGkBK + kk) * kGkBM + part * 4, A + (ok ? m0 + part * 4 + static_cast<int64_t>(k) * a.sak : 0), ok);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // B: 32 k x 32 chunks
      const int c = tid + i * kGkThreads;
      const int kk = c >> 5, part = c & 31;
      const bool ok = kb + kk < count && n0 + part * 4 < a.N;
      const int k = ok ? __ldg(klist + kb + kk) : 0;
      cp16(Bs + (buf * kGkBK + kk) * kGkBN + part * 4, B + (ok ? static_cast<int64_t>(k) * a.ldb + n0 + part * 4 : 0), ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

#pragma unroll
  for (int st = 0; st < kGkStages - 1; ++st) {
    if (st < nsteps) load_stage(st, st);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int step = 0; step < nsteps; ++step) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kGkStages - 2) : "memory");
    __syncthreads();  // stage `step` landed for every thread; the buffer refilled below is free
    const int nxt = step + kGkStages - 1;
    if (nxt < nsteps) load_stage(nxt, nxt % kGkStages);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const int buf = step % kGkStages;
    const float* as = As + buf * kGkBK * kGkBM + ty * 4;
    const float* bs = Bs + buf * kGkBK * kGkBN + tx * 4;
    const int kn = min(kGkBK, count - step * kGkBK);
    for (int kk = 0; kk < kn; ++kk) {
      const float4 av = *reinterpret_cast<const float4*>(as + kk * kGkBM);
      const float4 bv = *reinterpret_cast<const float4*>(bs + kk * kGkBN);
      const float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
  }
  const int64_t n = n0 + tx * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    if (r >= rows || n >= a.N) continue;
    float* dst = C + (m0 + r) * a.ldc + n;
    if (n + 4 <= a.N) *reinterpret_cast<float4*>(dst) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    else for (int j = 0; j < 4 && n + j < a.N; ++j) dst[j] = acc[i][j];
  }
}

bool gk_simt_f32_ok(const SpmmArgs& a) {
  // whole 16-byte row quads only (M, t0 multiples of 4: a strip load never reads past A)
  return a.plan == kPlanPitK && a.dtype == kDtypeF32 && a.batch <= 1 && a.sam == 1 && (a.sak % 4) == 0 &&
         (a.M % 4) == 0 &&
         (a.ldb % 4) == 0 && (a.ldc % 4) == 0 && (a.N % 4) == 0 && (a.t0 % 4) == 0 &&
         (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(a.B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && getenv_int("PIT_SIMT_GK", 1) != 0;
}

int run_gk_simt_f32(const SpmmArgs& a, cudaStream_t s) {
  const int64_t ytiles = a.n_groups * ceil_div(a.t0, kGkBM);
  const int64_t xtiles = ceil_div(a.N, kGkBN);
  if (ytiles == 0 || xtiles == 0) return kOk;
  if (ytiles > 65535 || xtiles > (1ll << 31) - 1) return kErrShape;
  constexpr int smem = kGkStages * kGkBK * (kGkBM + kGkBN) * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gk_simt_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  gk_simt_f32_kernel<<<dim3(static_cast<unsigned>(xtiles), static_cast<unsigned>(ytiles)), kGkThreads, smem, s>>>(a);
  note_launch();
  return cuda_status();
}

template <typename T, typename Acc>
int run_simt(const SpmmArgs& a, cudaStream_t s) {
  int64_t ytiles;
  if (a.plan == kPlanPitK) {
    ytiles = a.n_groups * ceil_div(a.t0, BM);
  } else {
    if (a.plan == kPlanPitM) {
      if (cudaMemset2DAsync(a.C, a.ldc * sizeof(T), 0, a.N * sizeof(T), a.M, s) != cudaSuccess) return cuda_status();
    }
    ytiles = ceil_div(a.plan == kPlanDense ? a.M : a.n_rows_host, BM);
  }
  const int64_t xtiles = ceil_div(a.N, BN);
  if (ytiles == 0 || xtiles == 0) return kOk;
  if (ytiles > 65535 || xtiles > (1ll << 31) - 1) return kErrShape;
  spmm_simt_kernel<T, Acc><<<dim3(static_cast<unsigned>(xtiles), static_cast<unsigned>(ytiles)), TPB, 0, s>>>(a);
  note_launch();
  return cuda_status();
}

}  // namespace

int launch_spmm_simt(const SpmmArgs& a, cudaStream_t s) {
  switch (a.dtype) {
    case kDtypeF32:
      return gk_simt_f32_ok(a) ? run_gk_simt_f32(a, s) : run_simt<float, float>(a, s);
    case kDtypeF64:
      return run_simt<double, double>(a, s);
    case kDtypeBF16:
      return run_simt<__nv_bfloat16, float>(a, s);
    case kDtypeF16:
      return run_simt<__half, float>(a, s);
    default:
      return kErrUnsupported;
  }
}

int launch_reduce_rows(const void* A, int dtype, int64_t P, int64_t L, int64_t lda, const uint32_t* occ, int64_t WG,
                       int mode, int block_l, void* out, cudaStream_t s) {
  if (P == 0) return kOk;
  const unsigned grid = static_cast<unsigned>(ceil_div(P * 32, 256));
  switch (dtype) {
    case kDtypeF32:
      reduce_rows_kernel<float, float><<<grid, 256, 0, s>>>(static_cast<const float*>(A), P, L, lda, occ, WG, mode,
                                                            block_l, static_cast<float*>(out));
      break;
    case kDtypeF64:
      reduce_rows_kernel<double, double><<<grid, 256, 0, s>>>(static_cast<const double*>(A), P, L, lda, occ, WG, mode,
                                                              block_l, static_cast<double*>(out));
      break;
    case kDtypeBF16:
      reduce_rows_kernel<__nv_bfloat16, float><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(A), P, L, lda,
                                                                    occ, WG, mode, block_l,
                                                                    static_cast<__nv_bfloat16*>(out));
      break;
    case kDtypeF16:
      reduce_rows_kernel<__half, float><<<grid, 256, 0, s>>>(static_cast<const __half*>(A), P, L, lda, occ, WG, mode,
                                                             block_l, static_cast<__half*>(out));
      break;
    default:
      return kErrUnsupported;
  }
  note_launch();
  return cuda_status();
}

int launch_dense_ref_f64(const double* A, int64_t s0, int64_t s1, const double* B, int64_t ldb, double* C, int64_t M,
                         int64_t N, int64_t K, cudaStream_t s) {
  if (M * N == 0) return kOk;
  dense_ref_f64_kernel<<<static_cast<unsigned>(ceil_div(M * N, 256)), 256, 0, s>>>(A, s0, s1, B, ldb, C, M, N, K);
  note_launch();
  return cuda_status();
}

int launch_sread(const GatherArgs& a, cudaStream_t s) {
  const int64_t n = a.TR * a.TC;
  if (n == 0) return kOk;
  const int zero_fill = a.zero_fill;
  const unsigned grid = static_cast<unsigned>(ceil_div(n, 256));
  switch (a.dtype) {
    case kDtypeF32:
      sread_kernel<float><<<grid, 256, 0, s>>>(a, zero_fill);
      note_launch();
      break;
    case kDtypeF64:
      sread_kernel<double><<<grid, 256, 0, s>>>(a, zero_fill);
      note_launch();
      break;
    case kDtypeBF16:
      sread_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(a, zero_fill);
      note_launch();
      break;
    case kDtypeF16:
      sread_kernel<__half><<<grid, 256, 0, s>>>(a, zero_fill);
      note_launch();
      break;
    default:
      return kErrUnsupported;
  }
  return cuda_status();
}

int launch_swrite(const GatherArgs& a, cudaStream_t s) {
  const int64_t n = a.TR * a.TC;
  if (n == 0) return kOk;
  const unsigned grid = static_cast<unsigned>(ceil_div(n, 256));
  switch (a.dtype) {
    case kDtypeF32:
      swrite_kernel<float><<<grid, 256, 0, s>>>(a);
      note_launch();
      break;
    case kDtypeF64:
      swrite_kernel<double><<<grid, 256, 0, s>>>(a);
      note_launch();
      break;
    case kDtypeBF16:
      swrite_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(a);
      note_launch();
      break;
    case kDtypeF16:
      swrite_kernel<__half><<<grid, 256, 0, s>>>(a);
      note_launch();
      break;
    default:
      return kErrUnsupported;
  }
  return cuda_status();
}

}  // namespace pit
