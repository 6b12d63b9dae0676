// K3s — pit:m products at very high micro-tile sparsity (C4: random 1x32 activation sparsity at 99%).
//
// The reference's _matmul_pit_m (executor.py:352-383) runs one dense tile per K-block group over that
// group's live rows and scatter-accumulates the result into C. With ~1% live (row, K-group) pairs,
// every 128-row tile of the masked dense kernels still holds a live row in ~all K-blocks, so they
// execute dense work. This path follows the reference's group-major order instead, on B200:
//
//   prep    a CTA per K-supergroup s (256 consecutive columns = 256/t1 K-groups): the union of its
//           groups' live rows (OR of the occupancy words), their ascending list and per-word prefix
//           counts. Every kernel of the path decides from the index counts (density <=
//           1/kSparseDen); prep also publishes the verdict in a device flag the masked dense
//           kernels read (no host round trip, CUDA-graph safe);
//   pack    SRead: row i of supergroup s -> packed row off[s] + i (256 columns, dead micro-tiles
//           written as zeros; packing one supergroup per CTA inside prep measured slower), so the
//           product reads its tokens by TMA;
//   product rowgemm2t (pit_spmm_tc.cu) with the supergroups as groups: D^T = W2_s^T . X_s^T on CTA
//           pairs, the partial sums of every (supergroup, live row) written in fp32 (no atomics);
//   reduce  a warp per output row sums its partials in ascending supergroup order (deterministic)
//           and writes C in the operand dtype; rows with no live micro-tile are exact zeros.
//
// Work: the tensor pipe executes union-row products (~8% of dense at 1% density); the traffic is
// the weights once, the packed rows, and the fp32 partials (~2.5 per output row at 1%).
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "pit_internal.h"

namespace pit {

namespace {

constexpr int kPrepThreads = 256;

int n_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

// Every kernel of the path decides for itself from the index counts (identical verdicts, no
// cross-kernel flag needed inside the path); the prep blocks also publish it for the masked kernels.
__device__ __forceinline__ bool sparse_verdict(const int32_t* __restrict__ counts, int nkg, int64_t M, int* red) {
  long long sum = 0;
  for (int g = threadIdx.x; g < nkg; g += blockDim.x) sum += __ldg(counts + g);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) reinterpret_cast<long long*>(red)[threadIdx.x >> 5] = sum;
  __syncthreads();
  long long total = 0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total += reinterpret_cast<long long*>(red)[w];
  __syncthreads();
  return total * kSparseDen <= M * static_cast<long long>(nkg);
}

// exclusive prefix of cnt[0..S) into soff[0..S] (shared), by the whole block
__device__ __forceinline__ void block_offsets(const int* __restrict__ cnt, int S, int* soff) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int running = 0;
    for (int s0 = 0; s0 < S; s0 += 32) {
      const int s = s0 + lane;
      const int c = s < S ? __ldcg(cnt + s) : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (s < S) soff[s] = running + incl - c;
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) soff[S] = running;
  }
  __syncthreads();
}

// One block per supergroup s: union words, per-word exclusive prefix, count, ascending row list.
__global__ void __launch_bounds__(kPrepThreads) gm_sparse_prep_kernel(
    const int32_t* __restrict__ counts, int nkg, int64_t M, int gps, int S, const uint32_t* __restrict__ occ,
    int64_t WG, int* __restrict__ flag, int* __restrict__ cnt, uint32_t* __restrict__ U, int* __restrict__ pre,
    int32_t* __restrict__ rows) {
  __shared__ int red[2 * kPrepThreads / 32];
  __shared__ int wsum[kPrepThreads / 32];
  const bool sparse = sparse_verdict(counts, nkg, M, red);
  const int s = blockIdx.x;
  if (s == 0 && threadIdx.x == 0) flag[0] = sparse ? 1 : 0;
  if (!sparse) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* Us = U + static_cast<int64_t>(s) * WG;
  int* pres = pre + static_cast<int64_t>(s) * WG;
  int32_t* out = rows + static_cast<int64_t>(s) * M;
  int base = 0;
  for (int64_t w0 = 0; w0 < WG; w0 += kPrepThreads) {
    const int64_t w = w0 + threadIdx.x;
    uint32_t u = 0;
    if (w < WG)
      for (int j = 0; j < gps; ++j) {
        const int64_t g = static_cast<int64_t>(s) * gps + j;
        if (g < nkg) u |= __ldg(occ + g * WG + w);
      }
    const int c = __popc(u);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int wb = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kPrepThreads / 32; ++i) {
      wb += i < warp ? wsum[i] : 0;
      tot += wsum[i];
    }
    int pos = base + wb + incl - c;
    if (w < WG) {
      Us[w] = u;
      pres[w] = pos;
      while (u) {
        const int b = __ffs(u) - 1;
        u &= u - 1;
        out[pos++] = static_cast<int32_t>(w * 32 + b);
      }
    }
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cnt[s] = base;
}

// SRead into packed rows: warp per packed row, a 16-byte chunk per lane (256 columns of 2-byte
// values); a chunk whose K-group is dead for the row is written as zeros. Packed row off[s] + i is
// row i of supergroup s (off: prefix of the counts, per block).
__global__ void __launch_bounds__(256) gm_sparse_pack_kernel(const int32_t* __restrict__ counts, int nkg,
                                                             const uint8_t* __restrict__ A, int64_t lda_bytes,
                                                             const int* __restrict__ cnt, int S,
                                                             const int32_t* __restrict__ rows, int64_t M,
                                                             const uint32_t* __restrict__ occ, int64_t WG, int lg_t1,
                                                             uint8_t* __restrict__ X, int64_t bound_rows, int sg) {
  extern __shared__ int soff[];  // [S + 1] packed offsets
  __shared__ int red[16];
  if (!sparse_verdict(counts, nkg, M, red)) return;
  block_offsets(cnt, S, soff);
  const int total = soff[S];
  const int lane = threadIdx.x & 31;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); j < total && j < bound_rows;
       j += static_cast<int64_t>(gridDim.x) * 8) {
    int lo = 0, hi = S;  // last s with soff[s] <= j
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (soff[mid] <= j) lo = mid; else hi = mid;
    }
    const int r = __ldcg(rows + lo * M + (j - soff[lo]));
    for (int c0 = 0; c0 < sg; c0 += 256) {  // 256 columns (32 lanes x 8) per pass
      const int64_t col = static_cast<int64_t>(lo) * sg + c0 + lane * 8;  // element column
      const int64_t kg = col >> lg_t1;
      const bool live = (__ldg(occ + kg * WG + (r >> 5)) >> (r & 31)) & 1u;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (live) v = __ldg(reinterpret_cast<const uint4*>(A + static_cast<int64_t>(r) * lda_bytes + col * 2));
      reinterpret_cast<uint4*>(X + j * (sg * 2) + c0 * 2)[lane] = v;
    }
  }
}

template <typename T>
__device__ __forceinline__ T cvt_out(float x);
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ __half cvt_out<__half>(float x) {
  return __float2half_rn(x);
}

// A block per 8 output rows: warp w lists row w's partial rows (the supergroups holding it, ascending:
// off[s] + rank_s(r)), then the 256 threads stream the 8 rows' partials column-wise (8 columns per
// thread, every row's loads in flight together) and write C in the operand dtype. Deterministic:
// each element is summed in ascending supergroup order. Rows with no partial are exact zeros.
constexpr int kMaxParts = 48;
constexpr int kRedRows = 8;
template <typename T>
__global__ void __launch_bounds__(256) gm_sparse_reduce_kernel(const int32_t* __restrict__ counts, int nkg,
                                                               const int* __restrict__ cnt, int S,
                                                               const uint32_t* __restrict__ U,
                                                               const int* __restrict__ pre, int64_t WG,
                                                               const float* __restrict__ part, int64_t N,
                                                               T* __restrict__ C, int64_t ldc, int64_t M) {
  extern __shared__ int soff[];  // [S + 1]
  __shared__ int red[16];
  __shared__ int64_t prow[kRedRows][kMaxParts];
  __shared__ int nparts[kRedRows];
  if (!sparse_verdict(counts, nkg, M, red)) return;
  block_offsets(cnt, S, soff);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRedRows; r0 < M; r0 += static_cast<int64_t>(gridDim.x) * kRedRows) {
    {
      const int64_t r = r0 + warp;
      int n = 0;
      if (r < M) {
        const int64_t w = r >> 5;
        const uint32_t bit = 1u << (r & 31);
        for (int s0 = 0; s0 < S; s0 += 32) {
          const int s = s0 + lane;
          const uint32_t u = s < S ? __ldcg(U + s * WG + w) : 0u;
          const uint32_t m = __ballot_sync(0xffffffffu, (u & bit) != 0u);
          if ((u & bit) != 0u) {
            const int slot = n + __popc(m & ((1u << lane) - 1u));
            if (slot < kMaxParts)
              prow[warp][slot] = (static_cast<int64_t>(soff[s]) + __ldcg(pre + s * WG + w) + __popc(u & (bit - 1u))) * N;
          }
          n += __popc(m);
        }
      }
      if (lane == 0) nparts[warp] = n < kMaxParts ? n : kMaxParts;
    }
    __syncthreads();
    const int rows = M - r0 < kRedRows ? static_cast<int>(M - r0) : kRedRows;
    for (int64_t e = threadIdx.x; e < rows * (N >> 3); e += 256) {
      const int i = static_cast<int>(e / (N >> 3));
      const int64_t c = (e - static_cast<int64_t>(i) * (N >> 3)) * 8;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const int np = nparts[i];
      for (int k0 = 0; k0 < np; k0 += 4) {
        // up to four partial rows' loads in flight before any is summed (ascending order kept)
        float4 a[4], b[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k0 + k < np) {
            a[k] = __ldcs(reinterpret_cast<const float4*>(part + prow[i][k0 + k] + c));
            b[k] = __ldcs(reinterpret_cast<const float4*>(part + prow[i][k0 + k] + c + 4));
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k0 + k < np) {
            acc[0] += a[k].x; acc[1] += a[k].y; acc[2] += a[k].z; acc[3] += a[k].w;
            acc[4] += b[k].x; acc[5] += b[k].y; acc[6] += b[k].z; acc[7] += b[k].w;
          }
        }
      }
      T h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = cvt_out<T>(acc[q]);
      *reinterpret_cast<uint4*>(C + (r0 + i) * ldc + c) = *reinterpret_cast<const uint4*>(h);
    }
    __syncthreads();
  }
}

}  // namespace

int64_t gm_sparse_bound_rows(int64_t M, int64_t nkg, int S) { return ceil_div(M * nkg, kSparseDen) + S; }

int gm_sg() {  // columns per supergroup: 256, or PIT_GM_SG=512 (A/B knob)
  static const int v = [] {
    const char* e = getenv("PIT_GM_SG");
    return e && atoi(e) == 512 ? 512 : 256;
  }();
  return v;
}

GmSparseWs gm_sparse_layout(int64_t M, int64_t N, int64_t WG, int S, int64_t bound_rows) {
  GmSparseWs w{};
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o += (bytes + 255) / 256 * 256;
    return at;
  };
  w.flag = take(16);
  w.cnt = take(4 * S);
  w.off = take(4 * (S + 1));
  w.U = take(4 * S * WG);
  w.pre = take(4 * S * WG);
  w.rows = take(4 * S * M);
  w.X = take(bound_rows * gm_sg() * 2);
  w.part = take(bound_rows * N * 4);
  w.bytes = o;
  return w;
}

int launch_gm_sparse_prep(const int32_t* counts, int nkg, int64_t M, int gps, int S, const uint32_t* occ, int64_t WG,
                          uint8_t* ws, const GmSparseWs& w, cudaStream_t s) {
  gm_sparse_prep_kernel<<<S, kPrepThreads, 0, s>>>(
      counts, nkg, M, gps, S, occ, WG, reinterpret_cast<int*>(ws + w.flag), reinterpret_cast<int*>(ws + w.cnt),
      reinterpret_cast<uint32_t*>(ws + w.U), reinterpret_cast<int*>(ws + w.pre), reinterpret_cast<int32_t*>(ws + w.rows));
  note_launch();
  return cuda_status();
}

int launch_gm_sparse_pack(const int32_t* counts, int nkg, const void* A, int64_t lda_bytes, int S, int64_t M,
                          const uint32_t* occ, int64_t WG, int t1, int64_t bound_rows, uint8_t* ws, const GmSparseWs& w,
                          cudaStream_t s) {
  const int64_t blocks = ceil_div(bound_rows, 8);
  const int64_t cap = static_cast<int64_t>(n_sms()) * 8;
  gm_sparse_pack_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, (S + 1) * sizeof(int), s>>>(
      counts, nkg, static_cast<const uint8_t*>(A), lda_bytes, reinterpret_cast<const int*>(ws + w.cnt), S,
      reinterpret_cast<const int32_t*>(ws + w.rows), M, occ, WG, t1 == 16 ? 4 : t1 == 32 ? 5 : 6, ws + w.X, bound_rows,
      gm_sg());
  note_launch();
  return cuda_status();
}

int launch_gm_sparse_reduce(const int32_t* counts, int nkg, int dtype, int S, int64_t WG, int64_t N, void* C,
                            int64_t ldc, int64_t M, uint8_t* ws, const GmSparseWs& w, cudaStream_t s) {
  const int64_t cap = static_cast<int64_t>(n_sms()) * 8, blocks = ceil_div(M, kRedRows);
  const unsigned grid = static_cast<unsigned>(blocks < cap ? blocks : cap);
  const size_t smem = (S + 1) * sizeof(int);
  const int* cnt = reinterpret_cast<const int*>(ws + w.cnt);
  const uint32_t* U = reinterpret_cast<const uint32_t*>(ws + w.U);
  const int* pre = reinterpret_cast<const int*>(ws + w.pre);
  const float* part = reinterpret_cast<const float*>(ws + w.part);
  if (dtype == kDtypeBF16)
    gm_sparse_reduce_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>(counts, nkg, cnt, S, U, pre, WG, part, N,
                                                                   static_cast<__nv_bfloat16*>(C), ldc, M);
  else
    gm_sparse_reduce_kernel<__half><<<grid, 256, smem, s>>>(counts, nkg, cnt, S, U, pre, WG, part, N,
                                                            static_cast<__half*>(C), ldc, M);
  note_launch();
  return cuda_status();
}

}  // namespace pit
