// L2 -> SM read ceiling on this part: the denominator for the gathered-K kernels' operand feed.
// One CTA per SM reads an L2-resident buffer (footprint well under the 126 MB L2, warmed first) as
// fast as the chosen path allows, no consumer work:
//   mode 0: TMA 1-D bulk copies (cp.async.bulk, 16 KB each) into a ring of 6 x 32 KB stages
//   mode 1: LDG.128 from every thread of 16 warps, 8 loads in flight per thread, summed (no smem)
//   mode 2: cp.async 16 B, 16 warps, contiguous 512 B rows into the same 6 x 32 KB ring
//   mode 3: cp.async 16 B, 16 warps, RANDOM 512 B rows (spmm_gk's B gather: one row per warp
//           instruction) of a matrix with row pitch `pitch` bytes, rows drawn from `nrows`
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2301_10936_b200/csrc l2_ceiling.cu -o l2_ceiling
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "pit_ptx.cuh"

using namespace pit;

constexpr int STAGES = 6;
constexpr int STAGE_BYTES = 32768;

__global__ void __launch_bounds__(512, 1) l2_read(const uint8_t* src, size_t footprint, int mode, int iters,
                                                   float* sink, int pitch = 16384, int nrows = 8192, int row_bytes = 512) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nchunks = footprint / STAGE_BYTES;
  if (mode == 1) {
    float acc = 0.f;
    const int4* p = reinterpret_cast<const int4*>(src);
    const size_t n16 = footprint / 16;
    size_t i = (static_cast<size_t>(blockIdx.x) * 4099 * 512 + threadIdx.x) % n16;
    for (int it = 0; it < iters * (STAGE_BYTES / 16 / 512); it += 8) {
      int4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + (i + static_cast<size_t>(j) * 512) % n16);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += __int_as_float(v[j].x ^ v[j].w);
      i = (i + 8 * 512) % n16;
    }
    if (acc == 1.2345f) sink[0] = acc;
    return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], mode == 0 ? 1 : 512);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  int stage = 0;
  size_t c = (static_cast<size_t>(blockIdx.x) * 37) % nchunks;
  for (int it = 0; it < iters; ++it) {
    if (it >= STAGES) mbar_wait(&full[stage], phase ^ 1);
    uint8_t* dst = smem + stage * STAGE_BYTES;
    const uint8_t* s = src + c * STAGE_BYTES;
    if (mode == 0) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&full[stage], STAGE_BYTES);
        for (int h = 0; h < 2; ++h)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(dst + h * 16384)),
              "l"(s + h * 16384), "r"(16384), "r"(smem_u32(&full[stage]))
              : "memory");
      }
    } else if (mode == 3) {
      const uint32_t d = smem_u32(dst);
      // 64 warp instructions of 512 B per stage; row_bytes / 512 consecutive instructions per row
      // (row_bytes and nrows powers of two: shifts and masks only, so the probe is not issue-bound)
      const int lg = __ffs(row_bytes / 512) - 1;
#pragma unroll
      for (int j = 0; j < STAGE_BYTES / 512 / 16; ++j) {
        const int ins = j * 16 + warp;
        const int row = ins >> lg, part = ins & ((1 << lg) - 1);
        const uint32_t k = ((static_cast<uint32_t>(it * 64 + row) + blockIdx.x * 7919u) * 2654435761u >> 7) & (nrows - 1);
        cp_async_16(d + (ins * 32 + lane) * 16, src + static_cast<size_t>(k) * pitch + part * 512 + lane * 16, 16);
      }
      cp_async_arrive_noinc(&full[stage]);
    } else {
      const uint32_t d = smem_u32(dst);
#pragma unroll
      for (int j = 0; j < STAGE_BYTES / 16 / 512; ++j)
        cp_async_16(d + (j * 512 + threadIdx.x) * 16, s + (j * 512 + threadIdx.x) * 16, 16);
      cp_async_arrive_noinc(&full[stage]);
    }
    c = (c + 148) % nchunks;
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  // drain
  for (int i = 0; i < STAGES; ++i) {
    mbar_wait(&full[stage], phase ^ 1);
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  (void)warp;
  (void)lane;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int smem = STAGES * STAGE_BYTES + 2048;
  cudaFuncSetAttribute(l2_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* sink;
  cudaMalloc(&sink, 4);
  const char* names[4] = {"tma_bulk_16KB", "ldg128_regs", "cp.async16_contig", "cp.async16_gather"};
  for (size_t mb : {16, 96}) {
    const size_t fp = mb << 20;
    uint8_t* buf;
    cudaMalloc(&buf, fp);
    cudaMemset(buf, 1, fp);
    for (int mode : {0, 1, 2}) {
      const int iters = 2000;
      l2_read<<<sms, 512, smem>>>(buf, fp, mode, 200, sink);  // warm L2
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      l2_read<<<sms, 512, smem>>>(buf, fp, mode, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = static_cast<double>(sms) * iters * STAGE_BYTES;
      const double gbs = bytes / (ms * 1e-3) / 1e9;
      printf("footprint %3zu MB  mode %d %-18s %9.1f GB/s  %6.2f B/cycle/SM (at %d MHz)  err=%s\n", mb, mode,
             names[mode], gbs, gbs * 1e9 / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(buf);
  }
  // random-row gathers: pitch and row-count sweep (the B slab of one n tile: 8192 rows)
  const size_t big = 160ull << 20;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  for (int rb : {512, 1024, 2048, 4096, 8192}) {
    const int nrows = 8192;
    for (int pitch : {16384}) {
      if (static_cast<size_t>(nrows) * pitch > big) continue;
      const int iters = 2000;
      l2_read<<<sms, 512, smem>>>(buf, big, 3, 200, sink, pitch, nrows, rb);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      l2_read<<<sms, 512, smem>>>(buf, big, 3, iters, sink, pitch, nrows, rb);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = static_cast<double>(sms) * iters * STAGE_BYTES / (ms * 1e-3) / 1e9;
      printf("gather rows=%5d pitch=%6d B row=%5d B  %9.1f GB/s  %6.2f B/cycle/SM  err=%s\n", nrows, pitch, rb, gbs,
             gbs * 1e9 / sms / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
