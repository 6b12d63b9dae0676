// Micro-probe: global->shared gather throughput on B200 for the three copy engines the PIT
// mainloops can use. One CTA per SM, a ring of STAGES x 32 KiB stages, no consumer: a stage is
// re-filled as soon as its previous fill has landed. Rows are random 128-byte windows of a
// 8192 x 8192 bf16 matrix (the B-gather pattern of spmm_gk).
//   mode 0: TMA tile::gather4 (4 rows x 128 B per instruction), issued by `warps` warps (lane 0)
//   mode 1: cp.async 16 B per thread, `warps` warps
//   mode 2: TMA 2-D tile (64 rows x 128 B per instruction, contiguous rows), `warps` warps
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2301_10936_b200/csrc copy_probe.cu -o copy_probe
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>

#include "pit_ptx.cuh"

using namespace pit;

constexpr int STAGES = 6;
constexpr int STAGE_BYTES = 32768;
constexpr int ROWS_PER_STAGE = STAGE_BYTES / 128;  // 256

__global__ void __launch_bounds__(512, 1) probe(const __grid_constant__ CUtensorMap tm, const __nv_bfloat16* B,
                                                  const int* rows, int nrows_total, int mode, int warps, int iters, int rshift, int nwin) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], mode == 20 ? 2 : (mode == 1 || mode >= 3) ? warps * 32 : warps);
    fence_mbar_init();
  }
  __syncthreads();
  if (mode == 20 && warp >= 2) return;
  if (warp >= warps) return;
  uint32_t phase = 0;
  int stage = 0;
  int rbase = (blockIdx.x * 977) % nrows_total;
  for (int it = 0; it < iters; ++it) {
    if (it >= STAGES) mbar_wait(&full[stage], phase ^ 1);
    uint8_t* dst = smem + stage * STAGE_BYTES;
    if (mode == 0) {
      const int quads = ROWS_PER_STAGE / 4;
      const int myq = (quads - warp + warps - 1) / warps;
      if (lane == 0) mbar_expect_tx(&full[stage], myq * 512);
      for (int q = warp; q < quads; q += warps) {
        const unsigned r = rbase + q * 4;
        const int r0 = ((r + 0) * 2654435761u) >> rshift, r1 = ((r + 1) * 2654435761u) >> rshift;
        const int r2 = ((r + 2) * 2654435761u) >> rshift, r3 = ((r + 3) * 2654435761u) >> rshift;
        if (lane == 0) tma_gather4(dst + q * 512, &tm, &full[stage], (blockIdx.x % (nwin * 4)) * 64, r0, r1, r2, r3);
      }
    } else if (mode == 3 || mode == 4) {
      // spmm_gk pattern: one 512-byte row per warp instruction (32 lanes x 16 B), zero-fill variant
      const uint32_t s = smem_u32(dst);
      const uint32_t nb = 16u - (lane == 99 ? 1u : 0u);  // opaque to the compiler: register src-size
      for (int row = warp; row < ROWS_PER_STAGE / 4; row += warps) {
        const int k = ((unsigned)(rbase + row) * 2654435761u) >> rshift;
        const int ch = lane;
        const uint32_t o = (ch >> 3) * (64 * 128) + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
        if (mode == 3)
          cp_async_16(s + o, B + (int64_t)k * 8192 + (blockIdx.x % nwin) * 256 + ch * 8, nb);
        else
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + o),
                       "l"(B + (int64_t)k * 8192 + (blockIdx.x % nwin) * 256 + ch * 8) : "memory");
      }
      cp_async_arrive_noinc(&full[stage]);
    } else if (mode == 5) {
      // spmm_gk footprint (64 rows x 512 B per stage) with 4 rows x 128 B per warp instruction
      const uint32_t s = smem_u32(dst);
      for (int it2 = warp; it2 < 64; it2 += warps) {  // 16 row quads x 4 column segments
        const int row = (it2 >> 2) * 4 + (lane >> 3);
        const int ch = (it2 & 3) * 8 + (lane & 7);
        const int k = ((unsigned)(rbase + row) * 2654435761u) >> rshift;
        const uint32_t o = (ch >> 3) * (64 * 128) + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
        cp_async_16(s + o, B + (int64_t)k * 8192 + (blockIdx.x % nwin) * 256 + ch * 8, 16u - (lane == 99 ? 1u : 0u));
      }
      cp_async_arrive_noinc(&full[stage]);
    } else if (mode == 20) {
      // TMA gather4 issued by EVERY lane: lane l of warp w fetches quad q = w*32 + l (4 rows x 128 B)
      const int quads = ROWS_PER_STAGE / 4;  // 64
      const int q = warp * 32 + lane;
      const bool act = q < quads;
      const uint32_t mine = __ballot_sync(0xffffffffu, act);
      if (lane == 0) mbar_expect_tx(&full[stage], __popc(mine) * 512);
      __syncwarp();
      if (act) {
        const unsigned r = rbase + q * 4;
        const int r0 = ((r + 0) * 2654435761u) >> rshift, r1 = ((r + 1) * 2654435761u) >> rshift;
        const int r2 = ((r + 2) * 2654435761u) >> rshift, r3 = ((r + 3) * 2654435761u) >> rshift;
        tma_gather4(dst + q * 512, &tm, &full[stage], (blockIdx.x % (nwin * 4)) * 64, r0, r1, r2, r3);
      }
    } else if (mode == 8 || mode == 9) {
      // spmm_gk row pattern (one 512 B row per warp instruction) but the row's four 128 B chunks at
      // byte offsets {0, 256, 1024, 1280} (mode 8) or {0, 128, 256, 384} contiguous (mode 9, = mode 3)
      const uint32_t s = smem_u32(dst);
      const int j = lane >> 3;
      const int off_el = mode == 8 ? ((j & 1) * 128 + (j >> 1) * 512) : j * 64;  // elements
      for (int row = warp; row < ROWS_PER_STAGE / 4; row += warps) {
        const int k = ((unsigned)(rbase + row) * 2654435761u) >> rshift;
        const int ch = lane;
        const uint32_t o = (ch >> 3) * (64 * 128) + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
        cp_async_16(s + o, B + (int64_t)k * 8192 + (blockIdx.x % nwin) * 1024 + off_el + (lane & 7) * 8,
                    16u - (lane == 99 ? 1u : 0u));
      }
      cp_async_arrive_noinc(&full[stage]);
    } else if (mode == 6 || mode == 7) {
      // 64 rows x 512 B per stage. mode 6: 4 rows x 128 B per warp instruction (segment-major);
      // mode 7: 4 rows x 128 B, row-quad-major
      const uint32_t s = smem_u32(dst);
#pragma unroll 4
      for (int q = warp; q < 64; q += warps) {
        const int rq = mode == 6 ? (q & 15) : (q >> 2), sg = mode == 6 ? (q >> 4) : (q & 3);
        const int row = rq * 4 + (lane >> 3);
        const int ch = sg * 8 + (lane & 7);
        const int k = ((unsigned)(rbase + row) * 2654435761u) >> rshift;
        const uint32_t o = sg * (64 * 128) + row * 128 + (((lane & 7) ^ (row & 7)) << 4);
        cp_async_16(s + o, B + (int64_t)k * 8192 + (blockIdx.x % nwin) * 256 + ch * 8, 16u - (lane == 99 ? 1u : 0u));
      }
      cp_async_arrive_noinc(&full[stage]);
    } else if (mode >= 10) {
      // 64 rows x 512 B per stage, R = 2^(mode-10) rows x (512/R) B per warp instruction
      const int R = 1 << (mode - 10), LPR = 32 / R;
      const uint32_t s = smem_u32(dst);
      for (int it2 = warp; it2 < 64; it2 += warps) {
        const int rg = it2 / R, sg = it2 % R;
        const int row = rg * R + lane / LPR;
        const int ch = sg * LPR + lane % LPR;
        const int k = ((unsigned)(rbase + row) * 2654435761u) >> rshift;
        const uint32_t o = (ch >> 3) * (64 * 128) + row * 128 + (((ch & 7) ^ (row & 7)) << 4);
        cp_async_16(s + o, B + (int64_t)k * 8192 + (blockIdx.x % nwin) * 256 + ch * 8, 16u - (lane == 99 ? 1u : 0u));
      }
      cp_async_arrive_noinc(&full[stage]);
    } else if (mode == 1) {
      const uint32_t s = smem_u32(dst);
      for (int row = warp * 4 + (lane >> 3); row < ROWS_PER_STAGE; row += warps * 4) {
        const int k = ((unsigned)(rbase + row) * 2654435761u) >> rshift;
        const int ch = lane & 7;
        cp_async_16(s + swz<7>(row * 128 + ch * 16), B + (int64_t)k * 8192 + (blockIdx.x % (nwin * 4)) * 64 + ch * 8, 16);
      }
      cp_async_arrive_noinc(&full[stage]);
    } else {
      const int tiles = ROWS_PER_STAGE / 64;
      const int myt = (tiles - warp + warps - 1) / warps;
      if (lane == 0) {
        mbar_expect_tx(&full[stage], myt * 8192);
        for (int t = warp; t < tiles; t += warps)
          tma_load_2d(dst + t * 8192, &tm, &full[stage], (blockIdx.x % (nwin * 4)) * 64, (rbase + t * 64) % 8000);
      }
    }
    rbase = (rbase + ROWS_PER_STAGE) % nrows_total;
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
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int row_bits = argc > 1 ? atoi(argv[1]) : 13, nwin = argc > 2 ? atoi(argv[2]) : 32;
  const int rshift = 32 - row_bits;
  printf("footprint: %d rows x %d windows x 512 B = %.1f MB\n", 1 << row_bits, nwin, (double)(1 << row_bits) * nwin * 512 / 1e6);
  const int R = 8192, C = 8192;
  __nv_bfloat16* B;
  cudaMalloc(&B, (size_t)R * C * 2);
  cudaMemset(B, 0, (size_t)R * C * 2);
  std::vector<int> h(1 << 20);
  srand(1);
  for (auto& x : h) x = rand() % R;
  int* rows;
  cudaMalloc(&rows, h.size() * 4);
  cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap tm_g, tm_t;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, str[1] = {(cuuint64_t)C * 2};
  cuuint32_t box_g[2] = {64, 1}, box_t[2] = {64, 64}, es[2] = {1, 1};
  enc(&tm_g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, dims, str, box_g, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tm_t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, dims, str, box_t, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int smem = STAGES * STAGE_BYTES + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[6] = {"tma_gather4", "cp.async16", "tma_tile2d", "cp.async512z", "cp.async512", "cp.async4x128"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 400;
  for (int mode : {0, 1, 9, 20}) {
    for (int warps : {4, 8, 16}) {
      if (mode == 2 && warps > 1) continue;
      const CUtensorMap& tm = mode == 2 ? tm_t : tm_g;
      probe<<<sms, 512, smem>>>(tm, B, rows, (int)h.size(), mode, warps, 20, rshift, nwin);
      cudaEventRecord(e0);
      probe<<<sms, 512, smem>>>(tm, B, rows, (int)h.size(), mode, warps, iters, rshift, nwin);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)sms * iters * STAGE_BYTES;
      double gbs = bytes / (ms * 1e-3) / 1e9;
      printf("mode %2d %-12s warps=%2d  %8.1f GB/s  %6.2f B/cycle/SM (at %d MHz)  err=%s\n", mode, mode < 6 ? names[mode] : (mode == 8 ? "512B-spread" : mode == 20 ? "gather4x32" : "512B-contig"), warps, gbs,
             gbs * 1e9 / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
