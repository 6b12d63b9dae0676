// Minimal reproducer for the compute-sanitizer racecheck report inside tmem_alloc2
// (csrc/pit_ptx.cuh, tcgen05.alloc.cta_group::2). No MMA, no TMA, no mbarriers: a cluster of two
// CTAs allocates TMEM exactly as rowgemm2 / spmm_gk2 do (allocator warp -> fence::before_thread_sync
// -> cluster barrier -> fence::after_thread_sync -> every thread reads the slot), then frees it.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o tmem_alloc2_race tmem_alloc2_race.cu
//   compute-sanitizer --tool racecheck ./tmem_alloc2_race [mode]
//
// mode 0: the slot is never written by threads (only by tcgen05.alloc)
// mode 1: thread 0 zeroes the slot first, __syncthreads, then the allocator warp allocates
// mode 2: cta_group::1 allocation (single CTA per cluster rank) for comparison
// mode 3: rowgemm2's prologue layout: 512 threads, 1024-aligned dynamic shared memory, the slot right
//         after the mbarriers, thread 0 initialising the mbarriers while warp 9 allocates
// If racecheck reports hazards for mode 0/1 with no other shared-memory traffic in the kernel, the
// report is about the allocator's own write to shared memory, not about the PIT kernels.
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) alloc2_kernel(int mode, uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (mode == 1) {
    if (threadIdx.x == 0) slot = 0;
    __syncthreads();
  }
  if (warp == 0) {
    if (mode == 2) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t base = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  fence_before();
  cluster_sync();
  if (warp == 0) {
    fence_after();
    if (mode == 2)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base));
  }
}

// variant bits: 1 = skip the mbarrier init, 2 = allocate from warp 0 instead of warp 9,
//               4 = static shared slot instead of the dynamic-smem slot
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) alloc2_dyn_kernel(uint32_t* out, int variant) {
  __shared__ uint32_t static_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * 32768);
  uint32_t* slot = (variant & 4) ? &static_slot : reinterpret_cast<uint32_t*>(bars + 6 * 4 + 4);
  const int warp = threadIdx.x / 32;
  const int alloc_warp = (variant & 2) ? 0 : 9;
  if (threadIdx.x == 0 && !(variant & 1)) {
    for (int i = 0; i < 6 * 4 + 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bars + i)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == alloc_warp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t base = *slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  fence_before();
  cluster_sync();
  if (warp == alloc_warp) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base));
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  uint32_t* d = nullptr;
  cudaMalloc(&d, 8 * sizeof(uint32_t));
  if (mode >= 3) {
    // modes 3..10: rowgemm2's prologue layout with variant = mode - 3 (see alloc2_dyn_kernel)
    const int smem = 6 * 32768 + 2048;
    cudaFuncSetAttribute(alloc2_dyn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    alloc2_dyn_kernel<<<8, 512, smem>>>(d, mode - 3);
  } else {
    alloc2_kernel<<<8, 128>>>(mode, d);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[8];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("mode %d: %s, tmem base cta0=%u cta1=%u\n", mode, cudaGetErrorString(e), h[0], h[1]);
  return e == cudaSuccess ? 0 : 1;
}
