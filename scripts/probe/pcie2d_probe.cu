// Pitched (column-slab) host<->device copies of a 8192 x 8192 bf16 matrix: copy-engine 2-D copies
// vs SM copy kernels that load / store mapped pinned host memory directly, alone and with the other
// direction running concurrently (the e2e path's B-slab upload beside its C-slab download).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/pcie2d scripts/probe/pcie2d_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// dst[r * dpitch + c] = src[r * spitch + c] for r < rows, c < width (bytes; all multiples of 16)
__global__ void copy2d_kernel(char* __restrict__ dst, size_t dpitch, const char* __restrict__ src, size_t spitch,
                              size_t width, int rows) {
  const int vw = static_cast<int>(width / 16);
  const long long total = static_cast<long long>(vw) * rows;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < total; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long j = i + u * stride;
      const int r = static_cast<int>(j / vw), c = static_cast<int>(j % vw);
      v[u] = *reinterpret_cast<const int4*>(src + r * spitch + c * 16);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long j = i + u * stride;
      const int r = static_cast<int>(j / vw), c = static_cast<int>(j % vw);
      *reinterpret_cast<int4*>(dst + r * dpitch + c * 16) = v[u];
    }
  }
  for (; i < total; i += stride) {
    const int r = static_cast<int>(i / vw), c = static_cast<int>(i % vw);
    *reinterpret_cast<int4*>(dst + r * dpitch + c * 16) = *reinterpret_cast<const int4*>(src + r * spitch + c * 16);
  }
}

static const int n = 8192;
static const size_t pitch = n * 2;

static void slabs(bool kernel, int ctas, char* dst, const char* src, int slab_cols, cudaStream_t s,
                  cudaMemcpyKind kind) {
  for (int j0 = 0; j0 < n; j0 += slab_cols) {
    if (kernel)
      copy2d_kernel<<<ctas, 512, 0, s>>>(dst + j0 * 2, pitch, src + j0 * 2, pitch, slab_cols * 2, n);
    else
      cudaMemcpy2DAsync(dst + j0 * 2, pitch, src + j0 * 2, pitch, slab_cols * 2, n, kind, s);
  }
}

int main() {
  char *h1, *h2, *d1, *d2;
  const size_t bytes = static_cast<size_t>(n) * n * 2;
  cudaHostAlloc(&h1, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&h2, bytes, cudaHostAllocDefault);
  cudaMalloc(&d1, bytes);
  cudaMalloc(&d2, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b, c;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreate(&c);
  struct Case {
    const char* name;
    bool up, down, kup, kdown;
    int cols, ctas;
  };
  const Case cases[] = {
      {"DMA up 1024-col slabs alone", true, false, false, false, 1024, 0},
      {"DMA down 1024-col slabs alone", false, true, false, false, 1024, 0},
      {"DMA up + DMA down 1024-col (current e2e)", true, true, false, false, 1024, 0},
      {"DMA up + DMA down 2048-col", true, true, false, false, 2048, 0},
      {"DMA up + DMA down 8192-col (contiguous)", true, true, false, false, 8192, 0},
      {"kernel up (16 CTAs) alone 1024-col", true, false, true, false, 1024, 16},
      {"kernel up (32 CTAs) alone 1024-col", true, false, true, false, 1024, 32},
      {"kernel up (64 CTAs) alone 1024-col", true, false, true, false, 1024, 64},
      {"kernel down (16 CTAs) alone 1024-col", false, true, false, true, 1024, 16},
      {"kernel down (32 CTAs) alone 1024-col", false, true, false, true, 1024, 32},
      {"kernel up + DMA down 1024-col (32)", true, true, true, false, 1024, 32},
      {"DMA up + kernel down 1024-col (32)", true, true, false, true, 1024, 32},
      {"kernel up + kernel down 1024-col (32+32)", true, true, true, true, 1024, 32},
      {"kernel up + kernel down 1024-col (16+16)", true, true, true, true, 1024, 16},
  };
  for (const Case& k : cases) {
    float best_up = 1e9f, best_dn = 1e9f, best_all = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s1);
      cudaStreamWaitEvent(s2, a, 0);
      if (k.up) slabs(k.kup, k.ctas, d1, h1, k.cols, s1, cudaMemcpyHostToDevice);
      cudaEventRecord(b, s1);
      if (k.down) slabs(k.kdown, k.ctas, h2, d2, k.cols, s2, cudaMemcpyDeviceToHost);
      cudaEventRecord(c, s2);
      cudaStreamWaitEvent(s1, c, 0);
      cudaDeviceSynchronize();
      float tu, td;
      cudaEventElapsedTime(&tu, a, b);
      cudaEventElapsedTime(&td, a, c);
      if (k.up) best_up = tu < best_up ? tu : best_up;
      if (k.down) best_dn = td < best_dn ? td : best_dn;
      const float tall = (k.up && k.down) ? (tu > td ? tu : td) : (k.up ? tu : td);
      best_all = tall < best_all ? tall : best_all;
    }
    printf("%-44s", k.name);
    if (k.up) printf("  up %6.3f ms %5.1f GB/s", best_up, bytes / best_up / 1e6);
    if (k.down) printf("  down %6.3f ms %5.1f GB/s", best_dn, bytes / best_dn / 1e6);
    if (k.up && k.down) printf("  both %6.3f ms %5.1f GB/s total", best_all, 2 * bytes / best_all / 1e6);
    printf("\n");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
