// Kernel-to-kernel cost inside a CUDA graph, with and without programmatic dependent launch (PDL).
// A chain of K dependent kernels (each reads the previous one's output) is captured from a stream,
// launched once per replay after an L2 flush; mean replay time over 200 replays.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/pdl_probe scripts/probe/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(const float* __restrict__ in, float* __restrict__ out, int n, int pdl, int setup_ns) {
  // "prologue" independent of the previous kernel (stands in for barrier init / TMEM alloc)
  if (setup_ns) {
    long long t0 = clock64();
    while (clock64() - t0 < (long long)setup_ns * 2) {
    }
  }
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (pdl & 2) asm volatile("griddepcontrol.launch_dependents;");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] + 1.0f;
}

__global__ void flush_kernel(float* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0.f;
}

static void launch(cudaStream_t s, const float* in, float* out, int n, int pdl, int setup_ns) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, step_kernel, in, out, n, pdl, setup_ns);
}

int main() {
  const int n = 148 * 256;
  float *a, *b, *fl;
  size_t fn = (size_t)256 << 20;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMalloc(&fl, fn * 4);
  cudaMemset(a, 0, n * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int setup : {0, 1500}) {
    for (int K : {1, 2, 4, 8}) {
      for (int pdl = 0; pdl < 4; pdl += (pdl == 0 ? 1 : 2)) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < K; ++k) launch(s, (k & 1) ? b : a, (k & 1) ? a : b, n, k > 0 ? pdl : (pdl & 2), setup);
        cudaStreamEndCapture(s, &g);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
          printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
          return 1;
        }
        for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
        double tot = 0;
        const int R = 200;
        for (int r = 0; r < R; ++r) {
          flush_kernel<<<592, 512, 0, s>>>(fl, fn);
          cudaEventRecord(e0, s);
          cudaGraphLaunch(ge, s);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          tot += ms;
        }
        printf("setup %4d ns  K=%d  pdl=%d  mean %.2f us\n", setup, K, pdl, tot / R * 1e3);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
