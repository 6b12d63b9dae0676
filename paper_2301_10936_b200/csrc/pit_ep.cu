// Expert-parallel MoE exchange over NVLink peer memory (SURVEY 8(b) pit_moe_dispatch, 8(e), C5).
//
// The reference has no multi-GPU code; its MoE view is one PIT index per expert over
// the routing one-hot (index.py:102-173 on from_mask(onehot,(1,1))). Across W ranks the
// expert groups are sharded, so the SRead that packs a group's token rows and the SWrite that
// scatters the expert outputs back cross GPUs. Here both are single kernels that move the rows over
// NVLink themselves, instead of a pack kernel + NCCL all-to-all-v + unpack:
//
//   dispatch  (pack + send, fused):  warp per token in expert order; the token row is stored
//             straight into the destination rank's receive region (peer pointer), at row
//             src_rank * cap + (position among the tokens this rank sends to that rank). The
//             per-expert counts go to the peers the same way. The last block to finish publishes
//             an epoch flag to every peer (fence.sc.sys, then st.release.sys).
//   recv plan (wait + plan):         each block waits for every peer's dispatch flag of this epoch,
//             then lists, per local expert, the receive rows (source-rank order, then token order).
//   signal                           after the expert FFNs wrote their outputs into the y region
//             (same row positions as the receive region), publish "y ready" to every peer.
//   combine   (pull + SWrite * gate, fused): wait for every peer's y flag, then each token pulls
//             its output row from the expert rank's y region over NVLink, scales it by the router
//             gate and stores it at its original position.
//
// No host round trip anywhere: split sizes never leave the device, so the layer is one stream of
// kernels and can be captured in a CUDA graph. Flags are monotonic epochs kept in device memory
// (every rank runs the same sequence of layers), so nothing is reset between calls. Reuse of the
// single receive / y buffers across consecutive layers is safe by construction: a rank's next
// dispatch into a peer only starts after its own combine, which waited for that peer's "y ready",
// which the peer publishes after its FFNs consumed the receive region; a rank overwrites its y only
// after every peer's next dispatch arrived, i.e. after every peer finished pulling.
//
// Every wait is bounded (20 s of globaltimer): on expiry the kernel sets
// the region's error word and returns, so a missing peer can never hang the GPU.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "pit_internal.h"

namespace pit {

namespace {

constexpr int kEpHeader = 256;
constexpr uint64_t kEpTimeoutNs = 20ull * 1000 * 1000 * 1000;

// region header (byte offsets)
constexpr int kOffEpoch = 0;     // u64: this rank's epoch, bumped by every dispatch
constexpr int kOffDone = 8;      // u32: dispatch blocks finished (last-arriver counter)
constexpr int kOffError = 12;    // u32: nonzero after a timed-out wait

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Layout {
  int64_t flags_d, flags_c, counts, recv, y, total;
};

__host__ __device__ inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

__host__ __device__ inline Layout ep_layout(int W, int64_t El, int64_t cap, int64_t row_bytes) {
  Layout L;
  L.flags_d = kEpHeader;
  L.flags_c = L.flags_d + 8 * W;
  L.counts = align256(L.flags_c + 8 * W);
  L.recv = align256(L.counts + 4 * W * El);
  L.y = align256(L.recv + W * cap * row_bytes);
  L.total = align256(L.y + W * cap * row_bytes);
  return L;
}

struct EpDev {
  int rank, W;
  int64_t El, cap, row_bytes;
  uint8_t* local;
  uint8_t* const* peers;  // device array [W]
  Layout L;
};

// Thread s < W of the block waits for flags[s] >= epoch (acquire, system scope); then the block syncs.
__device__ void wait_flags(const EpDev& d, int64_t flag_off, uint64_t epoch) {
  if (threadIdx.x < d.W) {
    const uint64_t* f = reinterpret_cast<const uint64_t*>(d.local + flag_off) + threadIdx.x;
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(f) < epoch) {
      if (globaltimer() - t0 > kEpTimeoutNs) {
        atomicExch(reinterpret_cast<unsigned*>(d.local + kOffError), 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// expert of sorted position i: largest e with offsets[e] <= i (offsets in shared memory, E+1 entries)
__device__ __forceinline__ int expert_of(const int32_t* so, int E, int i) {
  int lo = 0, hi = E;  // invariant: so[lo] <= i < so[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (so[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) ep_dispatch_kernel(EpDev d, const uint8_t* __restrict__ x, int64_t ldx_bytes,
                                                          int64_t T, const int32_t* __restrict__ perm,
                                                          const int32_t* __restrict__ offsets,
                                                          const int32_t* __restrict__ counts) {
  extern __shared__ int32_t so[];  // offsets [E+1]
  const int E = static_cast<int>(d.W * d.El);
  for (int e = threadIdx.x; e <= E; e += blockDim.x) so[e] = offsets[e];
  __syncthreads();
  // per-expert counts into every destination rank's counts region: peer r, row [rank], column el
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int r = static_cast<int>(e / d.El), el = static_cast<int>(e % d.El);
      int32_t* c = reinterpret_cast<int32_t*>(d.peers[r] + d.L.counts) + d.rank * d.El + el;
      *c = counts[e];
    }
  }
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t vec = d.row_bytes >> 4;  // 16-byte chunks per row (row_bytes % 16 == 0)
  for (int64_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < T; i += warps) {
    const int e = expert_of(so, E, static_cast<int>(i));
    const int r = static_cast<int>(e / d.El);
    const int64_t pos = i - so[r * d.El];
    const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(perm[i]) * ldx_bytes);
    uint4* dst = reinterpret_cast<uint4*>(d.peers[r] + d.L.recv + (d.rank * d.cap + pos) * d.row_bytes);
    for (int64_t c = lane; c < vec; c += 32) dst[c] = __ldg(src + c);
  }
  // last block to finish publishes the epoch to every peer (every thread fences its own stores)
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* done = reinterpret_cast<unsigned*>(d.local + kOffDone);
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0;
      uint64_t* ep = reinterpret_cast<uint64_t*>(d.local + kOffEpoch);
      const uint64_t epoch = *ep + 1;
      *ep = epoch;
      __threadfence_system();
      for (int r = 0; r < d.W; ++r)
        st_release_sys(reinterpret_cast<uint64_t*>(d.peers[r] + d.L.flags_d) + d.rank, epoch);
    }
  }
}

// Wait for every peer's dispatch of this epoch, then the receive plan of local expert blockIdx.y:
// rows[e * stride + j] = receive row of its j-th token (source-rank order), counts[e].
__global__ void __launch_bounds__(256) ep_recv_plan_kernel(EpDev d, int32_t* __restrict__ rows, int64_t stride,
                                                           int32_t* __restrict__ counts) {
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(d.local + kOffEpoch);
  wait_flags(d, d.L.flags_d, epoch);
  const int e = blockIdx.y;
  const int32_t* rc = reinterpret_cast<const int32_t*>(d.local + d.L.counts);  // [W][El]
  int out = 0;
  for (int s = 0; s < d.W; ++s) {
    int before = 0;
    for (int x = 0; x < e; ++x) before += __ldcv(rc + s * d.El + x);
    const int n = __ldcv(rc + s * d.El + e);
    const int64_t base = s * d.cap + before;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
      rows[static_cast<int64_t>(e) * stride + out + j] = static_cast<int32_t>(base + j);
    out += n;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[e] = out;
}

__global__ void ep_signal_kernel(EpDev d) {
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(d.local + kOffEpoch);
  __threadfence_system();
  for (int r = threadIdx.x; r < d.W; r += blockDim.x)
    st_release_sys(reinterpret_cast<uint64_t*>(d.peers[r] + d.L.flags_c) + d.rank, epoch);
}

__device__ __forceinline__ uint4 scale8_bf16(uint4 v, float g) {
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 f = __bfloat1622float2(h[k]);
    h[k] = __floats2bfloat162_rn(f.x * g, f.y * g);
  }
  return v;
}
__device__ __forceinline__ uint4 scale8_f16(uint4 v, float g) {
  __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 f = __half22float2(h[k]);
    h[k] = __floats2half2_rn(f.x * g, f.y * g);
  }
  return v;
}
__device__ __forceinline__ uint4 scale4_f32(uint4 v, float g) {
  float* f = reinterpret_cast<float*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) f[k] *= g;
  return v;
}

// Wait for every peer's "y ready", then out[perm[i]] = gate[perm[i]] * y_peer(r)[rank * cap + pos].
__global__ void __launch_bounds__(256) ep_combine_kernel(EpDev d, int dtype, int64_t T,
                                                         const int32_t* __restrict__ perm,
                                                         const int32_t* __restrict__ offsets,
                                                         const float* __restrict__ gate, uint8_t* __restrict__ out,
                                                         int64_t ldo_bytes) {
  extern __shared__ int32_t so[];
  const int E = static_cast<int>(d.W * d.El);
  for (int e = threadIdx.x; e <= E; e += blockDim.x) so[e] = offsets[e];
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(d.local + kOffEpoch);
  wait_flags(d, d.L.flags_c, epoch);  // includes __syncthreads
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t vec = d.row_bytes >> 4;
  for (int64_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < T; i += warps) {
    const int e = expert_of(so, E, static_cast<int>(i));
    const int r = static_cast<int>(e / d.El);
    const int64_t pos = i - so[r * d.El];
    const int t = perm[i];
    const float g = gate ? gate[t] : 1.0f;
    // peer data written by another device before its release flag: plain (coherent) loads
    const uint4* src = reinterpret_cast<const uint4*>(d.peers[r] + d.L.y + (d.rank * d.cap + pos) * d.row_bytes);
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(t) * ldo_bytes);
    for (int64_t c = lane; c < vec; c += 32) {
      uint4 v = __ldcv(src + c);
      v = dtype == kDtypeBF16 ? scale8_bf16(v, g) : dtype == kDtypeF16 ? scale8_f16(v, g) : scale4_f32(v, g);
      dst[c] = v;
    }
  }
}

EpDev make_dev(const EpArgs& a) {
  EpDev d;
  d.rank = a.rank;
  d.W = a.world;
  d.El = a.experts_local;
  d.cap = a.capacity;
  d.row_bytes = a.row_bytes;
  d.local = static_cast<uint8_t*>(a.local);
  d.peers = reinterpret_cast<uint8_t* const*>(a.peers);
  d.L = ep_layout(a.world, a.experts_local, a.capacity, a.row_bytes);
  return d;
}

int row_blocks(int64_t T) {
  const int64_t b = ceil_div(T, 8);  // 8 warps per block, one row per warp per step
  const int64_t cap = 4ll * 148;
  return static_cast<int>(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

void ep_region_layout(int W, int64_t El, int64_t cap, int64_t row_bytes, int64_t out[6]) {
  const Layout L = ep_layout(W, El, cap, row_bytes);
  out[0] = L.flags_d;
  out[1] = L.flags_c;
  out[2] = L.counts;
  out[3] = L.recv;
  out[4] = L.y;
  out[5] = L.total;
}

int launch_ep_dispatch(const EpArgs& a, const void* x, int64_t ldx_bytes, int64_t T, const int32_t* perm,
                       const int32_t* offsets, const int32_t* counts, cudaStream_t s) {
  const EpDev d = make_dev(a);
  const int E = static_cast<int>(a.world * a.experts_local);
  ep_dispatch_kernel<<<row_blocks(T), 256, sizeof(int32_t) * (E + 1), s>>>(d, static_cast<const uint8_t*>(x),
                                                                          ldx_bytes, T, perm, offsets, counts);
  note_launch();
  return cuda_status();
}

int launch_ep_recv_plan(const EpArgs& a, int32_t* rows, int64_t stride, int32_t* counts, cudaStream_t s) {
  const EpDev d = make_dev(a);
  const int64_t per = ceil_div(a.capacity, 256);
  dim3 grid(static_cast<unsigned>(per < 8 ? (per > 0 ? per : 1) : 8), static_cast<unsigned>(a.experts_local));
  ep_recv_plan_kernel<<<grid, 256, 0, s>>>(d, rows, stride, counts);
  note_launch();
  return cuda_status();
}

int launch_ep_signal(const EpArgs& a, cudaStream_t s) {
  ep_signal_kernel<<<1, 32, 0, s>>>(make_dev(a));
  note_launch();
  return cuda_status();
}

int launch_ep_combine(const EpArgs& a, int dtype, int64_t T, const int32_t* perm, const int32_t* offsets,
                      const float* gate, void* out, int64_t ldo_bytes, cudaStream_t s) {
  if (dtype != kDtypeBF16 && dtype != kDtypeF16 && dtype != kDtypeF32) return kErrUnsupported;
  const EpDev d = make_dev(a);
  const int E = static_cast<int>(a.world * a.experts_local);
  ep_combine_kernel<<<row_blocks(T), 256, sizeof(int32_t) * (E + 1), s>>>(d, dtype, T, perm, offsets, gate,
                                                                         static_cast<uint8_t*>(out), ldo_bytes);
  note_launch();
  return cuda_status();
}

}  // namespace pit
