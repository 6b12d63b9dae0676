// Output-sparse matmul (SDDMM): C = A . B restricted to the live micro-tiles of an
// output annotation, on tcgen05.
//
// The reference documents the output-side plans (the matmul n-axis plan as "the exact mirror of m",
// pkg/README.md:150-153) but does not wire them; this is the B200 form of the output-
// sparse plan the paper uses for attention scores (S = Q.K^T only inside the block mask) and for the
// ReLU-masked activation gradient dH = (dY . W2^T) * 1[H > 0].
//
// Layout. A row-major [rows, K] (slices stacked along rows), B column-major per slice, i.e. B^T
// row-major [batch * N, K] (the mirror of pit:m's row-major A: the operand on the permuted axis is
// the K-contiguous one), C row-major [rows, N]. Both MMA operands are K-major.
//
// Work. Two indexes of the output annotation, both built by K1 from the same bits:
//   * the unit index at micro (128, 64), PIT axis = columns: per 128-row tile, the ascending list of
//     64-column blocks holding any live element. A unit is a tile and up to four of its live column
//     blocks (not necessarily adjacent): D[128, 64 * nb] = A_tile . B_blocks^T in TMEM, the B
//     blocks gathered by TMA boxes from their rows of B^T.
//   * the fine occupancy bitmap at the annotation's micro-tile (g0, g1): the epilogue stores a
//     16-byte chunk (8 columns of one row) only if its micro-tile is live. Dead micro-tiles of C are
//     never written (SWrite semantics: a downstream PIT product reads only live micro-tiles).
// Optional elementwise gate (ReLU-masked gradients): a stored element is zeroed where gate <= 0.
//
// Roofline. Head dim 64 attention scores: 64 MACs per output element, i.e. bound by writing the live
// output (2 bytes per element) plus reading Q, K once: HBM. Large K (dH): tensor pipe.
//
// Warp roles (384 threads): warp 0 TMA producer (lane b fetches column block b's index entry; the
// next unit's table entry is prefetched a unit ahead), warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4-11 epilogue, two per TMEM lane quadrant (warp % 4), splitting the unit's column blocks.
// TMEM: two 256-column fp32 accumulators. A 32 x 64 box whose items are all live leaves by one TMA
// tile store from the swizzled staging box; partially live boxes by predicated 16-byte stores.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "pit_internal.h"
#include "pit_ptx.cuh"

// Diagnostics (compiled in with -DPIT_DIAG=1 only): PIT_SD_DIAG bits 0-3 drop the stores / TMEM loads /
// TMA loads / MMAs, bit 4 records CTA 0's unit timeline (globaltimer; scripts/sddmm_trace.py).
#ifndef PIT_DIAG
#define PIT_DIAG 0
#endif
__device__ unsigned long long g_sd_trace[8 * 64];

namespace pit {

namespace {

__device__ __forceinline__ unsigned long long sd_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SD_STAMP(row, idx)                                                                  \
  do {                                                                                      \
    if (PIT_DIAG && (p.diag & 16) && blockIdx.x == 0 && (idx) < 64) g_sd_trace[(row) * 64 + (idx)] = sd_timer(); \
  } while (0)

constexpr int kSdThreads = 384;
constexpr int kSdEpiWarps = 8;
constexpr int kSdStages = 3;
constexpr int kSdA = 128 * 128;          // A tile: 128 rows x 64 k (bf16) = 16 KB
constexpr int kSdBBox = 64 * 128;        // one B column block: 64 rows x 64 k = 8 KB
constexpr int kSdStage = kSdA + 4 * kSdBBox;
constexpr int kSdEpi = 32 * 128;         // per epilogue warp: 32 rows x 64 columns bf16
constexpr int kSdSmem = kSdStages * kSdStage + kSdEpiWarps * kSdEpi + 4 * 32 + 1024 + 256;

struct SddmmParams {
  void* C;
  int64_t ldc;
  int64_t M, N, K;  // per slice
  int batch;
  int tiles_per_slice;
  const int32_t* ucounts;
  const int32_t* uslots;
  int64_t ustride;
  const int32_t* unit_off;  // [G + 1] prefix of ceil(ucounts / 4)
  const int* unit_tab;      // [units][8] {group, nb, slice, 0, cb0..cb3} (sddmm_plan_kernel)
  int G;
  int lg0, lg1;             // log2(g0), log2(g1) when powers of two, else -1
  int box_uniform;          // every 32 x 64 box lies inside one annotation block (and inside C)
  int diag;
  const uint32_t* occ;  // fine bitmap, groups = row blocks of g0 (stacked), words per group WG
  int64_t WG;
  int g0, g1;
  const void* gate;
  int64_t ldg;
};

template <bool kBF16>
__device__ __forceinline__ uint32_t gate_mask_pair(uint32_t g2) {
  // keep mask (0xffff per element) for two packed 16-bit gate values: keep where value > 0
  uint32_t m = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint16_t v = static_cast<uint16_t>(g2 >> (16 * h));
    float f;
    if (kBF16) {
      f = __uint_as_float(static_cast<uint32_t>(v) << 16);
    } else {
      __half_raw r;
      r.x = v;
      f = __half2float(__half(r));
    }
    if (f > 0.0f) m |= 0xffffu << (16 * h);
  }
  return m;
}

// Per-unit metadata the producer hands to the epilogue through a shared-memory ring (group, column
// blocks), so the epilogue can look up the NEXT unit's fine-bitmap words while it stores the
// current one (looked up just in time they were an un-overlapped L2 round trip per unit).
struct SdMeta {
  int g, nb, slice, boxes;  // boxes: box-uniform liveness, bit 4 * column block + row quadrant
  int cb[4];
};
constexpr int kSdMeta = 4;

template <bool kBF16>
__global__ void __launch_bounds__(kSdThreads, 1)
    sddmm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const SddmmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi = smem + kSdStages * kSdStage;
  SdMeta* meta = reinterpret_cast<SdMeta*>(epi + kSdEpiWarps * kSdEpi);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(meta + kSdMeta);
  uint64_t* empty_bar = full_bar + kSdStages;
  uint64_t* tfull_bar = empty_bar + kSdStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* mfull_bar = tempty_bar + 2;
  uint64_t* mempty_bar = mfull_bar + kSdMeta;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mempty_bar + kSdMeta);
  int* stage_nb = reinterpret_cast<int*>(tmem_slot + 1);  // [kSdStages]: column blocks of the stage's unit

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int units = __ldg(p.unit_off + p.G);
  const int kblocks = static_cast<int>((p.K + 63) / 64);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSdStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kSdEpiWarps);
    }
    for (int m = 0; m < kSdMeta; ++m) {
      mbar_init(&mfull_bar[m], 32);
      mbar_init(&mempty_bar[m], kSdEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer: metadata + TMA
    // lane l < 8 holds word l of the descriptors of the next three units (no dependent loads on the
    // producer's path: a unit's group, width and column blocks come in one 32-byte entry)
    int u = blockIdx.x;
    const int G3 = static_cast<int>(gridDim.x);
    auto desc = [&](int x) { return x < units && lane < 8 ? __ldg(p.unit_tab + 8 * static_cast<int64_t>(x) + lane) : 0; };
    int d0 = desc(u), d1 = desc(u + G3), d2 = desc(u + 2 * G3);
    // box-uniform masks: lane l < 16 looks up the bit of box (column block l / 4, row quadrant l % 4) of
    // the NEXT unit (issued one unit ahead, consumed by a ballot on the next iteration)
    auto box_bit = [&](int word_desc) -> uint32_t {
      const int g = __shfl_sync(0xffffffffu, word_desc, 0);
      const int nb = __shfl_sync(0xffffffffu, word_desc, 1);
      const int cb = __shfl_sync(0xffffffffu, word_desc, 4 + ((lane >> 2) & 3));
      const int b = lane >> 2, q = lane & 3;
      if (!p.box_uniform || lane >= 16 || b >= nb) return 0u;
      const int row = g * 128 + 32 * q;
      const int rb = p.lg0 >= 0 ? (row >> p.lg0) : row / p.g0;
      const int cg = p.lg1 >= 0 ? ((cb * 64) >> p.lg1) : (cb * 64) / p.g1;
      return __ldg(p.occ + static_cast<int64_t>(rb) * p.WG + (cg >> 5)) >> (cg & 31);
    };
    uint32_t bits_next = u < units ? box_bit(d0) : 0u;
    int stage = 0, ms = 0;
    uint32_t phase = 0, mphase = 0;
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
    }
    for (; u < units; u += G3) {
      const int word = d0;
      const uint32_t bits_cur = bits_next;
      d0 = d1;
      d1 = d2;
      d2 = desc(u + 3 * G3);
      bits_next = u + G3 < units ? box_bit(d0) : 0u;
      const int g = __shfl_sync(0xffffffffu, word, 0);
      const int nb = __shfl_sync(0xffffffffu, word, 1);
      const int slice = __shfl_sync(0xffffffffu, word, 2);
      const int cbl = __shfl_sync(0xffffffffu, word, 4 + (lane & 3));
      mbar_wait(&mempty_bar[ms], mphase ^ 1);
      const int ui = (u - static_cast<int>(blockIdx.x)) / G3;
      if (lane == 0) SD_STAMP(0, ui);
      const uint32_t boxes = __ballot_sync(0xffffffffu, bits_cur & 1u) & 0xffffu;  // bit 4b + q
      if (lane < 8) reinterpret_cast<int*>(&meta[ms])[lane] = lane == 3 ? static_cast<int>(boxes) : word;
      mbar_arrive(&mfull_bar[ms]);
      if (++ms == kSdMeta) {
        ms = 0;
        mphase ^= 1;
      }
      const int brow = slice * static_cast<int>(p.N) + 64 * cbl;
      const int b0 = __shfl_sync(0xffffffffu, brow, 0), b1 = __shfl_sync(0xffffffffu, brow, 1);
      const int b2 = __shfl_sync(0xffffffffu, brow, 2), b3 = __shfl_sync(0xffffffffu, brow, 3);
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (lane == 0) {
          uint8_t* sA = smem + stage * kSdStage;
          stage_nb[stage] = nb;
          if (PIT_DIAG && (p.diag & 4)) {
            mbar_arrive(&full_bar[stage]);
          } else {
          mbar_expect_tx(&full_bar[stage], kSdA + nb * kSdBBox);
          tma_load_2d(sA, &tmA, &full_bar[stage], kb * 64, g * 128);
          tma_load_2d(sA + kSdA, &tmB, &full_bar[stage], kb * 64, b0);
          if (nb > 1) tma_load_2d(sA + kSdA + kSdBBox, &tmB, &full_bar[stage], kb * 64, b1);
          if (nb > 2) tma_load_2d(sA + kSdA + 2 * kSdBBox, &tmB, &full_bar[stage], kb * 64, b2);
          if (nb > 3) tma_load_2d(sA + kSdA + 3 * kSdBBox, &tmB, &full_bar[stage], kb * 64, b3);
          }
        }
        __syncwarp();
        if (++stage == kSdStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) SD_STAMP(1, ui);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const int ui = (u - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x);
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0 && kb == 0) SD_STAMP(2, ui);
        if (lane == 0) {
          const uint32_t idesc = idesc_f16(128, 64 * stage_nb[stage], kBF16, false, false);
          const uint32_t sA = smem_u32(smem + stage * kSdStage);
          const uint32_t sB = sA + kSdA;
#pragma unroll
          for (int ks = 0; ks < ((PIT_DIAG && (p.diag & 8)) ? 0 : 4); ++ks) {
            const uint64_t adesc = smem_desc(sA + ks * 32, 16, 1024, kSw128);
            const uint64_t bdesc = smem_desc(sB + ks * 32, 16, 1024, kSw128);
            umma_f16(tmem_base + static_cast<uint32_t>(acc * 256), adesc, bdesc, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (kb == kblocks - 1) {
            umma_commit(&tfull_bar[acc]);
            SD_STAMP(3, ui);
          }
        }
        __syncwarp();
        if (++stage == kSdStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue (SWrite)
    // two warps per TMEM lane quadrant (warp % 4): warp pair half h takes column blocks h, h + 2
    const int quad = warp & 3;
    const int half = (warp - 4) >> 2;
    const uint32_t sbuf = smem_u32(epi + (warp - 4) * kSdEpi);
    int acc = 0, ms = 0;
    uint32_t acc_phase = 0, mphase = 0;
    const int sub_row = lane >> 3;  // store phase: 4 rows x 8 chunks per instruction
    const int chunk = lane & 7;
    // the lane's row (row_base + lane) words of the fine bitmap for this warp's two column blocks
    struct Look {
      int g, nb, slice_end, boxes, cb[2];
      uint32_t w[2][2];
    };
    auto lookup = [&](int slot) {
      const SdMeta& md = meta[slot];
      Look L;
      L.g = md.g;
      L.nb = md.nb;
      L.slice_end = (md.slice + 1) * static_cast<int>(p.M);
      L.boxes = md.boxes;
      const int row = min(L.g * 128 + 32 * quad + lane, L.slice_end - 1);
      const int rb = p.lg0 >= 0 ? (row >> p.lg0) : row / p.g0;
      const uint32_t* wp = p.occ + static_cast<int64_t>(rb) * p.WG;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b = half + 2 * q;
        L.cb[q] = md.cb[b];
        const int col0 = L.cb[q] * 64;
        const int clast = min(col0 + 63, static_cast<int>(p.N) - 1);
        const int cg0 = p.lg1 >= 0 ? (col0 >> p.lg1) : col0 / p.g1;
        const int cg1 = p.lg1 >= 0 ? (clast >> p.lg1) : clast / p.g1;
        const bool need = !p.box_uniform && b < L.nb;
        L.w[q][0] = need ? __ldg(wp + (cg0 >> 5)) : 0u;
        L.w[q][1] = need && (cg1 >> 5) != (cg0 >> 5) ? __ldg(wp + (cg1 >> 5)) : L.w[q][0];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mempty_bar[slot]);
      return L;
    };
    // 8-bit chunk mask of the lane's row for column block q of a looked-up unit
    auto chunk_mask = [&](const Look& L, int q) -> uint32_t {
      const int b = half + 2 * q;
      if (b >= L.nb || L.g * 128 + 32 * quad + lane >= L.slice_end) return 0u;
      if (p.box_uniform) return ((L.boxes >> (4 * b + quad)) & 1u) ? 0xffu : 0u;
      const int col0 = L.cb[q] * 64;
      const int cg0 = p.lg1 >= 0 ? (col0 >> p.lg1) : col0 / p.g1;
      uint32_t m = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = col0 + 8 * c;
        const int cg = p.lg1 >= 0 ? (col >> p.lg1) : col / p.g1;
        const uint32_t w = (cg >> 5) == (cg0 >> 5) ? L.w[q][0] : L.w[q][1];
        m |= static_cast<uint32_t>(col < p.N && ((w >> (cg & 31)) & 1u)) << c;
      }
      return m;
    };
    Look cur{};
    if (static_cast<int>(blockIdx.x) < units) {
      mbar_wait(&mfull_bar[ms], mphase);
      cur = lookup(ms);
      if (++ms == kSdMeta) {
        ms = 0;
        mphase ^= 1;
      }
    }
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int g = cur.g, nb = cur.nb;
      const int row_base = g * 128 + 32 * quad;  // stacked row of this warp's TMEM lane 0
      const int cbv[2] = {cur.cb[0], cur.cb[1]};
      const uint32_t mrow[2] = {chunk_mask(cur, 0), chunk_mask(cur, 1)};
      if (u + static_cast<int>(gridDim.x) < units) {  // next unit's bitmap words, in flight while storing
        mbar_wait(&mfull_bar[ms], mphase);
        cur = lookup(ms);
        if (++ms == kSdMeta) {
          ms = 0;
          mphase ^= 1;
        }
      }
      const int ui = (u - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x);
      if (lane == 0 && warp == 4) SD_STAMP(4, ui);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (lane == 0 && warp == 4) SD_STAMP(5, ui);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b = half + 2 * q;
        if (b >= nb) break;
        const int cb = cbv[q];
        if (__all_sync(0xffffffffu, mrow[q] == 0u)) continue;  // no live item in this warp's box
        // TMEM -> registers: lane = row, 64 fp32 columns (both loads in flight) -> packed pairs -> staging
        uint32_t v0[32], v1[32];
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * quad) << 16) + static_cast<uint32_t>(acc * 256 + b * 64);
        if (PIT_DIAG && (p.diag & 2)) continue;
        tmem_ld32(taddr, v0);
        tmem_ld32(taddr + 32, v1);
        bulk_wait_read<0>();  // the previous TMA store no longer reads the staging box
        __syncwarp();
        tmem_wait_ld();
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          const uint32_t* v = c16 < 4 ? v0 : v1;
          const int q8 = (c16 & 3) * 8;
          uint32_t w[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const float lo = __uint_as_float(v[q8 + 2 * x]), hi = __uint_as_float(v[q8 + 2 * x + 1]);
            if (kBF16) {
              __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
              w[x] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __half2 h = __floats2half2_rn(lo, hi);
              w[x] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          // 128B-swizzled row (the layout of a SWIZZLE_128B TMA box [64 cols x 32 rows])
          st_shared_v4(sbuf + lane * 128 + ((c16 ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
        }
        const int col = cb * 64 + chunk * 8;
        if (PIT_DIAG && (p.diag & 1)) continue;
        if (__all_sync(0xffffffffu, mrow[q] == 0xffu) && p.gate == nullptr) {
          // every item of the 32 x 64 box is live: one TMA tile store
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, sbuf, cb * 64, row_base);
            bulk_commit();
          }
        } else {
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + sub_row;
            const uint32_t m = __shfl_sync(0xffffffffu, mrow[q], r);
            if (!((m >> chunk) & 1u)) continue;  // dead micro-tile (or outside C): never written
            const int64_t crow = row_base + r;
            uint4 val = ld_shared_v4(sbuf + r * 128 + ((chunk ^ (r & 7)) << 4));
            if (p.gate) {
              const uint4 gv = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(p.gate) +
                                                                    (crow * p.ldg + col) * 2));
              val.x &= gate_mask_pair<kBF16>(gv.x);
              val.y &= gate_mask_pair<kBF16>(gv.y);
              val.z &= gate_mask_pair<kBF16>(gv.z);
              val.w &= gate_mask_pair<kBF16>(gv.w);
            }
            *reinterpret_cast<uint4*>(static_cast<uint8_t*>(p.C) + (crow * p.ldc + col) * 2) = val;
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (lane == 0 && warp == 4) SD_STAMP(6, ui);
      if (lane == 0 && warp == 11) SD_STAMP(7, ui);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// unit_off[g] = sum_{g' < g} ceil(counts[g'] / 4) (single block, chunked scan), then the unit table
// tab[unit_off[g] + j] = {g, j}
__global__ void sddmm_plan_kernel(const int32_t* __restrict__ counts, int G, int32_t* __restrict__ unit_off,
                                  const int32_t* __restrict__ slots, int64_t stride, int tiles_per_slice,
                                  int* __restrict__ tab) {
  __shared__ int32_t s[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int g0 = 0; g0 < G; g0 += blockDim.x) {
    const int g = g0 + threadIdx.x;
    const int v = g < G ? (counts[g] + 3) / 4 : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < blockDim.x; o <<= 1) {
      const int add = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += add;
      __syncthreads();
    }
    if (g < G) unit_off[g] = carry + s[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += s[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) unit_off[G] = carry;
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const int o = unit_off[g], n = (counts[g] + 3) / 4;
    const int c = counts[g];
    for (int j = 0; j < n; ++j) {
      int* t = tab + 8 * static_cast<int64_t>(o + j);
      const int nb = min(4, c - 4 * j);
      *reinterpret_cast<int4*>(t) = make_int4(g, nb, g / tiles_per_slice, 0);
      const int32_t* sl = slots + static_cast<int64_t>(g) * stride + 4 * j;
      *reinterpret_cast<int4*>(t + 4) = make_int4(sl[0], nb > 1 ? sl[1] : 0, nb > 2 ? sl[2] : 0, nb > 3 ? sl[3] : 0);
    }
  }
}

int sd_num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

}  // namespace

int64_t sddmm_max_units(const SddmmArgs& a) { return a.n_unit_groups * ceil_div(ceil_div(a.N, 64), 4); }
int64_t sddmm_tab_offset(const SddmmArgs& a) { return (4 * (a.n_unit_groups + 1) + 31) & ~int64_t(31); }
int64_t sddmm_workspace_bytes(const SddmmArgs& a) { return sddmm_tab_offset(a) + 32 * sddmm_max_units(a); }

int launch_sddmm(const SddmmArgs& a, cudaStream_t s) {
  if (a.dtype != kDtypeBF16 && a.dtype != kDtypeF16) return kErrUnsupported;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.batch <= 0) return kOk;
  const int64_t tiles = ceil_div(a.M, 128);
  if (a.n_unit_groups != a.batch * tiles) return kErrShape;
  if (!a.workspace || a.workspace_bytes < sddmm_workspace_bytes(a)) return kErrArg;
  const CUtensorMapDataType dt = a.dtype == kDtypeBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmA, tmB, tmC;
  // A [batch * M, K] (stacked), B^T [batch * N, K]: 64-deep K boxes, 128B swizzle (K-major UMMA operands)
  if (encode_tensor_map_2d(&tmA, dt, a.A, static_cast<uint64_t>(a.K), static_cast<uint64_t>(a.batch * a.M),
                           static_cast<uint64_t>(a.lda) * 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  if (encode_tensor_map_2d(&tmB, dt, a.B, static_cast<uint64_t>(a.K), static_cast<uint64_t>(a.batch * a.N),
                           static_cast<uint64_t>(a.ldb) * 2, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  // C [batch * M, N]: 32-row x 64-column boxes, 128B swizzle (the epilogue's staging layout)
  if (encode_tensor_map_2d(&tmC, dt, a.C, static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.batch * a.M),
                           static_cast<uint64_t>(a.ldc) * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  int32_t* unit_off = static_cast<int32_t*>(a.workspace);
  int* tab = reinterpret_cast<int*>(static_cast<uint8_t*>(a.workspace) + sddmm_tab_offset(a));
  if (a.batch * a.M + 256 >= (1ll << 31) || a.batch * a.N >= (1ll << 31)) return kErrShape;  // 32-bit rows
  sddmm_plan_kernel<<<1, 1024, 0, s>>>(a.unit_counts, static_cast<int>(a.n_unit_groups), unit_off, a.unit_slots,
                                       a.unit_slot_stride, static_cast<int>(ceil_div(a.M, 128)), tab);
  note_launch();
  if (int st = cuda_status()) return st;
  SddmmParams p{};
  p.C = a.C;
  p.ldc = a.ldc;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.batch = static_cast<int>(a.batch);
  p.tiles_per_slice = static_cast<int>(tiles);
  p.ucounts = a.unit_counts;
  p.uslots = a.unit_slots;
  p.ustride = a.unit_slot_stride;
  p.unit_off = unit_off;
  p.unit_tab = tab;
  p.G = static_cast<int>(a.n_unit_groups);
  p.lg0 = (a.g0 & (a.g0 - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(a.g0)) : -1;
  p.lg1 = (a.g1 & (a.g1 - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(a.g1)) : -1;
  p.box_uniform = a.g0 % 32 == 0 && a.g1 % 64 == 0 && a.M % 32 == 0 && a.N % 64 == 0;
  p.diag = PIT_DIAG && getenv("PIT_SD_DIAG") ? atoi(getenv("PIT_SD_DIAG")) : 0;
  p.occ = a.occ;
  p.WG = a.words_per_group;
  p.g0 = a.g0;
  p.g1 = a.g1;
  p.gate = a.gate;
  p.ldg = a.ldgate;
  const int64_t max_units = sddmm_max_units(a);
  const int sms = sd_num_sms();
  const int grid = static_cast<int>(max_units < sms ? (max_units > 0 ? max_units : 1) : sms);
  auto kern = a.dtype == kDtypeBF16 ? sddmm_kernel<true> : sddmm_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSdSmem);
  kern<<<grid, kSdThreads, kSdSmem, s>>>(tmA, tmB, tmC, p);
  note_launch();
  return cuda_status();
}

}  // namespace pit

extern "C" __attribute__((visibility("default"))) int pit_debug_sddmm_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_sd_trace, sizeof(g_sd_trace)) == cudaSuccess ? 0 : 5;
}
