// Internal launcher interfaces shared by the .cu files and the C-ABI layer (pit_capi.cu).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pit {

// dtype codes shared with include/pit_b200.h
enum : int {
  kDtypeF32 = 0,
  kDtypeF64 = 1,
  kDtypeBF16 = 2,
  kDtypeF16 = 3,
  kDtypeU8 = 4,
};

// status codes shared with include/pit_b200.h
enum : int {
  kOk = 0,
  kErrArg = 1,
  kErrShape = 2,
  kErrLayout = 3,
  kErrRange = 4,
  kErrCuda = 5,
  kErrUnsupported = 6,
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int dtype_bytes(int dtype) {
  switch (dtype) {
    case kDtypeF32:
      return 4;
    case kDtypeF64:
      return 8;
    case kDtypeBF16:
    case kDtypeF16:
      return 2;
    case kDtypeU8:
      return 1;
    default:
      return 0;
  }
}

int cuda_status();  // maps cudaGetLastError() to kOk / kErrCuda and records the message
void note_launch(int n = 1);  // process-wide count of kernels this library launched

// ------------------------------------------------------------------ K1 detect
struct DetectValuesArgs {
  const void* x;  // physical row-major [R, C], row pitch ld elements
  int dtype;
  int64_t R, C, ld;
  int tr, tc;    // micro-tile in physical orientation
  int pit_phys;  // 0: coordinates run along physical rows (groups = micro-columns); 1: along columns
  uint32_t* occ; // [n_groups][WG] group-major bitmap, fully overwritten
};

struct DetectBitsArgs {
  const uint8_t* packed;  // MSB-first packed block bits, row-major over the block grid
  int64_t s0, s1;         // logical tensor shape
  int g0, g1;             // block granularity
  int t0, t1;             // micro-tile
  int pit_dim;            // 0 or 1 (logical)
  uint32_t* occ;
};

int launch_detect_values(const DetectValuesArgs& a, cudaStream_t s);
int launch_detect_bits(const DetectBitsArgs& a, cudaStream_t s);
// detect_bits + compact; one launch when the geometry allows (power-of-two, coordinate blocks >= 32
// coordinates wide)
int launch_index_from_bits(const DetectBitsArgs& a, int32_t* counts, int32_t* slots, int64_t slot_stride,
                           cudaStream_t s);
int launch_compact(const uint32_t* occ, int64_t n_groups, int64_t WG, int32_t* counts, int32_t* slots,
                   int64_t slot_stride, cudaStream_t s);
int launch_union(const uint32_t* occ, int64_t n_groups, int64_t WG, uint32_t* uni, cudaStream_t s);
int launch_occ_counts(const uint32_t* occ, int64_t n_groups, int64_t WG, int32_t* counts, cudaStream_t s);
int launch_slots_to_occ(const int32_t* counts, const int32_t* slots, int64_t slot_stride, int64_t n_groups,
                        int64_t WG, int64_t pit_grid, uint32_t* occ, int* bad, cudaStream_t s);

// ---------------------------------------------------------- K5 SRead / SWrite
struct GatherArgs {
  void* src_or_dst;     // tensor, logical [R, C], element (i,j) at i*st0 + j*st1
  void* tile;           // tile buffer, row-major [TR, TC] (contiguous)
  int dtype;
  int64_t R, C, st0, st1;
  int64_t TR, TC;
  int t_d, t_o;          // micro extent along the gather axis / the other axis
  int d;                 // logical gather axis (pit_dim)
  const int32_t* coords; // device, n_coords entries (already offset by start)
  int64_t n_coords;
  int64_t off_o;         // element offset along the other axis (group * t_o)
  int accumulate;        // swrite only
  int zero_fill;         // sread only: clear slots that receive no data (executor.py:195-198)
};
int launch_sread(const GatherArgs& a, cudaStream_t s);
int launch_swrite(const GatherArgs& a, cudaStream_t s);

// ------------------------------------------------------------------- SpMM
enum : int { kPlanDense = 0, kPlanPitM = 1, kPlanPitK = 2 };

struct SpmmArgs {
  int plan;     // kPlanDense / kPlanPitM / kPlanPitK
  int dtype;    // operands and C share a dtype; accumulation fp32 (fp64 for f64)
  int64_t M, N, K;
  const void* A;  // logical [M,K]; element (m,k) at A + m*sam + k*sak
  int64_t sam, sak;
  const void* B;  // row-major [K,N], pitch ldb
  int64_t ldb;
  void* C;        // row-major [M,N], pitch ldc; fully written by the call
  int64_t ldc;
  int t0, t1;     // plan micro-tile (logical)
  // index (device): pit:k groups = M-blocks (coords = k), pit:m groups = K-blocks (coords = rows)
  const int32_t* counts;
  const int32_t* slots;
  int64_t slot_stride;
  int64_t n_groups;
  const uint32_t* occ;      // group-major bitmap [n_groups][WG] (pit:m)
  int64_t WG;
  const int32_t* rows;      // pit:m union rows (ascending), n_rows entries
  const int32_t* n_rows;    // device scalar
  int64_t n_rows_host;      // upper bound used for the grid (<= M)
  int64_t batch = 1;        // pit:k slices stacked along M (see pit_spmm_args)
  int64_t b_batch_stride = 0;
  void* ws = nullptr;       // caller scratch (split gathered-K units), may be null
  int64_t ws_bytes = 0;
};

int launch_spmm_simt(const SpmmArgs& a, cudaStream_t s);
int launch_reduce_rows(const void* A, int dtype, int64_t P, int64_t L, int64_t lda, const uint32_t* occ, int64_t WG,
                       int mode, int block_l, void* out, cudaStream_t s);
int launch_dense_ref_f64(const double* A, int64_t s0, int64_t s1, const double* B, int64_t ldb, double* C, int64_t M,
                         int64_t N, int64_t K, cudaStream_t s);
int launch_spmm_tc(const SpmmArgs& a, cudaStream_t s);  // bf16 / fp16 tcgen05 paths
bool spmm_tc_supported(const SpmmArgs& a);
int64_t spmm_tc_workspace_bytes(const SpmmArgs& a);  // scratch the tcgen05 path can use (0: none)
int gk2_trace_read(unsigned long long* host);  // diagnostic timeline (PIT_GK2_DIAG bit 4)

// ----------------------------------------- K3s: pit:m at very high sparsity (pit_gm_sparse.cu)
// The sparse path runs when live micro-tiles <= 1/kSparseDen of the (row, K-group) grid (decided on
// the device from the index counts).
constexpr int kSparseDen = 48;
struct GmSparseWs {  // byte offsets into the caller's workspace
  int64_t flag, cnt, off, U, pre, rows, X, part, bytes;
};
int64_t gm_sparse_bound_rows(int64_t M, int64_t nkg, int S);
int gm_sg();  // columns per supergroup (256; PIT_GM_SG=512)
GmSparseWs gm_sparse_layout(int64_t M, int64_t N, int64_t WG, int S, int64_t bound_rows);
int launch_gm_sparse_prep(const int32_t* counts, int nkg, int64_t M, int gps, int S, const uint32_t* occ, int64_t WG,
                          uint8_t* ws, const GmSparseWs& w, cudaStream_t s);
int launch_gm_sparse_pack(const int32_t* counts, int nkg, const void* A, int64_t lda_bytes, int S, int64_t M,
                          const uint32_t* occ, int64_t WG, int t1, int64_t bound_rows, uint8_t* ws, const GmSparseWs& w,
                          cudaStream_t s);
int launch_gm_sparse_reduce(const int32_t* counts, int nkg, int dtype, int S, int64_t WG, int64_t N, void* C,
                            int64_t ldc, int64_t M, uint8_t* ws, const GmSparseWs& w, cudaStream_t s);

// Grouped gathered-row GEMM (MoE experts, batched per-slice plans): see rowgemm in pit_spmm_tc.cu.
struct GroupedGemmArgs {
  int dtype;
  const void* A;  // row-major [rows_a, K], pitch lda
  int64_t lda, rows_a;
  const void* B;  // stacked row-major [G, K, N], pitch ldb
  int64_t ldb;
  void* C;        // row-major, pitch ldc
  int64_t ldc;
  int64_t N, K, G;
  const int32_t* counts;        // [G]
  const int32_t* offsets;       // [G+1]
  const int32_t* tile_offsets;  // [G+1]
  const int32_t* row_src;
  int64_t src_stride;
  const int32_t* row_dst;
  int64_t dst_stride;
  const float* row_scale;
  int act;
  int64_t max_tiles;
  int64_t rows_hint;  // expected total rows (0: rows_a)
};
int launch_rowgemm(const GroupedGemmArgs& g, cudaStream_t s);

// ------------------------------------------------------------------- MoE dispatch
int launch_moe_route(const void* logits, int dtype, int64_t T, int E, int32_t* expert, float* gate, uint32_t* occ,
                     int32_t* counts, int32_t* slots, cudaStream_t s);
int launch_moe_plan(const int32_t* counts, int G, const int32_t* slots, int64_t stride, int32_t* offsets,
                    int32_t* tile_offsets, int32_t* perm, int64_t max_count, cudaStream_t s);
int launch_moe_recv_plan(const int32_t* rc, int W, int El, int32_t* rows, int64_t stride, int32_t* counts,
                         cudaStream_t s);
int launch_gather_rows(const void* src, int64_t ld_src_bytes, const int32_t* rows, int64_t n, int64_t row_bytes,
                       void* dst, int64_t ld_dst_bytes, cudaStream_t s);
int launch_pack_groups(const void* src, int64_t ld_src_bytes, const int32_t* rows, int64_t stride,
                       const int32_t* counts, const int32_t* offsets, int64_t G, int64_t max_count, int64_t row_bytes,
                       void* dst, int64_t ld_dst_bytes, cudaStream_t s);
int launch_scatter_rows_scaled(const void* src, int dtype, int64_t ld_src, const int32_t* rows, int64_t n,
                               int64_t width, const float* scale, void* dst, int64_t ld_dst, cudaStream_t s);

// ------------------------------------------- expert-parallel exchange over peer memory (pit_ep.cu)
struct EpArgs {
  int rank, world;
  int64_t experts_local, capacity, row_bytes;
  void* local;              // this rank's region
  void* const* peers;       // device array [world]: every rank's region as mapped here (peers[rank] = local)
};
void ep_region_layout(int W, int64_t El, int64_t cap, int64_t row_bytes, int64_t out[6]);
int launch_ep_dispatch(const EpArgs& a, const void* x, int64_t ldx_bytes, int64_t T, const int32_t* perm,
                       const int32_t* offsets, const int32_t* counts, cudaStream_t s);
int launch_ep_recv_plan(const EpArgs& a, int32_t* rows, int64_t stride, int32_t* counts, cudaStream_t s);
int launch_ep_signal(const EpArgs& a, cudaStream_t s);
int launch_ep_combine(const EpArgs& a, int dtype, int64_t T, const int32_t* perm, const int32_t* offsets,
                      const float* gate, void* out, int64_t ldo_bytes, cudaStream_t s);

// ------------------------------------------------------- output-sparse matmul (pit_sddmm.cu)
struct SddmmArgs {
  int dtype;
  const void* A;  // [batch * M, K] row-major, pitch lda
  int64_t lda;
  const void* B;  // B^T [batch * N, K] row-major (B column-major per slice), pitch ldb
  int64_t ldb;
  void* C;        // [batch * M, N] row-major, pitch ldc
  int64_t ldc;
  int64_t M, N, K, batch;
  const int32_t* unit_counts;  // index of C at micro (128, 64), pit axis = columns
  const int32_t* unit_slots;
  int64_t unit_slot_stride, n_unit_groups;
  const uint32_t* occ;  // C's annotation occupancy at micro (g0, g1), groups = row blocks
  int64_t words_per_group;
  int g0, g1;
  const void* gate;  // optional [batch * M, N], pitch ldgate: stored elements zeroed where gate <= 0
  int64_t ldgate;
  void* workspace;
  int64_t workspace_bytes;
};
int64_t sddmm_workspace_bytes(const SddmmArgs& a);
int launch_sddmm(const SddmmArgs& a, cudaStream_t s);

// Driver entry point for cuTensorMapEncodeTiled (resolved through the runtime, no -lcuda).
CUresult encode_tensor_map_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                              uint64_t outer, uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                              CUtensorMapSwizzle swizzle);
CUresult encode_tensor_map_3d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
                              uint64_t d2, uint64_t pitch1_bytes, uint64_t pitch2_bytes, uint32_t box0, uint32_t box1,
                              CUtensorMapSwizzle swizzle);

}  // namespace pit
