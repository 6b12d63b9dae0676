/*
 * pit_b200.h — C ABI of the B200-native PIT hot path (libpit_b200.so).
 *
 * Drop-in boundary for the reference `pittile` operator API (pkg/src/pittile/__init__.py:9-76).
 * Every entry point is extern "C", takes plain device pointers / sizes, is stream-ordered on the
 * caller's cudaStream_t (passed as void*), never allocates, and returns a pit_status; the message of
 * the last failure on the calling thread is available from pit_last_error().
 *
 * Index layout on the device (replaces MicroTileIndex, index.py:32-50):
 *   counts  int32 [n_groups]                live coordinates per group
 *   slots   int32 [n_groups * pit_grid]     group g's coordinates at slots[g*pit_grid + 0 .. counts[g])
 *                                           in ascending order (== reference workers=1 order)
 *   occ     uint32 [n_groups * words]       group-major occupancy bitmap, words = ceil(pit_grid/32),
 *                                           bit b of word w of group g <=> coordinate 32w+b is live
 * Groups run along the non-PIT micro grid; pit_dim 0 ("m"/"p") or 1 ("k"/"l") (index.py:25).
 */
#ifndef PIT_B200_H
#define PIT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PIT_API __attribute__((visibility("default")))
#else
#define PIT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PIT_OK = 0,
  PIT_ERR_ARG = 1,         /* maps to ValueError subclasses (ExecError / IndexBuildError) */
  PIT_ERR_SHAPE = 2,       /* "shape mismatch" */
  PIT_ERR_LAYOUT = 3,      /* LayoutError */
  PIT_ERR_RANGE = 4,       /* "out of range" */
  PIT_ERR_CUDA = 5,        /* CUDA runtime / driver failure */
  PIT_ERR_UNSUPPORTED = 6  /* combination not implemented on this path */
} pit_status;

typedef enum { PIT_F32 = 0, PIT_F64 = 1, PIT_BF16 = 2, PIT_F16 = 3, PIT_U8 = 4 } pit_dtype;

typedef enum { PIT_PLAN_DENSE = 0, PIT_PLAN_PIT_M = 1, PIT_PLAN_PIT_K = 2 } pit_plan;

/* Last error message of the calling thread (static storage, never NULL). */
PIT_API const char* pit_last_error(void);

/* ABI version (major*100 + minor). */
PIT_API int pit_abi_version(void); /* 104: pit_pack_groups; 103: pit_sddmm; 102: pit_grouped_gemm_args.rows_hint, pit_ep_* / pit_moe_dispatch */

/* Number of kernels this library has launched in the process (monotonic; for launch accounting). */
PIT_API long long pit_kernel_launches(void);

/* Micro-grid geometry of a (s0 x s1) operand under micro-tile (t0,t1) and PIT dim. */
PIT_API int pit_index_geometry(int64_t s0, int64_t s1, int t0, int t1, int pit_dim, int64_t* n_groups, int64_t* pit_grid,
                       int64_t* words_per_group);

/*
 * Online detection from raw values: an element is live iff value != 0.0 (sign bit ignored, so -0.0 is
 * dead; NaN / inf / denormals live). Replaces build_index_from_tensor (index.py:164-173).
 * values(i,j) lives at values + (i*stride0 + j*stride1) * sizeof(dtype); stride1 == 1 (row-major) or
 * stride0 == 1 (column-major) are accepted.
 */
PIT_API int pit_build_index_from_tensor(const void* values, int dtype, int64_t s0, int64_t s1, int64_t stride0,
                                int64_t stride1, int t0, int t1, int pit_dim, uint32_t* occ, int32_t* counts,
                                int32_t* slots, void* stream);

/*
 * Detection from a block annotation: packed = np.packbits of the row-major block grid (MSB first),
 * granularity (g0,g1). Replaces build_index (index.py:102-161) over a SparsityAnnotation
 * (sparsity.py:27-65). counts = slots = NULL: only the occupancy bitmap (no compaction launch).
 */
PIT_API int pit_build_index(const uint8_t* packed, int64_t s0, int64_t s1, int g0, int g1, int t0, int t1, int pit_dim,
                    uint32_t* occ, int32_t* counts, int32_t* slots, void* stream);

/* Plan-selection cover counts (policy.py:129-136 cover_group_counts, for every candidate of
 * selection_candidates policy.py:241-276 at once): for candidate c = (t0, t1, pit_dim) given in the
 * HOST array candidates[3c..3c+2], writes its n_groups live-micro-tile counts to the device array
 * counts, candidates back to back in order. occ_ws is a device scratch of ws_words 32-bit words
 * (at least max_c n_groups*words_per_group, see pit_index_geometry). */
PIT_API int pit_cover_counts(const uint8_t* packed, int64_t s0, int64_t s1, int g0, int g1, int n_candidates,
                             const int32_t* candidates, uint32_t* occ_ws, int64_t ws_words, int32_t* counts,
                             void* stream);

/* Occupancy bitmap from an arbitrary (e.g. reordered) index; *bad set to 1 on a coordinate out of
 * range (sread's "micro-tile coordinate out of range", executor.py:192-193). occ is overwritten. */
PIT_API int pit_index_occupancy(const int32_t* counts, const int32_t* slots, int64_t n_groups, int64_t pit_grid,
                        uint32_t* occ, int32_t* bad, void* stream);

/* Union of live coordinates over all groups, ascending: rows[0..*n_rows). union_ws: words uint32. */
PIT_API int pit_index_union(const uint32_t* occ, int64_t n_groups, int64_t pit_grid, uint32_t* union_ws, int32_t* rows,
                    int32_t* n_rows, void* stream);

/*
 * SRead (executor.py:170-208): gather coords[0..n_coords) of one group into tile (row-major
 * [tile_rows, tile_cols], contiguous). tensor is row-major [s0, s1] with pitch ld (stride1 == 1) or
 * column-major (ld = pitch of a column, pass col_major = 1). zero_fill clears unfilled tile slots.
 */
PIT_API int pit_sread(const void* tensor, int dtype, int64_t s0, int64_t s1, int64_t ld, int col_major, void* tile,
              int64_t tile_rows, int64_t tile_cols, int t0, int t1, int pit_dim, int64_t group,
              const int32_t* coords, int64_t n_coords, int zero_fill, void* stream);

/* SWrite (executor.py:211-264): mirror scatter; accumulate != 0 adds instead of assigning. */
PIT_API int pit_swrite(const void* tile, void* tensor, int dtype, int64_t s0, int64_t s1, int64_t ld, int col_major,
               int64_t tile_rows, int64_t tile_cols, int t0, int t1, int pit_dim, int64_t group,
               const int32_t* coords, int64_t n_coords, int accumulate, void* stream);

/* Sparse matmul against a prebuilt device index (run_matmul_with_index, executor.py:464-516). */
typedef struct {
  int plan;  /* pit_plan */
  int dtype; /* pit_dtype of A, B and C */
  int64_t M, N, K;
  const void* A; /* element (m,k) at A + m*sam + k*sak; pit:k needs sam == 1, pit:m/dense sak == 1 */
  int64_t sam, sak;
  const void* B; /* row-major [K,N], pitch ldb */
  int64_t ldb;
  void* C; /* row-major [M,N], pitch ldc; every element is written */
  int64_t ldc;
  int t0, t1; /* plan micro-tile */
  const int32_t* counts; /* pit:k: required; pit:m: optional (enables global dead-K-block skipping) */
  const int32_t* slots;
  int64_t slot_stride; /* = pit_grid */
  int64_t n_groups;
  const uint32_t* occ; /* pit:m: group-major occupancy */
  int64_t words_per_group;
  const int32_t* rows;   /* pit:m: union rows (pit_index_union) */
  const int32_t* n_rows; /* pit:m: device scalar */
  int64_t n_rows_bound;  /* pit:m: host upper bound on *n_rows (M is always safe) */
  int force_simt;        /* 1: CUDA-core path even for bf16/fp16 */
  /* Batched product over a prevalent axis (heads / slices), pit:k and dense only.
   * batch <= 1: a single product. batch > 1: M is the per-slice extent; A and C hold the slices
   * stacked along M ([batch*M, K] col-major / [batch*M, N] row-major), slice b of B starts at
   * B + b*b_batch_stride elements, and the pit:k index is the stacked one (n_groups = batch*M/t0,
   * so M must be a multiple of t0) -- what one detection pass over the stacked A produces. */
  int64_t batch;
  int64_t b_batch_stride;
  /* Caller-owned device scratch (may be NULL / 0): the gathered-K path for few, unequal groups
   * (e.g. attention with global query rows) splits long groups over several CTAs and reduces their
   * partial tiles; without scratch it runs unsplit. Size from pit_spmm_workspace_bytes. */
  void* workspace;
  int64_t workspace_bytes;
} pit_spmm_args;

PIT_API int pit_spmm(const pit_spmm_args* args, void* stream);

/* Scratch bytes pit_spmm can use for these arguments (0: none needed). Host-only, no GPU work. */
PIT_API int64_t pit_spmm_workspace_bytes(const pit_spmm_args* args);

/* 1 if the tcgen05 tensor-core path covers these arguments, else 0 (CUDA-core path). */
PIT_API int pit_spmm_uses_tensor_cores(const pit_spmm_args* args);

/*
 * Grouped gathered-row GEMM (batched / per-expert PIT plans). G groups; group g has
 * counts[g] rows, packed at offsets[g] (offsets[G+1]); tile_offsets[G+1] = prefix of ceil(counts/128).
 * Row i of group g reads A row row_src[g*src_stride + i] (or offsets[g]+i when row_src is NULL) and
 * writes C row row_dst[g*dst_stride + i] (or offsets[g]+i), against rows [g*K, (g+1)*K) of the stacked
 * B [G*K, N]. Epilogue: act (0 none, 1 ReLU) then * row_scale[C row] (if non-NULL). bf16 / fp16 only.
 */
typedef struct {
  int dtype;
  const void* A;
  int64_t lda, rows_a;
  const void* B;
  int64_t ldb;
  void* C;
  int64_t ldc;
  int64_t N, K, G;
  const int32_t* counts;
  const int32_t* offsets;
  const int32_t* tile_offsets;
  const int32_t* row_src;
  int64_t src_stride;
  const int32_t* row_dst;
  int64_t dst_stride;
  const float* row_scale;
  int act;
  int64_t max_tiles; /* host upper bound on tile_offsets[G] (e.g. ceil(total_rows/128) + G) */
  int64_t rows_hint; /* expected total rows when rows_a is only a capacity (0: rows_a); picks the kernel */
} pit_grouped_gemm_args;

PIT_API int pit_grouped_gemm(const pit_grouped_gemm_args* args, void* stream);

/*
 * MoE routing as a PIT index: top-1 argmax of logits [T, E] (ties -> lowest expert), softmax
 * probability of the winner as gate[T], expert[T], and the expert -> token index of the one-hot
 * routing mask (== build_index(from_mask(onehot,(1,1)),(1,1),"m")): counts[E], slots[E*T] ascending.
 * occ: workspace of E*ceil(T/32) words.
 */
PIT_API int pit_moe_route(const void* logits, int dtype, int64_t T, int64_t E, int32_t* expert, float* gate,
                          uint32_t* occ, int32_t* counts, int32_t* slots, void* stream);

/* offsets[G+1], tile_offsets[G+1] from counts[G]; if perm != NULL also the flattened token order
 * perm[offsets[g]+i] = slots[g*stride+i] (max_count = an upper bound on any counts[g]). */
PIT_API int pit_moe_plan(const int32_t* counts, int64_t G, const int32_t* slots, int64_t stride, int32_t* offsets,
                         int32_t* tile_offsets, int32_t* perm, int64_t max_count, void* stream);

/* Expert-parallel receive plan: rc[W*El] = tokens received from rank r for local expert e (rank-major
 * receive buffer). rows[e*stride + i] = receive-buffer row of the i-th token of local expert e; counts[El]. */
PIT_API int pit_moe_recv_plan(const int32_t* rc, int64_t W, int64_t El, int32_t* rows, int64_t stride,
                              int32_t* counts, void* stream);

/* SRead of whole rows: dst row i = src row rows[i] (row_bytes each; pitches in bytes). */
PIT_API int pit_gather_rows(const void* src, int64_t ld_src_bytes, const int32_t* rows, int64_t n, int64_t row_bytes,
                            void* dst, int64_t ld_dst_bytes, void* stream);

/* Group-wise SRead with device counts (the MoE FFN1 input in expert order, so the grouped GEMM reads it by TMA):
 * dst row offsets[g] + i = src row rows[g*stride + i] for i < counts[g], g < G; max_count bounds every count.
 * 16-byte aligned rows and pitches (bytes). */
PIT_API int pit_pack_groups(const void* src, int64_t ld_src_bytes, const int32_t* rows, int64_t stride,
                            const int32_t* counts, const int32_t* offsets, int64_t G, int64_t max_count,
                            int64_t row_bytes, void* dst, int64_t ld_dst_bytes, void* stream);

/* SWrite of whole rows with a per-destination-row scale (MoE combine): dst[rows[i]] = scale[rows[i]] * src[i]. */
PIT_API int pit_scatter_rows_scaled(const void* src, int dtype, int64_t ld_src, const int32_t* rows, int64_t n,
                                    int64_t width, const float* scale, void* dst, int64_t ld_dst, void* stream);

/*
 * Output-sparse matmul (SDDMM): C = A . B computed and stored only inside the live
 * micro-tiles of C's annotation. No reference counterpart is wired: the reference documents the
 * output-side (n-axis) plan as the mirror of pit:m and leaves it unimplemented (pkg/README.md:150-153,
 * SPEC.md:496). A row-major [batch*M, K]; B column-major per slice, passed as B^T row-major
 * [batch*N, K]; C row-major [batch*M, N]. unit_* = index of C's annotation at micro (128, 64) with the
 * column axis permuted (build_index(ann, (128, 64), "k")); occ = its occupancy at micro (g0, g1) (the
 * annotation granularity, g1 % 8 == 0). Elements of dead micro-tiles of C are never written. gate
 * (optional, same layout as C): a stored element is zeroed where gate <= 0 (ReLU-masked gradient).
 * bf16 / fp16; M % 128 == 0 when batch > 1; N, K, pitches multiples of 8. Workspace:
 * pit_sddmm_workspace_bytes.
 */
typedef struct {
  int dtype;
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  void* C;
  int64_t ldc;
  int64_t M, N, K, batch;
  const int32_t* unit_counts;
  const int32_t* unit_slots;
  int64_t unit_slot_stride, n_unit_groups;
  const uint32_t* occ;
  int64_t words_per_group;
  int g0, g1;
  const void* gate;
  int64_t ldgate;
  void* workspace;
  int64_t workspace_bytes;
} pit_sddmm_args;

PIT_API int64_t pit_sddmm_workspace_bytes(const pit_sddmm_args* args);
PIT_API int pit_sddmm(const pit_sddmm_args* args, void* stream);

/*
 * Expert-parallel MoE exchange over NVLink peer memory (SURVEY 8(b) pit_moe_dispatch, 8(e)). No reference
 * counterpart: the reference has no multi-GPU code; this is the cross-GPU form of the SRead that packs an
 * expert group's token rows and of the SWrite that scatters its outputs (index.py:102-173 routing index,
 * executor.py:170-264 gather/scatter semantics). One region per rank (pit_ep_region_alloc), exported to the
 * other ranks of the node through CUDA IPC; every call is stream-ordered with no host synchronisation
 * (CUDA-graph capturable). Region layout (pit_ep_region_layout): header, dispatch flags[W], combine
 * flags[W], counts[W][El] (received per source rank and local expert), recv[W*cap rows], y[W*cap rows]
 * (row r of source s at s*cap + position).
 */
typedef struct {
  int rank, world;
  int64_t experts_local; /* El: experts per rank; global expert e lives on rank e / El */
  int64_t capacity;      /* max tokens any rank sends per layer (its T) */
  int64_t row_bytes;     /* d_model * element size, multiple of 16 */
  void* local;           /* this rank's region */
  void* const* peers;    /* DEVICE array [world] of region pointers as mapped in this process */
} pit_ep_args;

/* out[6] = byte offsets {dispatch flags, combine flags, counts, recv, y, total size}. */
PIT_API int pit_ep_region_layout(int64_t world, int64_t experts_local, int64_t capacity, int64_t row_bytes,
                                 int64_t* out);
/* cudaMalloc + zero a region of `bytes` on the current device (flags and epochs start at 0). */
PIT_API int pit_ep_region_alloc(int64_t bytes, void** out);
PIT_API int pit_ep_region_free(void* region);
/* CUDA IPC: 64-byte handle of a region; open a peer's handle in this process (close with pit_ep_ipc_close). */
PIT_API int pit_ep_ipc_handle(void* region, void* handle64);
PIT_API int pit_ep_ipc_open(const void* handle64, void** out);
PIT_API int pit_ep_ipc_close(void* mapped);
/* nonzero if a wait in this region timed out (a peer never arrived); synchronous read. */
PIT_API int pit_ep_error(void* region, int* out);

/* Dispatch = pack + send fused: token perm[i] (expert order, expert prefix offsets[E+1], E = world*El) is
 * stored straight into rank (e/El)'s recv region over NVLink; counts[E] go to the peers' counts rows;
 * the last block publishes this rank's epoch to every peer. x: [T, row] with row pitch ldx_bytes. */
PIT_API int pit_moe_dispatch(const pit_ep_args* ep, const void* x, int64_t ldx_bytes, int64_t T, const int32_t* perm,
                             const int32_t* offsets, const int32_t* counts, void* stream);
/* Wait for every peer's dispatch of this epoch, then rows[e*stride + j] = recv row of local expert e's j-th
 * token (source-rank order), counts[El]. */
PIT_API int pit_moe_recv_plan_ep(const pit_ep_args* ep, int32_t* rows, int64_t stride, int32_t* counts, void* stream);
/* Publish "y ready" (the expert outputs are in this rank's y region) to every peer. */
PIT_API int pit_moe_signal(const pit_ep_args* ep, void* stream);
/* Combine = pull + SWrite * gate fused: wait for every peer's y flag, then out[perm[i]] = gate[perm[i]] *
 * y(rank e/El)[rank*cap + position]. dtype bf16 / f16 / f32. */
PIT_API int pit_moe_combine(const pit_ep_args* ep, int dtype, int64_t T, const int32_t* perm, const int32_t* offsets,
                            const float* gate, void* out, int64_t ldo_bytes, void* stream);

/*
 * Sparse row reduction (run_sparse_reduce_sum, executor.py:540-613): out[r] = sum of A[r, l] (row-major,
 * pitch lda) over live micro-tiles. mode 0 dense; mode 1 pit:l (occ groups = rows, micro (1,1));
 * mode 2 pit:p (occ groups = l-blocks of block_l columns, coordinates = rows). Dead rows are exact 0.
 */
PIT_API int pit_reduce_rows(const void* A, int dtype, int64_t P, int64_t L, int64_t lda, const uint32_t* occ,
                            int64_t words_per_group, int mode, int block_l, void* out, void* stream);

/* Pitched host<->device copy on the caller's stream (cudaMemcpy2DAsync, direction inferred): moves
 * column slabs of row-major operands for the pipelined host-buffer path. */
PIT_API int pit_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                             int64_t height, void* stream);

/* f64 verification oracle: C = A @ B with multiply-then-add in ascending k (no FMA), bit-identical to
 * the reference's run_dense_reference (executor.py:267-283). A(i,k) at A + i*s0 + k*s1. */
PIT_API int pit_dense_reference_f64(const double* A, int64_t s0, int64_t s1, const double* B, int64_t ldb, double* C,
                            int64_t M, int64_t N, int64_t K, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PIT_B200_H */
