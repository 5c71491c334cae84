/* spdistal_b200.h -- C-ABI of the B200-native SpDISTAL leaf/partition backend.
 *
 * This is the drop-in boundary under the reference's runtime
 * (dspar, /root/reference/proj/core).  The reference's hot path is
 *
 *   Plan plan(const ScheduledStatement&, const TensorSet&)         planner.hpp:42
 *   ExecResult execute(const Plan&, const TensorSet&, const MachineGrid&,
 *                      const Residency&, ExecMode)                  sim.hpp:121-122
 *
 * and the level-function "plugin" interface of the format abstraction
 * (LevelPartitioner, partition_from_parent/child, level_partition.hpp:23-85).
 * The entry points below replace, one for one, the pieces of that path that
 * move to the GPU: tensor storage (tensor.hpp:54-114), the universe / nonzero
 * level partitions (level_partition.cpp:134-212, deppart.cpp:15-53,
 * planner.cpp:10-69), the six leaf kernels executed by LeafRun
 * (sim.cpp:258-494), the deterministic reduce_combine (sim.cpp:791-811) and the
 * two-phase output assembly (sim.cpp:647-789).  INTEGRATION.md shows the
 * ExecMode::Gpu adapter a maintainer adds to sim.cpp to call them.
 *
 * Conventions
 *  - Plain C types only: int64_t coordinates/positions, double values, opaque
 *    handles.  No torch or CUDA types appear in a signature (streams are
 *    passed as void*).
 *  - Every function returns an int status mirroring the reference's error
 *    classes and the CLI's exit-code mapping (cli.cpp:297-319):
 *      SPD_OK (0); SPD_ERR_RUNTIME (1) = std::runtime_error / logic_error /
 *      ClosureViolation; SPD_ERR_VALIDATION (2) = ValidationError /
 *      ParseError / std::invalid_argument.  spd_last_error() returns the
 *      thread-local message of the last failure.
 *  - Device storage format: a compressed level is an int64 row pointer
 *    (parent positions + 1 entries), lossless versus the reference's inclusive
 *    (lo,hi) pos pairs because pos tiles [0,nnz) with canonical empties
 *    (tensor.cpp:258-281); crd int64; vals fp64.  Dense levels store nothing
 *    but their extents (dom), as in the reference.
 *  - Asynchrony: calls are enqueued on the context's stream; functions that
 *    return host data synchronise that stream.  Nothing falls back to the CPU:
 *    without a CUDA device every compute entry point fails with SPD_ERR_RUNTIME.
 */
#ifndef SPDISTAL_B200_H
#define SPDISTAL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPD_OK 0
#define SPD_ERR_RUNTIME 1
#define SPD_ERR_VALIDATION 2

#define SPD_DENSE 0      /* LevelKind::Dense,      tensor.hpp:13 */
#define SPD_COMPRESSED 1 /* LevelKind::Compressed, tensor.hpp:13 */

typedef struct spd_context spd_context;
typedef struct spd_tensor spd_tensor;

/* CoordRange (index_space.hpp:12-23): inclusive [lo, hi], empty iff lo > hi. */
typedef struct spd_range {
  int64_t lo, hi;
} spd_range;

/* One colour of one distributed loop (PlanLoop, plan.hpp:49-62) in compact
 * range form -- what the reference materialises as index sets (Partition,
 * partition.hpp:16-46) is, for the contiguous partitions of these schedules,
 * fully described by these spans:
 *   color:  PlanLoop::color_bounds[c] (coordinates for a universe split,
 *           positions for a nonzero split)
 *   q:      leaf-level crd/vals positions owned (image of the rows /
 *           the nonzero entry itself)
 *   par:    span of the split level's pos partition: the parent entries whose
 *           range meets q (preimage colours only the non-empty ones,
 *           deppart.cpp:46)
 *   top:    top-level coordinate bounds: the universe entry, or
 *           project_to_universe's [min,max] (planner.cpp:50-69) for a nonzero
 *           split -- the bounds other tensors (the output) are partitioned by. */
typedef struct spd_color {
  spd_range color, q, par, top;
} spd_color;

/* Stats (sim.hpp:25-36) of one execute. */
typedef struct spd_stats {
  int64_t workers;
  int64_t combines; /* extra contributions summed by reduce_combine */
  double imbalance; /* max work * workers / total work; 1 when no work */
  double kernel_ms; /* device time of the leaf + combine launches (CUDA events) */
  int64_t launches; /* kernels launched by this call */
} spd_stats;

/* ---- errors ----------------------------------------------------------- */
const char* spd_last_error(void);
/* Semantic version of this ABI (major*10000 + minor*100 + patch). */
int spd_abi_version(void);

/* ---- (1) context: one per GPU (one process per GPU) -------------------- */
/* Number of CUDA devices visible to this process (0 without a GPU). */
int spd_device_count(int* count);
/* device: CUDA ordinal.  stream: a cudaStream_t to enqueue on (cudaStreamLegacy
 * (0x1) selects the legacy default stream), or NULL for a context-owned
 * non-blocking stream. */
int spd_context_create(int device, void* stream, spd_context** out);
int spd_context_destroy(spd_context* ctx);
int spd_context_synchronize(spd_context* ctx);
/* Multi-GPU: rank/world of this context inside one NCCL communicator over
 * NVLink.  `unique_id` is the 128-byte ncclUniqueId created by rank 0
 * (spd_nccl_unique_id) and broadcast by the host's launcher.  Collective
 * calls check their arguments before the first collective they enqueue, and
 * spd_tensor_place broadcasts the root's input status first, so argument
 * errors fail on every rank together; a runtime failure on one rank after
 * the others entered a collective leaves them waiting -- spd_context_abort
 * on the waiting ranks ends it (their calls return an error), then destroy
 * the contexts. */
int spd_nccl_unique_id(void* out128);
int spd_context_init_comm(spd_context* ctx, const void* unique_id128, int rank, int world);
int spd_context_rank(const spd_context* ctx, int* rank, int* world);
/* Aborts the context's communicator (ncclCommAbort): collectives this rank
 * has queued stop waiting for their peers and the calls blocked on them
 * return an error.  For a host that runs several ranks in one process (the
 * drop-in's one thread per GPU): when one rank fails, abort the others'
 * communicators instead of leaving them waiting.  The context stays usable
 * without a communicator; destroy it afterwards. */
int spd_context_abort(spd_context* ctx);
/* In-place all-gather over the context's communicator (NVLink): rank r's
 * `bytes_per_rank` bytes at dev_buf + r*bytes_per_rank are gathered into every
 * rank's dev_buf.  Places a replicated dense operand (x / C / D) from a
 * block-distributed one -- the only data-path collective besides the
 * boundary-row exchange of the leaf ops. */
int spd_allgather(spd_context* ctx, void* dev_buf, int64_t bytes_per_rank);

/* ---- (2) tensors: the coordinate-tree encoding (tensor.hpp:54-114) ------ */
/* Upload from the reference's own host storage, SparseTensor::from_parts
 * (tensor.cpp:184-197): per stored level, dense levels pass NULL; compressed
 * levels pass inclusive (lo,hi) pos pairs (2*npos int64) and crd.  Stored
 * levels follow the format's level grouping (consecutive dense modes collapse,
 * tensor.cpp:30-41).  kinds/mode_order describe the FormatSpec (one entry per
 * mode).  The pairs are staged with cudaMemcpyAsync, converted to row
 * pointers and checked against SparseTensor::validate (tensor.cpp:241-286) on
 * the GPU; a violated invariant returns SPD_ERR_VALIDATION. */
int spd_tensor_upload(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                      const int* mode_order, const int64_t* const* pos_pairs,
                      const int64_t* const* crd, const double* vals, spd_tensor** out);
/* Re-stages an uploaded tensor from new host arrays of the same geometry
 * (same format, dims and per-level position counts; new pos pairs, crd and
 * vals), into its existing device buffers: the per-step upload of a stream of
 * same-shaped problems, with no device allocation.  Validated like
 * spd_tensor_upload; derived indices (compacted rows, hot columns) are
 * rebuilt on next use; a partition of this tensor on ctx is dropped.  A
 * position count that differs returns SPD_ERR_VALIDATION. */
int spd_tensor_restage(spd_context* ctx, spd_tensor* t, const int64_t* const* pos_pairs,
                       const int64_t* const* crd, const double* vals);
/* Mismatched placement: moves a piece (spd_tensor_place /
 * spd_tensor_upload_piece, split 1 rows or 2 nonzeros) to colour `rank` of
 * the compute partition need_split -- the data the reference's ledger
 * charges (spd_ledger_bytes).  Every GPU derives every GPU's held and needed
 * leaf position spans from the row pointer it holds; the overlaps travel as
 * grouped NCCL send/recv of crd and vals.  Collective over the communicator.
 * *bytes_in = crd + vals bytes this GPU received. */
int spd_tensor_repartition(spd_context* ctx, const spd_tensor* piece, int need_split,
                           spd_tensor** out, int64_t* bytes_in);
/* The reference's communication ledger for a CSR-like tensor (transfer_bytes,
 * sim.cpp:134-147, over residency_from_placements :547-566; 16 B per pos
 * range, 8 B per crd, 8 B per val, sim.hpp:21-23): bytes_out[w] for worker w
 * of `pieces` = the bytes of colour w of the compute partition (need_split:
 * 1 row split, 2 nonzero split)
 * that colour w of the placement (held_split: 1 rows "B(x,y) onto M(x)",
 * 2 nonzeros "... fuse(x,y->f) onto M(~f)", 3 replicated) does not hold.
 * A matched placement (need == held) charges 0.  Leaves the
 * compute partition on ctx. */
int spd_ledger_bytes(spd_context* ctx, const spd_tensor* t, int need_split, int held_split,
                     int64_t pieces, int64_t* bytes_out);
/* The ledger's primitive for arbitrary placements: missing_count of
 * transfer_bytes (sim.cpp:76-84, 134-147) evaluated on the GPU for `npairs`
 * pairs of sorted, duplicate-free int64 index sets in host memory --
 * missing[p] = |{ i in needed[p] : i not in held[p] }|.  The integration
 * adapter feeds it the needed sets of every (worker, tensor, region) of a
 * plan and the Residency's held sets, so execute_gpu's bytes_by_tensor is
 * the reference's ledger (replaces the accounting loop of execute,
 * sim.cpp:868-887). */
int spd_ledger_missing(spd_context* ctx, int64_t npairs, const int64_t* const* needed,
                       const int64_t* n_needed, const int64_t* const* held, const int64_t* n_held,
                       int64_t* missing);
/* This GPU's piece of a CSR-like ("ds") matrix staged from host arrays: the
 * whole pos level (pairs, O(rows)) is uploaded, converted and checked, the
 * compute partition (split 1 = rows, 2 = nonzeros; spd_partition_universe /
 * spd_partition_nonzero over the communicator's GPUs, one colour per GPU) is
 * computed on the GPU, and only this GPU's colour of crd / vals is copied
 * from `crd[1]` / `vals` (whole host arrays, indexed by global position) --
 * the matched placement of lower_tdn (planner.cpp:361-439) for which the
 * ledger charges 0 bytes, read from host memory.  Leaves the
 * partition on ctx; the piece runs every leaf op for this GPU's colour and
 * can be re-staged with spd_tensor_restage (a row split's range may move).
 * order 3 (dss / sss 3-tensors, the CSF of SpTTV / SpMTTKRP): the upper
 * levels and the leaf pos are staged whole, the leaf crd / vals as this
 * GPU's colour of the leaf-level nonzero split (2) or of the top-level row
 * split (1); such pieces are not re-stageable.
 * Without a communicator (world 1) the piece is the whole tensor. */
int spd_tensor_upload_piece(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                            const int* mode_order, const int64_t* const* pos_pairs,
                            const int64_t* const* crd, const double* vals, int split,
                            spd_tensor** out);
/* Same as spd_tensor_upload, with host row pointers (device format) instead
 * of pos pairs. */
int spd_tensor_upload_rowptr(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                             const int* mode_order, const int64_t* const* rowptr,
                             const int64_t* const* crd, const double* vals, int validate,
                             spd_tensor** out);
/* Zero-copy wrap of device-resident arrays in device format (the caller keeps
 * ownership and must keep them alive; for device-resident pipelines). */
int spd_tensor_wrap_device(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                           const int* mode_order, int64_t* const* rowptr_dev,
                           int64_t* const* crd_dev, double* vals_dev, spd_tensor** out);
int spd_tensor_destroy(spd_tensor* t);
/* Geometry: stored levels, per level kind / parent positions / positions
 * (level_positions, tensor.hpp:80-82) and the leaf (vals) count. */
int spd_tensor_num_levels(const spd_tensor* t, int* nlevels);
int spd_tensor_level(const spd_tensor* t, int level, int* kind, int64_t* parent_positions,
                     int64_t* positions);
int spd_tensor_nvals(const spd_tensor* t, int64_t* nvals);
/* Device pointers of a level / of vals (NULL where the level stores nothing). */
int spd_tensor_device_ptrs(const spd_tensor* t, int level, int64_t** rowptr, int64_t** crd);
int spd_tensor_vals_ptr(const spd_tensor* t, double** vals);
/* SparseTensor::pack (tensor.cpp:94-182) on the GPU: `nentries` COO entries
 * (coords[m] = the coordinates of logical mode m, values) -> the coordinate
 * tree of the format.  Duplicates are summed in input order from 0.0 and
 * kept when zero; out-of-range coordinates return SPD_ERR_VALIDATION.
 * on_device: 0 host pointers (staged with cudaMemcpyAsync), 1 device pointers.
 * Device-side construction is SURVEY 8f row 1 (the reference's pack runs on
 * one CPU thread through a std::map). */
int spd_tensor_pack(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                    const int* mode_order, int64_t nentries, const int64_t* const* coords,
                    const double* values, int on_device, spd_tensor** out);

/* load_tensor (tensor_io.cpp:136-142): a .tns or MatrixMarket file parsed on
 * all host threads into pinned staging, then spd_tensor_pack.  dims NULL:
 * from the MatrixMarket header, or the per-mode maximum of a .tns file;
 * dims_out (order entries, may be NULL) receives the dimensions used.
 * Malformed files return SPD_ERR_VALIDATION with the reference's message. */
int spd_tensor_load(spd_context* ctx, const char* path, int order, const int* kinds,
                    const int* mode_order, const int64_t* dims, spd_tensor** out, int64_t* dims_out);

/* write_tensor (tensor_io.cpp:145-155): every stored leaf, sorted by logical
 * coordinates, 1-indexed, value as %.17g. */
int spd_tensor_store(const spd_tensor* t, const char* path);

/* Download (synchronises): pos as (lo,hi) pairs, or row pointers. */
int spd_tensor_download_level(const spd_tensor* t, int level, int64_t* pos_pairs, int64_t* crd);
int spd_tensor_download_rowptr(const spd_tensor* t, int level, int64_t* rowptr);
int spd_tensor_download_vals(const spd_tensor* t, double* vals);
int spd_tensor_download_vals_range(const spd_tensor* t, int64_t first, int64_t count, double* vals);

/* ---- (3) partitioning: level functions on the GPU ---------------------- */
/* Universe partition of the top Dense level by divide_bounds(dim, pieces)
 * (planner.cpp:10-20, level_partition.cpp:142-181) derived down the tree by
 * partition_from_parent (copy + image, :214-232).  `colors_out` (host, pieces
 * entries) may be NULL when only the device copy is wanted. */
int spd_partition_universe(spd_context* ctx, const spd_tensor* t, int64_t pieces,
                           spd_color* colors_out);
/* Nonzero partition of compressed level `level` (entries divide_bounds(nnz,
 * pieces), level_partition.cpp:186-211), preimages up the tree
 * (partition_from_child :234-251, deppart.cpp:33-53) and projected top bounds
 * (planner.cpp:50-69).  The owner searches run warp-parallel on the GPU. */
int spd_partition_nonzero(spd_context* ctx, const spd_tensor* t, int level, int64_t pieces,
                          spd_color* colors_out);
/* ---- General dependent partitioning over materialised partitions (device
 * arrays): replaces image / preimage / partition_by_bounds
 * (deppart.cpp:15-31, 33-53, 55-91) for arbitrary -- non-contiguous,
 * overlapping -- colour subsets.  A partition is (pieces, off[pieces+1],
 * idx[off[pieces]]): colour c's subset is idx[off[c] .. off[c+1]), sorted and
 * unique as Partition holds it (partition.cpp:10-24); unsorted / out-of-range
 * input returns SPD_ERR_VALIDATION (the reference throws invalid_argument).
 * `ranges` is a range region: n inclusive (lo,hi) pairs into [0, dest_extent)
 * (Region::ranges, region.cpp:33-46; lo > hi is empty).  Outputs: out_off
 * (pieces+1, device) always; out_idx only when it fits `cap` (call with cap 0
 * to size it); *total = out_off[pieces]; *disjoint = Partition::disjoint()
 * (-1 when out_idx was not written). */
int spd_deppart_image(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                      int64_t pieces, const int64_t* off, const int64_t* idx, int64_t* out_off,
                      int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint);
int spd_deppart_preimage(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                         int64_t pieces, const int64_t* dest_off, const int64_t* dest_idx,
                         int64_t* out_off, int64_t* out_idx, int64_t cap, int64_t* total,
                         int* disjoint);
/* partition_by_bounds: colour c (0 <= c < pieces) is the box
 * bounds[(c*rank + d)*2 + {0,1}] = (lo,hi) per dimension d of a row-major
 * space `extents` (host arrays), enumerated row-major; a box with an empty
 * dimension colours nothing; a bound outside the space is a validation error. */
int spd_deppart_by_bounds(spd_context* ctx, int rank, const int64_t* extents, int64_t pieces,
                          const int64_t* bounds, int64_t* out_off, int64_t* out_idx, int64_t cap,
                          int64_t* total, int* disjoint);
/* Host-memory variants of image / preimage (same arguments and semantics,
 * every array in host memory) for host callers such as the reference's own
 * planner (integration/deppart_gpu.cpp): the inputs are staged once, the
 * operator runs on the GPU, out_off / out_idx are written in host memory
 * (out_idx when cap >= *total). */
int spd_deppart_image_host(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                           int64_t pieces, const int64_t* off, const int64_t* idx, int64_t* out_off,
                           int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint);
int spd_deppart_preimage_host(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                              int64_t pieces, const int64_t* dest_off, const int64_t* dest_idx,
                              int64_t* out_off, int64_t* out_idx, int64_t cap, int64_t* total,
                              int* disjoint);
int spd_deppart_by_bounds_host(spd_context* ctx, int rank, const int64_t* extents, int64_t pieces,
                               const int64_t* bounds, int64_t* out_off, int64_t* out_idx, int64_t cap,
                               int64_t* total, int* disjoint);
/* Test support (K2m): materialise colour `color`'s subset of a bundle region
 * exactly as the reference's Partition holds it (sorted unique indices).
 *   which: 0 dom, 1 pos, 2 crd of `level`; 3 vals.
 * Uses the colours of the last spd_partition_* call on this context.  Writes
 * up to `cap` indices and returns the count in *count. */
int spd_partition_materialize(spd_context* ctx, const spd_tensor* t, int level, int which,
                              int64_t color, int64_t* out, int64_t cap, int64_t* count);
/* Universe split of an inner compressed level (LevelPartitioner::finalize,
 * compressed universe entry, level_partition.cpp:193-205; bucketCoords in the
 * rendered plan): colour c holds the positions of `level` whose coordinate
 * lies in divide_bounds(the level mode's extent, pieces)[c] -- coordinate
 * buckets, not contiguous position spans; the second distributed mode of a
 * 2-D grid (rows over M.x, the columns j of SDDMM or SpTTV over M.y).
 * Bucketed on the GPU (a stable radix sort of the positions by colour, so a
 * colour's positions stay ascending).  counts_out[c] = |colour c| (pieces
 * entries, may be NULL).  The split stays on the context for: */
int spd_partition_bucket(spd_context* ctx, const spd_tensor* t, int level, int64_t pieces, int64_t* counts_out);
/* the positions of one colour (host copy, ascending; count = its size) -- the
 * crd partition of the reference's bundle; */
int spd_bucket_positions(spd_context* ctx, int64_t color, int64_t* out, int64_t cap, int64_t* count);
/* and, for `nspans` spans [lo, hi] of the bucketed level's positions (the row
 * blocks of the grid's first loop), the leaf positions of every (span,
 * colour) cell: out[x * pieces + y] -- the 2-D grid's per-worker work. */
int spd_bucket_grid_work(spd_context* ctx, const int64_t* spans, int64_t nspans, int64_t* out);

/* ---- (4) leaf kernels + combine (one execute of a plan) ---------------- */
/* Every op runs the colours [first_color, first_color + ncolors) of the last
 * spd_partition_* on this context on this GPU, combines overlapping partials
 * deterministically in ascending colour order (reduce_combine,
 * sim.cpp:791-811) and writes the output.  With a communicator and
 * ncolors == 1 per rank, boundary partials are exchanged with NCCL.
 * Dense outputs are row-major device arrays; untouched entries are 0.0
 * (assemble_output's all-dense path, sim.cpp:665-674).  `stats` may be NULL. */
int spd_spmv(spd_context* ctx, const spd_tensor* B, const double* c_dev, double* a_dev,
             int64_t first_color, int64_t ncolors, spd_stats* stats);
/* A(i,j) = B(i,k) * C(k,j), C dense K x N row-major (format dd). */
int spd_spmm(spd_context* ctx, const spd_tensor* B, const double* C_dev, int64_t N,
             double* A_dev, int64_t first_color, int64_t ncolors, spd_stats* stats);
/* A(i,j) = B(i,j) * C(i,k) * D(k,j): output vals on B's pattern (pattern
 * reuse, sim.cpp:571-606).  D(k,j) is read at D[k*dk + j*dj]. */
int spd_sddmm(spd_context* ctx, const spd_tensor* B, const double* C_dev, const double* D_dev,
              int64_t K, int64_t dk, int64_t dj, double* Avals_dev, int64_t first_color,
              int64_t ncolors, spd_stats* stats);
/* A(i,j) = B(i,j,k) * c(k) on a dss CSF; output vals on B's first two levels. */
int spd_spttv(spd_context* ctx, const spd_tensor* B, const double* c_dev, double* Avals_dev,
              int64_t first_color, int64_t ncolors, spd_stats* stats);
/* A(i,l) = B(i,j,k) * C(j,l) * D(k,l) on a dss CSF; C: J x R, D: K x R, A: I x R. */
int spd_spmttkrp(spd_context* ctx, const spd_tensor* B, const double* C_dev,
                 const double* D_dev, int64_t R, double* A_dev, int64_t first_color,
                 int64_t ncolors, spd_stats* stats);
/* A = B + C + D over CSR operands with identical dims, row split: two-phase
 * assembly (count -> scan -> fill, sim.cpp:676-788) producing a new CSR
 * tensor with the structural-union pattern.  With a communicator and one
 * colour per GPU, each GPU assembles the rows of its colour (other rows are
 * empty in its piece) and the per-GPU nnz are all-gathered so every piece
 * knows its global pos offset (spd_tensor_global_span). */
int spd_spadd3(spd_context* ctx, const spd_tensor* B, const spd_tensor* C, const spd_tensor* D,
               spd_tensor** A_out, int64_t first_color, int64_t ncolors, spd_stats* stats);

/* Row block [row_lo, row_hi], first global position and global nnz of a
 * tensor piece (a whole tensor: all rows, 0, nnz). */
int spd_tensor_global_span(const spd_tensor* t, int64_t* row_lo, int64_t* row_hi,
                           int64_t* pos_base, int64_t* global_positions);

/* Collective, data placement (lower_tdn + residency_from_placements,
 * planner.cpp:361-439, sim.cpp:547-566) of a CSR matrix by its compute
 * partition: split 1 = row (universe) split, 2 = nonzero split of the leaf
 * level, one colour per GPU.  `whole` is read on `root` only (NULL
 * elsewhere).  Every GPU receives the row pointer and its colour's crd/vals
 * (NCCL broadcast + send/recv) as a piece tensor that the leaf ops accept for
 * that colour (the matched distribution: compute moves 0 bytes of it); the
 * context's partition is left set to the piece.  *bytes_in = bytes received. */
int spd_tensor_place(spd_context* ctx, int root, const spd_tensor* whole, int split,
                     spd_tensor** piece, int64_t* bytes_in);
/* Positions [lo, hi] a (piece) tensor holds; a whole tensor: [0, nvals-1]. */
int spd_tensor_piece_span(const spd_tensor* t, int64_t* lo, int64_t* hi);

/* Collective: gathers the row-block pieces of a distributed CSR output on
 * GPU `root` (grouped NCCL send/recv; the reference assembles one Region per
 * output, sim.cpp:676-788).  *out is the whole tensor on root, NULL on the
 * other ranks. */
int spd_gather_rows(spd_context* ctx, const spd_tensor* A, int root, spd_tensor** out);

/* Colour blocks per GPU.  With a communicator rank r runs one contiguous
 * block of colours; by default [r * ceil(P / world), ...).  A plan with more
 * colours than GPUs (over-decomposition) can install its own blocks -- e.g.
 * balanced by a cost model -- as bounds[0..world] (bounds[0] = 0, bounds[world]
 * = pieces, every block non-empty); they apply to partitions of `pieces`
 * colours and must be the same on every rank (the boundary combine's
 * all-gather layout follows them).  bounds NULL restores the default.  The
 * reference maps colours to processors in its mapper (sim.cpp:833-847); the
 * partition itself (its bounds) is unchanged by the blocks. */
int spd_context_set_colour_blocks(spd_context* ctx, int64_t pieces, const int64_t* bounds);
/* The blocks a `pieces`-colour partition runs with on this context. */
int spd_context_colour_blocks(spd_context* ctx, int64_t pieces, int64_t* bounds);
/* Host-only (no GPU needed): contiguous blocks of near-equal total cost, the
 * boundary r at the cost prefix nearest r / world of the total. */
int spd_split_colour_blocks(const double* cost, int64_t pieces, int world, int64_t* bounds);
/* Per colour of the current partition of the ds matrix t: its positions, the
 * output rows it stores (W_c) and how many of those rows
 * are non-empty -- the inputs of a cost model for the blocks above. */
int spd_colour_costs(spd_context* ctx, const spd_tensor* t, int64_t* positions, int64_t* rows,
                     int64_t* nonempty);

/* Per-colour Stats::PerWorker::work of the last op (sim.cpp:352), `pieces`
 * entries. */
int spd_last_work(spd_context* ctx, int64_t* work, int64_t pieces);

/* Output rows (fibres for SpTTV) that colours [first, first + count) stored in
 * the last SpMV / SpMM / SpTTV / SpMTTKRP: the union of their write ranges W_c
 * (DESIGN.md section 5), lo > hi when none -- what a caller copies back from
 * this GPU's output buffer when the colours ran on several GPUs. */
int spd_last_owned(spd_context* ctx, int64_t first, int64_t count, int64_t* lo, int64_t* hi);

/* CUDA graphs: capture the ops enqueued on `ctx` between begin and end
 * (e.g. spd_partition_* with colors_out NULL + a leaf op with stats NULL)
 * and replay them with one launch.  The context must own an explicit
 * stream.  Ops that need a host read-back fail the capture, and so does the
 * first use of a derived per-tensor index that sizes itself on the host
 * (the compacted-column SpMV index): run the op once before capturing. */
typedef struct spd_graph spd_graph;
int spd_capture_begin(spd_context* ctx);
int spd_capture_end(spd_context* ctx, spd_graph** out);
int spd_graph_launch(spd_graph* g, spd_context* ctx);
int spd_graph_destroy(spd_graph* g);

/* ---- (5) instrumentation ----------------------------------------------- */
/* Records a CUDA-event pair around every leaf kernel launched on the
 * context's stream while enabled (no host synchronisation). */
int spd_context_timing(spd_context* ctx, int enable);
/* Synchronises, returns up to `cap` recorded leaf-kernel durations (ms) in
 * launch order via *n, and clears the record. */
int spd_context_read_timing(spd_context* ctx, double* leaf_ms, int64_t cap, int64_t* n);
/* Kernels launched by this context since it was created. */
int spd_context_launches(const spd_context* ctx, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif
