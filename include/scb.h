/*
 * scb.h -- C ABI of the B200-native single-cell hot path (libscb_b200.so).
 *
 * The reference (arxiv/paper_2605_13928, /root/reference) defines no compute API for
 * this path: the pipeline is out of its scope and exists only as the
 * Table-1 step list and the marker labels qc / norm_hvg / regress /
 * pca / knn (pkg/tests/helpers.py:31-36).  Each entry point below replaces one
 * Scanpy / rapids-singlecell step the paper's R script called through reticulate
 * (PAPER.md:23,62); the Scanpy function each mirrors is named in its comment, and the
 * Python step functions in paper_2605_13928_b200/pp.py keep Scanpy's names.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer owned by the caller unless noted; the library
 *     allocates only scratch held in the context;
 *   - work is ordered on `stream` (a cudaStream_t passed as void*); no host sync
 *     unless a function says so;
 *   - CSR = indptr int64[n_rows+1], indices int32[nnz] (sorted within a row), data
 *     float32[nnz];
 *   - return 0 (SCB_OK) or a negative SCB_ERR_*; scb_last_error() gives the message
 *     (thread-local);
 *   - one context per GPU, used by one host thread at a time.
 *   - "gene sums" are integer fixed-point accumulators: u64 [n_stats][2 limbs][n],
 *     value = limb0 + limb1 * 2^32, scaled by 2^-frac_bits.  They
 *     add exactly across shards, so multi-GPU callers all-reduce them as int64 SUM.
 */
#ifndef SCB_H_
#define SCB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCB_OK 0
#define SCB_ERR_ARG -1
#define SCB_ERR_CUDA -2
#define SCB_ERR_UNSUPPORTED -3
#define SCB_ERR_DATA -4
#define SCB_ERR_NOMEM -5

#define SCB_ABI_VERSION 1

/* fixed-point fractional bits of the gene-sum accumulators */
#define SCB_FX_Y 28      /* sum of normalized counts y            */
#define SCB_FX_Y2 24     /* sum of y^2                            */
#define SCB_FX_L 28      /* sum of log1p values l                 */
#define SCB_FX_L2 24     /* sum of l^2                            */

#if defined(__GNUC__)
#define SCB_API __attribute__((visibility("default")))
#else
#define SCB_API
#endif

typedef struct scb_ctx scb_ctx;

SCB_API int scb_abi_version(void);
SCB_API const char* scb_last_error(void);
/* number of kernels this library has launched in the process (for launch accounting) */
SCB_API unsigned long long scb_launch_count(void);
SCB_API int scb_ctx_create(int device, scb_ctx** out);
SCB_API int scb_ctx_destroy(scb_ctx* ctx);
/* on != 0: scb_qc_metrics no longer waits for its data-validity check (one host round trip);
 * the flag is returned in n_kept[3] of the next scb_filter_masks instead. */
SCB_API int scb_ctx_set_deferred_checks(scb_ctx* ctx, int32_t on);
/* stream-ordered copy of the ctx's current data-error flag (set by a deferred scb_qc_metrics) to
 * a device int32 -- e.g. to keep each chunk's check when QC runs chunk by chunk. */
SCB_API int scb_ctx_copy_data_flag(scb_ctx* ctx, int32_t* dst, void* stream);

/* ---- multi-GPU: a ctx that owns an NCCL communicator over `world`
 * ranks (one process per GPU).  Rank 0 makes the 128-byte id with scb_nccl_unique_id and
 * shares it (e.g. through the torch.distributed store); every rank then calls
 * scb_ctx_create_comm(its device, id, rank, world).  libnccl.so.2 is loaded on first use
 * (SCB_ERR_UNSUPPORTED without it).  The collectives are stream-ordered and in place:
 *   scb_comm_allreduce: dtype 0 int64, 1 float64, 2 float32, 3 int32; op 0 sum, 1 max;
 *   scb_comm_broadcast: `bytes` from `root`;
 *   scb_comm_allgather: recv[r * bytes_per_rank ...] = rank r's send buffer.
 * On a ctx without a communicator they are the world-size-1 identities. */
SCB_API int scb_nccl_unique_id(uint8_t* id_out);
SCB_API int scb_ctx_create_comm(int device, const uint8_t* nccl_id, int32_t rank, int32_t world, scb_ctx** out);
SCB_API int scb_comm_info(scb_ctx* ctx, int32_t* rank, int32_t* world);
SCB_API int scb_comm_allreduce(scb_ctx* ctx, void* buf, int64_t count, int32_t dtype, int32_t op, void* stream);
SCB_API int scb_comm_broadcast(scb_ctx* ctx, void* buf, int64_t bytes, int32_t root, void* stream);
SCB_API int scb_comm_allgather(scb_ctx* ctx, const void* send, void* recv, int64_t bytes_per_rank, void* stream);

/* ---- f1 ingest (sc.read_10x_mtx / sc.read_mtx): MatrixMarket coordinate data lines -> COO
 * on the device.  text holds the whole file (16-byte aligned, readable up to
 * roundup(n_bytes, 16)); data_offset = first data line (the host parses the banner, comments
 * and size line); field 0 = integer, 1 = real, 2 = pattern.  row/col receive 0-based file
 * coordinates in file order, val the values as float32.  SCB_ERR_DATA if the number of data
 * lines differs from nnz or a line is malformed / out of range. */
SCB_API int scb_mtx_parse(scb_ctx* ctx, const char* text, int64_t data_offset, int64_t n_bytes, int32_t field,
                  int64_t nnz, int64_t n_file_rows, int64_t n_file_cols, int32_t* row, int32_t* col,
                  float* val, void* stream);

/* ---- COO -> CSR over `major` (cells = file columns of a 10x matrix.mtx): indptr
 * int64[n_major+1], indices (minor, ascending within each row), data.  Input already in CSR
 * order (major non-decreasing, minor strictly increasing within a row) is converted without
 * moving entries (indices/data may alias minor/val); otherwise a counting scatter plus a
 * per-row sort (rows <= 8192 entries).  Duplicate (major, minor) entries: SCB_ERR_DATA. */
SCB_API int scb_coo_to_csr(scb_ctx* ctx, const int32_t* major, const int32_t* minor, const float* val, int64_t nnz,
                   int32_t n_major, int64_t* indptr, int32_t* indices, float* data, void* stream);

/* ---- a1: sc.pp.calculate_qc_metrics(qc_vars=["mt"], percent_top=None, log1p=False)
 * Per cell: n_genes_by_counts, total_counts, total_counts_mt, pct_counts_mt.
 * Per gene: n_cells_by_counts, total_counts (exact; counts must be non-negative
 * integers < 2^24 stored as float32, otherwise SCB_ERR_DATA). */
SCB_API int scb_qc_metrics(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* data,
                   int64_t n_rows, int32_t n_cols, const uint8_t* mt_mask,
                   int32_t* n_genes_by_counts, double* total_counts, double* total_counts_mt,
                   double* pct_counts_mt, int32_t* n_cells_by_counts, double* gene_total_counts,
                   int32_t* hvg_row_splits, void* stream);

/* Number of gene tiles T the HVG column pass uses for n_cols genes.  If T > 1, passing
 * hvg_row_splits (int32 [n_rows][T-1]) to scb_qc_metrics records, per row, how many entries
 * have a gene index below each tile boundary; scb_hvg_gene_sums then streams every nonzero
 * exactly once (otherwise each tile re-reads whole rows); rows whose column indices are not
 * sorted are detected there and the pass is redone without splits.  indices/data arrays of
 * every CSR entry point must be 16-byte aligned. */
SCB_API int32_t scb_hvg_tiles(int32_t n_cols);

/* ---- a2: sc.pp.filter_cells(min_genes, max_genes) + pct_counts_mt < max_pct_mt, and
 * sc.pp.filter_genes(min_cells).  max_genes < 0 disables the upper bound.
 * n_kept (device int64[4]) receives {kept cells, kept genes, nonzeros of the kept rows (if
 * indptr != NULL, else 0), the QC data-error flag (nonzero: scb_qc_metrics saw invalid counts
 * or column indices while the ctx defers checks, see scb_ctx_set_deferred_checks)}. */
SCB_API int scb_filter_masks(scb_ctx* ctx, const int32_t* n_genes_by_counts, const double* pct_counts_mt,
                     int64_t n_rows, const int32_t* n_cells_by_counts, int32_t n_cols,
                     int32_t min_genes, int32_t max_genes, double max_pct_mt, int32_t min_cells,
                     const int64_t* indptr, uint8_t* cell_mask, uint8_t* gene_mask, int64_t* n_kept, void* stream);

/* ---- a2 pass 1 when EVERY gene is kept (n_kept[1] == n_cols): no pass over the nonzeros --
 * gene_remap = identity, new_indptr from the kept rows' lengths, row_scale / row_scale_orig =
 * float32(target_sum / total_counts) (QC's exact totals; 1 for empty rows), i.e. exactly what
 * scb_subset_count computes in that case. */
SCB_API int scb_subset_rows_all_genes(scb_ctx* ctx, const int64_t* indptr, int64_t n_rows, int32_t n_cols,
                              const uint8_t* cell_mask, const double* total_counts, double target_sum,
                              int32_t* gene_remap, int64_t* new_indptr, float* row_scale, float* row_scale_orig,
                              void* stream);

/* ---- a2: adata[cell_mask, gene_mask] -- pass 1.  Builds gene_remap (new column or -1),
 * new_indptr (int64[n_kept_cells+1]; new_indptr[n_kept] = kept nnz) and, if
 * row_scale != NULL, the per-KEPT-row normalize_total factor float32(target_sum/total)
 * (fused count pass of the pipeline; target_sum ignored when row_scale == NULL).
 * If row_scale_orig != NULL it also receives the factor per ORIGINAL row (0 = dropped). */
SCB_API int scb_subset_count(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* data,
                     int64_t n_rows, int32_t n_cols, const uint8_t* cell_mask,
                     const uint8_t* gene_mask, int32_t* gene_remap, int64_t* new_indptr,
                     double target_sum, float* row_scale, float* row_scale_orig, void* stream);

/* ---- a2 pass 2: writes the compacted CSR.  If row_scale != NULL the values written are
 * log1p(x * row_scale[kept_row]) (fused normalize_total + log1p), else raw x. */
SCB_API int scb_subset_fill(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* data,
                    int64_t n_rows, int32_t n_cols, const uint8_t* cell_mask, const int32_t* gene_remap,
                    const int64_t* new_indptr, const float* row_scale, int32_t* new_indices,
                    float* new_data, void* stream);

/* ---- a2 pass 2 fused with a6's statistics: as scb_subset_fill with row_scale (log1p values),
 * and sums u64[2][2][n_slots] += the fixed-point Σl, Σl² of the HVG columns (slot: int32 per
 * OUTPUT gene, -1 = not an HVG) -- the numbers scb_scale_gene_sums would compute from the
 * written matrix, without re-reading it.  Requires n_cols <= 32767 (else SCB_ERR_UNSUPPORTED).
 * new_indices may be NULL when every row and every gene is kept: the output then shares the
 * input's indices (no copy; a kernel trap if a row or gene turns out to be dropped). */
SCB_API int scb_subset_fill_scale_sums(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* data,
                               int64_t n_rows, int32_t n_cols, const uint8_t* cell_mask, const int32_t* gene_remap,
                               const int64_t* new_indptr, const float* row_scale, const int32_t* slot,
                               int32_t n_slots, int32_t* new_indices, float* new_data, uint64_t* sums,
                               void* stream);

/* ---- a3+a4: sc.pp.normalize_total(target_sum) + sc.pp.log1p, out of place (out may
 * alias data).  row_scale receives float32(target_sum / row total) (1 for empty rows). */
SCB_API int scb_normalize_log1p(scb_ctx* ctx, const int64_t* indptr, const float* data, int64_t n_rows,
                        double target_sum, float* out, float* row_scale, void* stream);

/* ---- a5 partial: per-gene fixed-point sums of y = x*row_scale[r] and y^2 over rows with
 * row_scale != 0, accumulated (+=) into sums u64[2][2][n_out_cols] (stat, limb, gene).
 * gene_remap (optional) maps input columns to output columns (-1 = skip). */
SCB_API int scb_hvg_gene_sums(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* data,
                      const float* row_scale, int64_t n_rows, int32_t n_cols,
                      const int32_t* gene_remap, int32_t n_out_cols, const int32_t* hvg_row_splits,
                      uint64_t* sums, void* stream);

/* ---- compact "u16" CSR input (lossless wire/HBM format for count matrices with
 * n_cols <= 65536 and integer counts): the same entry points with uint16_t column indices and
 * uint16_t counts -- half the bytes per nonzero for every pass over the raw matrix and for
 * the host->device copy.  A stored count of 65535 is an escape: the entry's true value
 * (>= 65535) is esc_val[i] where esc_pos[i] (sorted, int64, device) is its position in the
 * arrays (n_esc entries; esc_pos/esc_val may be NULL when n_esc == 0).  Semantics, outputs and error codes are
 * those of the 32-bit entry points above (the kept matrix written by the subset fill passes
 * is int32/float32 in both cases).  Arrays must be 16-byte aligned. */
SCB_API int scb_qc_metrics_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices, const uint16_t* data,
                   int64_t n_rows, int32_t n_cols, const uint8_t* mt_mask,
                   int32_t* n_genes_by_counts, double* total_counts, double* total_counts_mt,
                   double* pct_counts_mt, int32_t* n_cells_by_counts, double* gene_total_counts,
                   int32_t* hvg_row_splits, const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                   void* stream);
SCB_API int scb_subset_count_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices, const uint16_t* data,
                     int64_t n_rows, int32_t n_cols, const uint8_t* cell_mask,
                     const uint8_t* gene_mask, int32_t* gene_remap, int64_t* new_indptr,
                     double target_sum, float* row_scale, float* row_scale_orig, const int64_t* esc_pos,
                     const float* esc_val, int64_t n_esc, void* stream);
SCB_API int scb_subset_fill_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices, const uint16_t* data,
                    int64_t n_rows, int32_t n_cols, const uint8_t* cell_mask, const int32_t* gene_remap,
                    const int64_t* new_indptr, const float* row_scale, int32_t* new_indices,
                    float* new_data, const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream);
SCB_API int scb_subset_fill_scale_sums_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices,
                               const uint16_t* data, int64_t n_rows, int32_t n_cols, const uint8_t* cell_mask,
                               const int32_t* gene_remap, const int64_t* new_indptr, const float* row_scale,
                               const int32_t* slot, int32_t n_slots, int32_t* new_indices, float* new_data,
                               uint64_t* sums, const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                               void* stream);
SCB_API int scb_hvg_gene_sums_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices, const uint16_t* data,
                      const float* row_scale, int64_t n_rows, int32_t n_cols,
                      const int32_t* gene_remap, int32_t n_out_cols, const int32_t* hvg_row_splits,
                      uint64_t* sums, const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream);

/* ---- f1 wire decode: compact u16 CSR (as above) -> int32 indices + float32 counts in HBM
 * (arrays 16-byte aligned; the output may then feed the 32-bit entry points).  4 B read + 8 B
 * written per nonzero; the escaped counts are scattered from (esc_pos, esc_val). */
SCB_API int scb_csr_u16_decode(scb_ctx* ctx, const uint16_t* indices16, const uint16_t* data16, int64_t nnz,
                               const int64_t* esc_pos, const float* esc_val, int64_t n_esc, int32_t* indices,
                               float* data, void* stream);

/* ---- f1 wire decode: byte-delta CSR -> int32 indices + float32 counts in HBM.  Per nonzero one
 * byte dgene = g - g_prev - 1 (g_prev = -1 at a row start; 255 = escape: the delta is
 * gesc_val at the sorted position gesc_pos) and one byte dcount = the count (255 = escape:
 * cesc_val at cesc_pos); rows as indptr (sorted, unique gene indices within a row).  2 B on the
 * wire per nonzero instead of 4 (u16) or 8 (int32 + float32); lossless (pp.DeltaCSR).
 * dgene / dcount 4-byte aligned, indices / data 16-byte aligned (else SCB_ERR_ARG). */
SCB_API int scb_csr_delta8_decode(scb_ctx* ctx, const int64_t* indptr, int64_t n_rows, const uint8_t* dgene,
                                  const uint8_t* dcount, int64_t nnz, const int64_t* gesc_pos,
                                  const int32_t* gesc_val, int64_t n_gesc, const int64_t* cesc_pos,
                                  const float* cesc_val, int64_t n_cesc, int32_t* indices, float* data,
                                  void* stream);

/* ---- a5: sc.pp.highly_variable_genes(flavor="seurat", n_top_genes, n_bins) from the
 * (all-reduced) gene sums.  Outputs per gene: means, variances, dispersions (log),
 * dispersions_norm, mean_bin; hvg_mask; hvg_index = sorted selected genes (int32[n_cols]
 * capacity).  ties = 1 (Scanpy): every gene with dispersions_norm >= the n_top-th largest
 * finite value (more than n_top only on exact ties); ties = 0: exactly min(n_top, #finite),
 * ties at the cutoff taken in gene-index order.  n_selected (device int32) = count. */
SCB_API int scb_hvg_select(scb_ctx* ctx, const uint64_t* sums, int32_t n_cols, int64_t n_cells,
                   int32_t n_top, int32_t n_bins, int32_t ties, double* means, double* variances,
                   double* dispersions, double* dispersions_norm, int32_t* mean_bin,
                   uint8_t* hvg_mask, int32_t* hvg_index, int32_t* n_selected, void* stream);

/* ---- a6 partial: fixed-point sums of l and l^2 for the selected genes
 * (gene_slot[g] = HVG slot or -1), accumulated into sums u64[2][2][n_slots]. */
SCB_API int scb_scale_gene_sums(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                        const float* logdata, int64_t n_rows, int32_t n_cols,
                        const int32_t* gene_slot, int32_t n_slots, uint64_t* sums, void* stream);

/* ---- a6: mean / inverse std (ddof=1, std==0 -> 1) from the all-reduced sums. */
SCB_API int scb_scale_finalize(scb_ctx* ctx, const uint64_t* sums, int32_t n_slots, int64_t n_cells,
                       double* mean, double* inv_std, void* stream);

/* ---- a6: sc.pp.scale(max_value) of the HVG columns into a dense row-major float32
 * matrix Z[n_rows][ldz]: column j < n_slots = float(max(min((l - mean)*inv_std, max_value),
 * min_value)) in fp64 (min_value = -max_value: Scanpy >= 1.10 / rapids-singlecell zero_center
 * clip; -inf: upper clip only, Scanpy <= 1.9);
 * column ones_col (if >= 0) = 1.0; other columns up to ldz = 0. */
SCB_API int scb_scale_dense(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                    const float* logdata, int64_t n_rows, int32_t n_cols, const int32_t* gene_slot,
                    int32_t n_slots, const double* mean, const double* inv_std, double max_value,
                    double min_value, float* Z, int64_t ldz, int32_t ones_col, void* stream);

/* ---- a6 in the pipeline's layout: the same z-scores written directly as BF16 planes
 * Z_hi = bf16(z), Z_lo = bf16(z - hi) (row-major [n_rows][ldz], ldz % 8 == 0; column ones_col =
 * 1) -- bit-identical to scb_scale_dense followed by scb_split_bf16, without the fp32 matrix.
 * The Gram (scb_gram_split) and the projection (scb_project_planes) read the planes. */
SCB_API int scb_scale_dense_planes(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* logdata,
                                   int64_t n_rows, int32_t n_cols, const int32_t* gene_slot, int32_t n_slots,
                                   const double* mean, const double* inv_std, double max_value, double min_value,
                                   uint16_t* Z_hi, uint16_t* Z_lo, int64_t ldz, int32_t ones_col, void* stream);

/* ---- f2 (optional, paper Table 1 step 4): sc.pp.regress_out(["total_counts",
 * "pct_counts_mt"]) fused with scale.  Replaces scale_gene_sums/finalize:
 *   1. scb_regress_cov_sums: sums6 = {n, Σtc, Σtc², Σpct, Σpct², Σtc·pct} over the kept
 *      cells (float64; all-reduced across ranks);
 *   2. scb_regress_design: standardised covariates design[2][n_kept] (kept-row order);
 *   3. scb_scale_dense with mean = 0, inv_std = 1, max_value = +inf -> Z holds l (dense);
 *   4. scb_regress_xty: xty[4][H] += {Σl, Σa1·l, Σa2·l, Σl²} per gene (all-reduced);
 *   5. scb_regress_finalize: beta[3][H] (OLS) and inv_std[H] of the residuals;
 *   6. scb_regress_apply: Z[:, :H] = clip((l - beta0 - a1 beta1 - a2 beta2) * inv_std, min, max). */
SCB_API int scb_regress_cov_sums(scb_ctx* ctx, const double* total_counts, const double* pct_counts_mt,
                         const uint8_t* cell_mask, int64_t n_rows, double* sums6, void* stream);
SCB_API int scb_regress_design(scb_ctx* ctx, const double* total_counts, const double* pct_counts_mt,
                       const uint8_t* cell_mask, int64_t n_rows, const double* sums6, int64_t n_kept,
                       double* design, void* stream);
SCB_API int scb_regress_xty(scb_ctx* ctx, const float* Z, int64_t n_rows, int64_t ld, int32_t n_slots,
                    const double* design, double* xty, void* stream);
SCB_API int scb_regress_finalize(scb_ctx* ctx, const double* xty, const double* sums6, int32_t n_slots,
                         double* beta, double* inv_std, void* stream);
SCB_API int scb_regress_apply(scb_ctx* ctx, float* Z, int64_t n_rows, int64_t ld, int32_t n_slots,
                      const double* design, const double* beta, const double* inv_std, double max_value,
                      double min_value, void* stream);

/* ---- f3 sc.pp.neighbors graph outputs (umap-learn fuzzy_simplicial_set on the exact kNN,
 * set_op_mix_ratio 1, local_connectivity 1).  knn_idx/knn_dist are [rows][k] as returned by
 * scb_knn (self included).  scb_knn_dist_sum: sum of all distances (the caller divides by
 * N*k for the global mean, all-reduced across ranks).  scb_umap_weights: per local row
 * sigma, rho and membership strengths w[rows][k] (row0 = global index of the first row).
 * scb_fuzzy_union_rows / _fill: rows [r0, r1) of C = W + Wᵀ - W∘Wᵀ (f32, scipy's evaluation
 * order) from the global (all-gathered) idx/w: indptr int64[r1-r0+1] first, then cols/vals
 * (sorted by column).  scb_knn_distances_csr: `distances` (non-zero kNN distances, sorted by
 * column; cols/vals need rows*k capacity). */
SCB_API int scb_knn_dist_sum(scb_ctx* ctx, const float* knn_dist, int64_t n, double* sum, void* stream);
SCB_API int scb_umap_weights(scb_ctx* ctx, const int32_t* knn_idx, const float* knn_dist, int64_t n_rows, int32_t k,
                     int64_t row0, const double* mean_dist, float* sigma, float* rho, float* w, void* stream);
SCB_API int scb_fuzzy_union_rows(scb_ctx* ctx, const int32_t* idx_all, const float* w_all, int64_t n_all, int32_t k,
                         int64_t r0, int64_t r1, int64_t* indptr, void* stream);
SCB_API int scb_fuzzy_union_fill(scb_ctx* ctx, const int32_t* idx_all, const float* w_all, int64_t n_all, int32_t k,
                         int64_t r0, int64_t r1, const int64_t* indptr, int32_t* cols, float* vals, void* stream);
SCB_API int scb_knn_distances_csr(scb_ctx* ctx, const int32_t* knn_idx, const float* knn_dist, int64_t n_rows,
                          int32_t k, int64_t* indptr, int32_t* cols, float* vals, void* stream);

/* ---- f3 sc.tl.umap layout: umap-learn optimize_layout_euclidean (2-D) on the connectivities
 * CSR (indptr/indices/weights, nnz entries, w_max = max weight), edge-parallel SGD for n_epochs
 * epochs from `init` (rows of >= 2 floats, stride init_ld; rescaled to [0, 10] as umap does);
 * a, b = the curve parameters of (min_dist, spread); emb receives float32 [n_vertices][2]. */
SCB_API int scb_umap_layout(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights,
                    int64_t n_vertices, int64_t nnz, float w_max, const float* init, int64_t init_ld,
                    int32_t n_epochs, float a, float b, int32_t neg_rate, uint64_t seed, float* emb, void* stream);

/* ---- f3 clustering on the neighbors graph (sc.tl.louvain / the local-moving + aggregation
 * core of sc.tl.leiden): multi-level modularity optimisation with resolution gamma on the
 * symmetric CSR (indptr/indices/weights), deterministic (2^-32 fixed-point weights, 8 hash-bucketed
 * synchronous moves, ties to the smaller community).  labels (device int32[n]) are numbered
 * by decreasing community size; n_communities / modularity are host outputs. */
SCB_API int scb_louvain(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights, int64_t n,
                int64_t nnz, double resolution, int32_t max_levels, int32_t max_iters, uint32_t seed,
                int32_t* labels, int32_t* n_communities, double* modularity, void* stream);
/* sc.tl.leiden: the same local moving, then Leiden's refinement of each level's partition
 * (singletons join well-connected sub-communities with the largest non-negative gain) and
 * aggregation by the refined partition, each aggregate node starting the next level in its
 * unrefined community (labels = that partition). */
SCB_API int scb_leiden(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights, int64_t n,
               int64_t nnz, double resolution, int32_t max_levels, int32_t max_iters, uint32_t seed,
               int32_t* labels, int32_t* n_communities, double* modularity, void* stream);

/* ---- f5 sc.tl.rank_genes_groups(method="t-test", reference="rest") on the log-normalized
 * kept matrix (CSR, ldata = log1p values) for cell labels 0..n_groups-1 (paper Table 1 step 9).
 * Outputs [n_groups][n_cols] float64: scores (Welch t), logfoldchanges, pvals, pvals_adj
 * (Benjamini-Hochberg per group); order int32 [n_groups][n_cols] = gene indices by decreasing
 * score (ties: smaller index). */
SCB_API int scb_rank_genes_groups(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* ldata,
                          int64_t n_rows, int32_t n_cols, const int32_t* labels, int32_t n_groups, double* scores,
                          double* logfoldchanges, double* pvals, double* pvals_adj, int32_t* order, void* stream);

/* ---- a7: partial Gram matrix C = Z^T Z (float64 [hp][hp], full symmetric) on the
 * 5th-gen tensor cores (tcgen05 kind::f16, "3xBF16": x = hi + lo with hi = bf16(x),
 * lo = bf16(x - hi), products hi*hi + hi*lo + lo*hi, <= 2^-16 relative each; FP32 accumulate
 * in TMEM per <=64k-cell K-slice, slices summed in float64; operands staged by TMA).
 * hp = ldz must be a multiple of 128; n_rows any. */
SCB_API int scb_gram(scb_ctx* ctx, const float* Z, int64_t n_rows, int32_t hp, double* C, void* stream);

/* ---- operand-plane format of this build: 0 = BF16 planes + three-product Gram (the default),
 * 2 = FP16 planes + three-product Gram, 1 = FP16 planes + one-product (hi x hi) Gram.  The
 * planes written by scb_split_bf16 / scb_scale_dense_planes and read by the Gram and the
 * projection are 16-bit values of that format. */
SCB_API int32_t scb_plane_format(void);

/* ---- a7 operand prep: BF16 planes Zhi = bf16(Z), Zlo = bf16(Z - Zhi) (uint16 storage,
 * [n_rows][ld], ld % 4 == 0) in one streaming pass. */
SCB_API int scb_split_bf16(scb_ctx* ctx, const float* Z, int64_t n_rows, int64_t ld, uint16_t* Zhi, uint16_t* Zlo,
                           void* stream);

/* ---- a7 from the BF16 planes of scb_split_bf16 (the same operands and MMA sequence as
 * scb_gram): TMA feeds the tensor cores directly, no in-kernel conversion. */
SCB_API int scb_gram_split(scb_ctx* ctx, const uint16_t* Zhi, const uint16_t* Zlo, int64_t n_rows, int32_t hp,
                           double* C, void* stream);

/* ---- a8: top-n_comps eigenpairs of the centred covariance
 * Cov = (C[:h,:h] - N m m^T)/(N-1), m = C[ones_col, :h]/N (column means of Z).
 * Outputs eigenvalues (desc, float64), components_t float32[n_comps_pad][hp] (row j =
 * component j, sign-canonical: largest |loading| positive, zero-padded), col_mean
 * float32[hp] and trace (float64, total variance).  Subspace iteration in float64. */
SCB_API int scb_pca_eig(scb_ctx* ctx, const double* C, int32_t h, int32_t hp, int32_t ones_col,
                int64_t n_cells, int32_t n_comps, int32_t n_comps_pad, double* eigenvalues,
                float* components_t, float* col_mean, double* trace, void* stream);

/* ---- a8: X_pca = (Z - m) V, float32 [n_rows][ld_out] (columns >= n_comps zeroed). */
SCB_API int scb_project(scb_ctx* ctx, const float* Z, int64_t n_rows, int32_t hp,
                const float* components_t, const float* col_mean, int32_t n_comps,
                int32_t n_comps_pad, float* X_pca, int32_t ld_out, void* stream);

/* ---- a8 from the BF16 planes: X_pca = (Z - m) V with Z = hi + lo (3xBF16 tcgen05 MMAs, the
 * Gram's operand scheme); same arguments and output as scb_project, hp % 64 == 0. */
SCB_API int scb_project_planes(scb_ctx* ctx, const uint16_t* Z_hi, const uint16_t* Z_lo, int64_t n_rows, int32_t hp,
                               const float* components_t, const float* col_mean, int32_t n_comps, int32_t n_comps_pad,
                               float* X_pca, int32_t ld_out, void* stream);

/* ---- a9: sc.pp.neighbors(n_neighbors=k, method exact, metric euclidean): for each query
 * row, the k nearest key rows (self included) ordered by (distance, index).  Candidate
 * scores on tcgen05 (kind::f16 operands, FP32 accumulate) with a fused per-row candidate
 * top-list, then exact FP32 re-rank.  k_cand (32 or 64, >= k) is the minimum candidate
 * count: k <= 16 keeps two 16-entry lists per row (one per key-column half; the top-k of
 * the union lies in the union of the per-half top-16), 16 < k <= 32 one 48-entry list,
 * k <= 64 one 64-entry list.  queries/keys float32 [n][ld] (d + 2 <= 64, columns >= d
 * ignored); for sharded queries pass the full key matrix (returned indices index keys). */
SCB_API int scb_knn(scb_ctx* ctx, const float* queries, int64_t n_queries, const float* keys,
            int64_t n_keys, int32_t d, int32_t ld, int32_t k, int32_t k_cand,
            int32_t* knn_index, float* knn_dist, void* stream);

/* ---- a9 with device timing: as scb_knn, and if ev_start / ev_end (cudaEvent_t) are
 * non-NULL they are recorded on `stream` immediately around the tcgen05 candidate kernel. */
SCB_API int scb_knn_timed(scb_ctx* ctx, const float* queries, int64_t n_queries, const float* keys, int64_t n_keys,
                          int32_t d, int32_t ld, int32_t k, int32_t k_cand, int32_t* knn_index, float* knn_dist,
                          void* stream, void* ev_start, void* ev_end);

/* ---- a9 with a caller-chosen scan order (queries == keys = x): order_key[i] (16-bit bucket)
 * replaces the built-in Morton bucket of row i; rows are scanned outward in bucket order. */
SCB_API int scb_knn_ordered(scb_ctx* ctx, const float* x, int64_t n, int32_t d, int32_t ld, int32_t k,
                            const uint16_t* order_key, int32_t* knn_index, float* knn_dist, void* stream,
                            void* ev_start, void* ev_end);

/* ---- synthetic negative-binomial counts (oracle/synth.py specification, generator v2), on
 * device; bit-identical to the CPU generator (fixed-order correctly rounded fp64 only).
 * scb_synth_logmean: logmean[c][g] = (log_s[c] + log_mu[g]) + L, L = A[cell_type[c]][g], then
 * L += U[c][r] * B[r][g] for r = 0..n_factors-1 (U f64 [n_rows][n_factors], B f64
 * [n_factors][n_genes], n_factors <= 64).
 * scb_synth_rows: rows [row0, row0+n_rows) given their logmean rows.  Pass 1 (indptr ==
 * NULL) writes nnz per row into row_nnz; pass 2 fills indices/data of a CSR whose indptr
 * (absolute offsets for these rows) the caller built from row_nnz. */
SCB_API int scb_synth_logmean(scb_ctx* ctx, int64_t n_rows, int32_t n_genes, int32_t n_factors, const double* log_mu,
                              const double* A, const int32_t* cell_type, const double* log_s, const double* U,
                              const double* B, double* logmean, void* stream);
SCB_API int scb_synth_rows(scb_ctx* ctx, uint64_t seed, int64_t row0, int64_t n_rows, int32_t n_genes,
                           const double* logmean, const int64_t* indptr, int64_t* row_nnz, int32_t* indices,
                           float* data, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SCB_H_ */
