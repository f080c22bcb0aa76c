/*
 * catgnn.h — C ABI of the B200-native CATGNN per-partition training step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/gnnpart/train.hpp, proj/src/train.cpp).  The
 * reference exposes a statically linked C++ namespace (`gnnpart::`) with no FFI
 * layer; every entry point below names the reference function it replaces.
 * INTEGRATION.md shows the binding a maintainer adds on the reference side.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *  - Return codes mirror the reference CLI's error categories
 *    (proj/include/gnnpart/common.hpp:16-24, proj/tools/gnnpart.cpp:387-399):
 *    0 ok, 2 ConfigError (bad parameters), 3 DataError (bad/inconsistent input),
 *    4 internal error (incl. CUDA failures).  The message of the last failure
 *    on the calling thread is returned by catgnn_last_error().  No exceptions
 *    cross the ABI.
 *  - The caller owns every host buffer it passes; the library owns device
 *    memory behind opaque handles, released by the matching *_destroy call.
 *  - All device work runs on the stream of the catgnn_ctx the object was
 *    created on.  A handle is not thread-safe.
 *  - Host float parameters/features are float32 row-major; the device computes
 *    in float32 (tensor-core GEMMs in TF32 with float32 accumulation).
 */
#ifndef CATGNN_H
#define CATGNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CATGNN_OK 0
#define CATGNN_ECONFIG 2
#define CATGNN_EDATA 3
#define CATGNN_EINTERNAL 4

typedef struct catgnn_ctx_s* catgnn_ctx;         /* device + stream + scratch */
typedef struct catgnn_artifact_s* catgnn_artifact; /* host view of a stored artifact */
typedef struct catgnn_shard_s* catgnn_shard;     /* device-resident shard (CSR, features, roles) */
typedef struct catgnn_model_s* catgnn_model;     /* GNN replica: params + optimizer state */
typedef struct catgnn_comm_s* catgnn_comm;       /* NCCL communicator (one rank per GPU) */
typedef struct catgnn_features_s* catgnn_features; /* device copy of the global feature matrix */
typedef struct catgnn_completion_s* catgnn_completion; /* per-partition edges + node tables */
typedef struct catgnn_index_s* catgnn_index;           /* GraphIndex: interned ids + degrees */

const char* catgnn_last_error(void);
int catgnn_version(void);

/* ---------------------------------------------------------------- context */
/* stream: a cudaStream_t to run on, or NULL to create a private stream. */
int catgnn_ctx_create(int device, void* stream, catgnn_ctx* out);
int catgnn_ctx_destroy(catgnn_ctx ctx);
int catgnn_ctx_synchronize(catgnn_ctx ctx);
/* Stream ordering between contexts of one device: work enqueued on `waiter`
 * after this call runs after everything enqueued on `producer` so far
 * (event record + stream wait; capturable into a CUDA graph).  Library calls
 * that read another context's objects (model averaging, parameter copies)
 * order themselves this way. */
int catgnn_ctx_wait(catgnn_ctx waiter, catgnn_ctx producer);
/* Persistent-grid budgets of this context's kernels: K2 aggregation grids
 * cover agg_sms SMs and K3 GEMM grids gemm_sms SMs (0 = all).  Budgets below
 * the SM count let shard lanes on other contexts' streams run beside them. */
int catgnn_ctx_set_sm_budget(catgnn_ctx ctx, int agg_sms, int gemm_sms);
/* Number of CUDA kernels this library launched on ctx since creation (evidence
 * for bench.py's gpu_launches; counts launches, not graph replays). */
uint64_t catgnn_ctx_launch_count(catgnn_ctx ctx);
/* Device time (ms) accumulated by the aggregation kernel (K2) and the GEMM
 * kernel (K3) while timing is enabled (CUDA events on ctx's stream). */
int catgnn_ctx_set_kernel_timing(catgnn_ctx ctx, int enable);
/* Diagnostics: per-label totals of the launches timed since the last
 * catgnn_ctx_set_kernel_timing (labels name the kernel and its shape).  Writes
 * record i as "label<TAB>ms_total<TAB>launches" into buf and the number of
 * records into *count (buf may be NULL to query the count).  No reference
 * counterpart (the reference has no device kernels). */
int catgnn_ctx_timing_record(catgnn_ctx ctx, uint32_t i, char* buf, uint32_t cap, uint32_t* count);
int catgnn_ctx_kernel_time(catgnn_ctx ctx, double* agg_ms, uint64_t* agg_launches,
                           double* gemm_ms, uint64_t* gemm_launches);

/* -------------------------------------------------- artifact (A1-A3 input) */
/* Reads manifest.json, part-<i>/{edges.bin,nodes.tsv}, labels.tsv and verifies
 * every count like read_partitions (proj/src/store.cpp:269-333). */
int catgnn_artifact_open(const char* dir, catgnn_artifact* out);
int catgnn_artifact_close(catgnn_artifact a);
typedef struct {
  uint32_t num_partitions;
  uint64_t num_nodes;
  uint64_t num_edges;
  uint32_t feature_dim;
  int has_features;
  int has_meta;
  int add_reverse;
  double replication_factor;          /* recomputed: metrics.cpp:9-12 */
  double manifest_replication_factor; /* as stored by write_partitions */
} catgnn_artifact_info;
int catgnn_artifact_get_info(catgnn_artifact a, catgnn_artifact_info* info);
/* Per-partition counts as in the manifest. */
int catgnn_artifact_part_counts(catgnn_artifact a, uint32_t part, uint64_t* nodes,
                                uint64_t* owned, uint64_t* edges);
/* Replica / halo map of one partition, in node-table (= local row) order:
 * external id, owner flag, role (0 none, 1 train, 2 val, 3 test) and the home
 * partition (owner partition of that node; == part for owners). */
int catgnn_artifact_replica_map(catgnn_artifact a, uint32_t part, uint64_t* ext_ids,
                                uint8_t* owner, uint8_t* role, uint32_t* home);

/* The same home map for a loaded partition shard, built on the shard's device
 * (K1's radix sort of every partition's owned ids, then a binary search of
 * the shard's replica table; completion.cpp:46-50): home[r] for each local
 * row (host array of rows entries, may be NULL) and the number of halo rows
 * (replicas this partition does not own).  Dense ids below 2^32. */
int catgnn_shard_halo_map(catgnn_shard s, catgnn_artifact a, uint32_t* home, uint64_t* n_halo);

/* ------------------------------------------------------------ shards (A3-A4) */
/* load_training_data (train.cpp:216-287) for one shard: part >= 0 is a
 * partition shard (local row i = i-th record of part-<i>/nodes.tsv; features
 * from part-<i>/features.bin or gathered from the global feature file);
 * part == -1 is the global shard (full edge stream, no dedup).  input/features
 * override the paths recorded in the manifest when non-NULL/non-empty. */
int catgnn_shard_load(catgnn_ctx ctx, catgnn_artifact a, int32_t part, const char* input,
                      const char* features, catgnn_shard* out);
/* build_adjacency (train.cpp:30-47) on the device from host local pairs
 * (pairs[2k], pairs[2k+1]) in edge order.  features may be NULL (dim 0). */
int catgnn_shard_create(catgnn_ctx ctx, uint32_t rows, const uint32_t* pairs, uint64_t num_edges,
                        const float* features, uint32_t dim, catgnn_shard* out);
/* Shard from an in-memory partition (what complete_edges produced): node table
 * (ascending external ids, owner flags, roles), external-id edges in stream
 * order, labels per local row, and features per local row (rows x dim). */
int catgnn_shard_create_from_part(catgnn_ctx ctx, uint64_t rows, const uint64_t* ext_ids,
                                  const uint8_t* owner, const uint8_t* role,
                                  const int32_t* labels, const uint64_t* edges_ext,
                                  uint64_t num_edges, const float* features, uint32_t dim,
                                  catgnn_shard* out);
int catgnn_shard_destroy(catgnn_shard s);
/* Labels and role rows in local row space (train rows = owner && role==train). */
int catgnn_shard_set_labels(catgnn_shard s, const int32_t* labels, const uint32_t* train_rows,
                            uint64_t n_train, const uint32_t* val_rows, uint64_t n_val,
                            const uint32_t* test_rows, uint64_t n_test);
/* Re-upload features (host rows x dim) into the resident device buffer. */
int catgnn_shard_upload_features(catgnn_shard s, const float* features, uint32_t dim);
/* Global feature matrix on the device (rows x dim f32, FEA1 row order, dense):
 * the source load_training_data gathers replica rows from when a partition has
 * no features.bin (proj/src/train.cpp:277-283).  upload copies host rows
 * [row_begin, row_begin+nrows) (pinned memory for full PCIe/C2C bandwidth);
 * gather sets the shard's input rows x[r] = F[ext_id(r)] on the device.
 * The store may live on another context (stream) of the same device: uploads
 * then run on that stream and are ordered against gathers by events (an upload
 * waits for the previous contents' gathers), so two stores can double-buffer
 * the host->device copy of the next step's features behind this step's work. */
int catgnn_features_create(catgnn_ctx ctx, uint64_t rows, uint32_t dim, catgnn_features* out);
int catgnn_features_destroy(catgnn_features f);
int catgnn_features_upload(catgnn_features f, const float* host, uint64_t row_begin, uint64_t nrows);
/* Forget the store's recorded upload / gather events; the caller orders its
 * producers and consumers by stream order from then on (before capturing a
 * CUDA graph that uploads into and gathers from the store). */
int catgnn_features_reset_deps(catgnn_features f);
/* split_features (proj/include/gnnpart/store.hpp:63, store.cpp:97-116): writes
 * <out_dir>/part-<s>/features.bin (FEA1) holding the rows of the global FEA1
 * matrix `features` named by partition s's node table, in node-table order —
 * byte-identical to the reference's files.  The matrix is read once and the
 * rows are gathered on the device instead of one seek per node record.
 * DataError (3) for a bad header or a node id past the matrix. */
int catgnn_split_features(catgnn_ctx ctx, catgnn_artifact a, const char* features, const char* out_dir,
                          uint32_t* files_written);
int catgnn_shard_gather_features(catgnn_shard s, catgnn_features f);
/* Device feature layout (no reference counterpart).  split_only = 1: gathers
 * write only the bf16x3 (hi, lo) copy that the GNN layers' tensor-core GEMMs
 * read (half the write traffic of keeping fp32 rows too); calls needing the
 * fp32 rows (SGC propagation, feature export, a model whose first layer is not
 * on the bf16x3 path) fail with ConfigError until the next upload. */
int catgnn_shard_set_feature_layout(catgnn_shard s, int split_only);
/* Multi-GPU refresh of a feature store: rank r uploads rows [r*R, (r+1)*R)
 * (catgnn_features_upload with row_begin = r*R), then this in-place NCCL
 * all-gather over NVLink completes every rank's copy (store rows >= R x ranks)
 * — each GPU's host link carries 1/N of the matrix.  Runs on the store's stream
 * (use a communicator created on that context). */
int catgnn_features_allgather(catgnn_features f, catgnn_comm c, uint64_t rows_per_rank);
typedef struct {
  uint64_t rows;
  uint64_t nnz;
  uint32_t dim;
  uint32_t classes; /* max(label)+1 over the shard, >= 1 */
  uint64_t n_train, n_val, n_test;
  uint64_t heavy_rows; /* rows split across several aggregation tasks */
  uint64_t tasks;      /* aggregation work items */
} catgnn_shard_info;
int catgnn_shard_get_info(catgnn_shard s, catgnn_shard_info* info);
/* The train-row views a train step aggregates its last layer over (no
 * reference counterpart; measurement): rows / neighbour entries of the train
 * rows' CSR rows and the neighbour entries that point at train rows (built if
 * needed; zeros when the shard has no train rows). */
int catgnn_shard_train_views(catgnn_shard s, uint64_t* sub_rows, uint64_t* sub_nnz, uint64_t* nbr_nnz);
/* Bit-exact export of the device CSR (offsets widened to u64). */
int catgnn_csr_export(catgnn_shard s, uint64_t* offsets, uint32_t* neighbors);
int catgnn_shard_role_rows(catgnn_shard s, int role, uint32_t* rows);
int catgnn_shard_labels(catgnn_shard s, int32_t* labels);
/* which: 0 = input features, 1 = SGC-propagated features. */
int catgnn_shard_export_features(catgnn_shard s, int which, float* out);

/* Device read bandwidth (GB/s) over a `bytes` buffer read `passes` times with
 * 128-bit L2-cached loads: < 126 MB measures L2, GBs measure HBM (roofline
 * denominators; not a reference function). */
int catgnn_probe_read_bandwidth(catgnn_ctx ctx, uint64_t bytes, int passes, double* gbs);

/* ------------------------------------------------ graph index (§8(f) row 3) */
/* compute_degrees (proj/src/edge_stream.cpp:192-215) on the device: external ids
 * interned in first-seen order (record (u, v): u first), degree per node with
 * self-loops counting 2, record and self-loop counts.  edges = 2 x num_edges
 * host ids in stream order. */
int catgnn_index_build(catgnn_ctx ctx, const uint64_t* edges, uint64_t num_edges, catgnn_index* out);
int catgnn_index_info(catgnn_index idx, uint64_t* num_nodes, uint64_t* num_edges, uint64_t* num_self_loops);
/* dense_to_ext[num_nodes], degree[num_nodes] (GraphIndex fields) */
int catgnn_index_export(catgnn_index idx, uint64_t* dense_to_ext, uint32_t* degree);
int catgnn_index_destroy(catgnn_index idx);

/* --------------------------------------------- neighbour completion (A1) */
/* complete_edges (proj/src/completion.cpp:130-171, PartitionBuilder :13-58) on
 * the device: edges = 2 x num_edges external ids in stream order, which must be
 * dense (every id in [0, num_nodes) a node of the stream, as
 * load_training_data requires, train.cpp:234-240); home[v] = SPRING's home
 * partition (HomeMap, completion.hpp:55-59); roles[v] = 0 none / 1 train /
 * 2 val / 3 test or NULL.  hops in {1,2,3}.  Per partition: one record per
 * unordered pair (first occurrence, original orientation, stream order) and the
 * node table (ascending ext id, owner flag, role on owners only).  Errors as
 * the reference: hops outside {1,2,3} -> 2, home out of range -> 3. */
int catgnn_complete_edges(catgnn_ctx ctx, const uint64_t* edges, uint64_t num_edges, const uint32_t* home,
                          const uint8_t* roles, uint64_t num_nodes, uint32_t p, uint32_t hops,
                          catgnn_completion* out);
/* Same over an edge file (EDG1 `.bin` streamed in chunks through one pinned
 * buffer — the stream never sits in host RAM; text files are read whole), with
 * EdgeReader's add_reverse expansion (edge_stream.cpp:138-148) done on the
 * device.  Identical results to reading the stream and calling
 * catgnn_complete_edges. */
int catgnn_complete_edges_file(catgnn_ctx ctx, const char* path, int add_reverse, const uint32_t* home,
                               const uint8_t* roles, uint64_t num_nodes, uint32_t p, uint32_t hops,
                               catgnn_completion* out);
/* Same for arbitrary 64-bit external ids: endpoints are routed through the
 * device graph index (GraphIndex::dense); home[] and roles[] are indexed by
 * dense id as the reference's HomeMap (completion.hpp:55-59) is. */
int catgnn_complete_edges_indexed(catgnn_ctx ctx, catgnn_index index, const uint64_t* edges, uint64_t num_edges,
                                  const uint32_t* home, const uint8_t* roles, uint32_t p, uint32_t hops,
                                  catgnn_completion* out);
int catgnn_completion_part_counts(catgnn_completion c, uint32_t part, uint64_t* edges, uint64_t* nodes,
                                  uint64_t* owned);
int catgnn_completion_part(catgnn_completion c, uint32_t part, uint64_t* edges, uint64_t* ext, uint8_t* owner,
                           uint8_t* role);
int catgnn_completion_destroy(catgnn_completion c);

/* ---------------------------------------------------------- SGC path (A5-A13) */
/* sgc_propagate (train.cpp:49-65): hops rounds of (x_i + sum_j x_j)/(1+deg_i),
 * stored in the shard's propagated buffer. */
int catgnn_sgc_propagate(catgnn_shard s, uint32_t hops);
/* softmax_loss / softmax_gradient (train.cpp:74-94) over the listed rows of the
 * propagated features.  W is dim x classes row-major, b is classes. */
int catgnn_softmax_loss(catgnn_shard s, const float* W, const float* b, uint32_t classes,
                        const uint32_t* rows, uint64_t n_rows, double* loss);
int catgnn_softmax_gradient(catgnn_shard s, const float* W, const float* b, uint32_t classes,
                            const uint32_t* rows, uint64_t n_rows, float* gW, float* gb);
/* train_epochs (train.cpp:96-128) for n replicas at once, one shard each:
 * W[i]/b[i] are host in/out parameter buffers; replica i uses seeds[i]. */
int catgnn_train_epochs(uint32_t n, const catgnn_shard* shards, float* const* W, float* const* b,
                        uint32_t classes, double lr, uint32_t batch, uint64_t epoch_begin,
                        uint64_t epoch_end, const uint64_t* seeds);
/* sync_weights (train.cpp:139-152). */
int catgnn_sync_weights(const uint64_t* counts, uint32_t n, double* alpha);
/* model_average (train.cpp:154-172) of n host parameter blocks of `count`
 * floats each (W and b flattened); result into out. */
int catgnn_model_average_host(catgnn_ctx ctx, uint32_t n, const float* const* params,
                              uint64_t count, const uint64_t* train_counts, float* out);
/* evaluate_micro_f1 (train.cpp:174-198) on the propagated features. */
int catgnn_evaluate_micro_f1(catgnn_shard s, const float* W, const float* b, uint32_t classes,
                             const uint32_t* mask_rows, uint64_t n_mask, double* f1);

typedef struct {
  uint32_t epochs;    /* TrainConfig (train.hpp:42-48) */
  double lr;
  uint32_t batch;
  uint32_t prop_hops;
  uint64_t seed;
} catgnn_train_config;
typedef struct {
  float* W;           /* out: dim x classes (caller-allocated, may be NULL) */
  float* b;           /* out: classes */
  uint32_t dim, classes;
  uint64_t* hist_epoch; uint64_t* hist_syncs; double* hist_val; double* hist_test;
  uint64_t hist_capacity;
  uint64_t n_hist;
  uint64_t averaging_ops;
} catgnn_dist_result;
/* distributed_train (train.cpp:289-340) over p partition shards + the global
 * shard for evaluation; workers q must divide p (results are independent of q). */
int catgnn_distributed_train(uint32_t p, const catgnn_shard* shards, catgnn_shard global,
                             uint32_t workers, uint32_t sync_interval,
                             const catgnn_train_config* cfg, catgnn_dist_result* result);

/* ------------------------------------------------- GNN models (north-star rows) */
#define CATGNN_MODEL_GCN 1  /* h' = D^-1/2 (A+I) D^-1/2 h W^T + b           */
#define CATGNN_MODEL_SAGE 2 /* h' = h W_s^T + mean_N(h) W_n^T + b          */
#define CATGNN_MODEL_GIN 3  /* h' = ((1+eps) h + sum_N h) W^T + b, eps = 0 */
/* h' = D~^-1 (A+I) h W^T + b, zero-initialised: with one layer this is the
 * reference's own model (sgc_propagate with prop_hops = 1, then softmax
 * regression, train.cpp:49-94, zero_params :67-72), here trained full-batch
 * through the GNN kernels (K2 + K3 + K4 + K5) so that machinery can be checked
 * against the compiled reference's distributed_train. */
#define CATGNN_MODEL_SGC 4
#define CATGNN_OPT_SGD 0
#define CATGNN_OPT_ADAM 1
typedef struct {
  int kind;
  uint32_t layers;
  uint32_t in_dim;
  uint32_t hidden;
  uint32_t classes;
  int optimizer;
  double lr;
  double beta1, beta2, eps; /* Adam */
  uint64_t seed;            /* init: splitmix of seed_for(seed, layer) */
} catgnn_model_config;
int catgnn_model_create(catgnn_ctx ctx, const catgnn_model_config* cfg, catgnn_model* out);
int catgnn_model_destroy(catgnn_model m);
/* Storage of the aggregation inputs (no reference counterpart; numerics only):
 * on (default, env CATGNN_ACT_F16=0 turns it off) the GCN backward gradients
 * and last-layer logits inputs are gathered as fp16 rows (fp32 accumulation,
 * ~2e-4 relative on gradients), off keeps every K2 input fp32. */
int catgnn_model_set_act_f16(catgnn_model m, int on);
uint64_t catgnn_model_num_params(catgnn_model m);
/* Flat parameter vector: per layer W (row-major, shape given by
 * catgnn_model_layer_shape) followed by b. */
int catgnn_model_layer_shape(catgnn_model m, uint32_t layer, uint32_t* w_rows, uint32_t* w_cols,
                             uint64_t* offset_w, uint64_t* offset_b);
int catgnn_model_get_params(catgnn_model m, float* out);
int catgnn_model_set_params(catgnn_model m, const float* in);
int catgnn_model_copy_params(catgnn_model dst, catgnn_model src);
int catgnn_model_get_grads(catgnn_model m, float* out);
/* One local iteration: full-batch forward + backward over the shard, loss on
 * the shard's train rows (mean CE), then one optimizer step.  loss may be NULL
 * (then no device->host read happens). */
int catgnn_model_train_step(catgnn_model m, catgnn_shard s, double* loss);
/* Loss of the last train_step (computed on the device either way); lets a
 * caller run several replicas' steps back to back and sync once. */
int catgnn_model_last_loss(catgnn_model m, double* loss);
/* Same, asynchronous: enqueues the copy of the loss sum into host_sum (pinned
 * host memory; capturable into a CUDA graph) and returns the train-row count
 * in *rows; the mean is *host_sum / *rows after the context synchronises. */
int catgnn_model_last_loss_async(catgnn_model m, double* host_sum, uint64_t* rows);
/* Forward + backward only (no update); gradients readable by get_grads. */
int catgnn_model_forward_backward(catgnn_model m, catgnn_shard s, double* loss);
/* Forward only; logits rows x classes into out (host) when out != NULL;
 * micro-F1 over role rows (2 val, 3 test) when f1 != NULL. */
int catgnn_model_forward(catgnn_model m, catgnn_shard s, float* logits, int role, double* f1);
/* Debug export of layer activations after forward/backward:
 * what 0 = layer output H_l (post activation), 1 = pre-activation Z_l,
 * 2 = dZ_l.  out holds rows x width(layer) floats. */
int catgnn_model_export(catgnn_model m, uint32_t layer, int what, float* out, uint32_t* width);
/* In-process model averaging (train.cpp:154-172): dst = sum_i alpha_i src_i,
 * alpha from sync_weights(train_counts); dst may alias one of src. */
int catgnn_model_average(uint32_t n, const catgnn_model* src, const uint64_t* train_counts,
                         catgnn_model dst);
/* Weighted sum with caller-supplied weights (model_average's loop,
 * train.cpp:164-169, with alpha from the GLOBAL sync_weights): a rank's share
 * of the cross-rank average before catgnn_model_allreduce.  Zero weights are
 * fine (a rank whose partitions hold no train rows contributes zeros). */
int catgnn_model_weighted_sum(uint32_t n, const catgnn_model* src, const double* alpha, catgnn_model dst);

/* ------------------------------------ GNN distributed training (north star) */
/* distributed_train (train.cpp:289-340, train.hpp:118-124) for the GNN models:
 * the artifact's partitions are loaded (load_training_data, train.cpp:216-287),
 * each trained full-batch (one local iteration = forward + backward + one
 * optimizer step), and every sync_interval iterations
 * (chunks of min(s, remaining), :315-316) the replicas restart from the
 * alpha-weighted average of all partitions (sync_weights over the partitions'
 * owner && train counts, :139-172).  After each average the val / test
 * micro-F1 of the averaged model on the global graph is recorded (:324-335)
 * when eval_global is set.
 * comm == NULL: this process trains every partition.  Otherwise rank r of the
 * communicator trains partitions r, r + nranks, ... and the
 * average is the alpha-prescaled weighted sum + ncclAllReduce over NVLink.
 * Errors as the reference: workers == 0 or p % workers != 0 or
 * sync_interval == 0 -> ConfigError (2); p % nranks != 0 -> ConfigError. */
typedef struct {
  catgnn_model_config model; /* in_dim 0 = the artifact's feature width; classes 0 = max label + 1 */
  uint32_t epochs;           /* local iterations */
  uint32_t sync_interval;
  uint32_t workers;          /* logical workers q (the reference's p % q check) */
  int eval_global;           /* record val/test micro-F1 on the global graph per sync */
} catgnn_gnn_train_config;
typedef struct {
  float* params;             /* out: logical flat parameters (catgnn_model_get_params layout) or NULL */
  uint64_t params_capacity;  /* floats available at params */
  uint64_t num_params;       /* out */
  double* losses;            /* out: per local iteration sum_i alpha_i mean-CE_i over ALL partitions */
  uint64_t loss_capacity;
  uint64_t n_losses;         /* out */
  uint64_t* hist_epoch; uint64_t* hist_syncs; double* hist_val; double* hist_test;
  uint64_t hist_capacity;
  uint64_t n_hist;           /* out */
  uint64_t averaging_ops;    /* out */
  uint32_t in_dim, classes;  /* out: resolved model widths */
  catgnn_model* model_out;   /* if non-NULL, receives the averaged model (destroy with catgnn_model_destroy) */
} catgnn_gnn_result;
int catgnn_gnn_distributed_train(catgnn_ctx ctx, const char* artifact_dir, const char* input,
                                 const char* features, const catgnn_gnn_train_config* cfg,
                                 catgnn_comm comm, catgnn_gnn_result* result);
/* train_local (train.cpp:130-137) on the device: zero_params + train_epochs
 * over the shard's train rows with cfg->seed, on the shard's features
 * propagated prop_hops times (the --compare-centralized path of train-sim,
 * gnnpart.cpp:330-339, calls it on the global shard).  W (dim x classes) and b
 * (classes) are outputs; classes = max label + 1 over the shard. */
int catgnn_train_local(catgnn_shard s, const catgnn_train_config* cfg, float* W, float* b, uint32_t* classes);

/* ---------------------------------------------------------- multi-GPU (C1) */
int catgnn_comm_unique_id(char id[128]);
int catgnn_comm_create(catgnn_ctx ctx, int nranks, int rank, const char id[128], catgnn_comm* out);
int catgnn_comm_destroy(catgnn_comm c);
/* Model averaging across ranks: params <- allreduce_sum(alpha * params) where
 * alpha = this rank's share (sum of its replicas' alphas is folded by the
 * caller via catgnn_model_scale). */
int catgnn_model_scale(catgnn_model m, double alpha);
int catgnn_model_allreduce(catgnn_model m, catgnn_comm c);

/* ------------------------------------------------------------- utilities */
/* Tensor-core GEMM test hook: C[M x N] = A[M x K] . B[N x K]^T (all host,
 * row-major float32), computed by the tcgen05 kernel; precision 1 = TF32,
 * 3 = 3xTF32 (split operands, ~fp32 accuracy); split_k 0 = automatic. */
int catgnn_gemm_tn(catgnn_ctx ctx, uint32_t M, uint32_t N, uint32_t K, const float* A,
                   const float* B, float* C, uint32_t split_k, int precision);
/* General form: A given as M x K (a_mn = 0) or K x M (a_mn = 1, read MN-major
 * by the tensor core), B as N x K or K x N; C[M x N] = A . B^T.  precision 4 =
 * bf16x3: both operands split on the device into bf16 (hi, lo) pairs and
 * multiplied as lo*hi + hi*lo + hi*hi with kind::f16 MMAs (~2^-16 relative). */
int catgnn_gemm(catgnn_ctx ctx, uint32_t M, uint32_t N, uint32_t K, const float* A, int a_mn,
                const float* B, int b_mn, float* C, uint32_t split_k, int precision);
/* Synthetic RMAT(a,b,c,1-a-b-c) stream of num_edges unique undirected pairs, no
 * self-loops, first-seen orientation, ids compacted to 0..|V|-1 (bench input
 * preparation).  out_edges holds 2*num_edges u64. */
int catgnn_synth_rmat(uint32_t scale, uint64_t num_edges, double a, double b, double c,
                      uint64_t seed, uint64_t* out_edges, uint64_t* num_nodes);

#ifdef __cplusplus
}
#endif
#endif /* CATGNN_H */
