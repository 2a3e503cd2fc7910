/* sfgpu — C ABI of the B200-native star-forest (PetscSF) communication layer.
 *
 * This is the drop-in boundary. Every entry point replaces one C++ entry of
 * the reference library (/root/reference/proj/include/sf/...), cited beside
 * it. Signatures carry only plain pointers, sizes and ints (no CUDA, NCCL or
 * torch types); `stream` is a cudaStream_t passed as void*. All functions
 * return SFG_OK or an error code, with the message in sfg_last_error()
 * (thread-local) — the C-ABI rendering of sf::Error / sf::TimeoutError
 * (errors.hpp:11-21). Messages match the reference's where the reference
 * defines one ("forest property", "root offset", ...).
 *
 * Data buffers (rootdata, leafdata, leafupdate, multirootdata) are device
 * pointers on the communicator's GPU. *_end() is stream-ordered: it enqueues
 * the completion of the operation on `stream` and returns; synchronise the
 * stream before reading results on the host (PETSc default-stream model,
 * PAPER.md:722-725). Begin/End calls must be issued in the same order on every
 * rank (they are collective, as in the reference).
 */
#ifndef SFGPU_H
#define SFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFGPU_VERSION 1

typedef struct sfg_world_s* sfg_world;   /* in-process rank world (harness.cpp:51-101) */
typedef struct sfg_comm_s* sfg_comm;     /* sf::Comm (comm.hpp:97-146) */
typedef struct sfg_sf_s* sfg_sf;         /* sf::StarForest (starforest.hpp:61-148) */
typedef struct sfg_handle_s* sfg_handle; /* sf::OpHandle (ops.hpp:31-51) */

enum sfg_status { SFG_OK = 0, SFG_ERR = 1, SFG_ERR_TIMEOUT = 2, SFG_ERR_CUDA = 3 };

/* sf::Kind (unit.hpp:14) */
enum sfg_kind { SFG_INT32 = 0, SFG_INT64 = 1, SFG_FLOAT64 = 2, SFG_BYTES = 3 };

/* sf::ReduceOp (unit.hpp:46) */
enum sfg_op {
  SFG_REPLACE = 0, SFG_SUM = 1, SFG_PROD = 2, SFG_MAX = 3, SFG_MIN = 4,
  SFG_LAND = 5, SFG_LOR = 6, SFG_BAND = 7, SFG_BOR = 8
};

/* sf::SetupAlg (starforest.hpp:41) */
enum sfg_setup_alg { SFG_SETUP_AUTO = 0, SFG_SETUP_DENSE = 1, SFG_SETUP_CONSENSUS = 2 };

/* sf::CommConfig (comm.hpp:54-66); backend/nranks are sfg_comm_create args. */
typedef struct sfg_config {
  int deterministic;             /* 1: reference fold order, bit-exact (default) */
  int debug_checksum;            /* verify begin/end source-buffer stability */
  int force_remote;              /* route self edges through the transport */
  int dense_discovery_threshold; /* kept for API parity; discovery is dense */
  uint64_t seed;
  double timeout_s;
} sfg_config;

/* State / shape of a forest (starforest.hpp:84-100). */
typedef struct sfg_sf_info {
  int state; /* 0 created, 1 graph-set, 2 set-up */
  int self_first;
  int contiguous_leaves;
  int n_root_groups;
  int n_leaf_groups;
  int64_t nroots;
  int64_t nleaves;
  int64_t leaf_index_bound;
} sfg_sf_info;

/* Pattern classification of one neighbor group (pattern.hpp:28-102 plus the
 * Affine3D class the planner infers). kind: 0 contiguous, 1 affine, 2 indexed. */
typedef struct sfg_pattern {
  int kind;
  int has_duplicates;
  int64_t count, start, dx, dy, dz, s1, s2, bound;
} sfg_pattern;

/* Copy instrumentation (pack.hpp:20-32 PackCounters, extended). */
typedef struct sfg_counters {
  uint64_t pack_copies, pack_elided, unpack_copies, unpack_elided;
  uint64_t replace_dup_collisions, kernel_launches, bytes_sent, bytes_recv, transport_calls;
} sfg_counters;

const char* sfg_last_error(void);
int sfg_version(void);
void sfg_config_default(sfg_config* cfg);

/* In-process world of `nranks` thread ranks (run_ranks, harness.hpp:58-72). */
int sfg_world_create(int nranks, double timeout_s, sfg_world* out);
int sfg_world_abort(sfg_world w); /* a failing rank aborts its peers (harness.cpp:75-79) */
int sfg_world_destroy(sfg_world w);

/* ncclUniqueId bytes (128) for one-process-per-GPU communicators. */
int sfg_nccl_unique_id(void* out, size_t bytes);

/* Create rank `rank` of an `nranks` communicator (sf::Comm, make_world
 * comm.cpp:138-143). world != NULL: ranks are threads of this process and the
 * control plane is in-process; world == NULL and nranks > 1: one process per
 * GPU, control plane over NCCL (nccl_id required). backend: "threads"
 * (stream-ordered peer copies, needs a world when nranks > 1), "nccl"
 * (grouped ncclSend/ncclRecv) or "p2p" (one-sided puts into the peer GPU's
 * staging mapped over NVLink with in-kernel flag signalling — the
 * reference's onesided engine, ops.cpp:91,160-246; one GPU per rank; NCCL
 * then only carries the control plane of process-per-GPU runs).
 * device < 0 creates a host-only communicator (set_graph/setup/degrees work,
 * operations do not). */
int sfg_comm_create(sfg_world world, int nranks, int rank, int device, const char* backend,
                    const void* nccl_id, const sfg_config* cfg, sfg_comm* out);
/* Control plane supplied by the caller (e.g. torch.distributed, MPI): the
 * host collectives SetUp and multi_sf need. Each returns 0 on success.
 * allgather: out[r*bytes ..] = rank r's `in`. alltoallv: send holds the
 * payloads for ranks 0..size-1 back to back (send_bytes[r] each), recv
 * receives rank r's payload at the prefix offset of recv_bytes. */
typedef struct sfg_ctrl_ops {
  void* ctx;
  int (*allgather)(void* ctx, const void* in, size_t bytes, void* out);
  int (*alltoallv)(void* ctx, const void* send, const int64_t* send_bytes, void* recv,
                   const int64_t* recv_bytes);
  int (*barrier)(void* ctx);
} sfg_ctrl_ops;
int sfg_comm_create_ext(int nranks, int rank, int device, const char* backend,
                        const void* nccl_id, const sfg_config* cfg, const sfg_ctrl_ops* ops,
                        sfg_comm* out);
int sfg_comm_destroy(sfg_comm c);
int sfg_comm_rank(sfg_comm c, int* rank, int* size, int* device);
/* Host allgather over the communicator's control plane (the reference's
 * Comm::allgather / allreduce building block, comm.hpp:118-127): `out`
 * receives size * bytes, rank r's `in` at r * bytes. Collective. */
int sfg_comm_allgather(sfg_comm c, const void* in, size_t bytes, void* out);

/* sf::StarForest(Comm) (starforest.hpp:64) */
int sfg_sf_create(sfg_comm c, sfg_sf* out);
int sfg_sf_destroy(sfg_sf sf);
/* StarForest::set_graph (starforest.hpp:71-74; starforest.cpp:29-76).
 * leaf_local may be NULL (leaves 0..nleaves-1); remote_rank/remote_off are
 * the RootRef{rank, offset} list split in two arrays. Host pointers. */
int sfg_sf_set_graph(sfg_sf sf, int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                     const int32_t* remote_rank, const int64_t* remote_off);
/* set_graph with the three arrays in the communicator's DEVICE memory (the
 * graph already lives in HBM): same contract, validation and
 * messages as sfg_sf_set_graph; sfg_sf_setup then plans on the GPU
 * (group lists stay in HBM, host copies are made only when asked for). */
int sfg_sf_set_graph_device(sfg_sf sf, int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                            const int32_t* remote_rank, const int64_t* remote_off);
/* StarForest::setup (starforest.hpp:79; starforest.cpp:82-161). Collective.
 * On a device communicator SetUp also builds the device plan, the
 * root-sorted fold plan (when a root has several leaves) and one staging slot
 * for 8-byte units, so no later Begin/End of an 8-byte unit allocates device
 * memory or synchronises the host. */
int sfg_sf_setup(sfg_sf sf, int alg);
/* The same for another unit (kind, blocklen): call before capturing a first
 * operation of that unit into a CUDA graph (Begin inside a capture fails
 * with a message naming this call otherwise). Collective on p2p.
 * Replays of a captured operation must be stream-ordered after eager
 * operations issued earlier on the same forest (they share its staging
 * slots and device message counters). No reference equivalent (the
 * reference has no device state). */
int sfg_sf_prepare(sfg_sf sf, int kind, int64_t blocklen);
int sfg_sf_get_info(sfg_sf sf, sfg_sf_info* out);
/* two_sided() groups: which = 0 root_ranks (items = leaf ordinals),
 * which = 1 leaf_ranks (items = root offsets) — starforest.hpp:47-55. */
int sfg_sf_group(sfg_sf sf, int which, int g, int* rank, int64_t* nitems, sfg_pattern* pat);
int sfg_sf_group_items(sfg_sf sf, int which, int g, int64_t* items);
/* StarForest::compute_degrees (starforest.hpp:105): out[nroots]. */
int sfg_sf_compute_degrees(sfg_sf sf, int64_t* out);
/* StarForest::multi_sf (starforest.hpp:110): borrowed, owned by sf. Collective. */
int sfg_sf_multi_sf(sfg_sf sf, sfg_sf* out);
/* graph_spec() (starforest.hpp:124): leaf indices and RootRefs per ordinal. */
int sfg_sf_graph(sfg_sf sf, int64_t* leaf_index, int32_t* remote_rank, int64_t* remote_off);

/* Split-phase operations (ops.hpp:57-94; ops.cpp:697-876). */
int sfg_bcast_begin(sfg_sf sf, int kind, int64_t blocklen, const void* rootdata, void* leafdata,
                    int op, void* stream, sfg_handle* out);
int sfg_bcast_end(sfg_handle h);
int sfg_reduce_begin(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata,
                     void* rootdata, int op, void* stream, sfg_handle* out);
int sfg_reduce_end(sfg_handle h);
int sfg_fetch_and_op_begin(sfg_sf sf, int kind, int64_t blocklen, void* rootdata,
                           const void* leafdata, void* leafupdate, int op, void* stream,
                           sfg_handle* out);
int sfg_fetch_and_op_end(sfg_handle h);
int sfg_gather_begin(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata,
                     void* multirootdata, void* stream, sfg_handle* out);
int sfg_gather_end(sfg_handle h);
int sfg_scatter_begin(sfg_sf sf, int kind, int64_t blocklen, const void* multirootdata,
                      void* leafdata, void* stream, sfg_handle* out);
int sfg_scatter_end(sfg_handle h);
/* One-shot operations (ops.hpp:60, 68, 79, 88, 94: bcast, reduce,
   fetch_and_op, gather, scatter), stream-ordered: Begin and End back to back
   on `stream` (synchronise it to get the reference's blocking behaviour).
   With nothing of the caller's between the halves, the p2p exchange runs on
   `stream` itself instead of a forked communicator stream. */
int sfg_bcast(sfg_sf sf, int kind, int64_t blocklen, const void* rootdata, void* leafdata, int op,
              void* stream);
int sfg_reduce(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata, void* rootdata, int op,
               void* stream);
int sfg_fetch_and_op(sfg_sf sf, int kind, int64_t blocklen, void* rootdata, const void* leafdata,
                     void* leafupdate, int op, void* stream);
int sfg_gather(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata, void* multirootdata,
               void* stream);
int sfg_scatter(sfg_sf sf, int kind, int64_t blocklen, const void* multirootdata, void* leafdata,
                void* stream);
/* Graph algebra (starforest.hpp:150-171). Collective over the operands'
 * communicator; the new forest is set up (identity: graph set, as the
 * reference's identity_sf). compose: roots of A, leaves of B, an edge where an
 * A leaf and a B root coincide; inverse != 0: compose_inverse (leaves of AB =
 * B's roots; B roots of degree <= 1, A's leaves covered by B's leaves).
 * embed: which = 0 keeps edges whose root is in sel (validated against
 * nroots), 1 edges whose leaf index is in sel (>= 0); indices not remapped. */
int sfg_sf_compose(sfg_sf a, sfg_sf b, int inverse, sfg_sf* out);
int sfg_sf_embed(sfg_sf sf, int which, const int64_t* sel, int64_t n, sfg_sf* out);
int sfg_sf_identity(sfg_comm c, int64_t n, sfg_sf* out);

/* Distributed SpMV over a ghost forest — the path's consumer
 * (spmv.hpp:147-169). A matrix block is uploaded once from host CSR arrays
 * (Csr<T>, spmv.hpp:31-78; kind SFG_FLOAT64 or SFG_INT64) to the
 * communicator's GPU. With ghost_sf = build_column_sf over the off-diagonal
 * block's garray (spmv.cpp:29-43; leaves = lvec, roots = owned x):
 *   sfg_spmv:            y = A x_owned + B lvec, the ghost Bcast overlapped
 *                        with the diagonal product (spmv.hpp:149-157);
 *   sfg_spmv_transpose:  y = A^T x_owned + Reduce_SUM(B^T x_owned)
 *                        (spmv.hpp:161-169).
 * Device pointers, stream-ordered like the operations; results are
 * bit-identical to the reference's Csr loops (no FMA contraction). */
typedef struct sfg_mat_s* sfg_mat;
int sfg_mat_create(sfg_comm c, int64_t rows, int64_t cols, const int64_t* rowptr,
                   const int64_t* colind, const void* vals, int kind, sfg_mat* out);
int sfg_mat_destroy(sfg_mat m);
int sfg_spmv(sfg_sf ghost_sf, sfg_mat diag, sfg_mat offdiag, const void* x_owned, void* lvec,
             void* y, void* stream);
int sfg_spmv_transpose(sfg_sf ghost_sf, sfg_mat diag, sfg_mat offdiag, const void* x_owned,
                       void* lvec, void* y, void* stream);

/* Handle introspection (OpHandle::kind/op/ended, ops.hpp:38-45) and release.
 * Freeing a handle that was begun but never ended fails on the p2p backend
 * (the staging slot is retired, the handle is still freed). */
int sfg_handle_info(sfg_handle h, int* opkind, int* op, int* ended);
int sfg_handle_free(sfg_handle h);

/* IndexPattern::analyze (pattern.hpp:52-53). infer_affine = 0 reproduces the
 * reference's classification; extents (X, XY) > 0 enable its strided path. */
int sfg_pattern_analyze(const int64_t* idx, int64_t n, int infer_affine, int64_t extents_x,
                        int64_t extents_xy, sfg_pattern* out);

int sfg_counters_get(sfg_counters* out);
int sfg_counters_reset(void);

/* Per-launch device timing: when enabled, CUDA events are recorded on the
 * launching stream around every kernel of the library; collect() waits for
 * them and aggregates per launch tag ("bcast_begin", "reduce_end", ...),
 * with the launch's algorithmic bytes (compulsory HBM traffic) and the bytes
 * it stored over NVLink into peer GPUs (one-sided puts of the p2p backend). */
typedef struct sfg_timing {
  char tag[32];
  uint64_t launches;
  double total_ms;
  double bytes;
  double link_bytes; /* bytes stored into peer GPUs' memory (p2p puts) */
} sfg_timing;
/* Debug: with SFG_TRACE_LAUNCHES=N in the environment, %globaltimer marks
 * of the first N multi-segment launches (put / receive CTA start and end,
 * LL data ready, launch end) are written to `path` as JSON lines. */
int sfg_trace_dump(const char* path);
int sfg_timing_enable(int on);
int sfg_timing_collect(sfg_timing* out, int cap, int* n);

#ifdef __cplusplus
}
#endif

#endif /* SFGPU_H */
