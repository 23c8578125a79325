/*
 * tileinv_b200.h -- C-ABI of the B200-native SPD tile inversion engine.
 *
 * Drop-in boundary for the reference package `tileinv`
 * (arxiv/paper_1002_4057, /root/reference/pkg/src/tileinv). The reference is
 * pure Python over numpy; its "FFI" for this path is the Python call surface
 * below, which the ctypes shim `paper_1002_4057_b200/_native.py` binds 1:1:
 *
 *   reference interface                                  replaced by
 *   -----------------------------------------------------------------------
 *   tile_matrix.from_dense(m, b)       tile_matrix.py:84-99   tinv_create + tinv_put_dense
 *   tile_matrix.to_dense(tm)           tile_matrix.py:102-114 tinv_get_dense(mode=LOWER)
 *   symmetrize_lower(to_dense(tm))     tile_matrix.py:117-119 tinv_get_dense(mode=SYMMETRIZE)
 *   tm.tile(i,j) / tm.set_tile(...)    tile_matrix.py:53-57   tinv_get_tile / tinv_put_tile
 *   taskgen.gen_step1/2/3, gen_inversion taskgen.py:230-269   tinv_gen_stream
 *   scheduler.build_dag                scheduler.py:101-153   tinv_dag_edges
 *   scheduler.execute(stream, a, w)    scheduler.py:261-351   tinv_plan_create + tinv_plan_exec
 *   scheduler.run_in_order(stream, a)  scheduler.py:248-258   same, flags |= TINV_SERIAL
 *   scheduler.run_task -> kernels.*    scheduler.py:206-235   executed on device per task kind
 *   ExecutionError(task, cause)        scheduler.py:185-190   tinv_err {task, kind, code, index}
 *
 * All arithmetic is IEEE FP64. Plain pointers and sizes only; no torch types.
 * Every call blocks until the device work it issued has finished.
 * A context is not thread-safe; use one context per host thread.
 */
#ifndef TILEINV_B200_H
#define TILEINV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TINV_ABI_VERSION 1

/* status codes */
#define TINV_OK 0
#define TINV_ERR_NOT_SPD 1     /* kernels.py:38-43  NotPositiveDefiniteError */
#define TINV_ERR_SINGULAR 2    /* kernels.py:46-51  SingularTileError        */
#define TINV_ERR_BAD_ARG 3     /* ValueError / InvalidSizeError               */
#define TINV_ERR_CUDA 4        /* CUDA runtime/driver failure                 */
#define TINV_ERR_STREAM 5      /* malformed stream (scheduler.py:274-276 and store KeyError) */
#define TINV_ERR_NO_DEVICE 6   /* no usable sm_100 device                     */
#define TINV_ERR_INTERNAL 7    /* executor watchdog / invariant violation     */

/* kernel kinds; COPY = taskgen.py:164-170, the rest = kernels.py:23-35 */
#define TINV_COPY 0
#define TINV_POTRF 1
#define TINV_TRSM 2
#define TINV_SYRK_SUB 3
#define TINV_SYRK_ADD_T 4
#define TINV_GEMM 5
#define TINV_TRTRI 6
#define TINV_TRMM_LEFT 7
#define TINV_TRMM_RIGHT_NEG 8
#define TINV_TRMM_LEFT_T 9
#define TINV_LAUUM 10

/* steps (taskgen.py:37-41); select the GEMM shape (scheduler.py:198-203) */
#define TINV_STEP_COPY 0
#define TINV_STEP_CHOLESKY 1
#define TINV_STEP_TRINV 2
#define TINV_STEP_PRODUCT 3

/* One task = TINV_TASK_FIELDS int32 (Task, taskgen.py:55-87):
 * kind, step, i, j, k, out_label, out_row, out_col, out_mode, nreads,
 * r0_label, r0_row, r0_col, r1_label, r1_row, r1_col.
 * Labels are small ints: 0 = the matrix being executed on (its TileMatrix
 * label), 1.. = working arrays (B, C, ...). out_mode: 1 = RW, 2 = W (COPY).
 * Unused index / read fields are -1. */
#define TINV_TASK_FIELDS 16

/* execution flags */
#define TINV_SERIAL 1u          /* chain tasks in stream order (run_in_order) */
#define TINV_TRACE 2u           /* record per-task device timestamps          */
#define TINV_KEEP_ON_FAILURE 4u /* snapshot the matrix; restore it if a task fails */
#define TINV_STREAM_IO 8u       /* plan for tinv_plan_exec_host: tile arrivals and departures are tasks */
#define TINV_SHARE_SLOTS 16u    /* memory-constrained renaming: working tiles (B / C copies, aux) share
                                   slots by live range in stream order, reuse ordered by added edges */

/* tinv_get_dense modes */
#define TINV_DENSE_LOWER_TILES 0 /* write only the lower tiles (to_dense on them) */
#define TINV_DENSE_SYMMETRIZE 1  /* full matrix: lower + mirrored upper          */

typedef struct tinv_err {
  int32_t task_id;  /* reference task id of the stream-order-first failure, -1 if none */
  int32_t kind;     /* its kernel kind                                             */
  int32_t code;     /* TINV_ERR_*                                                  */
  int32_t index;    /* tile-local index (pivot / zero diagonal), -1 if n/a         */
} tinv_err;

typedef struct tinv_ctx tinv_ctx;
typedef struct tinv_plan tinv_plan;

int tinv_abi_version(void);
/* number of usable devices (sm_100), or a negative TINV_ERR_* */
int tinv_device_count(void);
/* last error message of a context (or the global one when ctx == NULL) */
const char* tinv_last_error(const tinv_ctx* ctx);

/* TileMatrix (tile_matrix.py:35-66): order n, tile order b, on `device`. */
int tinv_create(tinv_ctx** ctx, int64_t n, int64_t b, int device);
/* A batch of `batch` independent order-n matrices in one device store
 * (BASELINE config 4). Dense transfers then move `batch` matrices stored back
 * to back (matrix m at offset m * n * lda); a plan made from a one-matrix
 * stream runs it on every matrix as one merged DAG (independent chains).
 * Error task ids are m * ntasks + task. Tile calls address matrix 0. */
int tinv_create_batch(tinv_ctx** ctx, int64_t batch, int64_t n, int64_t b, int device);
int tinv_destroy(tinv_ctx* ctx);
int tinv_shape(const tinv_ctx* ctx, int64_t* n, int64_t* b, int64_t* t, int64_t* padded_b);
/* bytes of the context's device tile store (grows to the largest plan run on it) */
int tinv_store_bytes(const tinv_ctx* ctx, int64_t* bytes);
/* run the context's device work on a caller-owned cudaStream_t (NULL restores
 * the context's own stream), so callers can time it with their own events */
int tinv_set_stream(tinv_ctx* ctx, void* cuda_stream);

/* dense row-major matrices (leading dimension lda >= n). `host` variants take
 * host pointers (pinned memory is faster, pageable works); `device` variants
 * take device pointers on the context's device. put copies only the lower
 * tiles (the authoritative ones, tile_matrix.py:62-66). */
int tinv_put_dense(tinv_ctx* ctx, const double* host, int64_t lda);
int tinv_get_dense(tinv_ctx* ctx, double* host, int64_t lda, int mode);
int tinv_put_dense_device(tinv_ctx* ctx, const double* dev, int64_t lda);
int tinv_get_dense_device(tinv_ctx* ctx, double* dev, int64_t lda, int mode);
/* one lower tile (i >= j) of the matrix, b*b row-major */
int tinv_put_tile(tinv_ctx* ctx, int64_t i, int64_t j, const double* host);
int tinv_get_tile(tinv_ctx* ctx, int64_t i, int64_t j, double* host);

/* Native stream generation (taskgen.py:178-269). steps: bit mask 1|2|4 for
 * steps 1,2,3; loops: 3 chars of 'U'/'D' (for a single-step stream only the
 * first char is used); out_of_place: Placement.OUT_OF_PLACE; pipelined: no
 * barriers between steps. If table is NULL only the counts are returned. */
int tinv_gen_stream(int32_t t, int32_t steps, const char* loops, int32_t out_of_place,
                    int32_t pipelined, int32_t* table, int64_t cap_tasks, int64_t* ntasks,
                    int64_t* barriers, int64_t cap_barriers, int64_t* nbarriers);

/* Hazard DAG of a stream (scheduler.py:101-153): edges (src, dst, kind) with
 * kind 0 RAW, 1 WAR, 2 WAW, 3 barrier; same multiset as the reference. */
int tinv_dag_edges(const int32_t* table, int64_t ntasks, const int64_t* barriers, int64_t nbar,
                   int32_t* src, int32_t* dst, int8_t* kind, int64_t cap, int64_t* nedges);

/* Longest paths of the hazard DAG (dag_analysis.py:46-118 semantics, over
 * the edges of tinv_dag_edges). weight[v]: cost of task v (NULL: 1 per kernel
 * task, 0 per COPY -- the paper's task count). Outputs (each may be NULL):
 * best[v] = heaviest path ending at v, v included; via[v] = its predecessor
 * on that path (-1 at a source; ties go to the smallest task id); depth[v] =
 * longest path ending at v counted in tasks, COPY included; *ncomp = weakly
 * connected components among kernel tasks (include_copies: among all). */
int tinv_dag_paths(const int32_t* table, int64_t ntasks, const int64_t* barriers, int64_t nbar,
                   const double* weight, int32_t include_copies, double* best, int32_t* via,
                   int32_t* depth, int64_t* ncomp);

/* Distribution over a P x Q device grid (2D block-cyclic owner-computes,
 * SURVEY.md §8(e)): owner(i, j) = (i mod P) * Q + (j mod Q) for every tile of
 * every label; a task runs on the owner of its output tile. The distributed
 * stream holds every task of `table` with reads of remotely owned tiles
 * redirected to receive tiles, plus one transfer per (tile version, consumer
 * rank): a COPY from the owner's tile into a fresh receive tile (label >=
 * TINV_RECV_LABEL0, so a receiver never waits on anti-dependences), emitted
 * right after the producing task (initial versions first). owner[k]: rank that
 * executes out task k (transfers: the sender); dest[k]: receiving rank of a
 * transfer, -1 otherwise; ref[k]: source task id, -1 for transfers. Executed
 * as one stream it is the loopback form of the distributed run; its per-rank
 * slices are the per-GPU streams. table NULL: count only. */
#define TINV_RECV_LABEL0 64
int tinv_dist_stream(const int32_t* table, int64_t ntasks, int32_t t, int32_t P, int32_t Q, int32_t* out,
                     int64_t cap, int64_t* nout, int32_t* owner, int32_t* dest, int32_t* ref);

/* Plan = the device-resident executable form of a stream on a context
 * (hazard DAG, renaming slots, priorities, ready queues). Reusable. */
int tinv_plan_create(tinv_ctx* ctx, const int32_t* table, int64_t ntasks, int32_t stream_t,
                     const int64_t* barriers, int64_t nbar, uint32_t flags, tinv_plan** plan,
                     tinv_err* err);
/* Plan with transfer pseudo-tasks (multi-GPU): kind 12 =
 * SEND (reads r0: the tile version; a CTA copies it into the receiver's pool
 * slot 2T + seq through peer memory and sets the receiver's inbox[seq]),
 * kind 13 = RECV (writes its receive tile, pinned at slot 2T + seq; completed
 * by the inbox poller when the data has arrived). aux[2k], aux[2k+1] = (dest
 * rank, seq) of task k; nrecv = inbox length. Without peers attached the
 * transfers loop back into this context (one-GPU execution of every rank). */
int tinv_plan_create_xfer(tinv_ctx* ctx, const int32_t* table, int64_t ntasks, int32_t stream_t,
                          const int32_t* aux, int64_t nrecv, uint32_t flags, tinv_plan** plan, tinv_err* err);
/* Ranks emulated in ONE launch on one B200 (the multi-GPU schedule on SM
 * groups): the transfer plan of tinv_plan_create_xfer (every rank's tasks,
 * SEND / RECV through the local pool) with rank_of[v] = the rank that runs
 * row v (its task owner; SEND: the sender; RECV: the receiver). CTA b of the
 * launch is rank b % nranks, each rank gets nsm / nranks CTAs and claims only
 * its own tasks from its own priority queues -- the distributed schedule of
 * scheduler.py:261-351 over P x Q GPUs, at 1/nranks of a B200 per rank.
 * nranks <= 8. */
int tinv_plan_create_ranks(tinv_ctx* ctx, const int32_t* table, int64_t ntasks, int32_t stream_t,
                           const int32_t* aux, int64_t nrecv, const int32_t* rank_of, int32_t nranks,
                           uint32_t flags, tinv_plan** out, tinv_err* err);

/* Load report of the last tinv_plan_exec* (SURVEY.md §8(f) row 1): per CTA
 * of the launch, the ns its scheduler warp waited for a claimable work item
 * (busy = kernel time - idle), and the rank it served. */
int tinv_plan_cta_idle(const tinv_plan* p, int64_t* idle_ns, int32_t* rank, int64_t cap, int64_t* nctas);

/* Schedule model (host only, no GPU needed; csrc/model.cu): discrete-event
 * simulation of the plan tinv_plan_create / _create_ranks would compile for
 * an n x n matrix of b x b tiles, run by nranks GPUs of sms_per_rank SMs
 * each with the executor's claim rules (per-rank level FIFOs, phase groups,
 * work items). flags: 0 or TINV_SHARE_SLOTS. aux / nrecv / rank_of as in tinv_plan_create_ranks (NULL and 0
 * for a single-GPU stream; rank_of NULL when nranks == 1). cost[9], in us:
 * block product (128^3), per-item overhead, 128-block Cholesky+inverse,
 * 128-block triangular inverse, 128-block copy, SEND per 128-block, link
 * latency, masked-block fraction, ready -> start latency of an item. out[0] = makespan (us), out[1..nranks] =
 * busy SM-us per rank, out[nranks+1] = tasks never run (0 unless deadlock),
 * out[nranks+2] = tile slots the plan's device store needs (2T + working).
 * crit_kind[17] (or NULL): the chain of releasing predecessors ending at the
 * last task to finish, its time (release -> finish) summed per task kind
 * (TINV_* kinds 0-10, then INV, SEND, RECV, ARRIVE, DEPART, POTRF_INV). */
int tinv_model_run(int64_t n, int64_t b, const int32_t* table, int64_t ntasks, int32_t stream_t,
                   const int64_t* barriers, int64_t nbar, const int32_t* aux, int64_t nrecv,
                   const int32_t* rank_of, int32_t nranks, int32_t sms_per_rank, uint32_t flags,
                   const double* cost, double* out, double* crit_kind);

/* Multi-process runs (one rank per B200 of a node): size the store for
 * `plan` and export this rank's pool and inbox as CUDA IPC handles (64 bytes
 * each); after the exchange, map every peer (handles in rank order). Call
 * tinv_ipc_reset on every rank, then a barrier across ranks, before each
 * tinv_plan_exec of a transfer plan. The store cannot grow once exported. */
int tinv_ipc_export(tinv_ctx* ctx, tinv_plan* plan, void* pool_handle, void* inbox_handle);
int tinv_ipc_open(tinv_ctx* ctx, int32_t rank, int32_t world, const void* pool_handles,
                  const void* inbox_handles);
int tinv_ipc_reset(tinv_ctx* ctx);
/* Several ranks in ONE process on one device (tests / emulation of the
 * multi-process runtime): after tinv_ipc_export on every rank's context,
 * tinv_peer_attach maps the peers' pools and inboxes by plain device pointer
 * (what tinv_ipc_open does with IPC handles across processes). */
int tinv_peer_attach(tinv_ctx* ctx, int32_t rank, int32_t world, tinv_ctx* const* peers);
/* A rank's store with slots only for the lower tiles it owns (owned[i * t + j]
 * != 0, i >= j; e.g. the 2D block-cyclic owner (i mod P) * Q + (j mod Q) ==
 * rank), their rename shadows, and its receive / working tiles -- instead of
 * the whole matrix twice. Plans may touch only owned matrix tiles (the
 * distributed stream of the rank does); not combinable with
 * TINV_KEEP_ON_FAILURE or TINV_STREAM_IO. put / get_dense skip other ranks'
 * tiles (get leaves them as they are in the destination). */
int tinv_create_owned(tinv_ctx** ctx, int64_t n, int64_t b, int device, const int32_t* owned);
/* receive-slot base of this store (SEND targets in it), and the peers' bases
 * for a multi-process run whose stores differ (exchange, then set; plain
 * pointers via tinv_peer_attach set them automatically) */
int tinv_recv_base(const tinv_ctx* ctx, int32_t* base);
int tinv_ipc_recv_bases(tinv_ctx* ctx, int32_t world, const int32_t* bases);
/* executor grid of this context: nsm CTAs (1 <= nsm <= the device's SMs;
 * default all). Ranks sharing one device each take a disjoint share, so their
 * persistent executors are co-resident. Set before creating plans. */
int tinv_set_sms(tinv_ctx* ctx, int32_t nsm);
/* run the plan on the context's matrix; blocks. ms (optional) = device time
 * of the executor launch measured with CUDA events. */
int tinv_plan_exec(tinv_plan* plan, tinv_err* err, double* ms);
/* End to end with host buffers, transfers overlapped with the computation
 * (replaces tinv_put_dense + tinv_plan_exec + tinv_get_dense, i.e.
 * from_dense -> execute -> [symmetrize_lower(]to_dense[)], tile_matrix.py:84-119
 * and scheduler.py:261). The plan must be made with TINV_STREAM_IO: the copy
 * engines move A's lower tiles host -> device in column order while the
 * executor already runs (a task reading a tile waits for its arrival), and
 * every result tile is written into `x` by the executor as soon as its last
 * writer is done (mode TINV_DENSE_*; SYMMETRIZE mirrors on the fly). `a`
 * should be page-locked for the copies to be asynchronous; `x` must be
 * page-locked (device-mapped) host memory, else TINV_ERR_BAD_ARG. Batched
 * stores: matrix m at a + m*n*lda and x + m*n*ldx. `a` is never written; on
 * failure `x` is unspecified. Not combinable with TINV_KEEP_ON_FAILURE. */
int tinv_plan_exec_host(tinv_plan* plan, const double* a, int64_t lda, double* x, int64_t ldx, int mode,
                        tinv_err* err, double* ms);
int tinv_plan_destroy(tinv_plan* plan);
/* plan statistics: exec tasks (incl. hidden INV tasks), work items, edges */
int tinv_plan_stats(const tinv_plan* plan, int64_t* exec_tasks, int64_t* items, int64_t* edges);
/* per reference task: device start/end (ns since launch) and SM id; TRACE only */
int tinv_plan_trace(const tinv_plan* plan, int64_t* start_ns, int64_t* end_ns, int32_t* sm,
                    int64_t ntasks);

/* convenience: plan_create + plan_exec + plan_destroy */
int tinv_run(tinv_ctx* ctx, const int32_t* table, int64_t ntasks, int32_t stream_t,
             const int64_t* barriers, int64_t nbar, uint32_t flags, tinv_err* err);

/* ---- batched small inversions (BASELINE config 4), no context ----------
 * For nb = n the reference runs gen_inversion(1) -- POTRF, TRTRI, LAUUM of
 * one tile (taskgen.py:178-223; kernels.py:59-76, 120-130, 148-151) -- and
 * then symmetrize_lower(to_dense(tm)) (tile_matrix.py:102-119), once per
 * matrix. These entry points run that per-matrix sequence fused into one
 * thread block per matrix (csrc/batched.cu), 1 <= n <= 256.
 *
 * tinv_batch_small_launch: device pointers; matrix k at dA + k * stride
 * (row-major, ld = n; only its lower triangle is read), its full symmetric
 * inverse to dX + k * stride (dX may equal dA). Asynchronous on cuda_stream
 * (null = legacy default stream). *dfail is a device u64 the caller sets to
 * all ones; it receives min over failing matrices of (k << 32 | column), the
 * column being POTRF's NotPositiveDefiniteError index (kernels.py:68-71).
 * For even n, dA and dX must be 16-byte aligned and stride even (16-byte row
 * accesses); otherwise the call returns TINV_ERR_BAD_ARG without launching. */
int tinv_batch_small_launch(const double* dA, double* dX, int64_t batch, int64_t n, int64_t stride,
                            void* cuda_stream, unsigned long long* dfail);
/* tinv_batch_small_host: host buffers (page-locked for overlap), blocking.
 * The batch streams through the device in chunks: host -> device copy,
 * kernel, device -> host copy on three streams, overlapped. On a failure
 * returns TINV_ERR_NOT_SPD with *fail_matrix / *fail_index set (else -1);
 * *ms (optional) = wall time of the device work. */
int tinv_batch_small_host(const double* hA, double* hX, int64_t batch, int64_t n, int device,
                          int64_t* fail_matrix, int64_t* fail_index, double* ms);
/* tinv_batch_small_engine: the engine the two calls above use (process-wide;
 * initial value from the environment, TINV_BSMALL_ENGINE=cta|pipe):
 *   TINV_BSMALL_CTA  (0) one thread block per matrix running the fused block
 *                        program (csrc/batched.cu), any 1 <= n <= 256;
 *   TINV_BSMALL_PIPE (1) one persistent block per SM keeping several matrices
 *                        in flight, their 64x64 block jobs scheduled over a
 *                        DAG in shared memory (csrc/batched_pipe.cu); even
 *                        64 <= n <= 256 (other n run on TINV_BSMALL_CTA).
 * engine < 0 only queries. Returns the engine in effect before the call. */
#define TINV_BSMALL_CTA 0
#define TINV_BSMALL_PIPE 1
int tinv_batch_small_engine(int engine);

#ifdef __cplusplus
}
#endif
#endif /* TILEINV_B200_H */
