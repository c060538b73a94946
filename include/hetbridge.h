/*
 * hetbridge — C-ABI of the B200-native boundary communicator.
 *
 * Drop-in boundary for the reference's hetsim::grid / hetsim::bridge API
 * (/root/reference/proj/core/include/hetsim/{grid,bridge}.hpp). The reference
 * is C++ with no FFI; each entry point below names the reference declaration
 * it replaces. Plain pointers and sizes only — no C++ or torch types.
 *
 * Status convention: 0 = OK; otherwise the reference ErrorCode ordinal + 1
 * (error.hpp:13-38: 1 RankOutOfModule, 2 CoordOutOfBounds, 3 IndivisibleBatch,
 * 4 PartialOverlap, 5 NonIntegerFan, 6 PlanInfeasible, 7 ShardIntervalMismatch,
 * 8 MissingSourceShard, 9 GradIntervalMismatch, 10 UnknownMicrobatch, ...,
 * 13 ShapeMismatch, 16 DivisibilityViolation, 20 NotColocated,
 * 24 InvalidArgument) and two device-runtime additions: 25 CudaError,
 * 26 Timeout. hb_last_error() returns the message of the calling thread's last
 * failure. No exception crosses this boundary.
 */
#ifndef HETBRIDGE_H_
#define HETBRIDGE_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_ERR_CUDA 25
#define HB_ERR_TIMEOUT 26

/* dtypes */
#define HB_BF16 0
#define HB_FP16 1
#define HB_FP32 2
#define HB_FP64 3

/* placement (grid.hpp:61) and DpKind (bridge.hpp:38) */
#define HB_COLOCATED 0
#define HB_NONCOLOCATED 1
#define HB_EQUAL 0
#define HB_FANIN 1
#define HB_FANOUT 2

/* per-logical-rank buffer slots */
#define HB_SLOT_SRC_ACT 0  /* source shard: forward input                     */
#define HB_SLOT_DST_ACT 1  /* destination shard / CP token slice: fwd output  */
#define HB_SLOT_DST_GRAD 2 /* destination gradient: backward input            */
#define HB_SLOT_SRC_GRAD 3 /* source gradient: backward output (accumulated)  */
#define HB_SLOT_TEXT 4     /* text embedding rows: splice forward input       */

/* splice text numbering */
#define HB_TEXT_FULL 0  /* text buffer row = global text index (-1-code)    */
#define HB_TEXT_SLICE 1 /* text buffer row = k-th text position of the slice */
#define HB_TEXT_INPLACE 2 /* no text buffer: the caller wrote the text rows into the
                           * destination slice; only vision rows are written (the
                           * masked scatter of VLM input embeddings)            */

typedef struct hb_plan hb_plan;
typedef struct hb_splice hb_splice;
typedef struct hb_exec hb_exec;

/* hetsim::grid::ModuleLayout (grid.hpp:16-31) */
typedef struct {
  const char* name;
  int tp, cp, pp, dp, rank_offset;
} hb_layout;

/* hetsim::grid::BoundaryEdge (grid.hpp:55-60) */
typedef struct {
  hb_layout source, dest;
  int global_batch;
  int feature_width;
} hb_edge;

/* ---- errors ---------------------------------------------------------------- */
size_t hb_last_error(char* buf, size_t cap);
const char* hb_error_name(int status); /* error.cpp error_code_name */
int hb_abi_version(void);

/* ---- grid (grid.hpp:64-92) --------------------------------------------------- */
int hb_coord_of_rank(const hb_layout* l, int rank, int coord4[4]);      /* grid.hpp:64 */
int hb_rank_of_coord(const hb_layout* l, const int coord4[4], int* rank); /* grid.hpp:67 */
int hb_partition_batch(int batch, int dp, int* start_len, int cap_pairs); /* grid.hpp:70 */
int hb_leader_rank(const hb_layout* l, int pp, int dp, int* rank);       /* grid.hpp:74 */
int hb_placement_of_edge(const hb_edge* e, int* placement);              /* grid.hpp:78 */
int hb_ranks_of_stage(const hb_layout* l, int pp, int* out, int cap, int* n); /* grid.hpp:82 */
int hb_replica_group(const hb_layout* l, int pp, int dp, int* out, int cap, int* n); /* :86 */
/* per-module process groups of `rank`: kind 0 TP, 1 CP, 2 PP, 3 DP (runtime rank-group setup) */
int hb_module_group(const hb_layout* l, int rank, int kind, int* out, int cap, int* n);

/* ---- plan (bridge.hpp:137-142) ----------------------------------------------- */
int hb_classify_dp_relation(const hb_edge* e, int* kind, int* factor); /* bridge.hpp:137 */
int hb_plan_create(const hb_edge* e, hb_plan** out);                   /* bridge.hpp:138 plan_bridge */
void hb_plan_destroy(hb_plan* p);
int hb_plan_export(const hb_plan* p, int elem_bytes, char* buf, size_t cap, size_t* len); /* :142 */
int hb_plan_info(const hb_plan* p, int* placement, int* kind, int* factor,
                 int* cross_boundary_messages, int* world); /* BridgePlan fields, :122-135 */

/* ---- configuration ingestion (SPEC cli module S:495-545: ExperimentConfig,
 *      parse_config; paper Appendix B module_parallelisms) -------
 * Grammar: `[module.<name>]` sections with tensor_model_parallel_size,
 * context_parallel_size, pipeline_model_parallel_size, data_parallel_size,
 * rank_offset; `[model]` and `[run]` sections (global_batch, num_microbatches,
 * steps, seed, tolerance, ...); `#` comments; integer or decimal values only.
 * Errors: 22 ParseError ("line N: ..."), 23 ValidationError (one "language"
 * module and >= 1 encoder; IndivisibleBatch; PartialOverlap). */
typedef struct hb_config hb_config;
int hb_config_parse(const char* text, hb_config** out); /* parse_config */
void hb_config_destroy(hb_config* c);
int hb_config_num_modules(const hb_config* c, int* n);
/* module i in file order; out->name stays valid while c lives */
int hb_config_module(const hb_config* c, int i, hb_layout* out, int* is_language);
int hb_config_run(const hb_config* c, int* global_batch, int* num_microbatches, int* steps,
                  long long* seed, double* tolerance);
/* encoder -> language edge of one microbatch (global_batch / num_microbatches samples) */
int hb_config_edge(const hb_config* c, const char* encoder, int feature_width, hb_edge* out);
/* canonical text (parse(render(c)) reproduces c) */
int hb_config_render(const hb_config* c, char* buf, size_t cap, size_t* len);

/* ---- splice (tinymodel.hpp:94-112) -------------------------------------------- */
int hb_cp_token_slice(int seq_len, int cp, int cp_idx, int* start, int* length); /* :95 */
/* codes[Q*S]: >= 0 vision row (local sample j)*S_v + token t; < 0 text row -1-code. */
int hb_splice_create(int Q, int S, int d_h, int S_v, int text_mode, const int* codes,
                     hb_splice** out);
void hb_splice_destroy(hb_splice* s);

/* ---- ownership index maps (host only; for inspection and tests) --------------- */
typedef struct {
  int src_rank, src_slot;
  long long src_off;
  int dst_rank, dst_slot;
  long long dst_off;
  long long n; /* elements */
} hb_copy_seg;
typedef struct {
  int rank, slot;
  long long off;
} hb_ref;
typedef struct {
  int dst_rank, dst_slot;
  long long dst_off;
  long long n;
  int nterms, term0;
} hb_reduce_seg;
int hb_index_forward(const hb_plan* p, const hb_splice* s, hb_copy_seg* out, size_t cap, size_t* n);
int hb_index_backward(const hb_plan* p, const hb_splice* s, hb_reduce_seg* out, size_t cap,
                      size_t* n, hb_ref* terms, size_t tcap, size_t* tn);
/* The backward map the device runtime executes by default (hb_exec_config.
 * strict_provenance = 0): terms read from the holder's tp replicas in turn. */
int hb_index_backward_balanced(const hb_plan* p, const hb_splice* s, hb_reduce_seg* out, size_t cap,
                               size_t* n, hb_ref* terms, size_t tcap, size_t* tn);
int hb_index_buffer_elems(const hb_plan* p, const hb_splice* s, int rank, int slot,
                          long long* elems);

/* ---- device execution (replaces BridgeRuntime, bridge.hpp:146-173, and the
 *      whole-edge bridge_forward/bridge_backward, :175-185) --------------------- */
typedef struct {
  int act_dtype;      /* HB_BF16 ... activations (source/destination shards)  */
  int grad_in_dtype;  /* destination gradients                                  */
  int grad_out_dtype; /* source gradients (fp32 recommended for accumulation)   */
  int mb_slots;       /* buffer sets for microbatches in flight                 */
  int internal_alloc; /* 1: allocate the IPC-exported device region            */
  int blocks_per_sm;
  int threads;
  double timeout_s; /* cross-GPU flag wait timeout                            */
  int fwd_mode;     /* forward: 0 auto, 1 consumers pull, 2 owners push         */
  int partition;    /* CTA work split: 0 auto, 1 contiguous, 2 interleaved      */
  /* 0 (default): the backward reads each gradient term from one of the holder's
   * tp replicas (the source rank itself if it is one, else replica j % tp), which
   * spreads NVLink egress; identical sums when tp replicas hold identical
   * gradients, the contract of bridge.hpp:33-36. 1: always the tp=0 copy, the
   * reference data path replica for replica (strict provenance). */
  int strict_provenance;
  /* 1 (splice edges): the TEXT slot holds int32 token ids, one per text row, and
   * the forward gathers each text row from the embedding table set with
   * hb_exec_set_text_embedding (the LLM's embedding lookup fused into the
   * splice). An id outside [0, vocab) makes hb_exec_status
   * return InvalidArgument (device error 2); that row is left unwritten. */
  int text_embedding;
  /* cap on every boundary kernel's grid (0 = fill the GPU): leaves SMs to
   * concurrent work such as pipeline P2P, and lets several execs of one group
   * share a device (hb_exec_open_peers_local). */
  int max_ctas;
  /* cap on the backward (gradient-return) grid alone; 0 = max_ctas. With a
   * forward and a backward in flight at once (the 1F1B-paired graph) the two
   * kinds can be sized separately so both grids fit on the GPU. */
  int max_ctas_bwd;
  /* TMA copy stage size in KiB (8, 16 or 32; 0 = HB_TMA_CHUNK_KB or 32): smaller
   * stages leave shared memory for a concurrent gradient-return grid. */
  int tma_chunk_kib;
} hb_exec_config;
void hb_exec_config_default(hb_exec_config* c);

/* rank_to_gpu[n_ranks]: the GPU (0..n_gpus-1) hosting each logical rank; this
 * process drives GPU my_gpu (the current CUDA device). Collective over the
 * processes of the exec group when n_gpus > 1. */
int hb_exec_create(const hb_plan* p, const hb_splice* s, int n_gpus, int my_gpu,
                   const int* rank_to_gpu, int n_ranks, const hb_exec_config* cfg,
                   hb_exec** out);
void hb_exec_destroy(hb_exec* x);
int hb_exec_ipc_handle(hb_exec* x, void* out64);
int hb_exec_open_peers(hb_exec* x, const void* handles, size_t nbytes); /* n_gpus*64 bytes */
/* Single-process form of the group setup (one host thread drives every GPU of
 * the group, as the reference's "one script per rank" collapsed into one
 * process): execs[g] = this process's exec of GPU g (n = n_gpus; execs[my_gpu]
 * ignored). Peer regions are used directly; peer access is enabled between
 * distinct devices; execs of one group may also share a device (set max_ctas
 * so their grids are co-resident). Every exec must outlive its peers' ops. */
int hb_exec_open_peers_local(hb_exec* x, hb_exec* const* execs, int n);
int hb_exec_buffer(hb_exec* x, int rank, int slot, int mb_slot, void** ptr, size_t* bytes);
/* Caller-owned device buffer for a resident rank's slot (replaces the
 * reference's ShardedTensor payload, bridge.hpp:47-57: the caller keeps
 * ownership, the library reads/writes it in place). ptr = NULL reverts to the
 * library's region. Rebinding rebuilds the device tables at the next op and
 * drops captured graphs (recapture them). Any GPU count: in a multi-process
 * group every process then calls hb_exec_export_bindings, all-gathers the
 * blobs and hb_exec_import_bindings each peer's blob before its next op. */
int hb_exec_bind(hb_exec* x, int rank, int slot, int mb_slot, void* ptr, size_t bytes);
/* As hb_exec_bind with a row stride in elements (DeviceShard.row_stride):
 * row i of the shard starts at element i*row_stride; rows are samples
 * (feature_width elements) or, for splice token slices / text rows, tokens
 * (d_h). 0 or the row width = packed. */
int hb_exec_bind_strided(hb_exec* x, int rank, int slot, int mb_slot, void* ptr, size_t bytes, long long row_stride);
/* Multi-process binding exchange: *len = blob size (buf may be NULL to query);
 * import a peer GPU's blob (CUDA IPC handles of the bound allocations). */
int hb_exec_export_bindings(hb_exec* x, void* buf, size_t cap, size_t* len);
int hb_exec_import_bindings(hb_exec* x, int gpu, const void* blob, size_t len);
/* forward: BridgeRuntime::forward_{source,dest,colocated} for every resident rank */
int hb_exec_forward(hb_exec* x, int mb, void* cuda_stream);
/* backward: BridgeRuntime::backward_* ; src_grad = beta*src_grad + returned gradient */
int hb_exec_backward(hb_exec* x, int mb, float beta, void* cuda_stream);
int hb_exec_seed_forward_record(hb_exec* x, int mb); /* bridge.hpp:165 */
/* 1F1B pair (no reference counterpart: the reference issues the two calls
 * one after the other): forward of fwd_mb and backward of bwd_mb in one launch
 * of the fused paired step kernel, as hb_exec_forward(fwd_mb) followed by
 * hb_exec_backward(bwd_mb, beta) would leave every buffer. Peers may issue the
 * same two ops as separate calls. *fused (may be NULL) = 1 if one launch ran. */
int hb_exec_paired(hb_exec* x, int fwd_mb, int bwd_mb, float beta, void* cuda_stream, int* fused);
/* Embedding table [vocab x d_h] (activation dtype, device memory of this GPU). */
int hb_exec_set_text_embedding(hb_exec* x, const void* table, long long vocab);
/* Vocab-parallel table (Megatron's VocabParallelEmbedding, the LLM side of
 * tinymodel.hpp:97-101): resident logical rank `rank` holds rows
 * [vocab_begin, vocab_begin + rows) of the [vocab x d_h] table at `shard`
 * (activation dtype, this GPU). The shards of a destination TP group are
 * equal-sized and ordered by tp index (vocab_begin = tp_idx * rows). The splice
 * then gathers each text row from the rank owning its id, on this GPU or a
 * peer's over NVSwitch, instead of a masked lookup and a TP all-reduce. Peers'
 * shards arrive with hb_exec_export_bindings / hb_exec_import_bindings. */
int hb_exec_set_text_embedding_shard(hb_exec* x, int rank, const void* shard, long long vocab_begin, long long rows,
                                     long long vocab);
/* CUDA graph of one buffer set's boundary ops; what: 0 forward, 1 forward +
 * backward(beta), 2 backward(beta), 3 forward + backward(beta) of every buffer
 * set in order (one launch replays mb_slots steps; mb_slot ignored), 4 the
 * 1F1B-paired cycle: step k runs the forward of set k concurrently with the
 * backward(beta) of set k-1 (a pipeline schedule call pairs them the same way;
 * mb_slots >= 2; size max_ctas so both grids fit on the GPU together), 5 the
 * same cycle with each pair in ONE warp-specialised launch (a TMA lane for the
 * forward, 15 warps for the gradient return; no co-residency condition). One
 * graph launch replays the ops; replays bypass the microbatch records. */
int hb_exec_graph_capture(hb_exec* x, int mb_slot, int what, float beta, void* cuda_stream);
int hb_exec_graph_launch(hb_exec* x, int mb_slot, int what, void* cuda_stream);
int hb_exec_status(hb_exec* x, unsigned* device_error);
/* Recovery after a Timeout (26) or GroupMismatch (12): zeroes the exec's launch
 * counters, claim queues, error word and signal pad and drops its microbatch
 * records; tables and captured graphs stay valid. Collective: every exec of
 * the group calls it with its device idle, between two group-wide barriers
 * (no reference counterpart; simnet aborts the whole fabric instead). */
int hb_exec_reset_protocol(hb_exec* x);
int hb_exec_stats(hb_exec* x, long long* fwd_segments, long long* bwd_segments,
                  long long* fwd_bytes, long long* bwd_elems, long long* launches);
/* Diagnostics (no reference counterpart): with HB_TRACE=1 in the environment
 * at hb_exec_create, every boundary launch records per-CTA %globaltimer stamps
 * (8 x u64 per CTA: entry, arrival resolved, peers confirmed, first chunk
 * landed, work done, exit, chunks, remote chunks). Copies the last launch of
 * kind (0 forward, 1 backward) into out[max_ctas x 8]; *n_ctas = CTAs copied
 * (0 when tracing is off), *grid = that launch's grid. Synchronises. */
int hb_exec_trace(hb_exec* x, int kind, unsigned long long* out, int max_ctas, int* n_ctas, int* grid);
/* Static race and bounds check (no reference counterpart; stands in for
 * compute-sanitizer, which this pool does not allow). Downloads every buffer
 * set's device tables and checks that each copy run, reduce term and
 * accumulator lies inside one planned buffer of its slot, that pull mode
 * writes only this GPU's destinations and the gradient return only its
 * accumulators, that no two writes of a launch overlap and no read overlaps a
 * write, that every run touching a peer is handed out behind the peer wait,
 * and that every chunk is handed out exactly once. *checks = items checked.
 * Returns ValidationError (23) with the first violation in hb_last_error(). */
int hb_exec_validate(hb_exec* x, long long* checks);

/* ---- projector GEMM with a boundary epilogue (the
 *      encoder projector of tinymodel.hpp:62) ----------------------------------
 * Y[M x N] = X[M x K] . W[N x K]^T on the sm_100a tensor cores (tcgen05, TMEM
 * accumulators, TMA-fed), bf16 in/out, fp32 accumulation. Output row m is
 * stored to every non-null row_dst[m*fan + f] (device array of pointers to N
 * bf16, local or peer-mapped), so the projector writes straight into the
 * boundary's destination rows. Needs N % 256 == 0, K % 64 == 0, 16-B aligned
 * operands and leading dimensions. */
int hb_projector_gemm(const void* x, long long ldx, const void* w, long long ldw, void* const* row_dst, int fan,
                      int M, int N, int K, void* cuda_stream);
/* Boundary forward with the projector fused in: x = the pre-projection token
 * rows of every local source rank stacked in ascending rank order [x_rows x K]
 * (x_rows must equal those ranks' token rows, else ShapeMismatch), w = the
 * projector weight [d_h x K]; each projected row is stored straight into
 * every destination row of the plan, local or on a peer GPU (push over
 * NVSwitch; the source shards are never written). Replaces forward_* for that
 * microbatch (records it like hb_exec_forward). Any GPU count, non-splice
 * edges, bf16 activations. */
int hb_exec_forward_projected(hb_exec* x, int mb, const void* act, long long x_rows, long long ldx, const void* w,
                              long long ldw, int d_h, int K, void* cuda_stream);

/* ---- graph-aware pipeline dispatch (SPEC.md:358-437
 *      `sched`: build_stage_graph, generate_1f1b_dispatch, validate_dispatch;
 *      the reference's sched.cpp is an empty stub) --------------------------- */
typedef struct hb_stage_graph hb_stage_graph;
/* cell ops */
#define HB_OP_COMPUTE 0
#define HB_OP_SEND_FWD 1
#define HB_OP_RECV_FWD 2
#define HB_OP_SEND_BWD 3
#define HB_OP_RECV_BWD 4
/* edge kinds */
#define HB_EDGE_P2P 0
#define HB_EDGE_NC 1
typedef struct {
  int row;  /* schedule call */
  int node; /* stage-graph node (module, pp) */
  int op;   /* HB_OP_* */
  int edge; /* stage-graph edge of a communication op (-1 for compute) */
  int kind; /* HB_EDGE_* */
  int mb;
  int bwd;  /* compute: 1 = backward */
} hb_cell;
/* modules[n_modules] with their rank ranges; module edges edge_src[i] ->
 * edge_dst[i] (indices into modules). Nodes are (module, pp) in module order;
 * edges: module chains (P2P) then one NC edge per module edge, from the source
 * module's last stage to the destination's first. Errors: CyclicGraph (17),
 * DanglingEdge (18), InfeasibleSchedule (19: not exactly one sink). */
int hb_stage_graph_create(const hb_layout* modules, int n_modules, const int* edge_src, const int* edge_dst,
                          int n_edges, hb_stage_graph** out);
void hb_stage_graph_destroy(hb_stage_graph* g);
/* out[3*i..] = {module, pp, distance to the sink}; out[4*i..] = {src node,
 * dst node, kind, module-edge index (-1 for P2P)} */
int hb_stage_graph_nodes(const hb_stage_graph* g, int* out, int cap, int* n);
int hb_stage_graph_edges(const hb_stage_graph* g, int* out, int cap, int* n);
/* 1F1B dispatch table (warmup = longest distance to the sink); *n cells,
 * *rows schedule calls; cells may be NULL to query the count. */
int hb_dispatch_generate(const hb_stage_graph* g, int nmb, hb_cell* cells, size_t cap, size_t* n, int* rows);
/* join readiness, edge identity, no double consumption; never fails on a bad
 * table: *n_violations and one line per violation in report */
int hb_dispatch_validate(const hb_stage_graph* g, const hb_cell* cells, size_t n, int nmb, char* report, size_t cap,
                         size_t* len, int* n_violations);
int hb_dispatch_render(const hb_stage_graph* g, int nmb, char* buf, size_t cap, size_t* len);
/* The NC cells of `node` in the order the host runtime issues them on its
 * boundary stream: by row, then module edge, then forward before backward —
 * one global order for every GPU, so each op's in-kernel rendezvous is met
 * (no reference counterpart; the execution rule of hb_runtime_step). */
int hb_dispatch_nc_order(const hb_stage_graph* g, int nmb, int node, hb_cell* cells, size_t cap, size_t* n);

/* ---- host-owned per-module runtime (per-module rank groups,
 *      communicators and streams; §8(f) row 2: executes the graph-aware
 *      dispatch table). One per process (one GPU), collective at create.
 *      Modules have disjoint rank ranges (the non-colocated topology). The
 *      runtime owns: the TP/CP/PP/DP groups of this rank (grid.cpp:41-53,
 *      87-106), an NCCL world communicator and each module's PP communicator
 *      (ncclCommSplit), one boundary exec per module edge (IPC handles
 *      exchanged over NCCL), a boundary stream at the highest priority, a PP
 *      stream and a compute stream. hb_runtime_step enqueues this rank's
 *      column of the 1F1B table: P2P cells as grouped ncclSend/ncclRecv on the
 *      PP stream, NC cells as the edge exec's forward/backward on the
 *      boundary stream, compute cells through `fn` on the compute stream,
 *      ordered by CUDA events. ---------------------------------------------- */
typedef struct hb_runtime hb_runtime;
typedef struct {
  int nmb;            /* microbatches per step */
  int max_ctas;       /* CTA cap of the boundary kernels (0 = fill the GPU) */
  long long pp_bytes; /* one microbatch's stage activation/gradient per rank (P2P) */
  int act_dtype, grad_in_dtype, grad_out_dtype;
  double timeout_s;
  int skip;           /* bit 0: NC cells, bit 1: P2P cells, bit 2: compute (overlap studies) */
} hb_runtime_config;
/* compute callback: stage-graph node, microbatch, 1 = backward, cudaStream_t */
typedef void (*hb_compute_fn)(void* user, int node, int mb, int bwd, void* stream);
int hb_nccl_unique_id(void* out128); /* rank 0 creates it; the caller broadcasts it */
void hb_runtime_config_default(hb_runtime_config* c);
int hb_runtime_create(const hb_layout* modules, int n_modules, const int* edge_src, const int* edge_dst, int n_edges,
                      int global_batch, int feature_width, int world, int my_rank, const void* nccl_id128,
                      const hb_runtime_config* cfg, hb_runtime** out);
void hb_runtime_destroy(hb_runtime* r);
/* this rank's stage-graph node (-1: none), module, node count, table rows */
int hb_runtime_info(const hb_runtime* r, int* node, int* module, int* n_nodes, int* rows);
int hb_runtime_group(const hb_runtime* r, int kind, int* out, int cap, int* n); /* 0 TP 1 CP 2 PP 3 DP */
/* the edge's exec (owned by the runtime: do not destroy): its buffers via hb_exec_buffer / hb_exec_bind */
int hb_runtime_edge_exec(hb_runtime* r, int module_edge, hb_exec** out);
/* which: 0 act_in (RecvFwd), 1 act_out (SendFwd), 2 grad_in (RecvBwd), 3 grad_out (SendBwd) */
int hb_runtime_stage_buffer(hb_runtime* r, int which, int mb, void** ptr, size_t* bytes);
int hb_runtime_stream(hb_runtime* r, int which, void** stream); /* 0 boundary, 1 PP, 2 compute */
int hb_runtime_step(hb_runtime* r, hb_compute_fn fn, void* user);
int hb_runtime_last_step_ms(hb_runtime* r, float* ms); /* synchronises; Timeout if a flag wait expired */
/* Boundary forward/backward pairs that shared one call of this rank's column
 * and went out as one hb_exec_paired launch (only with HB_RT_PAIRED=1), all steps. */
int hb_runtime_paired_ops(const hb_runtime* r, long long* n);

#ifdef __cplusplus
}
#endif

#endif /* HETBRIDGE_H_ */
