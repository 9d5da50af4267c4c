/*
 * tg_abi.h — C-ABI of the B200 mini-batch gradient oracle.
 *
 * The reference (BurTorch/tapegrad, /root/reference/proj) is a header-only
 * C++20 library with no FFI: user code records one sample on a
 * tapegrad::Tape (tape.hpp:68-353), calls backward_with_scratch
 * (backprop.hpp:139-184) per sample, accumulates parameter gradients and runs
 * sgd_step.  This header is the boundary that replaces that
 * per-sample loop: a recorded tape is described in plain arrays
 * (tg_tape_desc), compiled once (tg_compile) and then evaluated for a whole
 * batch on the GPU (tg_forward_backward), followed by the GD update
 * (tg_gd_update).  Every entry point cites the reference interface it
 * replaces.  No C++ exception crosses this boundary; failures return a
 * tg_status and set a thread-local message (tg_last_error).
 *
 * Layouts (all device pointers unless stated otherwise):
 *   inputs        [n_inputs][ld]        scalar (dtype), struct-of-arrays
 *   index_inputs  [n_index_inputs][ld]  int32, struct-of-arrays
 *   params        [n_params]            scalar
 *   loss_out      [batch]               scalar, per-sample root value f_i
 *   input_grad_out[n_inputs][ld]        scalar, per-sample d f_i / d input
 *   grad_sum      [n_params]            scalar, sum_i d f_i / d params
 * ld == batch for every SoA array.
 */
#ifndef TG_ABI_H
#define TG_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status (maps reference exceptions, errors.hpp:9-36, ops.hpp:16-32) ---- */
typedef enum tg_status {
  TG_OK = 0,
  TG_INVALID_ARGUMENT = 1,  /* std::invalid_argument (ops.hpp:41-42, :153-157, :226-229) */
  TG_CAPACITY = 2,          /* CapacityError (tape.hpp:278-282, :291-295)              */
  TG_INVALID_HANDLE = 3,    /* InvalidHandle (tape.hpp:268-273)                          */
  TG_INVALID_CHECKPOINT = 4,/* InvalidCheckpoint (tape.hpp:236-239)                      */
  TG_DOMAIN = 5,            /* std::domain_error (ops.hpp:16-20)                         */
  TG_FORMAT = 6,            /* FormatError (errors.hpp:29-31)                            */
  TG_IO = 7,                /* IoError (errors.hpp:34-36)                                */
  TG_CUDA = 8,              /* CUDA runtime failure (no reference equivalent)            */
  TG_UNSUPPORTED = 9,       /* program shape outside what a kernel path supports         */
  TG_NCCL = 10              /* NCCL failure or NCCL not loadable (no reference equivalent) */
} tg_status;

typedef enum tg_dtype { TG_F64 = 0, TG_F32 = 1 } tg_dtype;

/* Opaque CUDA stream (cudaStream_t); NULL = legacy default stream. */
typedef void* tg_stream_t;

/* Thread-local message of the last failing call on this thread.  Domain
 * errors reproduce the reference text, ops.hpp:17-19:
 * "<op_name>: input <to_string(value)> is outside the operator domain". */
const char* tg_last_error(void);
const char* tg_status_name(tg_status s);
/* Opcode mnemonic, op_kind.hpp:89-123 (extensions: "stopGradMax"). */
const char* tg_op_name(uint8_t op);

/* ---- tape description (what the compiler reads from a recorded tape) ---- */

/* Leaf classes.  The reference has one leaf kind (OpKind::Leaf); which leaves
 * are trainable parameters, per-sample inputs or constants is implicit in user
 * code (SPEC.md:262-271 ParamRange).  The recorder makes it explicit. */
enum { TG_NODE_OP = 0, TG_LEAF_PARAM = 1, TG_LEAF_INPUT = 2, TG_LEAF_CONST = 3 };

/* Extension opcode (not in op_kind.hpp): non-differentiable max over its
 * children, the softmax max-shift "treated as a non-differentiable
 * stabilization constant".  On a reference tape it is a
 * Leaf whose value is that max. */
#define TG_OP_STOPGRAD_MAX 64u

/* A child entry with this bit set is a data-dependent reference (token-id
 * gather): child = gathers[id].first_node + stride * idx[s][index_col] + offset
 * where idx[s][col] is the sample's int32 index input, 0 <= idx < n_rows. */
#define TG_GATHER_FLAG 0x80000000u

typedef struct tg_gather {
  uint32_t first_node;   /* raw node index of table row 0, element 0 */
  uint32_t stride;       /* nodes per table row                       */
  uint32_t n_rows;       /* valid index range                         */
  uint32_t index_col;    /* which int32 index input selects the row   */
  uint32_t offset;       /* element within the row                    */
} tg_gather;

typedef struct tg_tape_desc {
  uint32_t n_nodes;             /* live nodes, Tape::size() (tape.hpp:101)         */
  tg_dtype dtype;               /* Tape<Scalar> (tape.hpp:68)                      */
  const uint8_t* op;            /* [n_nodes] OpKind numbering (op_kind.hpp:10-44)  */
  const uint64_t* child_offset; /* [n_nodes+1] CSR over the child pool            */
  const uint32_t* child;        /* [child_offset[n_nodes]] (tape.hpp:257-260)      */
  const double* constant;       /* [n_nodes] constant slot (tape.hpp:223), nullable */
  const uint8_t* leaf_class;    /* [n_nodes] TG_NODE_OP / TG_LEAF_*                */
  const uint32_t* leaf_index;   /* [n_nodes] PARAM: param id, INPUT: input column  */
  const double* leaf_value;     /* [n_nodes] CONST value / initial PARAM value     */
  uint32_t n_gathers;
  const tg_gather* gathers;
  uint32_t root;                /* backward root (backprop.hpp:140)                */
  uint32_t n_params;
  uint32_t n_inputs;
  uint32_t n_index_inputs;
} tg_tape_desc;

/* ---- recorder: the reference's recording surface behind a C-ABI ---------- */
/* Replaces Tape::leaf / emplace and the ops.hpp free functions for non-C++
 * callers (ctypes); C++ callers use tg::Tape in tg_recorder.hpp directly.     */
typedef struct tg_recorder* tg_recorder_t;

tg_status tg_recorder_new(tg_dtype dtype, size_t capacity, tg_recorder_t* out);
void tg_recorder_free(tg_recorder_t r);
tg_status tg_rec_param(tg_recorder_t r, double value, uint32_t* node_out);
tg_status tg_rec_input(tg_recorder_t r, uint32_t col, double template_value, uint32_t* node_out);
tg_status tg_rec_const(tg_recorder_t r, double value, uint32_t* node_out);
/* Declares a gather reference; template_index picks the row used for the
 * recorder's eager values.  Returns a child reference with TG_GATHER_FLAG. */
tg_status tg_rec_gather(tg_recorder_t r, uint32_t first_node, uint32_t stride, uint32_t n_rows,
                        uint32_t index_col, uint32_t offset, int32_t template_index,
                        uint32_t* ref_out);
/* Appends op over children with the reference's eager semantics and checks
 * (ops.hpp:38-307): arity errors -> TG_INVALID_ARGUMENT, domain -> TG_DOMAIN. */
tg_status tg_rec_op(tg_recorder_t r, uint8_t op, const uint32_t* children, uint32_t n_children,
                    double constant, uint32_t* node_out);
tg_status tg_rec_value(tg_recorder_t r, uint32_t ref, double* value_out);
tg_status tg_rec_set_root(tg_recorder_t r, uint32_t node);
/* Fills desc with views into the recorder (valid until the next mutation). */
tg_status tg_rec_describe(tg_recorder_t r, tg_tape_desc* desc);

/* Fixed-capacity recorder (TapeConfig{capacity, fixed_capacity, child_capacity},
 * tape.hpp:40-53, :79-81): no storage growth after construction; exceeding
 * either capacity is TG_CAPACITY with the reference's message (tape.hpp:278-295).
 * child_capacity 0 selects 8 x capacity, as the reference does.              */
tg_status tg_recorder_new_fixed(tg_dtype dtype, size_t capacity, size_t child_capacity, tg_recorder_t* out);

/* Checkpoint / rewind (Tape::checkpoint / rewind, tape.hpp:228-242).  Rewind
 * discards every node at index >= mark; surviving values and the child-pool
 * cursor are restored exactly, handles into the discarded range become
 * TG_INVALID_HANDLE, and the next node reuses index mark.  A mark ahead of the
 * live size is TG_INVALID_CHECKPOINT with the reference's message.           */
typedef struct tg_checkpoint {
  uint32_t mark;          /* live node count at capture                       */
  uint32_t params;        /* parameter leaves at capture (recorder extension) */
  uint64_t child_mark;    /* child-pool cursor at capture                      */
  uint32_t gathers;       /* gather references at capture (extension)          */
  uint32_t reserved;
} tg_checkpoint;
tg_status tg_rec_checkpoint(tg_recorder_t r, tg_checkpoint* out);
tg_status tg_rec_rewind(tg_recorder_t r, const tg_checkpoint* cp);

/* Recorder size and high-water marks (Tape::size / peak_nodes / child_pool_size
 * / peak_children / peak_arena_bytes / max_arity, tape.hpp:98-125).          */
typedef struct tg_rec_stats {
  uint32_t size;
  uint32_t peak_nodes;
  uint64_t child_pool_size;
  uint64_t peak_children;
  uint64_t peak_arena_bytes;
  uint32_t max_arity;
  uint32_t n_params;
} tg_rec_stats;
tg_status tg_rec_get_stats(tg_recorder_t r, tg_rec_stats* out);

/* ---- built-in workloads (BASELINE.json configs) -------------------------- */
typedef enum tg_model {
  TG_MODEL_FIG1 = 1,     /* cfg1: Fig. 1 tiny graph            */
  TG_MODEL_LISTING1 = 2, /* Listing-1 small graph             */
  TG_MODEL_MOONS_MLP = 3,/* cfg2: scalar MLP 2-16-16-1, hinge + 1e-4 L2      */
  TG_MODEL_CHAR_MLP = 4, /* cfg3: Bengio char-MLP 27/3/10/200                */
  TG_MODEL_GPT = 5,      /* cfg4: mini GPT (dims in tg_model_args)           */
  TG_MODEL_WIDE_MLP = 6  /* cfg5: 784-1024-1024-10 relu MLP (dims in args)   */
} tg_model;

typedef struct tg_model_args {
  uint32_t dims[8];   /* model-specific sizes; zeros select BASELINE.json sizes */
  tg_dtype dtype;
} tg_model_args;

/* Records one template sample of `model` (parameters initialised from seed). */
tg_status tg_build_model(tg_model model, const tg_model_args* args, uint64_t seed,
                         tg_recorder_t* out);
/* Host-side synthetic batch (SURVEY.md §8d generators, mt19937_64 TestRng
 * stream as in testing_support.hpp:49-58).  Host pointers. */
tg_status tg_synth_batch(tg_model model, const tg_model_args* args, uint64_t seed, size_t batch,
                         void* inputs, int32_t* index_inputs);

/* Counter-based synthetic batches (the on-device input
 * pipeline).  Same columns, layouts and per-sample draw order as
 * tg_synth_batch, but draw j of global sample s comes from Philox4x32-10
 * keyed by `seed` at counter (s, j/2), so samples [first_sample,
 * first_sample + batch) are generated independently of one another: the host
 * version and the device version (written into device arrays on `stream`, no
 * host traffic) give identical bits, for any split of the sample range across
 * calls, chunks or ranks.  Zipf vocabularies up to 1024 ids on the device. */
tg_status tg_synth_ctr(tg_model model, const tg_model_args* args, uint64_t seed, uint64_t first_sample, size_t batch,
                       void* inputs, int32_t* index_inputs);
tg_status tg_synth_ctr_device(tg_model model, const tg_model_args* args, uint64_t seed, uint64_t first_sample,
                              size_t batch, void* inputs, int32_t* index_inputs, tg_stream_t stream);

/* ---- compile and run ------------------------------------------------------ */
typedef struct tg_program* tg_program_t;

typedef struct tg_program_info {
  uint32_t n_params, n_inputs, n_index_inputs;
  uint32_t n_sample_nodes;   /* per-sample op nodes evaluated on device  */
  uint32_t n_uniform_nodes;  /* sample-invariant op nodes (hoisted)      */
  uint32_t n_dense_groups;   /* inner-product groups lowered to dense ops */
  uint32_t n_fwd_instr, n_bwd_instr;
  uint64_t n_edges;          /* per-sample child references              */
  uint32_t tile_samples;     /* samples per CTA tile                     */
  uint32_t smem_bytes;       /* dynamic shared memory per CTA            */
  uint32_t storage;          /* 0 = shared-memory tile interpreter,
                                1 = HBM SoA interpreter,
                                2 = register-resident specialised kernel,
                                3 = staged (HBM rows, dense layers as GEMMs) */
  tg_dtype dtype;
  uint32_t n_attn_heads;     /* softmax attention heads fused from the scalar graph */
  uint32_t n_layer_norms;    /* layer normalisations fused from the scalar graph */
  uint32_t fused_mlp;        /* 1: the staged tape runs as one embedding-MLP / softmax-CE kernel */
} tg_program_info;

/* Lowers the tape to the device program (replaces the per-sample DFS of
 * backward_with_scratch, backprop.hpp:150-175: topology is sample-invariant,
 * so the reverse order is computed once here). */
tg_status tg_compile(const tg_tape_desc* desc, tg_program_t* out);
tg_status tg_program_info_get(tg_program_t p, tg_program_info* info);
/* Recorded-order topology for tests: processing order of backward_with_scratch
 * (backprop.hpp:183), host array of n_order entries. */
tg_status tg_program_order(tg_program_t p, const uint32_t** order, uint32_t* n_order);
/* Caller-allocated device workspace (zero allocation on the hot path,
 * PAPER.md:1357-1359). */
tg_status tg_workspace_size(tg_program_t p, size_t batch, size_t* bytes);

/* Sequential-accumulation memory mode (
 * SURVEY.md §8f row 1): the staged tier streams the batch through its
 * HBM-resident rows in chunks of samples whose rows fit `bytes`, summing the
 * gradient chunk by chunk, so tg_workspace_size stops growing with the batch
 * once the batch exceeds one chunk.  0 restores the default (64 GB, or env
 * TG_STAGED_MB in MiB).  Set it before sizing the workspace.  Other tiers
 * keep their rows in registers / shared memory (workspace bounded by the grid
 * already). */
tg_status tg_set_memory_budget(tg_program_t p, size_t bytes);
/* Samples per chunk that tg_forward_backward will use for `batch` (the batch
 * itself for tiers without chunking). */
tg_status tg_chunk_samples(tg_program_t p, size_t batch, size_t* samples);

/* Forward sweep + reverse sweep + batch reduction for `batch` samples:
 * replaces, per sample, rewind/build (tape.hpp:235-242), zero_grads
 * (backprop.hpp:100-109), backward_with_scratch (backprop.hpp:139-184) and
 * the accumulator add of train_step.  grad_sum receives the
 * sum (not the mean) over the batch.  loss_out / input_grad_out may be NULL. */
tg_status tg_forward_backward(tg_program_t p, const void* inputs, const int32_t* index_inputs,
                              size_t batch, const void* params, void* loss_out,
                              void* input_grad_out, void* grad_sum, void* workspace,
                              size_t workspace_bytes, tg_stream_t stream);

/* params -= gamma * grad_sum / global_batch (sgd_step).
 * With several GPUs the caller all-reduces grad_sum first. */
tg_status tg_gd_update(tg_program_t p, void* params, const void* grad_sum, double gamma,
                       size_t global_batch, tg_stream_t stream);

/* ---- data parallelism over NCCL (north_star (d)) -------
 * One process per GPU; the batch is sharded, parameters are replicated.  After
 * tg_forward_backward of its shard, every rank calls tg_allreduce_gd_step:
 * one in-place ncclAllReduce(sum) of grad_sum (n_params scalars, the
 * tape dtype) on `stream`, then params -= gamma * grad_sum / global_batch
 * (sgd_step) on every rank, so replicas stay identical
 * without a broadcast.  comm == NULL is the single-GPU case (the update only).
 * NCCL is bound at run time (dlopen: the already-loaded libnccl.so.2 first,
 * then TG_NCCL_LIB, then the system soname); TG_NCCL when absent or failing.
 * Communicators come from tg_nccl_comm_init (rank 0's tg_nccl_get_unique_id
 * bytes shared with every rank out of band) or are any ncclComm_t. */
typedef void* tg_comm_t;   /* ncclComm_t */
#define TG_NCCL_UNIQUE_ID_BYTES 128
tg_status tg_nccl_get_unique_id(void* id_out /* TG_NCCL_UNIQUE_ID_BYTES */);
tg_status tg_nccl_comm_init(int nranks, const void* id, int rank, tg_comm_t* out);
tg_status tg_nccl_comm_destroy(tg_comm_t comm);
/* NCCL_VERSION_CODE of the bound library, 0 when none could be bound. */
int tg_nccl_version(void);
tg_status tg_allreduce_gd_step(tg_program_t p, void* params, void* grad_sum, double gamma, size_t global_batch,
                               tg_comm_t comm, tg_stream_t stream);

/* ---- fused exchange + GD over symmetric peer memory ----
 * A window is NCCL symmetric memory for the d-length gradient sum
 * (ncclMemAlloc + ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC) + the NCCL
 * >= 2.28 device API): every rank's buffer is load/store reachable from every
 * rank over NVLink, and with TG_WINDOW_MULTIMEM (fp32) on an NVSwitch fabric
 * that supports it, through one multicast (NVLS) address.  Collective: every
 * rank calls create / allreduce_gd / destroy in the same order.
 * tg_window_buffer is this rank's gradient buffer: pass it as grad_sum to
 * tg_forward_backward, then tg_window_allreduce_gd replaces
 * tg_allreduce_gd_step with ONE kernel: sum over ranks (switch-side
 * multimem.ld_reduce + multimem.st, or peer loads summed in rank order and
 * stored back to every rank), then x -= gamma * g / global_batch on `params`
 * (the sgd_step of SPEC.md:424-430; equal to tg_gd_update bit for bit on one
 * rank).  On return the window holds the global sum on every rank.
 * Replaces, with tg_allreduce_gd_step, the reference's sequential
 * GradAccumulator + sgd_step at N > 1.                    */
typedef struct tg_window* tg_window_t;
#define TG_WINDOW_MULTIMEM 1
tg_status tg_window_create(tg_comm_t comm, tg_dtype dtype, size_t count, int flags, tg_window_t* out);
tg_status tg_window_destroy(tg_window_t w);
void* tg_window_buffer(tg_window_t w);
int tg_window_multimem(tg_window_t w);
tg_status tg_window_allreduce_gd(tg_window_t w, void* params, double gamma, size_t global_batch, tg_stream_t stream);

/* Fused single-GPU step: forward_backward + gd_update. */
tg_status tg_train_step(tg_program_t p, const void* inputs, const int32_t* index_inputs,
                        size_t batch, void* params, void* loss_out, void* grad_sum,
                        double gamma, void* workspace, size_t workspace_bytes,
                        tg_stream_t stream);

/* ---- host-buffer training loop -----------------------------------------------
 * The reference's calling convention: each step's samples arrive in host
 * memory and its per-sample losses go back to host memory (train_step,
 * SPEC.md:431-439, the loop of PAPER.md:1357-1359).  A pipeline owns the
 * device staging for `depth` in-flight steps (4; env TG_PIPE_DEPTH).  Step i's host->device input copy
 * runs on a copy stream while step i-1 computes.  Step i's losses return on
 * a second copy stream while step i+1 computes.  Parameters stay resident on
 * the device (`params`, updated in place by the fused GD).
 * Host buffers passed to step i may be reused once step i+depth has been
 * submitted or after tg_pipeline_sync; h_loss of step i is valid after
 * tg_pipeline_sync.  Pinned host memory (tg_host_alloc) gives overlapped
 * copies; pageable memory is accepted but the copies serialise. */
typedef struct tg_pipeline* tg_pipeline_t;
tg_status tg_pipeline_new(tg_program_t p, size_t batch, void* params, tg_stream_t stream, tg_pipeline_t* out);
/* One training step over host buffers: inputs [n_inputs][batch],
 * index_inputs [n_index_inputs][batch] (may be NULL if unused), h_loss
 * [batch] (may be NULL).  Returns after enqueueing. */
tg_status tg_pipeline_step(tg_pipeline_t pl, const void* h_inputs, const int32_t* h_index_inputs, void* h_loss,
                           double gamma);
/* Makes `stream` wait for every enqueued step (copies included), without
 * blocking the host. */
tg_status tg_pipeline_join(tg_pipeline_t pl, tg_stream_t stream);
/* Blocks the host until every enqueued step has finished. */
tg_status tg_pipeline_sync(tg_pipeline_t pl);
/* Device pointer of the batch-summed gradient of the last completed step. */
tg_status tg_pipeline_grad_sum(tg_pipeline_t pl, void** grad_sum);
void tg_pipeline_free(tg_pipeline_t pl);
tg_status tg_host_alloc(size_t bytes, void** out);
void tg_host_free(void* ptr);

/* ---- bit-exact serialization of value / gradient ranges ----
 * Raw range format: headerless, count x scalar, little-endian IEEE-754 (width
 * 4 or 8), values then gradients when given: bytes = width * count * (1 or 2)
 * (7 fp64 values = 56 bytes, Table 4).  Snapshot format: "BTSG",
 * version u32 (1), precision u8 (0 fp32 / 1 fp64), flags u8 (bit 0: grads),
 * count u64, values, then grads.  NaN payloads travel verbatim.  values /
 * grads may be device or host pointers (grads NULL: values only); byte
 * buffers are host memory.  Loads check the byte count / header first and
 * never apply partially (TG_FORMAT on a mismatch). */
size_t tg_range_bytes(tg_dtype dtype, size_t count, int with_grads);
tg_status tg_save_range(tg_dtype dtype, const void* values, const void* grads, size_t count, void* out, size_t out_bytes,
                        size_t* written);
tg_status tg_load_range(tg_dtype dtype, void* values, void* grads, size_t count, const void* in, size_t in_bytes);
size_t tg_snapshot_bytes(tg_dtype dtype, size_t count, int with_grads);
tg_status tg_save_snapshot(tg_dtype dtype, const void* values, const void* grads, size_t count, void* out,
                           size_t out_bytes, size_t* written);
/* Reads the header, checks it against the target range (`dtype`, room for
 * `capacity` scalars of that dtype in values / grads) before writing anything
 * (a precision mismatch is TG_FORMAT, a larger count TG_CAPACITY), then writes
 * values (and grads when present and grads != NULL) and reports the count and
 * grads flag. */
tg_status tg_load_snapshot(const void* in, size_t in_bytes, tg_dtype dtype, void* values, void* grads,
                           size_t capacity, size_t* count_out, int* with_grads_out);

/* Synchronises `stream` and reports the first per-sample domain violation
 * seen since the last check as TG_DOMAIN with the reference message. */
tg_status tg_check_device_error(tg_program_t p, tg_stream_t stream, int64_t* sample_out,
                                uint32_t* node_out);

/* Kernel-level timing: when enabled, CUDA events bracket the per-sample tape
 * kernel on the launch stream; tg_profile_read synchronises and returns the
 * accumulated milliseconds and launch count since the last read. */
tg_status tg_profile_enable(tg_program_t p, int on);
tg_status tg_profile_read(tg_program_t p, double* tape_ms, uint64_t* tape_launches);

/* The dense-layer matrix product of the staged path (exposed for testing):
 *   C[m][n] (+)= sum_k A(m,k) B(k,n),   m < M, n < N, k < K
 *   A(m,k) = a_kmajor ? A[m*lda + k] : A[k*lda + m]
 *   B(k,n) = b_nmajor ? B[k*ldb + n] : B[n*ldb + k]
 * engine 0: SIMT register-tiled (fp32 / fp64); 1: tcgen05 tensor cores,
 * 3xTF32 (fp32 only; CTA pairs with 256 x 256 tiles when M > 128); 2: the
 * same with single-CTA 128 x 128 tiles only.  accumulate != 0 adds into C.
 * Device pointers. */
tg_status tg_gemm(tg_dtype dtype, int engine, uint32_t M, uint32_t N, uint32_t K, const void* A, size_t lda,
                  int a_kmajor, const void* B, size_t ldb, int b_nmajor, void* C, size_t ldc, int accumulate,
                  tg_stream_t stream);

/* Short tapes are specialised into a register-resident kernel (NVRTC,
 * sm_100a) on first use.  Returns its CUDA source and compiler log;
 * TG_UNSUPPORTED when the program runs on the interpreter kernel instead.
 * Requires a device.  Set TG_JIT=0 to force the interpreter. */
tg_status tg_program_jit(tg_program_t p, const char** source, const char** log, double* compile_ms);

/* Number of kernel launches issued by this program since creation. */
uint64_t tg_launch_count(tg_program_t p);
void tg_program_free(tg_program_t p);

#ifdef __cplusplus
}
#endif
#endif /* TG_ABI_H */
