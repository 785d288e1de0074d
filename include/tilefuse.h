/*
 * tilefuse — C ABI of the B200-native (sm_100a) fused-collective library.
 *
 * This is the drop-in boundary under the reference package's Python primitive
 * and operator API (overlapsim, arXiv 2605.02953).  Every entry point below
 * names the reference interface it replaces (path:line relative to
 * /root/reference/pkg/src/overlapsim/).  Plain pointers and sizes only: no
 * torch types cross this boundary.  Streams are cudaStream_t passed as void*.
 *
 * Status codes (also the Python exception mapping in errors.py):
 *   0 OK, 1 INVALID_ARG -> ValueError, 2 CONFIG -> ConfigError,
 *   3 ALLOC -> AllocationError, 4 PROTOCOL -> ProtocolError,
 *   5 CUDA -> RuntimeError, 6 TIMEOUT -> DeadlockError.
 * The message for the last failure on the calling thread is tf_last_error().
 *
 * Asynchrony: every data-path call is enqueued on the given stream(s) and
 * returns immediately; argument validation is synchronous.  Device-side spin
 * timeouts are latched into the team's error word; tf_team_check() reads it.
 */
#ifndef TILEFUSE_H_
#define TILEFUSE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_MAX_WORLD 16

enum {
  TF_OK = 0,
  TF_ERR_INVALID = 1,
  TF_ERR_CONFIG = 2,
  TF_ERR_ALLOC = 3,
  TF_ERR_PROTOCOL = 4,
  TF_ERR_CUDA = 5,
  TF_ERR_TIMEOUT = 6,
};

enum { TF_DTYPE_BF16 = 0, TF_DTYPE_F32 = 1 };
enum { TF_REDUCE_RING = 0, TF_REDUCE_ASCENDING = 1 };
/* phases of a per-rank collective call */
enum { TF_PHASE_PRE = 1, TF_PHASE_MAIN = 2, TF_PHASE_POST = 4, TF_PHASE_FINAL = 8,
       TF_PHASE_ALL = 15 };

typedef struct tf_team tf_team;

/* Message of the last failed call on this thread ("" if none). */
const char* tf_last_error(void);
/* Library version / build string. */
const char* tf_version(void);

/* ------------------------------------------------------------------ tile order
 * Host-side tile tables, bit-identical to the reference swizzles.
 * tf_tile_map: entry j = row tile computed at step j.
 *   mode 0 = gather  (ag_gemm_tile_map,  swizzle.py:178-180, 144-175, 109-141)
 *   mode 1 = scatter (gemm_rs_tile_map,  swizzle.py:183-185)
 * tf_swizzle_2d: grouped order (swizzle_2d, swizzle.py:76-88).
 */
int tf_tile_map(int64_t m, int rank, int world, int nnodes, int block_m, int mode,
                int32_t* out, int64_t out_len);
int tf_swizzle_2d(int64_t pid, int64_t num_pid_m, int64_t num_pid_n, int group_m,
                  int64_t* pid_m, int64_t* pid_n);
/* MoE dynamic schedule (swizzle_ag_moe, swizzle.py:225-286).  counts is
 * [world, n_experts] row-major.  Output arrays are length >= *ntiles; call
 * with out arrays NULL to query ntiles. */
int tf_moe_schedule(const int64_t* counts, int world, int n_experts, int rank, int local_world,
                    int block_m, int64_t* ntiles, int64_t* expert_id, int64_t* tiled_m,
                    int64_t* segment_start, int64_t* segment_end, int64_t* stage);

/* ------------------------------------------------------------------ team / heap
 * Replaces SymmetricHeap (shmem.py:87-165).  A team is `world` PEs, each with a
 * symmetric data region of heap_bytes and signal_slots uint64 flags.
 *
 * tf_team_create_local: all PEs live in this process.  devices[pe] is the CUDA
 *   device of PE pe; devices may repeat (several PEs on one GPU: the
 *   single-device emulation used for parity tests when fewer GPUs exist).
 * tf_team_create_ipc: one PE per process (torchrun).  Allocates this rank's
 *   region; exchange tf_team_export_handle() blobs out of band (the Python side
 *   uses torch.distributed) and call tf_team_open_peers() with all of them.
 */
int tf_team_create_local(int world, const int* devices, size_t heap_bytes, size_t signal_slots,
                         tf_team** out);
int tf_team_create_ipc(int world, int rank, int device, size_t heap_bytes, size_t signal_slots,
                       tf_team** out);
int tf_team_export_handle(tf_team* t, void* blob, size_t blob_len); /* blob_len >= 128 */
int tf_team_open_peers(tf_team* t, const void* blobs, size_t blob_len);
int tf_team_destroy(tf_team* t);
int tf_team_world(tf_team* t, int* world);
int tf_team_device(tf_team* t, int pe, int* device);
/* Reads and clears the device error word of every PE this process owns and reports
 * the first one set: TF_ERR_TIMEOUT if a spin timed out, TF_ERR_PROTOCOL for a double
 * scoreboard release, TF_ERR_INVALID for a MoE receive-buffer overflow (a destination
 * row >= max_recv; those rows were not written) or an expert id outside [-1, E). */
int tf_team_check(tf_team* t);

/* alloc (shmem.py:109-121): identical offset on every PE, bump allocator. */
int tf_heap_alloc(tf_team* t, size_t nbytes, size_t align, uint64_t* offset);
/* alloc_signals (shmem.py:132-139). */
int tf_signal_alloc(tf_team* t, size_t nslots, uint64_t* base);
/* symm_at / remote_ptr / view (shmem.py:143-165): device pointer of PE pe's copy. */
int tf_heap_ptr(tf_team* t, int pe, uint64_t offset, void** ptr);
int tf_signal_ptr(tf_team* t, int pe, uint64_t slot, uint64_t** ptr);
/* sig_view (shmem.py:155-157): synchronous copy of n slots to host. */
int tf_signal_read(tf_team* t, int pe, uint64_t base, size_t n, uint64_t* host_out);
/* zero n slots of PE pe (stream-ordered). */
int tf_signal_reset(tf_team* t, int pe, uint64_t base, size_t n, void* stream);

/* ------------------------------------------------------------------ one-sided ops
 * Host-initiated, stream-ordered (copy engine where the driver uses one).
 * putmem / getmem (shmem.py:239-251), putmem_signal (shmem.py:301-310):
 * the signal on to_pe lands after the payload (release ordering). */
int tf_putmem(tf_team* t, int to_pe, uint64_t dst_off, const void* src, size_t nbytes,
              void* stream);
int tf_getmem(tf_team* t, int from_pe, uint64_t src_off, void* dst, size_t nbytes, void* stream);
int tf_putmem_signal(tf_team* t, int to_pe, uint64_t dst_off, const void* src, size_t nbytes,
                     uint64_t sig_slot, uint64_t value, int op_add, void* stream);
/* multimem_ld_reduce (shmem.py:335-351): out[i] = sum over the team's PEs, in
 * ascending rank order, of the element at `offset` + i in each PE's heap copy;
 * dtype 0 bf16 (fp32 accumulation, bf16 out), 1 fp32, 2 int64 (exact).  `out` is a
 * device buffer on the caller's device; peers are read over P2P (NVLink).
 * multimem_st (shmem.py:353-361): copy `src` into every PE's copy at `offset`
 * (one copy-engine transfer per PE).  Both stream-ordered on `stream`. */
int tf_team_reduce(tf_team* t, int pe, uint64_t offset, int dtype, int64_t count, void* out,
                   void* stream);
int tf_team_broadcast(tf_team* t, int from_pe, uint64_t offset, const void* src, size_t nbytes,
                      void* stream);
/* atomic_cas (shmem.py:196-206): acq_rel compare-and-swap of a signal slot; the
 * old value is returned in *old_out (synchronous: the stream is drained). */
int tf_signal_cas(tf_team* t, int pe, uint64_t slot, uint64_t cmp, uint64_t value, uint64_t* old_out,
                  void* stream);
/* putmem_strided (shmem.py:253-268): rows of row_bytes from src (src_pitch apart)
 * into PE to_pe's heap at dst_off, dst_pitch bytes apart (one 2-D copy). */
int tf_putmem_strided(tf_team* t, int to_pe, uint64_t dst_off, size_t dst_pitch, const void* src,
                      size_t src_pitch, size_t row_bytes, size_t rows, void* stream);
/* st / notify / atomic_add on a signal slot of PE pe (shmem.py:174-194). */
int tf_signal_op(tf_team* t, int pe, uint64_t slot, uint64_t value, int op_add, void* stream);
/* wait (shmem.py:208-235): stream waits until all n slots >= value (epoch flags). */
int tf_signal_wait(tf_team* t, int pe, uint64_t slot, size_t n, uint64_t value, void* stream);
/* wait with an explicit comparison: TF_CMP_EQ is the reference's semantics
 * (shmem.py:223-224, every slot == value); TF_CMP_GE the epoch-flag form. */
#define TF_CMP_GE 0
#define TF_CMP_EQ 1
int tf_signal_wait_cmp(tf_team* t, int pe, uint64_t slot, size_t n, uint64_t value, int cmp,
                       void* stream);
/* atomic_add returning the old value (shmem.py:184-194); synchronous like
 * tf_signal_cas.  tf_signal_op(op_add=1) is the stream-ordered, no-return form. */
int tf_signal_fetch_add(tf_team* t, int pe, uint64_t slot, uint64_t value, uint64_t* old_out,
                        void* stream);
/* barrier_all (shmem.py:319-322), split so a single host thread can drive
 * several PEs that share one stream: arrive, then wait. */
int tf_barrier_arrive(tf_team* t, int rank, void* stream);
int tf_barrier_wait(tf_team* t, int rank, void* stream);
int tf_barrier_all(tf_team* t, int rank, void* stream);

/* ------------------------------------------------------------------ float32 operands
 * The reference's float32 contract (oracles.py:12-27; tests/test_kernels.py:365-381
 * pin unordered float paths to norm-relative 1e-5).  Splits fp32 rows [rows, k]
 * (ld_src elements apart) into three bf16 terms and writes the 6-term K-expanded
 * operand [rows, 6*kp] bf16 (role 0 = A order a0 a0 a1 a0 a1 a2, role 1 = B order
 * b0 b1 b0 b2 b1 b0; columns k..kp zero), so the bf16 GEMM of the expanded
 * operands is the fp32 product up to ~2^-24 relative terms.  Stream-ordered. */
int tf_split_f32_bf16x3(const float* src, int64_t rows, int64_t k, int64_t ld_src, void* dst, int64_t kp,
                        int role, void* stream);

/* ------------------------------------------------------------------ GEMM tile
 * Core GEMM (the tile body of ag_gemm.py:93-94 / gemm_rs.py:123): persistent,
 * warp-specialised tcgen05 kernel, C[m,n] = sum_k A[m,k] * B[n,k], bf16 inputs,
 * fp32 accumulation in TMEM, bf16 or fp32 output.  Tile order: linear step ->
 * swizzle_2d(group_m) -> tile_map[pid_m] (ag_gemm.py:81-84). */
typedef struct tf_gemm_args {
  const void* a; /* [m, k] bf16, row stride lda elements (lda*2 % 16 == 0) */
  const void* b; /* [n, k] bf16, row stride ldb elements */
  void* c;       /* [m, n] out_dtype, row stride ldc elements */
  int64_t m, n, k, lda, ldb, ldc;
  int32_t out_dtype;   /* TF_DTYPE_BF16 or TF_DTYPE_F32 */
  int32_t block_m;     /* 128 (tensor-core tile rows) */
  int32_t block_n;     /* 128 or 256 */
  int32_t block_k;     /* 64 */
  int32_t group_m;     /* swizzle_2d group */
  int32_t num_gemm_sms;/* persistent CTAs; 0 = all SMs (minus num_comm_sms) */
  int32_t num_comm_sms;/* CTAs left free for reduce/pack kernels */
  int32_t swizzle;     /* 1 = apply the gather/scatter tile map */
  int32_t fuse_scatter;/* gemm_rs only; 1 = epilogue stores into owners' slots */
  int32_t reduce_order;/* TF_REDUCE_* */
  const int32_t* tile_map; /* optional device [ceil(m/block_m)] table; NULL = identity */
  int32_t nnodes;      /* gemm_rs unfused: nodes of the topology (0/1 = one node) */
  int32_t ring_links;  /* gemm_rs unfused: 1 = assume_full_mesh_links=False (ring order in a node) */
} tf_gemm_args;

int tf_gemm(const tf_gemm_args* args, void* stream);

/* ------------------------------------------------------------------ fused collectives
 * AllGather+GEMM (ag_gemm.py:20-94).  Per rank: a = local A shard [m/world, k],
 * b = local B shard [n_local, k], c = [m, n_local].  The team owns the gather
 * workspace (double-buffered) and arrival flags.  phase selects TF_PHASE_*:
 *   PRE  = local copy into own workspace slot + arrival flag + barrier arrive
 *   MAIN = barrier wait + peer pulls (rank+i)%w with per-chunk flags on
 *          comm_stream, tile GEMM waiting per tile on covering chunks on stream
 *   POST = nothing (flags are epoch-valued) unless reset_signals.
 * args->m is the GATHERED row count. */
int tf_ag_gemm(tf_team* t, int rank, const tf_gemm_args* args, int phase, void* stream,
               void* comm_stream);
/* GEMM+ReduceScatter (gemm_rs.py:31-338).  Per rank: a = input shard [m, k_local],
 * b = weight shard [n, k_local], c = output [m/world, n].
 *   fuse_scatter=1: epilogue stores row-slices into owner slot [rank] and bumps
 *   per-row-tile arrival counters (gemm_rs.py:135-162); the owner reduces its
 *   world slots in ascending or ring order in fp32 (gemm_rs.py:325-338).
 *   fuse_scatter=0: local GEMM + per-segment counters, owner pull-reduce
 *   (gemm_rs.py:107-132, 177-196).
 * phases: PRE = barrier arrive; MAIN = barrier wait + GEMM (+ overlapped reduce
 * on comm_stream when overlap is possible); POST = reduce (if not overlapped)
 * + counter reset. */
int tf_gemm_rs(tf_team* t, int rank, const tf_gemm_args* args, int phase, void* stream,
               void* comm_stream);

/* GEMM+AllReduce (gemm_ar.py:25-153).  Per rank: a = [m, k] and b = [n, k]
 * partial operands, c = [m, n] = sum over ranks of a_r . b_r^T (same on every rank).
 * The GEMM writes its partial into the symmetric workspace and bumps a
 * per-128-row-block counter (epoch-valued, never reset: target = epoch*tiles).
 * two_shot = 0: every rank pulls every block from all peers and reduces it in
 *   ascending rank order (gemm_ar.py:95-102).
 * two_shot = 1: block b is owned by rank b % world; the owner reduces it and
 *   P2P-stores the result into every peer's result buffer, then releases a
 *   per-block flag (multimem_st analogue, gemm_ar.py:103-133); every rank copies
 *   the result once all blocks are flagged.
 * phases as tf_gemm_rs: PRE = barrier arrive, MAIN = barrier wait + GEMM (+
 * overlapped reduce when no other rank shares the device), POST = reduce,
 * FINAL = two-shot result gather (after every rank's POST). */
int tf_gemm_ar(tf_team* t, int rank, const tf_gemm_args* args, int two_shot, int phase,
               void* stream, void* comm_stream);

/* ------------------------------------------------------------------ NVLS multicast region
 * The B200 form of multimem_ld_reduce / multimem_st (shmem.py:335-385): one
 * multicast object over every PE's copy of an `nvls` region, reached with
 * multimem.ld_reduce (sum of all copies, reduced in the NVSwitch) and
 * multimem.st (write every copy).  Opt-in: tf_nvls_supported probes
 * CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED; creation failures return
 * TF_ERR_CONFIG and callers keep the P2P paths.
 *   local team: tf_team_nvls_create does everything (fd_out = -1).
 *   IPC team  : rank 0 tf_team_nvls_create -> POSIX fd (pass it to the peers
 *               over a Unix socket, SCM_RIGHTS); the others tf_team_nvls_import;
 *               then every rank tf_team_nvls_add_device, a barrier, and
 *               tf_team_nvls_bind. */
int tf_nvls_supported(int device, int* supported);
int tf_team_nvls_create(tf_team* t, size_t bytes, int* fd_out);
int tf_team_nvls_import(tf_team* t, size_t bytes, int fd);
int tf_team_nvls_add_device(tf_team* t);
int tf_team_nvls_bind(tf_team* t);
int tf_nvls_enabled(tf_team* t, int* enabled, size_t* bytes);
int tf_nvls_alloc(tf_team* t, size_t nbytes, size_t align, uint64_t* offset);
int tf_nvls_ptr(tf_team* t, int pe, uint64_t offset, void** uc, void** mc);
/* out[0:count) = sum over PEs of region[offset:...] (dtype 0 bf16 with fp32
 * accumulation, 1 f32, 2 int64); device out, stream-ordered on PE pe's device. */
int tf_nvls_reduce(tf_team* t, int pe, uint64_t offset, int dtype, int64_t count, void* out, void* stream);
/* every PE's region[offset:offset+bytes) = src (device, 16-byte aligned). */
int tf_nvls_broadcast(tf_team* t, int pe, uint64_t offset, const void* src, size_t bytes, void* stream);

/* ------------------------------------------------------------------ SP attention scores
 * AllGather-KV fused with Q.K^T (BASELINE config 3): structurally
 * ag_gemm (ag_gemm.py:20-94) with the gathered operand on the N (key) side.
 * Per rank: q = [s_local, hq, d] queries, k = [s_local, hkv, d] keys (GQA,
 * hq % hkv == 0); scores[h] = q[:, h, :] . K_all[:, h / (hq/hkv), :]^T, i.e.
 * scores = [hq, s_local, world * s_local].  The key shards are pulled into the
 * symmetric workspace with per-chunk flags; every head's GEMM acquire-waits on
 * the key chunks its tiles cover, in gather-swizzled key-tile order. */
typedef struct tf_attn_args {
  const void* q;
  const void* k;
  void* scores;
  int64_t s_local, hq, hkv, d;  /* d % 8 == 0 */
  int32_t out_dtype, block_m, block_n, group_m, num_gemm_sms, swizzle;
  const int32_t* key_tile_map;  /* optional device [ceil(S/block_n)] permutation */
} tf_attn_args;
int tf_ag_kv_scores(tf_team* t, int rank, const tf_attn_args* a, int phase, void* stream,
                    void* comm_stream);

/* AG-KV fused with the flash-attention forward (config 3):
 * O[q, h, :] = softmax(q[q, h, :] . K_all[:, g(h), :]^T * scale) . V_all[:, g(h), :]
 * for this rank's queries against every rank's keys/values, never
 * materialising the scores.  q/out: [s_local, hq, 128] bf16; k/v: [s_local, hkv,
 * 128] bf16 shards; s_local % 128 == 0.  Same phases as tf_ag_gemm. */
typedef struct tf_attn_fwd_args {
  const void* q;
  const void* k;
  const void* v;
  void* out;
  int64_t s_local, hq, hkv, d;
  float scale;
} tf_attn_fwd_args;
int tf_ag_kv_attention(tf_team* t, int rank, const tf_attn_fwd_args* a, int phase, void* stream,
                       void* comm_stream);

/* ------------------------------------------------------------------ MoE (expert parallel)
 * Not in the reference as an all-to-all; what the reference pins
 * is the layout: the [world, E] routing-count matrix (ag_moe.py:28-33) and the
 * expert-major, then source-rank, then source-order receive layout
 * (gather_tokens_by_expert, oracles.py:38-50).  Rank d owns experts
 * [d*E/world, (d+1)*E/world).
 *
 * Routing: top-k of logits per token, descending, ties to the lower expert id;
 * weights = softmax of the selected logits (fp32). */
int tf_moe_topk(const float* logits, int64_t tokens, int n_experts, int k, int32_t* topk_idx,
                float* topk_w, void* stream);
/* This rank's routing row and send order: counts[e] = #(token, slot) routed to
 * expert e; sorted_pos[t*k+j] = position of (t, j) in the rank's expert-sorted
 * chunk (stable: expert, then token, then slot).  Deterministic (no atomics
 * decide positions).  scratch: >= tf_moe_count_scratch_bytes(tokens*k, n_experts). */
int64_t tf_moe_count_scratch_bytes(int64_t entries, int n_experts);
int tf_moe_count(const int32_t* topk_idx, int64_t tokens, int k, int n_experts, int32_t* counts,
                 int32_t* sorted_pos, void* scratch, void* stream);

typedef struct tf_moe_args {
  int64_t tokens;         /* T: tokens on this rank */
  int64_t hidden;         /* H (multiple of 8) */
  int32_t k;              /* top-k */
  int32_t n_experts;      /* E, divisible by world */
  int64_t max_recv;       /* receive capacity in rows on every rank */
  const void* x;          /* [T, H] bf16 dispatch input */
  const int32_t* topk_idx;/* [T, k] */
  const float* topk_w;    /* [T, k] combine weights */
  void* out;              /* [T, H] bf16 combine output */
  int32_t* counts;        /* [world, E] device: full routing matrix (filled by dispatch) */
  int32_t* sorted_pos;    /* [T, k] device: from tf_moe_count */
  int32_t* dest_row;      /* [T, k] device: receive row of (t, j) on its owner (filled by dispatch) */
  int64_t* recv_rows;     /* [1] device: rows received by this rank (filled by dispatch) */
  const float* logits;    /* optional [T, E] fp32 router logits: dispatch computes the top-k
                             itself (ties -> lower expert) into topk_idx / topk_w */
} tf_moe_args;

/* Device pointers of this rank's receive buffer [max_recv, H] bf16 and expert
 * output buffer [max_recv, H] bf16 inside the symmetric heap. */
int tf_moe_buffers(tf_team* t, int rank, const tf_moe_args* a, void** recv, void** expert_out);
/* Dispatch (EP all-to-all).  When the caller passes PRE|MAIN in one call (one
 * rank per GPU), both run as ONE persistent launch (routing, counts, count
 * exchange, layout and scatter, with a grid-wide wait in between); PRE and MAIN
 * called separately (several ranks sharing a GPU) are one launch each.
 *   PRE  = routing counts + send order of this rank (as tf_moe_count, into
 *          a->sorted_pos), count row pushed to every peer's matrix + flag;
 *   MAIN = wait for all rows, copy the full matrix to a->counts, compute
 *          a->dest_row / a->recv_rows, 16-byte vector scatter of token rows into
 *          the owners' receive buffers, release a per-source flag on each owner;
 *   POST = wait until every source has delivered to this rank. */
int tf_moe_dispatch(tf_team* t, int rank, const tf_moe_args* a, int phase, void* stream);
/* Combine: PRE = announce this rank's expert outputs ready; MAIN = wait all
 * owners, pull the k expert rows of every token over NVLink and reduce
 * out[t] = sum_j w[t,j] * y[row(t,j)] in fp32 (slot order), bf16 out. */
int tf_moe_combine(tf_team* t, int rank, const tf_moe_args* a, int phase, void* stream);

/* AllGather + grouped GEMM for expert-routed tokens (ag_moe_group_gemm,
 * ovs/kernels/ag_moe.py:20-142).  Per rank: tokens = this rank's rows [rows_r, k]
 * bf16 grouped by expert (rows_r = sum(routing[rank])), weights = this rank's
 * stacked expert shards [n_experts, n, k] bf16, out = [total_rows, n]
 * expert-major (row expert_base[e] + source-major offset).  routing is a HOST
 * [world, n_experts] int64 count matrix, identical on every rank.
 *   PRE  = tile schedule (swizzle_ag_moe order, swizzle.py:225-286, or plain tile
 *          order when swizzle = 0) and piece tables to the device; local rows ->
 *          own workspace at their expert-major rows; own arrival counter :=
 *          target; barrier arrive                        (ag_moe.py:104-108)
 *   MAIN = barrier wait, then ONE launch: num_comm_sms pull-engine CTAs copy the
 *          peers' pieces in (rank+i)%w order and release a per-source arrival
 *          counter (ag_moe.py:109-117); the grouped tcgen05 GEMM CTAs walk the
 *          schedule and acquire-wait sources [segment_start, segment_end] of
 *          each tile before its TMA loads (ag_moe.py:120-142).
 * max_rows bounds total_rows (workspace sizing; 0 = this call's total).
 * block_m 128 (one CTA) or 256 (CTA pair); n % 8 == 0, k % 8 == 0. */
typedef struct tf_agmoe_args {
  const void* tokens;
  const void* weights;
  void* out;
  const int64_t* routing;
  int64_t n_experts, n, k, max_rows, lda, ldo;
  int32_t out_dtype, block_m, block_n, num_gemm_sms, num_comm_sms, swizzle;
} tf_agmoe_args;
int tf_ag_moe_group_gemm(tf_team* t, int rank, const tf_agmoe_args* a, int phase, void* stream);

/* ------------------------------------------------------------------ task-level megakernel
 * Executor for the reference's task graphs (ovs/megakernel/):
 * queues = int32 [slots][num_sms][30] task records (encoding.py:20-166),
 * counts = int32 [num_sms], deps = int32 [n][3] (producer, first tile, end),
 * layer_cfg = int32 [layers][4] (op 0 linear / 1 add / 2 allreduce, block_m,
 * block_n, block_rows), all device pointers.  Scoreboard flags live in every PE's
 * signal space at flag_base + task * max_tiles + tile and are set to `epoch`.
 * All ranks of the (local, single-device) team run co-resident in one launch:
 * world * num_sms CTAs.  Tensors: fp32 [rows, cols] at each io slot's offset. */
typedef struct tf_mega_args {
  const int32_t* queues;
  const int32_t* counts;
  const int32_t* deps;
  const int32_t* task_ops; /* reserved */
  const int32_t* layer_cfg;
  int32_t num_sms, slots, max_tiles, num_layers;
  uint64_t flag_base, epoch, timeout_ns;
} tf_mega_args;
int tf_megakernel_run(tf_team* t, const tf_mega_args* a, void* stream);

/* ------------------------------------------------------------------ fused-layer megakernel (bf16)
 * Same task records / queues / dependency rows / scoreboard as tf_megakernel_run
 * (ovs/megakernel/encoding.py:20-166, builders.py:105-162, scoreboard.py:33-56),
 * for the bf16 transformer-layer ops (BASELINE config 5): layer_cfg = int32
 * [layers][16] = {op (1 rmsnorm, 2 linear, 3 attention, 4 allreduce_residual),
 * block_m, block_n, block_rows, epilogue (0 none, 1 rope, 2 silu_mul), tensor map
 * of A / qkv, tensor map of B, heads_q, heads_kv, seq_len, softmax scale (f32
 * bits), rms eps (f32 bits), causal, rope columns, output io slot, 0}.
 * map_specs (HOST) = int64 [num_maps][8] {heap offset, ndims, dims[3] innermost
 * first, box[3]}: bf16 128-byte-swizzled TMA maps encoded against every launched
 * rank's heap base.  Local team: rank = -1, every rank co-scheduled on one
 * device (world * num_sms CTAs).  IPC team: rank = this process's rank (num_sms
 * CTAs; peers reached through the IPC-mapped heaps). */
typedef struct tf_layer_args {
  const int32_t* queues;
  const int32_t* counts;
  const int32_t* deps;
  const int32_t* layer_cfg;
  const int64_t* map_specs;
  int32_t num_maps, num_sms, max_tiles, num_layers;
  uint64_t flag_base, epoch, timeout_ns;
  /* optional device trace, [ctas][slots][4] u64 (NULL = off): per task the
   * %globaltimer ns when warp 0 (tensor tasks) / warps 2-5 (elementwise) picked
   * it up, when its dependencies were satisfied, when its flag was released,
   * and task_id << 32 | tile */
  uint64_t* trace;
  int32_t trace_slots; /* queue slots per CTA in the trace layout */
} tf_layer_args;
int tf_layer_megakernel_run(tf_team* t, int rank, const tf_layer_args* a, void* stream);

/* ------------------------------------------------------------------ device tracing
 * Per-tile device events (%globaltimer ns) from the GEMM kernels on `device`,
 * the hardware analogue of the reference's Trace / TraceEvent
 * (simengine.py:56-73, export_chrome_trace :372-389).  Record = 4 x u64:
 *   [0] kind << 56 | rank << 48 | cta << 32 | tile   (kind 1 wait_chunks, 2 gemm_tile, 3 epilogue)
 *   [1] t_start  [2] t_end  [3] payload (wait: first_chunk << 32 | num_slots;
 *   tiles: pid_m << 32 | pid_n).  tf_trace_read copies and clears the buffer. */
int tf_trace_enable(int device, int64_t capacity);
int tf_trace_disable(int device);
int tf_trace_read(int device, uint64_t* host, int64_t capacity, int64_t* count);

/* ------------------------------------------------------------------ device topology
 * Die (L2 partition) of every SM of `device`, measured once per process by
 * first-touch load latency (no reference counterpart: it feeds the persistent
 * GEMM's die-ranked tile order, TF_GEMM_DIE).  out[smid] = 0 / 1 for smid <
 * *n_sms; *n_sms = 0 when no two-die structure was found. */
int tf_sm_die_map(int device, uint8_t* out, int cap, int* n_sms);

#ifdef __cplusplus
}
#endif
#endif /* TILEFUSE_H_ */
