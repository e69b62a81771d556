/*
 * shmem_b200.h — C ABI of the B200-native fused AllGather+GEMM / GEMM+ReduceScatter
 * path (symmetric heap over NVLink + sm_100a tcgen05 kernels).
 *
 * This is the drop-in boundary for the reference package `minishmem`
 * (/root/reference/pkg/src/minishmem).  Every entry point below replaces one
 * reference interface; the Python mirror in paper_2504_19442_b200/ binds
 * these with ctypes exactly as a maintainer would from the reference side
 * (see INTEGRATION.md).
 *
 * Conventions
 *   - every function returns int status: SH_OK (0) or one of SH_ERR_*; the
 *     message of the last failure on the calling thread is sh_last_error().
 *   - pointers are device pointers on the rank's GPU unless stated; sizes in
 *     bytes; matrices are row-major, dtype bf16 (SH_DTYPE_BF16) or fp16.
 *   - `stream` is a cudaStream_t (may be NULL = legacy default stream); all
 *     device work is enqueued on it (stream-ordered, asynchronous).
 *     sh_gemm / sh_ag_gemm / sh_gemm_rs refuse a stream under CUDA graph
 *     capture (SH_ERR_STATE): their epochs are baked into each launch.
 *   - signals are u64 words in a pad at the tail of each rank's slab; a
 *     signal index `sig` addresses slab + heap_bytes + 8*sig on every rank
 *     (reference core.py:242-261).
 */
#ifndef SHMEM_B200_H
#define SHMEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SH_OK 0
#define SH_ERR_ARG 1     /* maps to ArgumentError       (reference errors.py:19)  */
#define SH_ERR_ALLOC 2   /* maps to AllocationError     (reference errors.py:15)  */
#define SH_ERR_TIMEOUT 3 /* maps to SynchronizationFault (reference errors.py:27) */
#define SH_ERR_CUDA 4    /* CUDA runtime/driver failure                           */
#define SH_ERR_STATE 5   /* maps to UsageError          (reference errors.py:31)  */
#define SH_ERR_CONFIG 6  /* maps to ConfigurationError  (reference errors.py:11)  */

#define SH_DTYPE_BF16 0
#define SH_DTYPE_FP16 1

#define SH_MAX_WORLD 16

typedef struct sh_world sh_world;

/* Library identity / diagnostics. */
int sh_version(void);
const char* sh_last_error(void);

/* World bring-up: replaces WorldSpec/World.__init__/init_world
 * (reference core.py:35-66, 151-187, 565-567).
 * Single-process world: rank r lives on devices[r] (ranks may share a GPU);
 * every slab is mapped into every rank (peer access over NVLink). */
int sh_world_create(int world_size, const int* devices, size_t heap_bytes, int signal_count,
                    double timeout_s, sh_world** out);
/* One process per GPU (torchrun): allocate this rank's slab; peers are
 * attached with sh_import_ipc_handles after an out-of-band all-gather. */
int sh_world_create_member(int world_size, int rank, int device, size_t heap_bytes,
                           int signal_count, double timeout_s, sh_world** out);
int sh_ipc_handle_size(void);
int sh_export_ipc_handle(sh_world* w, void* handle_out);
int sh_import_ipc_handles(sh_world* w, const void* handles /* world_size * handle_size */);
int sh_world_destroy(sh_world* w);

/* Symmetric allocation: replaces World.alloc_symmetric / alloc_signals
 * (reference core.py:211-237).  Same offset / base on every rank. */
int sh_alloc(sh_world* w, size_t nbytes, size_t align, size_t* offset);
int sh_alloc_signals(sh_world* w, int count, int* base);

/* Address resolution: replaces World._abs / _sig_abs (reference core.py:254-261).
 * Pointer to `peer`'s replica as seen from `rank`'s device. */
int sh_heap_ptr(sh_world* w, int rank, int peer, size_t offset, void** ptr);
int sh_signal_ptr(sh_world* w, int rank, int peer, int sig, void** ptr);

/* Signal maintenance: replaces sig_read / _reset_own_signals / tuning.reset_signals
 * (reference core.py:263-301, collectives.py:67-69, tuning.py:79-91). */
int sh_read_signals(sh_world* w, int rank, int base, int count, uint64_t* out_host);
int sh_reset_signals(sh_world* w, int rank, int base, int count, void* stream);

/* Release-store `value` into signals [base, base+count) of `rank`'s own pad
 * on `stream` (recovery: saturating the words satisfies every pending >= wait
 * of a world whose peer never signalled; World.recover). */
int sh_fill_signals(sh_world* w, int rank, int base, int count, uint64_t value, void* stream);

/* Device-side timeouts (bounded spins) land in a host-mapped error word per
 * rank; nonzero => SynchronizationFault (reference sched.py:227-238). */
int sh_poll_error(sh_world* w, int rank, int* code);
/* Clears the error word and the kernels' retired-CTA counters (the last-CTA
 * flag release); call with the rank's device drained (World.recover). */
int sh_clear_error(sh_world* w, int rank);

/* Fused AllGather+GEMM for rank `rank`: replaces pipelines.ag_gemm
 * (reference pipelines.py:97-150) including its comm half
 * allgather_push_intra(wait_all=False) (collectives.py:83-102).
 *   a_shard : (m/W, k) this rank's rows        b : (k, n)        c : (m, n) out
 *   gathered_off : offset of the symmetric (W*m/W*k) gather buffer
 *   ready_base   : W signals; ready[src] counts src's landed row ranges:
 *                  (epoch-1)*S + j once range j of S landed (S = sh_ag_subchunks)
 *   done_base    : W signals; done[p] = epoch once rank p finished reading its
 *                  gather buffer (stored into every peer by the GEMM's last
 *                  retiring CTA; SHB_EXIT_RELEASE=0: stream writes after it)
 *   chunk_order  : W ints, a permutation (first-visit order of the TileSchedule)
 *   epoch        : monotone call counter (>= 1), identical on every rank */
int sh_ag_gemm(sh_world* w, int rank, const void* a_shard, const void* b, void* c,
               size_t gathered_off, int ready_base, int done_base, int m, int n, int k, int dtype,
               const int* chunk_order, uint64_t epoch, void* stream);

/* Fused GEMM+ReduceScatter for rank `rank`: replaces pipelines.gemm_rs
 * (reference pipelines.py:179-216) with rs_intra_streams (collectives.py:131-175).
 *   a : (m, k)   b : (k, n)   out : (m/W, n) = row block `rank` of sum_r a_r @ b_r
 *   staging_off   : offset of the symmetric W*(m/W)*n staging buffer
 *   producer_base : W signals; producer[d] = epoch once rank d reduced this call
 *                   (stored by the last retiring CTA of the reducing kernel)
 *   reduction_base: W signals; reduction[s] counts elements delivered by s */
int sh_gemm_rs(sh_world* w, int rank, const void* a, const void* b, void* out,
               size_t staging_off, int producer_base, int reduction_base, int m, int n, int k,
               int dtype, const int* chunk_order, uint64_t epoch, void* stream);

/* Phased variants.  SH_PHASE_ALL is the fused call above.  A call split into
 * SH_PHASE_COMM then SH_PHASE_COMPUTE (same epoch) never waits on the device
 * for work a peer has not issued yet, provided every rank's COMM phase has
 * completed (stream drained + host barrier) before any COMPUTE phase is
 * enqueued -- the protocol World uses for ranks that share a process when a
 * kernel-serialising tool (ncu, compute-sanitizer, CUDA_LAUNCH_BLOCKING) is
 * attached.
 *   AG: COMM = the shard pushes and their ready flags (on `stream`);
 *       COMPUTE = the GEMM (flags already set) and the done flags.
 *   RS: COMM = the GEMM with every tile scattered into its owner's staging
 *       slot plus the arrival counters (no fused reduction);
 *       COMPUTE = the ascending-source reduction and the producer flags.
 * subchunks (AG): row ranges per pushed shard, each with its own flag value
 * (0 = library policy, sh_ag_subchunks); must agree on every rank. */
#define SH_PHASE_ALL 0
#define SH_PHASE_COMM 1
#define SH_PHASE_COMPUTE 2
int sh_ag_gemm_ex(sh_world* w, int rank, const void* a_shard, const void* b, void* c,
                  size_t gathered_off, int ready_base, int done_base, int m, int n, int k,
                  int dtype, const int* chunk_order, uint64_t epoch, int subchunks, int phase,
                  void* stream);
int sh_gemm_rs_ex(sh_world* w, int rank, const void* a, const void* b, void* out,
                  size_t staging_off, int producer_base, int reduction_base, int m, int n, int k,
                  int dtype, const int* chunk_order, uint64_t epoch, int phase, void* stream);
/* Default sub-chunk count of an AG shard of (m/world, k) (1 = whole shard). */
int sh_ag_subchunks(int m, int k, int world, int* subchunks);

/* One-sided primitives, stream-ordered on the rank's stream: the Table-1
 * subset the standalone collectives are composed of (reference
 * primitives.py:126-257).  putmem copies nbytes from the rank's device memory
 * into `peer`'s replica at dst_off (copy engine over NVLink); getmem the
 * reverse.  signal_op: op 0 = SET (stream write, release), 1 = ADD (device
 * red.release.sys).  signal_wait: cond 0 EQ, 1 NE, 2 GE, 3 GT, 4 LE, 5 LT on the
 * rank's own pad (EQ/GE on the GPU front end, others a one-thread bounded spin). */
#define SH_SIG_SET 0
#define SH_SIG_ADD 1
int sh_putmem(sh_world* w, int rank, int peer, size_t dst_off, const void* src, size_t nbytes,
              void* stream);
int sh_getmem(sh_world* w, int rank, void* dst, int peer, size_t src_off, size_t nbytes,
              void* stream);
int sh_signal_op(sh_world* w, int rank, int peer, int sig, int op, uint64_t value, void* stream);
int sh_signal_wait(sh_world* w, int rank, int sig, int cond, uint64_t value, void* stream);

/* out[i] = sum over s = 0..nslots-1 (ascending) of slot s of the rank's own
 * replica at staging_off (reduce half of rs_intra_streams, collectives.py:163-171).
 * dtype: SH_DTYPE_BF16 / FP16 (fp32 accumulate), SH_DTYPE_FP32, SH_DTYPE_I32,
 * SH_DTYPE_I64 (accumulate in the element type, like numpy's `acc +=`). */
#define SH_DTYPE_FP32 2
#define SH_DTYPE_I32 3
#define SH_DTYPE_I64 4
int sh_reduce_slots(sh_world* w, int rank, size_t staging_off, int nslots, size_t slot_elems,
                    int dtype, void* out, void* stream);

/* Node-scope multimem (reference Pe.multimem_st / Pe.multimem_ld_reduce,
 * primitives.py:291-315), over the node's ranks [first, first + count):
 * sh_multimem_st replicates the caller's bytes [offset, offset + nbytes) of
 * its own replica into every other node rank's replica (one read, count-1
 * NVLink stores per 16 B); sh_multimem_ld_reduce writes into the device
 * buffer `out` the element-wise sum of the node's replicas in ascending rank
 * order, computed like numpy's `out += replica` in the element type (floats
 * round per step, integers wrap).  dtype: SH_DTYPE_BF16, FP16, FP32, I32,
 * I64, U8, I8; nbytes must be a multiple of the element size.  Both are
 * stream-ordered: the caller orders them after the peers' writes (barrier). */
#define SH_DTYPE_U8 5
#define SH_DTYPE_I8 6
int sh_multimem_st(sh_world* w, int rank, int first, int count, size_t offset, size_t nbytes,
                   void* stream);
int sh_multimem_ld_reduce(sh_world* w, int rank, int first, int count, size_t offset,
                          size_t nbytes, int dtype, void* out, void* stream);

/* Timeline evidence (reference World.start_trace/stop_trace, core.py:434-444,
 * and Timeline.to_chrome_trace, costmodel.py:185-190): while enabled, every
 * fused launch of `rank` records %globaltimer stamps per CTA -- chunk-flag
 * waits, per-tile epilogue windows, peer-arrival waits, CTA lifetime -- into
 * a ring of `max_launches` launch slots.  sh_trace_read copies the ring
 * (words = max_launches*grid*records_per_cta*4) and fills info =
 * {launches recorded, slots, grid, records_per_cta, mode of slot 0..}. */
int sh_trace_enable(sh_world* w, int rank, int records_per_cta, int max_launches);
int sh_trace_read(sh_world* w, int rank, uint64_t* out_host, size_t out_words, int* info);

/* The GEMM core alone (TP=1, no symmetric heap): c(m,n) = a(m,k) @ b(k,n).
 * `workspace` (device, 16-B aligned, sh_gemm_workspace_bytes() bytes, may be
 * NULL when that is 0) holds the stream-K partials; with a NULL / short
 * workspace the kernel falls back to whole tiles.  Stream-ordered like the
 * rest, so a caching allocator may hand the same block to the next call. */
int sh_gemm_workspace_bytes(int m, int n, int k, size_t* bytes);
int sh_gemm(const void* a, const void* b, void* c, int m, int n, int k, int dtype, void* workspace,
            size_t workspace_bytes, void* stream);

/* Tile override for tuning: bn in {0 (auto), 128, 224, 256, 512}; cta_group in {0 (auto),
 * 1, 2} (224 and 512 need cta_group 2; 512 = the single-buffered 256x512 pair tile). */
int sh_set_tile_config(int bn, int cta_group);
/* Tile-order override for tuning: stream_k -2 unset (env SHB_SK, else auto),
 * -1 auto (split the last waves when they would leave CTA pairs idle), 0 off,
 * 1 always; group_m -1 unset (env SHB_GROUP_M, else auto), 0 auto (L2 budget)
 * or the number of m-blocks walked per n-block. */
int sh_set_schedule_config(int stream_k, int group_m);
/* Data-parallel tile hand-out: -1 default (env SHB_DYN, else static), 0 static
 * stride schedule, 1 dynamic (global atomic counter, one tile fetched ahead). */
int sh_set_dynamic_tiles(int mode);
/* Launch config chosen for a problem (for the bench's roofline bookkeeping). */
int sh_query_tile_config(int rows, int world, int n, int* bn, int* cta_group, int* grid);

/* Single-GPU TP proxy (measurement only; no reference counterpart): treat
 * `rank` as the only rank on its device (full persistent grid, overlapped
 * side-stream pushes) while its peers are emulated by feeder streams that do
 * not launch GEMMs; solo=0 restores the device-sharing bookkeeping. */
int sh_set_rank_solo(sh_world* w, int rank, int solo);
/* Stream memory operations on any 8-byte word (device memory, or pinned host
 * memory under UVA): a front-end write / a GEQ wait, no SM involved. */
int sh_stream_write_word(void* word, uint64_t value, void* stream);
int sh_stream_wait_word(const void* word, uint64_t value, void* stream);
/* Host pacer: spin until *origin >= origin_value, then store tick_base+i+1
 * into *tick at origin + deltas_ns[i] (host monotonic clock).  Blocking. */
int sh_pace_host(const void* origin, uint64_t origin_value, void* tick, uint64_t tick_base,
                 const uint64_t* deltas_ns, int n, double timeout_s);
#ifdef __cplusplus
}
#endif
#endif /* SHMEM_B200_H */
