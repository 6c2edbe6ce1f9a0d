/*
 * hod.h — C ABI of the Holmes Overlapped Distributed-optimizer (HOD) data path
 * on B200 (sm_100a).
 *
 * The reference (arXiv 2312.03549, /root/reference/pkg) has NO native optimizer:
 * it only PRICES the data-parallel gradient synchronisation of a pipeline stage
 * as reduce-scatter + all-gather of the stage's gradient bytes
 *   - CostModel.reduce_scatter / CostModel.all_gather   simulator.py:81-89
 *   - dp_sync per stage (max over the stage's DP rows)  simulator.py:327-333
 *   - post-flush placement                              simulator.py:445-452
 *   - gradient-set size                                 simulator.py:268-280
 * and imports the real optimizer from Megatron-LM / Megatron-LLaMA.
 * Every entry point below is the device-side operation behind one of those
 * priced terms.  A host binding (ctypes, cgo,
 * JNI, ...) needs nothing but this header: plain pointers, sizes, and a
 * cudaStream_t passed as void*.
 *
 * Conventions
 *   - return 0 on success; a non-zero value is a cudaError_t / ncclResult_t /
 *     HOD_E* code and hod_last_error() returns a thread-local message.
 *   - every buffer is caller-owned device memory (allocated by PyTorch); the
 *     library never allocates persistent device memory (NCCL's internal
 *     buffers excepted) and never synchronises the host inside a step.
 *   - "bf16" buffers are uint16_t bit patterns; rounding is IEEE RNE.
 *   - all kernels are compiled for sm_100a only; there is no CPU fallback.
 */
#ifndef HOD_H_
#define HOD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 3: hod_adamw_tma removed (the TMA-fed path is the span kernel of
 *    hod_p2p_step), hod_set_span_tma added */
#define HOD_ABI_VERSION 3

/* library-level error codes (outside the cudaError_t / ncclResult_t ranges) */
#define HOD_OK 0
#define HOD_EINVAL 10001   /* bad argument (null pointer, negative size, ...) */
#define HOD_EALIGN 10002   /* a buffer violates the documented alignment     */
#define HOD_ETIMEOUT 10003 /* a cross-GPU wait exceeded its spin budget      */
#define HOD_ENCCL 10004    /* NCCL returned an error (message has details)   */
#define HOD_ESPAN 10005    /* ranks met at a barrier slot with different tags,
                              i.e. closed a span over different buckets     */

/* source dtype of a gradient tensor fed to the packer */
#define HOD_DTYPE_BF16 0
#define HOD_DTYPE_F32 1

/* maximum tensors in one hod_pack_bf16 call (larger tables are split) */
#define HOD_PACK_MAX_ENTRIES 64

/* number of per-bucket partial sums written by hod_sumsq_bf16 */
#define HOD_SUMSQ_PARTIALS 296

/* One gradient tensor of a bucket: `numel` elements of `src` (dtype given to
 * the call) land at bucket[dst_offset .. dst_offset+numel).  Entries must be
 * sorted by dst_offset and must not overlap; elements of the bucket covered
 * by no entry (alignment gaps, tail padding) are written as +0.0. */
typedef struct hod_pack_entry {
  const void* src;
  int64_t numel;
  int64_t dst_offset;
} hod_pack_entry;

/* AdamW arithmetic: EXACT = IEEE operations in the oracle's order (bit-exact
 * against oracle/hod_oracle.c; ~90 instructions per element); FAST = the same
 * algebra with FMAs and MUFU sqrt/reciprocal (~25 instructions per element),
 * within the north star's 1e-6 (1 step) / 1e-5 (100 steps) tolerance. */
#define HOD_ADAMW_EXACT 0
#define HOD_ADAMW_FAST 1

/* AdamW hyper-parameters for one step.  The library folds them into fp32
 * constants exactly as documented in DESIGN.md §K2 (decoupled weight decay,
 * torch.optim.AdamW algebra). */
typedef struct hod_adamw_params {
  double lr;
  double beta1;
  double beta2;
  double eps;
  double weight_decay;
  int64_t step; /* 1-based step count used for bias correction */
  int32_t mode; /* HOD_ADAMW_EXACT (default) or HOD_ADAMW_FAST */
  int32_t reserved;
} hod_adamw_params;

/* ---- version / errors ---------------------------------------------------- */
int hod_abi_version(void);
const char* hod_last_error(void);
/* number of kernels this library has launched in the process (all streams) */
long long hod_launch_count(void);
/* Cap every subsequent launch of the process (all threads: autograd issues
 * hook-driven launches from its own device thread) at `max_ctas` CTAs
 * (0 = no cap).  The overlapped optimizer sets it while backward GEMMs run.
 * A cap <= 148 (one CTA per SM) is the CO-RESIDENT mode: the launchers also
 * pick register-light kernel variants, so that every optimizer CTA fits on an
 * SM beside a resident cuBLAS GEMM CTA and the two share the SM (tensor
 * cores vs HBM/NVLink) instead of time-slicing it.  Every kernel prefers the
 * maximum shared-memory carveout for the same reason (HOD_CARVEOUT=0 turns
 * that off).  Partial-sum kernels use min(cap, HOD_SUMSQ_PARTIALS) CTAs and
 * zero the unused partial slots. */
int hod_set_grid_limit(int max_ctas);

/* ---- K1: bucket pack + dp-scale + bf16 cast ---------------
 * bucket[dst_offset + i] = bf16_rne(float(src[i]) * scale), zeros elsewhere.
 * `entries` is a HOST array (copied into the kernel's parameter space).
 * Replaces the reference's implicit "gradient bytes of a stage"
 * (simulator.py:268-280) with the actual flattened bucket. */
int hod_pack_bf16(const hod_pack_entry* entries, int n_entries, uint16_t* bucket,
                  int64_t bucket_numel, float scale, int src_dtype, void* stream);

/* ---- K1+K2 fused for d == 1 (no collective between pack and update) ------
 * For every element of the bucket range [0, bucket_numel): g = bf16_rne(src*scale)
 * (0 where no entry covers it), (* *clip_coef), AdamW on master/exp_avg/exp_avg_sq
 * (bucket-indexed, bucket_numel elements each) and param = bf16_rne(master).
 * Bit-identical to hod_pack_bf16 followed by hod_adamw_bf16 on the bucket;
 * 28 B/element instead of 32. */
int hod_pack_adamw(const hod_pack_entry* entries, int n_entries, int64_t bucket_numel,
                   float scale, int src_dtype, float* master, float* exp_avg,
                   float* exp_avg_sq, uint16_t* param, const hod_adamw_params* hp,
                   const float* clip_coef, void* stream);

/* Sum of squares of the values the packed bucket would hold (bf16_rne(src*scale),
 * 0 in gaps), read straight from the tensors: HOD_SUMSQ_PARTIALS fixed-grid
 * partials (longer tables are split into windows of HOD_PACK_MAX_ENTRIES whose
 * sums are added per partial slot in window order).  d == 1 with clipping:
 * norm pass (2 B/element) then hod_pack_adamw with the clip coefficient. */
int hod_pack_sumsq(const hod_pack_entry* entries, int n_entries, int64_t bucket_numel,
                   float scale, int src_dtype, float* partials, void* stream);

/* ---- K3: deterministic sum of squares of a bf16 shard -----
 * Writes HOD_SUMSQ_PARTIALS fp32 partial sums to partials[0..HOD_SUMSQ_PARTIALS)
 * (fixed grid, fixed order => bit-reproducible for a given n). */
int hod_sumsq_bf16(const uint16_t* x, int64_t n, float* partials, void* stream);

/* Sums `n_partials` fp32 partials in fixed order (fp64 accumulator) and writes
 * the fp32 result to *out. */
int hod_sum_partials(const float* partials, int64_t n_partials, float* out,
                     void* stream);

/* coef = min(1, max_norm / (sqrt(*sumsq) + 1e-6)); *norm = sqrt(*sumsq).
 * torch.nn.utils.clip_grad_norm_ convention. */
int hod_clip_coef(const float* sumsq, float max_norm, float* coef, float* norm,
                  void* stream);

/* ---- K2: fused sharded AdamW ------------------------------
 * For i in [0,n): g = float(grad[i]) (* *clip_coef if clip_coef != NULL);
 * master/m/v updated in place; param[i] = bf16_rne(master[i]).
 * 28 bytes of HBM traffic per element.  clip_coef is a DEVICE pointer. */
int hod_adamw_bf16(float* master, float* exp_avg, float* exp_avg_sq,
                   const uint16_t* grad, uint16_t* param, int64_t n,
                   const hod_adamw_params* hp, const float* clip_coef, void* stream);

/* The SURVEY §8b scalar-argument spelling of K2 (same kernel, same bits as
 * hod_adamw_bf16 with hp = {lr, beta1, beta2, eps, weight_decay, step}). */
int hod_adamw(float* master, float* exp_avg, float* exp_avg_sq, const uint16_t* grad,
              uint16_t* param, int64_t n, float lr, float beta1, float beta2, float eps,
              float weight_decay, int64_t step, const float* clip_coef, void* stream);

/* The SURVEY §8b accumulating spelling of K3: *out += sum(x^2) (fp32 result of
 * the fixed-grid partials summed in fixed order, so bit-reproducible).  Uses a
 * per-device scratch array inside the library: calls on two streams of one
 * device must not run concurrently (use hod_sumsq_bf16 + caller partials then). */
int hod_sumsq(const uint16_t* x, int64_t n, float* out, void* stream);

/* Same update reading an fp32 gradient (fp32 reduce-scatter parity mode). */
int hod_adamw_f32(float* master, float* exp_avg, float* exp_avg_sq,
                  const float* grad, uint16_t* param, int64_t n,
                  const hod_adamw_params* hp, const float* clip_coef, void* stream);

/* ---- C1-C3: NCCL collectives over NVLink (§8e) ---------
 * Communicators are built from GroupPlan DP rows (groups.py:137-148), ranks
 * converted 1-based -> 0-based by the host. */
int hod_nccl_unique_id(uint8_t out[128]);
int hod_nccl_comm_init(const uint8_t id[128], int nranks, int rank, void** comm);
int hod_comm_destroy(void* comm);
/* HOD_OK, or HOD_ENCCL with the communicator's asynchronous error (a peer
 * failure, a network error) in hod_last_error(): ncclCommGetAsyncError,
 * polled by the host between steps without synchronising. */
int hod_comm_async_error(void* comm);
/* sum-reduce-scatter: recv (recvcount bf16) = sum over ranks of
 * send[rank*recvcount .. (rank+1)*recvcount).  In-place allowed when
 * recv == send + rank*recvcount. (prices: simulator.py:81-84) */
int hod_reduce_scatter_bf16(const void* send, void* recv, size_t recvcount, void* comm,
                            void* stream);
/* all-gather: recv[r*sendcount ..] = rank r's send.  In-place allowed when
 * send == recv + rank*sendcount. (prices: simulator.py:86-89) */
int hod_all_gather_bf16(const void* send, void* recv, size_t sendcount, void* comm,
                        void* stream);
int hod_all_reduce_f32(float* buf, size_t n, void* comm, void* stream);

/* ---- Fused collectives over NVLink peer memory (the B200-native path) ------
 * The DP row's gradient-bucket and param buffers are symmetric allocations:
 * every rank maps every peer's buffer (p2p) and an NVLS multicast range
 * (nvls).  Per bucket one kernel does cross-GPU arrival barrier +
 * reduce-scatter + AdamW + all-gather (HOD_P2P_FUSED); with clipping the RS
 * half (HOD_P2P_RS, writes reduced_out + sum-of-squares partials) and the
 * update half (HOD_P2P_ADAMW_AG, reads reduced_out, scales by *clip_coef) run
 * on either side of hod_p2p_norm.  Replaces what the reference prices as
 * reduce_scatter + all_gather (simulator.py:81-89, 327-333) and places after
 * the flush (simulator.py:445-452), overlapped per bucket instead.
 * p2p: fp32 rank-order sum, one bf16 rounding (bit-exact vs the oracle).
 * nvls: multimem.ld_reduce.add.acc::f32 + multimem.st (switch-side reduce and
 * replicate; one bf16 rounding, switch summation order). */
#define HOD_P2P_MAX_RANKS 8
#define HOD_P2P_FUSED 0
#define HOD_P2P_RS 1
#define HOD_P2P_ADAMW_AG 2

#define HOD_P2P_MAX_SPAN 32

/* A span of consecutive buckets (1..HOD_P2P_MAX_SPAN) handled by one launch. */
typedef struct hod_p2p_span {
  uint16_t* grad[HOD_P2P_MAX_RANKS];  /* rank q's flat grad-bucket buffer; nvls: [0] = multicast base */
  uint16_t* param[HOD_P2P_MAX_RANKS]; /* rank q's flat param buffer; nvls: [0] = multicast base */
  uint64_t* flags[HOD_P2P_MAX_RANKS]; /* rank q's flag array: [slot][HOD_P2P_MAX_RANKS] u64,
                                         value = epoch << 32 | tag */
  uint16_t* local_grad;   /* this rank's flat grad buffer: the reduced bf16 shard of bucket k is
                             kept in place at bucket_start[k] + rank*shard_numel[k] (RS: out,
                             ADAMW_AG: in, FUSED: only when keep_reduced) */
  float* master;          /* this rank's state for the span's shards, back to back */
  float* exp_avg;
  float* exp_avg_sq;
  float* partials;        /* RS: HOD_SUMSQ_PARTIALS sums of squares for the span (optional) */
  const float* clip_coef; /* ADAMW_AG: device clip coefficient (optional) */
  uint32_t* err;          /* device error word (HOD_ETIMEOUT on a barrier timeout) */
  int64_t bucket_start[HOD_P2P_MAX_SPAN]; /* element offset of bucket k in the flat buffers */
  int64_t shard_numel[HOD_P2P_MAX_SPAN];  /* bucket k's numel / d (multiple of 8) */
  int n_buckets;
  int d;
  int rank;
  int nvls;
  int keep_reduced;
  int slot;               /* barrier slot (index of the span's first bucket) */
  uint32_t epoch;         /* monotonically increasing per step, > 0 */
  uint32_t tag;           /* span identity checked at the barrier (HOD_SPAN_TAG(first, last)):
                             a peer arriving at `slot` with the same epoch and another tag
                             records HOD_ESPAN in *err and the launch skips its work */
  unsigned long long timeout_ns; /* barrier spin budget (0 = 20 s) */
} hod_p2p_span;

#define HOD_SPAN_TAG(first, last) ((uint32_t)(first) | ((uint32_t)(last) << 16))
#define HOD_NORM_TAG 0x4e4f524du /* tag of the norm-exchange barrier */

/* p2p launches with the whole GPU run the TMA-fed kernel (cp.async.bulk peer
 * reads / peer writes through a shared-memory ring, one CTA per SM); under a
 * co-resident grid cap (hod_set_grid_limit <= 148) the register-streaming
 * kernel, which fits beside a GEMM CTA.  Same results, bit for bit (RS
 * partial sums: same value within fp32 summation order).  hod_set_span_tma
 * (initial value: env HOD_SPAN_TMA): 0 = never, 1 = default, 2 = also under
 * a cap.
 * Errors inside a launch go to the device word *err (HOD_ETIMEOUT, HOD_ESPAN).
 * Fail-stop: once *err is nonzero every later barrier, span and update launch
 * of this rank returns at entry without signalling its peers (which then time
 * out in turn); the host reads the word and raises. */
int hod_p2p_step(const hod_p2p_span* span, int mode, const hod_adamw_params* hp, void* stream);
int hod_set_span_tma(int mode);

/* stand-alone cross-GPU barrier on `slot` (1 CTA): signal (epoch, tag) then wait
 * for all d ranks; a different tag at the same epoch records HOD_ESPAN */
int hod_p2p_barrier(uint64_t* const* flags, int d, int rank, int slot, uint32_t epoch, uint32_t tag,
                    unsigned long long timeout_ns, uint32_t* err, void* stream);

/* One-directional hand-off between two GPUs (pipeline activations, §8f.3):
 * hod_p2p_signal stores `epoch` into a peer-mapped flag once all prior work of
 * `stream` is complete (system fence); hod_p2p_wait makes `stream` wait (1
 * thread, bounded spin, HOD_ETIMEOUT into *err) until the local flag >= epoch. */
int hod_p2p_signal(uint32_t* peer_flag, uint32_t epoch, void* stream);
int hod_p2p_wait(const uint32_t* flag, uint32_t epoch, unsigned long long timeout_ns, uint32_t* err,
                 void* stream);

/* global norm over d ranks through peer memory: fixed-order sum of this rank's
 * partials, publish to xchg[q][rank] (fp64) of every rank, barrier, rank-order
 * sum => identical deterministic coef/norm on all ranks. */
int hod_p2p_norm(const float* partials, int64_t n_partials, double* const* xchg,
                 uint64_t* const* flags, int d, int rank, int slot, uint32_t epoch,
                 unsigned long long timeout_ns, uint32_t* err, float max_norm, float* coef,
                 float* norm, float* sumsq, void* stream);

/* ---- copy-engine transfer (peer-mapped addresses, no SMs used) ---------- */
int hod_ce_copy(void* dst, const void* src, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HOD_H_ */
