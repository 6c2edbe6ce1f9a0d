// hod_p2p.cu — the B200-native collectives of the optimizer step, fused with
// the update, over NVLink 5 / NVSwitch peer memory.
//
// The gradient-bucket buffer and the param buffer of every rank of a DP row
// are symmetric allocations (one virtual range per rank, mapped into every
// peer; plus an NVLS multicast range).  A launch covers a SPAN of consecutive
// buckets (1 .. HOD_P2P_MAX_SPAN): per-bucket launches while backward is still
// producing buckets, coalesced spans when many buckets are ready at once
// (fewer barriers and launch tails, longer NVLink streams).
//
//   FUSED (no clip): ONE kernel per span —
//       cross-GPU arrival barrier (peer flag stores, acquire spin);
//       reduce-scatter: rank r sums shard r of every bucket of every peer
//         p2p : d 16-byte P2P loads, fp32 sum in rank order 0..d-1, one RNE
//               rounding to bf16  -> bit-exact with oracle_rs_sum;
//         nvls: one multimem.ld_reduce.add.acc::f32 per 8 elements (the
//               switch reduces: ingress per GPU drops from 2P(d-1)/d to 2P/d);
//       AdamW on the fp32 master/m/v shard (local HBM, 24 B/elem);
//       all-gather: the bf16 param vector is stored to every peer's param
//         buffer (p2p: d stores) or once to the multicast range (nvls:
//         multimem.st, the switch replicates).
//   RS (+sum-of-squares partials) / ADAMW_AG (clip): the two halves as two
//       kernels with the global norm exchanged over peer memory in between;
//       the reduced bf16 shard lives in place in the own-shard region of the
//       local grad buffer (only this rank ever reads that region).
//
// Barriers are monotonic epoch flags: rank r writes `epoch` into slot
// [slot][r] of every peer's flag array (st.release.sys) and waits until its own
// [slot][q] >= epoch for all q (ld.acquire.sys).  Every CTA signals (idempotent
// store), so progress never depends on which CTAs are resident.  Spins are
// bounded by a %globaltimer budget; on timeout the kernel records HOD_ETIMEOUT
// in the caller's device error word and skips its work instead of hanging.
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "hod_common.cuh"

namespace hod {

constexpr int kMaxRanks = HOD_P2P_MAX_RANKS;
constexpr int kMaxSpan = HOD_P2P_MAX_SPAN;

struct PeerTable {
  uintptr_t p[kMaxRanks];
};

struct BarrierArgs {
  PeerTable flags;          // flags[q] = base of rank q's flag array (device ptrs)
  uint32_t* local_flags;    // this rank's flag array
  uint32_t* err;            // device error word (nullable)
  int slot;
  uint32_t epoch;
  unsigned long long timeout_ns;
};

struct SpanArgs {
  PeerTable grad;           // p2p: rank q's flat grad buffer; nvls: grad[0] = multicast base
  PeerTable param;          // same for the param buffer
  uint16_t* local_grad;     // this rank's flat grad buffer (in-place reduced shards)
  float* master;            // state of the span's first shard (shards are back to back)
  float* m;
  float* v;
  float* partials;          // optional: HOD_SUMSQ_PARTIALS per-CTA sums of squares
  const float* coef;        // optional clip coefficient (device)
  int64_t own_off[kMaxSpan];     // element offset of this rank's shard of bucket k
  int64_t item_end[kMaxSpan];    // prefix (inclusive) of shard items (8 elements) over the span
  int n_buckets;
  int d;
  int keep_reduced;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Signal arrival at `slot` to every rank and wait for all of them.  Returns
// false (and records the error) on timeout.  Must be called by all threads.
__device__ bool cross_gpu_barrier(const BarrierArgs& b, int d, int rank) {
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < d) {
    const int q = threadIdx.x;
    uint32_t* peer = reinterpret_cast<uint32_t*>(b.flags.p[q]) + b.slot * kMaxRanks + rank;
    st_release_sys(peer, b.epoch);
    const uint32_t* mine = b.local_flags + b.slot * kMaxRanks + q;
    const unsigned long long t0 = globaltimer();
    while (static_cast<int32_t>(ld_acquire_sys(mine) - b.epoch) < 0) {
      if (globaltimer() - t0 > b.timeout_ns) {
        atomicExch(&timed_out, 1);
        if (b.err) atomicExch(b.err, static_cast<uint32_t>(HOD_ETIMEOUT));
        break;
      }
      __nanosleep(100);
    }
  }
  __syncthreads();
  return timed_out == 0;
}

__device__ __forceinline__ uint4 ld_reduce_bf16x8(const uint16_t* mc) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}

__device__ __forceinline__ void st_multicast16(uint16_t* mc, const uint4& q) {
  // .v4 multimem stores take a float vector; the 16 bytes are moved bit-for-bit
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc),
               "f"(__uint_as_float(q.x)), "f"(__uint_as_float(q.y)), "f"(__uint_as_float(q.z)),
               "f"(__uint_as_float(q.w))
               : "memory");
}

__device__ __forceinline__ float block_sum_f(float x) {
  __shared__ float part[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = x;
  __syncthreads();
  float s = 0.0f;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += part[w];
  return s;
}

// One thread's 8-element work item, split into a load phase and a compute /
// store phase so that U items can have all their loads in flight at once.
template <int D, bool kNVLS>
struct Item {
  static constexpr int kRaw = kNVLS ? 1 : (D > 0 ? D : kMaxRanks);
  uint4 raw[kRaw];     // peers' bucket vectors (p2p), the switch-reduced vector (nvls),
                       // or the local reduced shard (mode 2, raw[0])
  float4 st[6];        // master, m, v (two float4 each)
  int64_t e;           // element offset in the flat buffers
  int64_t s;           // element offset in the span's state
};

// Map a span item index to (flat element offset, state offset); `k` is the
// caller's monotonically advancing bucket cursor.
__device__ __forceinline__ void locate(const SpanArgs& a, int64_t iv, int& k, int64_t& e, int64_t& s) {
  while (k < a.n_buckets - 1 && iv >= a.item_end[k]) ++k;
  const int64_t first = k ? a.item_end[k - 1] : 0;
  e = a.own_off[k] + (iv - first) * 8;
  s = iv * 8;
}

template <int D, bool kNVLS, int kMode>
__device__ __forceinline__ void load_item(const SpanArgs& a, Item<D, kNVLS>& it) {
  const int64_t e = it.e;
  if (kMode == 2) {
    it.raw[0] = *reinterpret_cast<const uint4*>(a.local_grad + e);
  } else if constexpr (kNVLS) {
    it.raw[0] = ld_reduce_bf16x8(reinterpret_cast<const uint16_t*>(a.grad.p[0]) + e);
  } else {
    const int dd = D > 0 ? D : a.d;
#pragma unroll
    for (int q = 0; q < Item<D, kNVLS>::kRaw; ++q)
      if (q < dd) it.raw[q] = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.grad.p[q]) + e);
  }
  if (kMode != 1) {
    const float4* p4 = reinterpret_cast<const float4*>(a.master + it.s);
    const float4* m4 = reinterpret_cast<const float4*>(a.m + it.s);
    const float4* v4 = reinterpret_cast<const float4*>(a.v + it.s);
    it.st[0] = p4[0]; it.st[1] = p4[1];
    it.st[2] = m4[0]; it.st[3] = m4[1];
    it.st[4] = v4[0]; it.st[5] = v4[1];
  }
}

template <int D, bool kNVLS>
__device__ __forceinline__ void gather_store8(const SpanArgs& a, int64_t e, const uint4& q8) {
  if constexpr (kNVLS) {
    st_multicast16(reinterpret_cast<uint16_t*>(a.param.p[0]) + e, q8);
  } else {
    const int dd = D > 0 ? D : a.d;
#pragma unroll
    for (int q = 0; q < (D > 0 ? D : kMaxRanks); ++q)
      if (q < dd) *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.param.p[q]) + e) = q8;
  }
}

template <int D, bool kNVLS, int kMode>
__device__ __forceinline__ void finish_item(const SpanArgs& a, const Item<D, kNVLS>& it,
                                            const AdamWConsts& c, float coef, float& ss) {
  float g[8];
  if (kMode == 2 || kNVLS) {
    unpack8(it.raw[0], g);
  } else {
    const int dd = D > 0 ? D : a.d;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
#pragma unroll
    for (int q = 0; q < Item<D, kNVLS>::kRaw; ++q) {
      if (q < dd) {
        float f[8];
        unpack8(it.raw[q], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = __fadd_rn(acc[k], f[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k] = bf16_to_f32(f32_to_bf16(acc[k]));
  }
  if (kMode != 2) {
    if (kMode == 1 || a.keep_reduced) *reinterpret_cast<uint4*>(a.local_grad + it.e) = pack8(g);
    if (kMode == 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) ss = __fadd_rn(ss, __fmul_rn(g[k], g[k]));
      return;
    }
  }
  float pf[8] = {it.st[0].x, it.st[0].y, it.st[0].z, it.st[0].w, it.st[1].x, it.st[1].y, it.st[1].z, it.st[1].w};
  float mf[8] = {it.st[2].x, it.st[2].y, it.st[2].z, it.st[2].w, it.st[3].x, it.st[3].y, it.st[3].z, it.st[3].w};
  float vf[8] = {it.st[4].x, it.st[4].y, it.st[4].z, it.st[4].w, it.st[5].x, it.st[5].y, it.st[5].z, it.st[5].w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float gk = (kMode == 2 && a.coef) ? __fmul_rn(g[k], coef) : g[k];
    adamw_elem(pf[k], mf[k], vf[k], gk, c);
  }
  float4* p4 = reinterpret_cast<float4*>(a.master + it.s);
  float4* m4 = reinterpret_cast<float4*>(a.m + it.s);
  float4* v4 = reinterpret_cast<float4*>(a.v + it.s);
  p4[0] = make_float4(pf[0], pf[1], pf[2], pf[3]);
  p4[1] = make_float4(pf[4], pf[5], pf[6], pf[7]);
  m4[0] = make_float4(mf[0], mf[1], mf[2], mf[3]);
  m4[1] = make_float4(mf[4], mf[5], mf[6], mf[7]);
  v4[0] = make_float4(vf[0], vf[1], vf[2], vf[3]);
  v4[1] = make_float4(vf[4], vf[5], vf[6], vf[7]);
  gather_store8<D, kNVLS>(a, it.e, pack8(pf));
}

// kMode: 0 = fused RS+AdamW+AG, 1 = RS only (+in-place reduced shard, partials),
// 2 = AdamW+AG from the in-place reduced shard.  U: items per thread in flight
// (memory-level parallelism for the NVLink loads).
template <int D, bool kNVLS, int kMode, int U>
__global__ void __launch_bounds__(kThreads) p2p_step_kernel(const __grid_constant__ SpanArgs a,
                                                             const BarrierArgs b, const AdamWConsts c,
                                                             int rank) {
  if (kMode != 2) {
    if (!cross_gpu_barrier(b, a.d, rank)) return;
  }
  const float coef = (kMode == 2 && a.coef) ? __ldg(a.coef) : 1.0f;
  const int64_t n_items = a.item_end[a.n_buckets - 1];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  float ss = 0.0f;
  int cur[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cur[u] = 0;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; base < n_items;
       base += stride * U) {
    Item<D, kNVLS> it[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t iv = base + u * stride;
      if (iv < n_items) {
        locate(a, iv, cur[u], it[u].e, it[u].s);
        load_item<D, kNVLS, kMode>(a, it[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * stride < n_items) finish_item<D, kNVLS, kMode>(a, it[u], c, coef, ss);
  }
  if (kMode == 1 && a.partials) {
    const float s = block_sum_f(ss);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = s;
    if (blockIdx.x == 0)
      for (int i = gridDim.x + threadIdx.x; i < HOD_SUMSQ_PARTIALS; i += blockDim.x) a.partials[i] = 0.0f;
  }
  if (kMode != 1) __threadfence_system();  // remote param stores performed before any later signal
}

__global__ void barrier_kernel(const BarrierArgs b, int d, int rank) {
  __threadfence_system();
  cross_gpu_barrier(b, d, rank);
}

// Global-norm exchange: one warp sums this rank's partials (lane-strided fp64,
// fixed shuffle tree => deterministic), publishes the value into slot `rank`
// of every peer's exchange array, then (after the barrier) sums all d slots in
// rank order -> identical, deterministic norm on every rank.
__global__ void norm_exchange_kernel(const float* partials, int64_t n_partials, PeerTable xchg,
                                     double* local_xchg, const BarrierArgs b, int d, int rank,
                                     float max_norm, float* coef, float* norm, float* sumsq_out) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n_partials; i += 32) s += static_cast<double>(partials[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x < d) {
    double* dst = reinterpret_cast<double*>(xchg.p[threadIdx.x]) + rank;
    *reinterpret_cast<volatile double*>(dst) = s;
  }
  __threadfence_system();
  __syncwarp();
  if (!cross_gpu_barrier(b, d, rank)) return;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < d; ++q) t += *reinterpret_cast<volatile double*>(local_xchg + q);
    const float s32 = static_cast<float>(t);
    const float nrm = __fsqrt_rn(s32);
    const float cf = __fdiv_rn(max_norm, __fadd_rn(nrm, 1e-6f));
    *coef = cf < 1.0f ? cf : 1.0f;
    if (norm) *norm = nrm;
    if (sumsq_out) *sumsq_out = s32;
  }
}

static int unroll_setting() {
  static int u = [] {
    const char* e = getenv("HOD_P2P_UNROLL");
    return e ? atoi(e) : 0;  // 0 = auto
  }();
  return u;
}

template <int D, bool kNVLS, int kMode>
static void launch_step(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank,
                        int grid, cudaStream_t s) {
  count_launch(1);
  // measured (tools/p2p_microbench.py): two items in flight per thread pay off
  // at d = 2 (one remote load each); at d >= 4 the register cost outweighs it
  const int u = unroll_setting();
  if (u >= 2 || (u == 0 && D == 2))
    p2p_step_kernel<D, kNVLS, kMode, 2><<<grid, kThreads, 0, s>>>(a, b, c, rank);
  else
    p2p_step_kernel<D, kNVLS, kMode, 1><<<grid, kThreads, 0, s>>>(a, b, c, rank);
}

template <bool kNVLS, int kMode>
static void dispatch_d(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank,
                       int grid, cudaStream_t s) {
  switch (kNVLS ? 0 : a.d) {
    case 2: launch_step<2, kNVLS, kMode>(a, b, c, rank, grid, s); break;
    case 4: launch_step<4, kNVLS, kMode>(a, b, c, rank, grid, s); break;
    case 8: launch_step<8, kNVLS, kMode>(a, b, c, rank, grid, s); break;
    default: launch_step<0, kNVLS, kMode>(a, b, c, rank, grid, s); break;
  }
}

static int fill_barrier(uint32_t* const* flags, int d, int rank, int slot, uint32_t epoch,
                        unsigned long long timeout_ns, uint32_t* err, BarrierArgs* b) {
  memset(b, 0, sizeof(*b));
  for (int q = 0; q < d; ++q) {
    b->flags.p[q] = reinterpret_cast<uintptr_t>(flags[q]);
    if (!b->flags.p[q]) { set_error("hod_p2p: null flag array %d", q); return HOD_EINVAL; }
  }
  b->local_flags = flags[rank];
  b->err = err;
  b->slot = slot;
  b->epoch = epoch;
  b->timeout_ns = timeout_ns ? timeout_ns : 20000000000ull;
  return HOD_OK;
}

static int fill_span(const hod_p2p_span* sp, SpanArgs* a, BarrierArgs* b) {
  if (!sp || sp->d < 1 || sp->d > kMaxRanks || sp->rank < 0 || sp->rank >= sp->d) {
    set_error("hod_p2p: bad group (d=%d rank=%d)", sp ? sp->d : -1, sp ? sp->rank : -1);
    return HOD_EINVAL;
  }
  if (sp->n_buckets < 1 || sp->n_buckets > kMaxSpan) {
    set_error("hod_p2p: span of %d buckets (1..%d)", sp->n_buckets, kMaxSpan);
    return HOD_EINVAL;
  }
  memset(a, 0, sizeof(*a));
  const int nptr = sp->nvls ? 1 : sp->d;
  for (int q = 0; q < nptr; ++q) {
    a->grad.p[q] = reinterpret_cast<uintptr_t>(sp->grad[q]);
    a->param.p[q] = reinterpret_cast<uintptr_t>(sp->param[q]);
    if (!a->grad.p[q] || !a->param.p[q] || (a->grad.p[q] & 15) || (a->param.p[q] & 15)) {
      set_error("hod_p2p: peer buffer %d null or not 16-byte aligned", q);
      return HOD_EALIGN;
    }
  }
  a->local_grad = sp->local_grad;
  if (!a->local_grad || (reinterpret_cast<uintptr_t>(a->local_grad) & 15)) {
    set_error("hod_p2p: local grad buffer null or misaligned"); return HOD_EALIGN;
  }
  int64_t items = 0;
  for (int k = 0; k < sp->n_buckets; ++k) {
    const int64_t n = sp->shard_numel[k];
    if (n < 8 || (n & 7) || sp->bucket_start[k] < 0 || (sp->bucket_start[k] & 7)) {
      set_error("hod_p2p: bucket %d: shard size/offset must be positive multiples of 8", k);
      return HOD_EALIGN;
    }
    a->own_off[k] = sp->bucket_start[k] + static_cast<int64_t>(sp->rank) * n;
    items += n / 8;
    a->item_end[k] = items;
  }
  a->master = sp->master;
  a->m = sp->exp_avg;
  a->v = sp->exp_avg_sq;
  a->partials = sp->partials;
  a->coef = sp->clip_coef;
  a->n_buckets = sp->n_buckets;
  a->d = sp->d;
  a->keep_reduced = sp->keep_reduced;
  return fill_barrier(sp->flags, sp->d, sp->rank, sp->slot, sp->epoch, sp->timeout_ns, sp->err, b);
}

}  // namespace hod

using namespace hod;

extern "C" {

int hod_p2p_step(const hod_p2p_span* sp, int mode, const hod_adamw_params* hp, void* stream) {
  SpanArgs a;
  BarrierArgs b;
  int rc = fill_span(sp, &a, &b);
  if (rc) return rc;
  if (mode < HOD_P2P_FUSED || mode > HOD_P2P_ADAMW_AG) { set_error("hod_p2p_step: bad mode %d", mode); return HOD_EINVAL; }
  if (mode != HOD_P2P_RS && (!hp || hp->step < 1)) { set_error("hod_p2p_step: bad hp/step"); return HOD_EINVAL; }
  if (mode != HOD_P2P_RS && (!a.master || !a.m || !a.v)) { set_error("hod_p2p_step: null state"); return HOD_EINVAL; }
  const AdamWConsts c = (mode != HOD_P2P_RS) ? fold_adamw(*hp) : AdamWConsts{};
  const int64_t items = a.item_end[a.n_buckets - 1];
  // RS keeps a FIXED grid so its sum-of-squares partials are reproducible
  const int grid = (mode == HOD_P2P_RS) ? partials_grid() : grid_for(items, kThreads, 4);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool nv = sp->nvls != 0;
  if (mode == HOD_P2P_FUSED) {
    if (nv) dispatch_d<true, 0>(a, b, c, sp->rank, grid, s); else dispatch_d<false, 0>(a, b, c, sp->rank, grid, s);
  } else if (mode == HOD_P2P_RS) {
    if (nv) dispatch_d<true, 1>(a, b, c, sp->rank, grid, s); else dispatch_d<false, 1>(a, b, c, sp->rank, grid, s);
  } else {
    if (nv) dispatch_d<true, 2>(a, b, c, sp->rank, grid, s); else dispatch_d<false, 2>(a, b, c, sp->rank, grid, s);
  }
  return cuda_status(cudaGetLastError(), "hod_p2p_step launch");
}

int hod_p2p_barrier(uint32_t* const* flags, int d, int rank, int slot, uint32_t epoch,
                    unsigned long long timeout_ns, uint32_t* err, void* stream) {
  if (!flags || d < 1 || d > kMaxRanks || rank < 0 || rank >= d || slot < 0) {
    set_error("hod_p2p_barrier: bad arguments"); return HOD_EINVAL;
  }
  BarrierArgs b;
  int rc = fill_barrier(flags, d, rank, slot, epoch, timeout_ns, err, &b);
  if (rc) return rc;
  count_launch(1);
  barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(b, d, rank);
  return cuda_status(cudaGetLastError(), "hod_p2p_barrier launch");
}

int hod_p2p_norm(const float* partials, int64_t n_partials, double* const* xchg, uint32_t* const* flags,
                 int d, int rank, int slot, uint32_t epoch, unsigned long long timeout_ns, uint32_t* err,
                 float max_norm, float* coef, float* norm, float* sumsq, void* stream) {
  if (!partials || !xchg || !flags || !coef || d < 1 || d > kMaxRanks || rank < 0 || rank >= d ||
      !(max_norm > 0.0f)) {
    set_error("hod_p2p_norm: bad arguments"); return HOD_EINVAL;
  }
  PeerTable x;
  memset(&x, 0, sizeof(x));
  for (int q = 0; q < d; ++q) x.p[q] = reinterpret_cast<uintptr_t>(xchg[q]);
  BarrierArgs b;
  int rc = fill_barrier(flags, d, rank, slot, epoch, timeout_ns, err, &b);
  if (rc) return rc;
  count_launch(1);
  norm_exchange_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      partials, n_partials, x, xchg[rank], b, d, rank, max_norm, coef, norm, sumsq);
  return cuda_status(cudaGetLastError(), "hod_p2p_norm launch");
}

}  // extern "C"
