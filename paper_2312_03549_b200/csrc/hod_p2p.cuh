// hod_p2p.cuh — pieces shared by the fused span kernels (hod_p2p.cu: the
// register-streaming kernel, p2p and NVLS; hod_span_tma.cu: the TMA-fed p2p
// kernel): peer tables, span/barrier arguments, the cross-GPU epoch barrier.
#pragma once

#include <stdint.h>

#include "hod_common.cuh"

namespace hod {

constexpr int kMaxRanks = HOD_P2P_MAX_RANKS;
constexpr int kMaxSpan = HOD_P2P_MAX_SPAN;
#ifndef HOD_P2P_MINB
#define HOD_P2P_MINB 1
#endif

struct PeerTable {
  uintptr_t p[kMaxRanks];
};

// Where the reduce-scatter reads the d contributions of an owned element:
enum : int {
  kSrcPeer = 0,    // pull from the d peers' packed buckets (p2p)
  kSrcNvls = 1,    // one multimem.ld_reduce through the switch (nvls; AG via multimem.st)
};

struct BarrierArgs {
  PeerTable flags;          // flags[q] = base of rank q's 64-bit flag array (device ptrs)
  uint64_t* local_flags;    // this rank's flag array
  uint32_t* err;            // device error word (nullable)
  int slot;
  uint32_t epoch;
  uint32_t tag;             // what the slot synchronises (must agree across ranks)
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
  int64_t elem_end[kMaxSpan];    // prefix (inclusive) of shard elements over the span
  int64_t chunk_end[kMaxSpan];   // prefix (inclusive) of 256-element chunks per bucket shard
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

__device__ __forceinline__ void st_release_sys64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Nonzero once any kernel of this rank recorded an error (fail-stop check at
// kernel entry; one load per CTA).
__device__ __forceinline__ bool rank_failed(const uint32_t* err) {
  return err && *reinterpret_cast<const volatile uint32_t*>(err) != 0u;
}

// Signal arrival at `slot` to every rank and wait for all of them.  Returns
// false (and records the error) on timeout or tag mismatch, and at once —
// without signalling — if the rank already failed.  Called by all threads.
static __device__ bool cross_gpu_barrier(const BarrierArgs& b, int d, int rank) {
  __shared__ int failed;
  if (threadIdx.x == 0) failed = rank_failed(b.err) ? 1 : 0;
  __syncthreads();
  if (failed) return false;
  if (threadIdx.x < d) {
    const int q = threadIdx.x;
    uint64_t* peer = reinterpret_cast<uint64_t*>(b.flags.p[q]) + b.slot * kMaxRanks + rank;
    st_release_sys64(peer, (static_cast<uint64_t>(b.epoch) << 32) | b.tag);
    const uint64_t* mine = b.local_flags + b.slot * kMaxRanks + q;
    const unsigned long long t0 = globaltimer();
    uint64_t v;
    while (static_cast<int32_t>(static_cast<uint32_t>((v = ld_acquire_sys64(mine)) >> 32) - b.epoch) < 0) {
      if (globaltimer() - t0 > b.timeout_ns) {
        atomicExch(&failed, 1);
        if (b.err) atomicExch(b.err, static_cast<uint32_t>(HOD_ETIMEOUT));
        break;
      }
      __nanosleep(100);
    }
    if (!failed && static_cast<uint32_t>(v >> 32) == b.epoch && static_cast<uint32_t>(v) != b.tag) {
      atomicExch(&failed, 1);
      if (b.err) atomicExch(b.err, static_cast<uint32_t>(HOD_ESPAN));
    }
  }
  __syncthreads();
  return failed == 0;
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

__device__ __forceinline__ uint2 ld_reduce_bf16x4(const uint16_t* mc) {
  uint2 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v2.bf16x2 {%0, %1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(mc)
               : "memory");
  return r;
}

__device__ __forceinline__ void st_multicast8(uint16_t* mc, const uint2& q) {
  asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(mc),
               "f"(__uint_as_float(q.x)), "f"(__uint_as_float(q.y))
               : "memory");
}

// TMA-fed p2p span kernel (hod_span_tma.cu): whether it takes this launch
// (HOD_SPAN_TMA, not under a co-resident grid cap by default), and the launch.
bool span_tma_applies();
int launch_span_tma(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank, int mode,
                    cudaStream_t s);

}  // namespace hod
