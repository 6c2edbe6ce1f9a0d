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
//         p2p : d 8-byte P2P loads per quad, fp32 sum in rank order 0..d-1, one
//               RNE rounding to bf16  -> bit-exact with oracle_rs_sum;
//         nvls: one multimem.ld_reduce.add.acc::f32 per 4 elements (the
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
// Barriers are monotonic epoch flags: rank r writes (epoch << 32 | tag) into
// slot [slot][r] of every peer's 64-bit flag array (st.release.sys) and waits
// until its own [slot][q] carries an epoch >= `epoch` for all q
// (ld.acquire.sys).  The tag names what the slot synchronises (a span's first
// and last bucket): a peer that arrives with the same epoch but another tag
// closed its span differently, which records HOD_ESPAN instead of reading a
// bucket the peer has not packed.  Every CTA signals (idempotent store), so
// progress never depends on which CTAs are resident.  Spins are bounded by a
// %globaltimer budget; on timeout the kernel records HOD_ETIMEOUT in the
// caller's device error word and skips its work instead of hanging.  Once the
// error word is set, every later barrier / update of the rank skips at entry
// without signalling (fail-stop: peers time out in turn, no rank proceeds on
// a half-finished step; the host surfaces the word as DeviceError).
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "hod_p2p.cuh"

namespace hod {

// One thread's work item: the two quads (4 elements each) it owns in a
// 256-element warp chunk of the span (lane*4 and 128 + lane*4, see kChunk in
// hod_common.cuh), so every warp-wide access is a fully used contiguous span.
// Quads never straddle buckets (shards are multiples of 16 elements); each
// quad is located on its own.  Split into a load phase and a compute/store
// phase so U items can have all their loads in flight at once.
template <int D, int kSrc, int W = 0>
struct Item {
  static constexpr int kRaw = kSrc == kSrcNvls ? 1 : (D > 0 ? D : kMaxRanks);
  // W (wide, p2p pull only): the peers' bucket vectors are pulled 16 bytes
  // per lane (8 contiguous elements, half the load instructions of two 8-byte
  // quads; measured d = 2 read+write ceiling 678 vs 641 GB/s), reduced, and
  // the reduced bf16 quads are shuffled to the quad-pair mapping of the state
  static constexpr bool kWide = W != 0 && kSrc == kSrcPeer;
  uint2 raw[2][kRaw];  // per quad: peers' bucket vectors (p2p), the switch-reduced
                       // vector (nvls) or the local reduced shard (mode 2, raw[h][0])
  uint4 raw8[kWide ? kRaw : 1];  // wide: the peers' 8-element vectors at e8
  int64_t e8;          // wide: element offset of this lane's 8 contiguous elements
  bool ok8;
  float4 st[2][3];     // per quad: master, m, v
  int64_t e[2];        // element offset in the flat buffers
  int64_t s[2];        // element offset in the span's state
  bool ok[2];
};

// Locate the two quads of this lane in warp chunk `ch`.  Chunks are counted
// per bucket shard (a chunk never straddles buckets), so the bucket lookup is
// warp-uniform and done once per chunk; `k` is the caller's monotonically
// advancing bucket cursor.  A quad past the shard end (last, partial chunk)
// is marked !ok (shards are multiples of 16, so quads are all-in or all-out).
template <typename ItemT>
__device__ __forceinline__ void locate_chunk(const SpanArgs& a, int64_t ch, int lane, int& k, ItemT& it) {
  if (ch >= a.chunk_end[a.n_buckets - 1]) {
    it.ok[0] = it.ok[1] = false;
    it.ok8 = false;
    return;
  }
  while (k < a.n_buckets - 1 && ch >= a.chunk_end[k]) ++k;
  const int64_t first_chunk = k ? a.chunk_end[k - 1] : 0;
  const int64_t first_elem = k ? a.elem_end[k - 1] : 0;
  const int64_t n = a.elem_end[k] - first_elem;
  const int64_t own = a.own_off[k];
  const int64_t base = (ch - first_chunk) * kChunk + lane * 4;
  it.e8 = own + (ch - first_chunk) * kChunk + lane * 8;
  it.ok8 = (ch - first_chunk) * kChunk + lane * 8 < n;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t off = base + h * 128;
    it.ok[h] = off < n;
    it.e[h] = own + off;
    it.s[h] = first_elem + off;
  }
}

template <int D, int kSrc, int kMode, int W>
__device__ __forceinline__ void load_item(const SpanArgs& a, Item<D, kSrc, W>& it, int rank) {
  using ItemT = Item<D, kSrc, W>;
  if constexpr (ItemT::kWide && kMode != 2) {
    if (it.ok8) {
      const int dd = D > 0 ? D : a.d;
#pragma unroll
      for (int q = 0; q < ItemT::kRaw; ++q)
        if (q < dd) it.raw8[q] = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.grad.p[q]) + it.e8);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!it.ok[h]) continue;
    const int64_t e = it.e[h];
    if (kMode == 2) {
      it.raw[h][0] = *reinterpret_cast<const uint2*>(a.local_grad + e);
    } else if constexpr (kSrc == kSrcNvls) {
      it.raw[h][0] = ld_reduce_bf16x4(reinterpret_cast<const uint16_t*>(a.grad.p[0]) + e);
    } else if constexpr (!ItemT::kWide) {
      const int dd = D > 0 ? D : a.d;
#pragma unroll
      for (int q = 0; q < ItemT::kRaw; ++q)
        if (q < dd) it.raw[h][q] = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(a.grad.p[q]) + e);
    }
    if (kMode != 1) {
      it.st[h][0] = *reinterpret_cast<const float4*>(a.master + it.s[h]);
      it.st[h][1] = *reinterpret_cast<const float4*>(a.m + it.s[h]);
      it.st[h][2] = *reinterpret_cast<const float4*>(a.v + it.s[h]);
    }
  }
}

template <int D, int kSrc>
__device__ __forceinline__ void gather_store4(const SpanArgs& a, int64_t e, const uint2& q4) {
  if constexpr (kSrc == kSrcNvls) {
    st_multicast8(reinterpret_cast<uint16_t*>(a.param.p[0]) + e, q4);
  } else {
    const int dd = D > 0 ? D : a.d;
#pragma unroll
    for (int q = 0; q < (D > 0 ? D : kMaxRanks); ++q)
      if (q < dd) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.param.p[q]) + e) = q4;
  }
}

template <int D, int kSrc, int kMode, int W, bool kFast>
__device__ __forceinline__ void finish_item(const SpanArgs& a, const Item<D, kSrc, W>& it,
                                            const AdamWConsts& c, float coef, float& ss) {
  using ItemT = Item<D, kSrc, W>;
  uint2 red[2];
  if constexpr (ItemT::kWide && kMode != 2) {
    // reduce this lane's 8 contiguous elements over the d peers (rank order,
    // fp32, one RNE rounding: the same per-element arithmetic as the quad
    // path), then lane l takes quad l from lane l/2 and quad 32+l from lane
    // 16+l/2 (half l&1 of the source's 8 elements).  Whole warp participates.
    uint4 r8 = make_uint4(0u, 0u, 0u, 0u);
    if (it.ok8) {
      const int dd = D > 0 ? D : a.d;
      float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int q = 0; q < ItemT::kRaw; ++q) {
        if (q < dd) {
          float f[8];
          unpack8(it.raw8[q], f);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] = __fadd_rn(acc[k], f[k]);
        }
      }
      r8 = pack8(acc);
    }
    const int lane = threadIdx.x & 31;
    const bool hi = lane & 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int src = h * 16 + (lane >> 1);
      const uint32_t x = __shfl_sync(0xffffffffu, r8.x, src), y = __shfl_sync(0xffffffffu, r8.y, src);
      const uint32_t z = __shfl_sync(0xffffffffu, r8.z, src), w = __shfl_sync(0xffffffffu, r8.w, src);
      red[h] = hi ? make_uint2(z, w) : make_uint2(x, y);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!it.ok[h]) continue;
    float g[4];
    if (kMode == 2 || kSrc == kSrcNvls) {
      unpack4(it.raw[h][0], g);
    } else if constexpr (ItemT::kWide) {
      unpack4(red[h], g);
    } else {
      const int dd = D > 0 ? D : a.d;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int q = 0; q < ItemT::kRaw; ++q) {
        if (q < dd) {
          float f[4];
          unpack4(it.raw[h][q], f);
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], f[k]);
        }
      }
      uint16_t r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        r[k] = f32_to_bf16(acc[k]);
        g[k] = bf16_to_f32(r[k]);
      }
      red[h] = make_uint2(r[0] | (static_cast<uint32_t>(r[1]) << 16), r[2] | (static_cast<uint32_t>(r[3]) << 16));
    }
    if (kMode != 2) {
      // red[h]: this quad's reduced bf16 bits (already rounded: no second pass)
      if (kMode == 1 || a.keep_reduced) *reinterpret_cast<uint2*>(a.local_grad + it.e[h]) =
          kSrc == kSrcNvls ? it.raw[h][0] : red[h];
      if (kMode == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) ss = __fadd_rn(ss, __fmul_rn(g[k], g[k]));
        continue;
      }
    }
    const float4 P = it.st[h][0], M = it.st[h][1], V = it.st[h][2];
    float pf[4] = {P.x, P.y, P.z, P.w};
    float mf[4] = {M.x, M.y, M.z, M.w};
    float vf[4] = {V.x, V.y, V.z, V.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gk = (kMode == 2 && a.coef) ? __fmul_rn(g[k], coef) : g[k];
      adamw_elem<kFast>(pf[k], mf[k], vf[k], gk, c);
    }
    *reinterpret_cast<float4*>(a.master + it.s[h]) = make_float4(pf[0], pf[1], pf[2], pf[3]);
    *reinterpret_cast<float4*>(a.m + it.s[h]) = make_float4(mf[0], mf[1], mf[2], mf[3]);
    *reinterpret_cast<float4*>(a.v + it.s[h]) = make_float4(vf[0], vf[1], vf[2], vf[3]);
    gather_store4<D, kSrc>(a, it.e[h], kFast ? pack4_hw(pf) : pack4(pf));
  }
}

// kMode: 0 = fused RS+AdamW+AG, 1 = RS only (+in-place reduced shard, partials),
// 2 = AdamW+AG from the in-place reduced shard.  U: items per thread in flight
// (memory-level parallelism for the NVLink loads).
template <int D, int kSrc, int kMode, int U, int W, bool kFast>
__global__ void __launch_bounds__(kThreads, HOD_P2P_MINB) p2p_step_kernel(const __grid_constant__ SpanArgs a,
                                                             const BarrierArgs b, const AdamWConsts c,
                                                             int rank) {
  if (kMode != 2) {
    if (!cross_gpu_barrier(b, a.d, rank)) return;
  } else {
    // the update half has no barrier of its own: it must not apply a clip
    // coefficient left over from a norm exchange that failed
    __shared__ int failed;
    if (threadIdx.x == 0) failed = rank_failed(b.err);
    __syncthreads();
    if (failed) return;
  }
  const float coef = (kMode == 2 && a.coef) ? __ldg(a.coef) : 1.0f;
  const int64_t n_chunks = a.chunk_end[a.n_buckets - 1];
  const int64_t n_warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  const int lane = threadIdx.x & 31;
  float ss = 0.0f;
  int cur[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cur[u] = 0;
  for (int64_t base = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; base < n_chunks;
       base += n_warps * U) {
    Item<D, kSrc, W> it[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t ch = base + u * n_warps;
      locate_chunk(a, ch, lane, cur[u], it[u]);
      load_item<D, kSrc, kMode, W>(a, it[u], rank);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) finish_item<D, kSrc, kMode, W, kFast>(a, it[u], c, coef, ss);
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

// One-directional hand-off for pipeline point-to-point transfers (§8f.3):
// the producer signals after its payload copy is complete (stream order +
// system fence), the consumer's stream waits until the flag reaches `epoch`.
__global__ void signal_kernel(uint32_t* peer_flag, uint32_t epoch) {
  __threadfence_system();
  st_release_sys(peer_flag, epoch);
}

__global__ void wait_kernel(const uint32_t* flag, uint32_t epoch, unsigned long long timeout_ns, uint32_t* err) {
  const unsigned long long t0 = globaltimer();
  while (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) < 0) {
    if (globaltimer() - t0 > timeout_ns) {
      if (err) atomicExch(err, static_cast<uint32_t>(HOD_ETIMEOUT));
      return;
    }
    __nanosleep(200);
  }
}

static int unroll_setting() {
  static int u = [] {
    const char* e = getenv("HOD_P2P_UNROLL");
    return e ? atoi(e) : 0;  // 0 = auto
  }();
  return u;
}

// 16-byte peer loads in the p2p pull reduce-scatter (Item::kWide): default
// on at d = 2 (measured: fused span kernel -2.3 %, LLaMA-7B RS -1 %; the
// d = 4 read ceiling is the same for 8- and 16-byte loads); env
// HOD_P2P_WIDE=0/1 forces it off/on
static int wide_setting() {
  static int w = [] {
    const char* e = getenv("HOD_P2P_WIDE");
    return e ? atoi(e) : -1;
  }();
  return w;
}

template <int D, int kSrc, int kMode, int U, int W>
static void launch_u_w(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank, int grid,
                       cudaStream_t s) {
  // the RS half has no update: only the exact instantiation exists
  if (kMode != 1 && c.fast) launch(p2p_step_kernel<D, kSrc, kMode, U, W, kMode != 1>, grid, kThreads, 0, s, a, b, c, rank);
  else launch(p2p_step_kernel<D, kSrc, kMode, U, W, false>, grid, kThreads, 0, s, a, b, c, rank);
}

template <int D, int kSrc, int kMode>
static void launch_step(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank,
                        int grid, cudaStream_t s) {
  count_launch(1);
  // measured (tools/p2p_microbench.py): two items in flight per thread pay off
  // at d = 2 (one remote load each); at d >= 4 the register cost outweighs it.
  // Co-resident launches (beside backward GEMMs) take the one-item variant:
  // <= 84 registers, so a CTA fits the 22.5 K registers a GEMM CTA leaves.
  const int u = unroll_setting();
  const bool two = !coresident() && (u >= 2 || (u == 0 && D == 2));
  const int w = wide_setting();
  if (kSrc == kSrcPeer && kMode != 2 && (w > 0 || (w < 0 && D == 2))) {
    if (two) launch_u_w<D, kSrc, kMode, 2, 1>(a, b, c, rank, grid, s);
    else launch_u_w<D, kSrc, kMode, 1, 1>(a, b, c, rank, grid, s);
  } else {
    if (two) launch_u_w<D, kSrc, kMode, 2, 0>(a, b, c, rank, grid, s);
    else launch_u_w<D, kSrc, kMode, 1, 0>(a, b, c, rank, grid, s);
  }
}

template <int kSrc, int kMode>
static void dispatch_d(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank,
                       int grid, cudaStream_t s) {
  switch (kSrc == kSrcNvls ? 0 : a.d) {
    case 2: launch_step<2, kSrc, kMode>(a, b, c, rank, grid, s); break;
    case 4: launch_step<4, kSrc, kMode>(a, b, c, rank, grid, s); break;
    case 8: launch_step<8, kSrc, kMode>(a, b, c, rank, grid, s); break;
    default: launch_step<0, kSrc, kMode>(a, b, c, rank, grid, s); break;
  }
}

static int fill_barrier(uint64_t* const* flags, int d, int rank, int slot, uint32_t epoch, uint32_t tag,
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
  b->tag = tag;
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
  int64_t elems = 0;
  for (int k = 0; k < sp->n_buckets; ++k) {
    const int64_t n = sp->shard_numel[k];
    if (n < 8 || (n & 7) || sp->bucket_start[k] < 0 || (sp->bucket_start[k] & 7)) {
      set_error("hod_p2p: bucket %d: shard size/offset must be positive multiples of 8", k);
      return HOD_EALIGN;
    }
    a->own_off[k] = sp->bucket_start[k] + static_cast<int64_t>(sp->rank) * n;
    a->chunk_end[k] = (k ? a->chunk_end[k - 1] : 0) + (n + kChunk - 1) / kChunk;
    elems += n;
    a->elem_end[k] = elems;
  }
  a->master = sp->master;
  a->m = sp->exp_avg;
  a->v = sp->exp_avg_sq;
  a->partials = sp->partials;
  a->coef = sp->clip_coef;
  a->n_buckets = sp->n_buckets;
  a->d = sp->d;
  a->keep_reduced = sp->keep_reduced;
  return fill_barrier(sp->flags, sp->d, sp->rank, sp->slot, sp->epoch, sp->tag, sp->timeout_ns, sp->err, b);
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
  const int64_t chunks = a.chunk_end[a.n_buckets - 1];
  // RS keeps a FIXED grid so its sum-of-squares partials are reproducible
  // 2 CTAs/SM measured best for the fused span kernel (tools/sweep_grid.sh, d = 2/4)
  static const int p2p_cps = [] {
    const char* e = getenv("HOD_P2P_CTAS_PER_SM");  // tuning override of the fused/AG grid
    return e ? atoi(e) : 2;
  }();
  const int grid = (mode == HOD_P2P_RS) ? partials_grid() : grid_for(chunks * 32, kThreads, p2p_cps);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int src = sp->nvls ? kSrcNvls : kSrcPeer;
  if (src == kSrcPeer && span_tma_applies()) return launch_span_tma(a, b, c, sp->rank, mode, s);
  if (mode == HOD_P2P_FUSED) {
    if (src == kSrcNvls) dispatch_d<kSrcNvls, 0>(a, b, c, sp->rank, grid, s);
    else dispatch_d<kSrcPeer, 0>(a, b, c, sp->rank, grid, s);
  } else if (mode == HOD_P2P_RS) {
    if (src == kSrcNvls) dispatch_d<kSrcNvls, 1>(a, b, c, sp->rank, grid, s);
    else dispatch_d<kSrcPeer, 1>(a, b, c, sp->rank, grid, s);
  } else {
    // the update half never reads the grad side: only the AG flavour matters
    if (src == kSrcNvls) dispatch_d<kSrcNvls, 2>(a, b, c, sp->rank, grid, s);
    else dispatch_d<kSrcPeer, 2>(a, b, c, sp->rank, grid, s);
  }
  return cuda_status(cudaGetLastError(), "hod_p2p_step launch");
}

int hod_p2p_signal(uint32_t* peer_flag, uint32_t epoch, void* stream) {
  if (!peer_flag) { set_error("hod_p2p_signal: null flag"); return HOD_EINVAL; }
  count_launch(1);
  launch(signal_kernel, 1, 1, 0, static_cast<cudaStream_t>(stream), peer_flag, epoch);
  return cuda_status(cudaGetLastError(), "hod_p2p_signal launch");
}

int hod_p2p_wait(const uint32_t* flag, uint32_t epoch, unsigned long long timeout_ns, uint32_t* err,
                 void* stream) {
  if (!flag) { set_error("hod_p2p_wait: null flag"); return HOD_EINVAL; }
  count_launch(1);
  launch(wait_kernel, 1, 1, 0, static_cast<cudaStream_t>(stream), flag, epoch,
         timeout_ns ? timeout_ns : 20000000000ull, err);
  return cuda_status(cudaGetLastError(), "hod_p2p_wait launch");
}

// Copy-engine transfer between a local and a peer-mapped (symmetric-memory)
// address: the GPU's copy engines move the bytes over NVLink while every SM
// stays with the GEMMs (pipeline stage hand-offs, the post-checkpoint
// all-gather of restored param shards).  One peer at a time reaches
// 718-755 GB/s per direction; three peers at once only 390-445 GB/s
// (profiles/r01_ce_probe.jsonl), so the optimizer's own collectives stay on
// SMs.
int hod_ce_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return HOD_OK;
  if (!dst || !src) { set_error("hod_ce_copy: null pointer"); return HOD_EINVAL; }
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)),
                     "hod_ce_copy");
}

int hod_p2p_barrier(uint64_t* const* flags, int d, int rank, int slot, uint32_t epoch, uint32_t tag,
                    unsigned long long timeout_ns, uint32_t* err, void* stream) {
  if (!flags || d < 1 || d > kMaxRanks || rank < 0 || rank >= d || slot < 0) {
    set_error("hod_p2p_barrier: bad arguments"); return HOD_EINVAL;
  }
  BarrierArgs b;
  int rc = fill_barrier(flags, d, rank, slot, epoch, tag, timeout_ns, err, &b);
  if (rc) return rc;
  count_launch(1);
  launch(barrier_kernel, 1, 32, 0, static_cast<cudaStream_t>(stream), b, d, rank);
  return cuda_status(cudaGetLastError(), "hod_p2p_barrier launch");
}

int hod_p2p_norm(const float* partials, int64_t n_partials, double* const* xchg, uint64_t* const* flags,
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
  int rc = fill_barrier(flags, d, rank, slot, epoch, HOD_NORM_TAG, timeout_ns, err, &b);
  if (rc) return rc;
  count_launch(1);
  launch(norm_exchange_kernel, 1, 32, 0, static_cast<cudaStream_t>(stream), 
      partials, n_partials, x, xchg[rank], b, d, rank, max_norm, coef, norm, sumsq);
  return cuda_status(cudaGetLastError(), "hod_p2p_norm launch");
}

}  // extern "C"
