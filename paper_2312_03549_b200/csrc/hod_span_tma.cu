// hod_span_tma.cu — the fused span kernel with TMA-fed data movement (p2p).
//
// Same work and the same arithmetic as p2p_step_kernel (hod_p2p.cu) — the
// cross-GPU arrival barrier, the reduce-scatter of this rank's shard of every
// bucket of the span (fp32 sum in rank order 0..d-1, one RNE rounding), the
// AdamW update and the all-gather of the bf16 params into every peer — but
// every byte moves on the Tensor Memory Accelerator:
//
//   producer warp (one elected lane): per 2048-element tile, cp.async.bulk of
//     the d peers' packed-gradient tiles (NVLink reads, straight into shared
//     memory) and of the master / m / v tiles, into a ring of stages, each
//     signalled by an mbarrier with the tile's byte count;
//   16 consumer warps: reduce + AdamW in shared memory (in place), each warp
//     signalling a per-stage mbarrier when its part of the tile is done;
//   storer warp (one elected lane): issues the bulk stores — master / m / v
//     back to HBM and the bf16 param tile into each peer's param buffer
//     (NVLink writes) — and recycles the stage once those stores have read it.
//     Consumers never wait for stores; the producer runs up to S - 1 tiles
//     ahead of the storer.
//
// Bytes in flight per SM are bounded by the ~185 KB ring instead of the
// register file: the register kernel holds <= 2 x 16 quads per thread in
// flight and needs 2 CTAs/SM x 116 registers to approach the NVLink ceiling,
// which also leaves no room for the pack kernel to co-run.  This kernel runs
// one CTA per SM with 576 threads.  Modes as hod_p2p_step: FUSED, RS (reduced
// shard in place + per-CTA sum-of-squares partials), ADAMW_AG (from the
// in-place reduced shard, clip coefficient applied).  Bit-identical to the
// register kernel in every mode but the RS partials' summation order (the
// norm is checked within tolerance; the coefficient is identical on every
// rank because the ranks exchange their local sums, hod_p2p_norm).
#include <stdint.h>
#include <stdlib.h>

#include <atomic>

#include "hod_p2p.cuh"
#include "hod_tma.cuh"

namespace hod {

constexpr int kTile = 2048;             // owned elements per tile
constexpr int kCons = 512;              // consumer threads (16 warps)
constexpr int kTmaBlock = kCons + 64;   // + a producer warp and a storer warp
constexpr int kSmemBudget = 200 * 1024;

template <int D, int kMode>
struct TmaSpanLayout {
  static constexpr int kSlots = kMode == 2 ? 1 : (D > 0 ? D : kMaxRanks);  // bf16 grad tiles per stage
  static constexpr bool kState = kMode != 1;
  static constexpr int kStateOff = kSlots * kTile * 2;                       // master | m | v (fp32)
  static constexpr int kOutOff = kStateOff + (kState ? 3 * kTile * 4 : 0);   // bf16 params
  static constexpr int kStageBytes = kOutOff + (kState ? kTile * 2 : 0);
  static constexpr int kStagesFit = kSmemBudget / kStageBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static_assert(kStages >= 3, "stage ring too shallow");
  static constexpr int kSmem = kStages * kStageBytes + 3 * kStages * 8;
};

struct TileLoc {
  int k;          // bucket of the span
  int64_t off;    // element offset inside the bucket's shard
  int len;        // elements (multiple of 16)
};

__device__ __forceinline__ TileLoc locate_tile(const SpanArgs& a, const int64_t* tile_end, int64_t j, int& k) {
  while (k < a.n_buckets - 1 && j >= tile_end[k]) ++k;
  const int64_t first = k ? tile_end[k - 1] : 0;
  const int64_t n = a.elem_end[k] - (k ? a.elem_end[k - 1] : 0);
  const int64_t off = (j - first) * kTile;
  const int64_t len = n - off < kTile ? n - off : kTile;
  return TileLoc{k, off, static_cast<int>(len)};
}

template <int D, int kMode, bool kFast>
__global__ void __launch_bounds__(kTmaBlock, 1) span_tma_kernel(const __grid_constant__ SpanArgs a,
                                                                const BarrierArgs b, const AdamWConsts c, int rank) {
  using Lay = TmaSpanLayout<D, kMode>;
  constexpr int S = Lay::kStages;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Lay::kStageBytes);   // loads landed
  uint64_t* computed = full + S;                                                 // consumers done
  uint64_t* empty = computed + S;                                                // stores read the stage
  __shared__ int64_t tile_end[kMaxSpan];
  __shared__ float red[kCons / 32];
  const int dd = D > 0 ? D : a.d;

  if (kMode != 2) {
    if (!cross_gpu_barrier(b, a.d, rank)) return;
  } else {
    // the update half has no barrier of its own: never apply a clip
    // coefficient left over from a norm exchange that failed
    __shared__ int failed;
    if (threadIdx.x == 0) failed = rank_failed(b.err);
    __syncthreads();
    if (failed) return;
  }
  if (threadIdx.x == 0) {
    int64_t t = 0, prev = 0;
    for (int k = 0; k < a.n_buckets; ++k) {
      t += (a.elem_end[k] - prev + kTile - 1) / kTile;
      prev = a.elem_end[k];
      tile_end[k] = t;
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&computed[s], kCons / 32);
      mbar_init(&empty[s], 1);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const int64_t n_tiles = tile_end[a.n_buckets - 1];

  if (threadIdx.x >= kCons) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < kCons + 32) {
      // ---------------- producer: one lane streams tiles into the ring
      if (lane != 0) return;
      int k = 0;
      int64_t i = 0;
      for (int64_t j = blockIdx.x; j < n_tiles; j += gridDim.x, ++i) {
        const int s = static_cast<int>(i % S);
        if (i >= S) mbar_wait(&empty[s], static_cast<uint32_t>((i / S - 1) & 1));
        const TileLoc L = locate_tile(a, tile_end, j, k);
        uint8_t* st = smem + s * Lay::kStageBytes;
        const uint32_t gb = static_cast<uint32_t>(L.len) * 2, sb = static_cast<uint32_t>(L.len) * 4;
        mbar_expect_tx(&full[s], (kMode == 2 ? gb : dd * gb) + (Lay::kState ? 3 * sb : 0u));
        const int64_t e = a.own_off[L.k] + L.off;
        if (kMode == 2) {
          bulk_g2s(st, a.local_grad + e, gb, &full[s]);
        } else {
#pragma unroll
          for (int q = 0; q < Lay::kSlots; ++q)
            if (q < dd) bulk_g2s(st + q * kTile * 2, reinterpret_cast<const uint16_t*>(a.grad.p[q]) + e, gb, &full[s]);
        }
        if constexpr (Lay::kState) {
          const int64_t si = (L.k ? a.elem_end[L.k - 1] : 0) + L.off;
          bulk_g2s(st + Lay::kStateOff, a.master + si, sb, &full[s]);
          bulk_g2s(st + Lay::kStateOff + kTile * 4, a.m + si, sb, &full[s]);
          bulk_g2s(st + Lay::kStateOff + 2 * kTile * 4, a.v + si, sb, &full[s]);
        }
      }
      return;
    }
    // ---------------- storer: one lane writes computed tiles back (HBM
    // state, NVLink params, the reduced shard) and recycles their stages
    if (lane != 0) return;
    int k = 0;
    int64_t i = 0;
    for (int64_t j = blockIdx.x; j < n_tiles; j += gridDim.x, ++i) {
      const int s = static_cast<int>(i % S);
      mbar_wait(&computed[s], static_cast<uint32_t>((i / S) & 1));
      const TileLoc L = locate_tile(a, tile_end, j, k);
      const uint8_t* st = smem + s * Lay::kStageBytes;
      const int64_t e = a.own_off[L.k] + L.off;
      const uint32_t gb = static_cast<uint32_t>(L.len) * 2, sb = static_cast<uint32_t>(L.len) * 4;
      if (kMode == 1 || (kMode == 0 && a.keep_reduced)) bulk_s2g(a.local_grad + e, st, gb);
      if constexpr (Lay::kState) {
        const int64_t si = (L.k ? a.elem_end[L.k - 1] : 0) + L.off;
        bulk_s2g(a.master + si, st + Lay::kStateOff, sb);
        bulk_s2g(a.m + si, st + Lay::kStateOff + kTile * 4, sb);
        bulk_s2g(a.v + si, st + Lay::kStateOff + 2 * kTile * 4, sb);
#pragma unroll
        for (int q = 0; q < (D > 0 ? D : kMaxRanks); ++q)
          if (q < dd) bulk_s2g(reinterpret_cast<uint16_t*>(a.param.p[q]) + e, st + Lay::kOutOff, gb);
      }
      bulk_commit();
      // one tile's stores stay in flight: release the previous tile's stage
      // once its stores have read it
      if (i >= 1) {
        bulk_wait_read<1>();
        mbar_arrive(&empty[(i - 1) % S]);
      }
    }
    bulk_wait_all();            // every store performed (peers' params included)
    fence_proxy_async_global();
    __threadfence_system();     // before any later signal of this rank
    return;
  }

  // ---------------- consumers: reduce + AdamW in shared memory
  const int t = threadIdx.x;
  const float coef = (kMode == 2 && a.coef) ? __ldg(a.coef) : 1.0f;
  float ss = 0.0f;
  int k = 0;
  int64_t i = 0;
  for (int64_t j = blockIdx.x; j < n_tiles; j += gridDim.x, ++i) {
    const int s = static_cast<int>(i % S);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const TileLoc L = locate_tile(a, tile_end, j, k);
    uint8_t* st = smem + s * Lay::kStageBytes;
    const int nq = L.len >> 2;
    for (int qd = t; qd < nq; qd += kCons) {
      float g[4];
      if (kMode == 2) {
        unpack4(reinterpret_cast<const uint2*>(st)[qd], g);
      } else {
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int q = 0; q < Lay::kSlots; ++q) {
          if (q < dd) {
            float f[4];
            unpack4(reinterpret_cast<const uint2*>(st + q * kTile * 2)[qd], f);
#pragma unroll
            for (int x = 0; x < 4; ++x) acc[x] = __fadd_rn(acc[x], f[x]);
          }
        }
        uint16_t r[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          r[x] = f32_to_bf16(acc[x]);
          g[x] = bf16_to_f32(r[x]);
        }
        // the reduced quad replaces slot 0 (stored to the own shard)
        if (kMode == 1 || a.keep_reduced)
          reinterpret_cast<uint2*>(st)[qd] = make_uint2(r[0] | (static_cast<uint32_t>(r[1]) << 16),
                                                        r[2] | (static_cast<uint32_t>(r[3]) << 16));
      }
      if constexpr (kMode == 1) {
#pragma unroll
        for (int x = 0; x < 4; ++x) ss = __fadd_rn(ss, __fmul_rn(g[x], g[x]));
      } else {
        float4* P = reinterpret_cast<float4*>(st + Lay::kStateOff);
        float4* M = P + kTile / 4;
        float4* V = M + kTile / 4;
        const float4 p4 = P[qd], m4 = M[qd], v4 = V[qd];
        float pf[4] = {p4.x, p4.y, p4.z, p4.w};
        float mf[4] = {m4.x, m4.y, m4.z, m4.w};
        float vf[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const float gx = (kMode == 2 && a.coef) ? __fmul_rn(g[x], coef) : g[x];
          adamw_elem<kFast>(pf[x], mf[x], vf[x], gx, c);
        }
        P[qd] = make_float4(pf[0], pf[1], pf[2], pf[3]);
        M[qd] = make_float4(mf[0], mf[1], mf[2], mf[3]);
        V[qd] = make_float4(vf[0], vf[1], vf[2], vf[3]);
        reinterpret_cast<uint2*>(st + Lay::kOutOff)[qd] = kFast ? pack4_hw(pf) : pack4(pf);
      }
    }
    // this warp's shared-memory writes -> visible to the storer's bulk copies
    fence_proxy_async_smem();
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(&computed[s]);
  }
  if constexpr (kMode == 1) {
    if (a.partials) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if ((t & 31) == 0) red[t >> 5] = ss;
      named_sync<kCons>(1);
      if (t == 0) {
        float tot = 0.0f;
        for (int w = 0; w < kCons / 32; ++w) tot += red[w];
        a.partials[blockIdx.x] = tot;
      }
      if (blockIdx.x == 0)
        for (int x = gridDim.x + t; x < HOD_SUMSQ_PARTIALS; x += kCons) a.partials[x] = 0.0f;
    }
  }
}

// 0 = off, 1 = full-GPU launches (default), 2 = also under a grid cap (the
// one-GPU rank emulation covers the kernel with it).  Initial value from env
// HOD_SPAN_TMA, then hod_set_span_tma.
static std::atomic<int> g_span_tma{[] {
  const char* e = getenv("HOD_SPAN_TMA");
  return e ? atoi(e) : 1;
}()};
static int span_tma_setting() { return g_span_tma.load(std::memory_order_relaxed); }

template <int D, int kMode, bool kFast>
static int launch_tma(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank, cudaStream_t s) {
  using Lay = TmaSpanLayout<D, kMode>;
  static const cudaError_t attr = cudaFuncSetAttribute(span_tma_kernel<D, kMode, kFast>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::kSmem);
  if (attr != cudaSuccess) return cuda_status(attr, "span_tma_kernel smem attribute");
  int64_t tiles = 0, prev = 0;
  for (int k = 0; k < a.n_buckets; ++k) {
    tiles += (a.elem_end[k] - prev + kTile - 1) / kTile;
    prev = a.elem_end[k];
  }
  int grid = static_cast<int>(tiles < kSMs ? tiles : kSMs);
  if (grid_limit() > 0 && grid_limit() < grid) grid = grid_limit();
  if (grid < 1) grid = 1;
  count_launch(1);
  return cuda_status(launch(span_tma_kernel<D, kMode, kFast>, grid, kTmaBlock, Lay::kSmem, s, a, b, c, rank),
                     "span_tma_kernel launch");
}

template <int D, int kMode>
static int launch_tma_fast(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank, cudaStream_t s) {
  if (kMode != 1 && c.fast) return launch_tma<D, kMode, kMode != 1>(a, b, c, rank, s);
  return launch_tma<D, kMode, false>(a, b, c, rank, s);
}

template <int kMode>
static int launch_tma_d(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank, cudaStream_t s) {
  switch (a.d) {
    case 2: return launch_tma_fast<2, kMode>(a, b, c, rank, s);
    case 4: return launch_tma_fast<4, kMode>(a, b, c, rank, s);
    case 8: return launch_tma_fast<8, kMode>(a, b, c, rank, s);
    default: return launch_tma_fast<0, kMode>(a, b, c, rank, s);
  }
}

bool span_tma_applies() {
  const int v = span_tma_setting();
  return v >= 2 || (v == 1 && !coresident());
}

int launch_span_tma(const SpanArgs& a, const BarrierArgs& b, const AdamWConsts& c, int rank, int mode,
                    cudaStream_t s) {
  if (mode == HOD_P2P_FUSED) return launch_tma_d<0>(a, b, c, rank, s);
  if (mode == HOD_P2P_RS) return launch_tma_d<1>(a, b, c, rank, s);
  return launch_tma_d<2>(a, b, c, rank, s);
}

}  // namespace hod

extern "C" int hod_set_span_tma(int mode) {
  if (mode < 0 || mode > 2) { hod::set_error("hod_set_span_tma: mode %d (0..2)", mode); return HOD_EINVAL; }
  hod::g_span_tma.store(mode, std::memory_order_relaxed);
  return HOD_OK;
}
