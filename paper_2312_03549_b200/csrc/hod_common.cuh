// hod_common.cuh — shared helpers for the HOD sm_100a kernels.
//
// Arithmetic here is written with explicit-rounding intrinsics (__fmul_rn,
// __fadd_rn, __fdiv_rn, __fsqrt_rn) so that nvcc cannot contract into FMA:
// the CPU oracle (oracle/hod_oracle.c, built with -ffp-contract=off) performs
// the identical IEEE operations in the identical order, which makes the
// device results bit-exact against it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/hod.h"

namespace hod {

// Thread-local error slot behind hod_last_error().
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
void count_launch(int n);  // feeds hod_launch_count()

constexpr int kThreads = 256;
constexpr int kSMs = 148;

__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float(static_cast<uint32_t>(h) << 16);
}

// IEEE round-to-nearest-even fp32 -> bf16 (NaN stays NaN, quieted).
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x0040u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Hardware RNE of two fp32 to bf16x2 (lo in bits 0-15).  A NaN becomes the
// canonical NaN, so use it only where NaN payload bits do not matter (norms).
__device__ __forceinline__ uint32_t cvt_bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Unpack 8 bf16 from a uint4 into floats.
__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = static_cast<uint32_t>(f32_to_bf16(f[2 * i])) |
           (static_cast<uint32_t>(f32_to_bf16(f[2 * i + 1])) << 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Warp-contiguous element mapping.  A warp owns a 256-element chunk; lane l
// handles the two quads at chunk*256 + 4l and chunk*256 + 128 + 4l, so every
// warp-wide 16-byte fp32 access (and 8-byte bf16 access) covers one fully
// used contiguous 512-byte (256-byte) span — no half-used sectors, no L1
// replays (ncu showed 61 % L1 hits from the previous lane-owns-8-contiguous
// mapping, i.e. every state load fetched twice the sectors it used).
constexpr int kChunk = 256;

// Which 256-element chunks this warp processes: all warps of the grid stride
// the range together.  (A blocked variant — each CTA streaming its own
// contiguous run — measured 4-12 % slower on B200; tools/sweep_grid.sh.)
struct ChunkRange {
  int64_t first, last, step;
};

__device__ __forceinline__ ChunkRange chunk_range(int64_t n_chunks) {
  const int64_t n_warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  return ChunkRange{(static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, n_chunks, n_warps};
}

__device__ __forceinline__ void ld_f32_quads(const float* p, int64_t e0, float (&x)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p + e0);
  const float4 b = *reinterpret_cast<const float4*>(p + e0 + 128);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

__device__ __forceinline__ void st_f32_quads(float* p, int64_t e0, const float (&x)[8]) {
  *reinterpret_cast<float4*>(p + e0) = make_float4(x[0], x[1], x[2], x[3]);
  *reinterpret_cast<float4*>(p + e0 + 128) = make_float4(x[4], x[5], x[6], x[7]);
}

__device__ __forceinline__ void unpack4(const uint2& q, float* f) {
  f[0] = __uint_as_float(q.x << 16);
  f[1] = __uint_as_float(q.x & 0xffff0000u);
  f[2] = __uint_as_float(q.y << 16);
  f[3] = __uint_as_float(q.y & 0xffff0000u);
}

__device__ __forceinline__ void ld_bf16_quads(const uint16_t* p, int64_t e0, float (&x)[8]) {
  unpack4(*reinterpret_cast<const uint2*>(p + e0), x);
  unpack4(*reinterpret_cast<const uint2*>(p + e0 + 128), x + 4);
}

__device__ __forceinline__ uint2 pack4(const float* f) {
  return make_uint2(static_cast<uint32_t>(f32_to_bf16(f[0])) | (static_cast<uint32_t>(f32_to_bf16(f[1])) << 16),
                    static_cast<uint32_t>(f32_to_bf16(f[2])) | (static_cast<uint32_t>(f32_to_bf16(f[3])) << 16));
}

// fast mode: hardware RNE (cvt.rn.bf16x2; NaN payloads are not preserved)
__device__ __forceinline__ uint2 pack4_hw(const float* f) {
  return make_uint2(cvt_bf16x2_rn(f[0], f[1]), cvt_bf16x2_rn(f[2], f[3]));
}

template <bool kHw = false>
__device__ __forceinline__ void st_bf16_quads(uint16_t* p, int64_t e0, const float (&x)[8]) {
  *reinterpret_cast<uint2*>(p + e0) = kHw ? pack4_hw(x) : pack4(x);
  *reinterpret_cast<uint2*>(p + e0 + 128) = kHw ? pack4_hw(x + 4) : pack4(x + 4);
}

// Fp32 AdamW constants folded on the host in double precision, then rounded
// once to fp32.
struct AdamWConsts {
  float decay;      // 1 - lr*wd
  float b1, omb1;   // beta1, 1-beta1
  float b2, omb2;   // beta2, 1-beta2
  float step_size;  // lr / (1 - beta1^t)
  float bc2_sqrt;   // sqrt(1 - beta2^t)
  float eps;
  float inv_bc2_sqrt;   // 1 / sqrt(1 - beta2^t)        (fast mode)
  float neg_step_size;  // -lr / (1 - beta1^t)          (fast mode)
  int fast;             // HOD_ADAMW_FAST: launchers pick the kFast kernels
};

AdamWConsts fold_adamw(const hod_adamw_params& hp);

// One element of the update.
//  exact (kFast = false): identical IEEE operations in the identical order as
//    oracle/hod_oracle.c (explicit _rn intrinsics, no FMA contraction, IEEE
//    sqrt and divisions): bit-exact against the oracle.
//  fast (kFast = true, HOD_ADAMW_FAST): the same algebra in ~10 FP operations —
//    FMAs, MUFU square root and reciprocal (sqrt.approx / rcp.approx, <= 2 ulp
//    each), the bias correction folded into constants.  The update term
//    lr*m/(sqrt(v)+eps) carries a few ulp of relative error, i.e. ~1e-9 of
//    |theta| at lr = 1e-4; m and v differ from the exact mode by <= 1 ulp per
//    step (FMA rounding): inside the north star's 1e-6 (1 step) / 1e-5
//    (100 steps) tolerance (tests/test_kernels_gpu.py measures it).
template <bool kFast = false>
__device__ __forceinline__ void adamw_elem(float& p, float& m, float& v, float g,
                                           const AdamWConsts& c) {
  if constexpr (kFast) {
    m = fmaf(c.b1, m, c.omb1 * g);
    v = fmaf(c.b2, v, (c.omb2 * g) * g);
    float s, r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(v));
    const float den = fmaf(s, c.inv_bc2_sqrt, c.eps);
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(den));
    p = fmaf(p, c.decay, c.neg_step_size * (m * r));
  } else {
    p = __fmul_rn(p, c.decay);
    m = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.omb1, g));
    v = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(c.omb2, __fmul_rn(g, g)));
    const float den = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), c.bc2_sqrt), c.eps);
    p = __fsub_rn(p, __fmul_rn(c.step_size, __fdiv_rn(m, den)));
  }
}

// CTA cap set by hod_set_grid_limit (0 = none): lets the optimizer's kernels
// co-run with the backward GEMMs.  A cap of at most one CTA per SM is the
// CO-RESIDENT mode: launchers then also pick their register-light variants so
// that one optimizer CTA (256 threads, <= 88 registers, no shared memory)
// fits beside a resident cuBLAS GEMM CTA (measured nvjet sm_100 kernels: 256
// threads x 168 registers, 213 KB shared memory, tools/corun_probe.py).
int grid_limit();
inline bool coresident() { return grid_limit() > 0 && grid_limit() <= kSMs; }

// Co-resident launches prefer the maximum shared-memory carveout.  An SM runs
// CTAs of one L1/shared split at a time: a kernel launched with the default
// (small) carveout keeps the SMs it occupies in that configuration, and a
// GEMM that needs 213 KB of shared memory cannot be placed there until they
// drain — the optimizer would then serialise with backward instead of
// sharing the SMs.  Measured (tools/corun_probe.py, profiles/r02_corun.jsonl):
// AdamW at one CTA/SM launched BEFORE a GEMM loop hides 0.72 of its time with
// the carveout vs 0.0 without.  Full-GPU launches keep the default split: the
// larger L1 holds more loads in flight (AdamW alone 6.3 vs 5.3 TB/s).
// HOD_CARVEOUT=0 disables it (A/B runs).
bool carveout_enabled();

// HOD_CTAS_PER_SM (env) overrides the per-kernel CTAs-per-SM cap (tuning runs).
int ctas_per_sm_override();

// Programmatic dependent launch for back-to-back bucket kernels (HOD_PDL=0 disables).
bool pdl_enabled();

// Device side: let the next PDL launch in the stream start while this grid
// drains.  Only for kernels whose successor never reads what they write
// (consecutive buckets: disjoint memory).
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Host side: launch with programmatic stream serialization, so the kernel may
// overlap the tail of the previous kernel in the stream IF that kernel called
// pdl_trigger(); after any other kernel the usual full dependency holds.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (pdl_enabled()) cfg.numAttrs = 1;
  if (coresident() && carveout_enabled()) {
    attr[cfg.numAttrs].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    attr[cfg.numAttrs].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
    ++cfg.numAttrs;
  }
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// <<<grid, block, smem, stream>>> with the co-resident carveout applied.
template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
  attr[0].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
  cfg.attrs = attr;
  cfg.numAttrs = (coresident() && carveout_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int grid_for(int64_t work_items, int per_block, int max_blocks_per_sm = 8) {
  int64_t need = (work_items + per_block - 1) / per_block;
  if (ctas_per_sm_override() > 0) max_blocks_per_sm = ctas_per_sm_override();
  int64_t cap = static_cast<int64_t>(kSMs) * max_blocks_per_sm;
  if (grid_limit() > 0 && grid_limit() < cap) cap = grid_limit();
  if (need < 1) need = 1;
  return static_cast<int>(need < cap ? need : cap);
}

// Grid of the kernels that emit HOD_SUMSQ_PARTIALS per-CTA partials: fixed
// (reproducible) for a given limit; CTA 0 zero-fills the unused slots.
inline int partials_grid() {
  const int lim = grid_limit();
  return (lim > 0 && lim < HOD_SUMSQ_PARTIALS) ? lim : HOD_SUMSQ_PARTIALS;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace hod
