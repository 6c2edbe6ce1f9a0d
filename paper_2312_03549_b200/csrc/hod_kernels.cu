// hod_kernels.cu — K1 (bucket pack/cast), K2 (fused sharded AdamW) and K3
// (deterministic grad sum-of-squares + clip coefficient) for sm_100a.
//
// All three are elementwise and HBM-bound: no tensor
// cores, 128-bit coalesced loads/stores, grid sized in multiples of the 148
// SMs and grid-strided.  See include/hod.h for the contracts.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <vector>

#include "hod_common.cuh"

namespace hod {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// process-wide: autograd runs post-accumulate-grad hooks (hence bucket
// launches) on its own device thread, which must see the same cap
static std::atomic<int> g_grid_limit{0};
int grid_limit() { return g_grid_limit.load(std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("HOD_PDL");
    return !e || atoi(e) != 0;
  }();
  return v;
}

// HOD_PACK_GENTLE=0: co-resident packs keep the full-GPU unroll (A/B runs)
static bool pack_gentle() {
  static const bool v = [] {
    const char* e = getenv("HOD_PACK_GENTLE");
    return !e || atoi(e) != 0;
  }();
  return v;
}

bool carveout_enabled() {
  static const bool v = [] {
    const char* e = getenv("HOD_CARVEOUT");
    return !e || atoi(e) != 0;
  }();
  return v;
}

int ctas_per_sm_override() {
  static const int v = [] {
    const char* e = getenv("HOD_CTAS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  return v;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return HOD_OK;
  set_error("%s: %s (%d)", what, cudaGetErrorString(e), static_cast<int>(e));
  return static_cast<int>(e);
}

AdamWConsts fold_adamw(const hod_adamw_params& hp) {
  AdamWConsts c;
  const double t = static_cast<double>(hp.step);
  const double bc1 = 1.0 - pow(hp.beta1, t);
  const double bc2 = 1.0 - pow(hp.beta2, t);
  c.decay = static_cast<float>(1.0 - hp.lr * hp.weight_decay);
  c.b1 = static_cast<float>(hp.beta1);
  c.omb1 = static_cast<float>(1.0 - hp.beta1);
  c.b2 = static_cast<float>(hp.beta2);
  c.omb2 = static_cast<float>(1.0 - hp.beta2);
  c.step_size = static_cast<float>(hp.lr / bc1);
  c.bc2_sqrt = static_cast<float>(sqrt(bc2));
  c.eps = static_cast<float>(hp.eps);
  c.inv_bc2_sqrt = static_cast<float>(1.0 / sqrt(bc2));
  c.neg_step_size = static_cast<float>(-hp.lr / bc1);
  c.fast = hp.mode == HOD_ADAMW_FAST;
  return c;
}

// ---------------------------------------------------------------------------
// K1: pack.  The table travels by value in the kernel parameter space
// (constant bank), so a CTA-uniform scan over it is a broadcast read.  Each
// CTA owns tiles of kPackTile destination elements; a tile that lies inside
// one tensor with a 16-byte-aligned source takes the vector path, the few
// tiles touching a tensor boundary or padding take the scalar path.
// ---------------------------------------------------------------------------
constexpr int kPackVec = 8;                          // elements per 16-byte bf16 store
constexpr int kPackUnroll = 8;
constexpr int kPackTile = kThreads * kPackVec * kPackUnroll;  // 8192 elements

struct PackTable {
  const void* src[HOD_PACK_MAX_ENTRIES];
  int64_t numel[HOD_PACK_MAX_ENTRIES];
  int64_t off[HOD_PACK_MAX_ENTRIES];
  uint64_t vec_ok;  // bit i: src[i] is 16-byte aligned
  int n;
};

template <typename SrcT>
__device__ __forceinline__ float load_src(const void* p, int64_t i) {
  if constexpr (sizeof(SrcT) == 2)
    return bf16_to_f32(static_cast<const uint16_t*>(p)[i]);
  else
    return static_cast<const float*>(p)[i];
}

template <typename SrcT>
__device__ __forceinline__ void load8(const void* p, int64_t i, float (&f)[8]) {
  if constexpr (sizeof(SrcT) == 2) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p) + i));
    unpack8(q, f);
  } else {
    const float4* s = reinterpret_cast<const float4*>(static_cast<const float*>(p) + i);
    const float4 a = __ldg(s), b = __ldg(s + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
}

// kUnroll: 16-byte vectors in flight per thread.  8 for full-GPU launches;
// co-resident launches (beside GEMMs) take 2 — a quarter of the memory
// pressure per SM, for a kernel that has the whole backward to finish.
template <typename SrcT, int kUnroll = kPackUnroll>
__global__ void __launch_bounds__(kThreads) pack_kernel(const __grid_constant__ PackTable t,
                                                         uint16_t* __restrict__ dst,
                                                         int64_t bucket_numel, float scale) {
  constexpr int kPackTile = kThreads * kPackVec * kUnroll;
  constexpr int kPackUnroll = kUnroll;
  pdl_trigger();  // the next bucket's pack touches disjoint memory
  const int64_t n_tiles = (bucket_numel + kPackTile - 1) / kPackTile;
  int e = 0;  // entry cursor; tiles visited by a CTA are increasing
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t a = tile * kPackTile;
    const int64_t b = min(a + kPackTile, bucket_numel);
    while (e < t.n && t.off[e] + t.numel[e] <= a) ++e;  // CTA-uniform
    const bool inside = e < t.n && t.off[e] <= a && b <= t.off[e] + t.numel[e];
    if (inside && ((t.vec_ok >> e) & 1ull) && (b - a) == kPackTile) {
      const int64_t s0 = a - t.off[e];
      float f[kPackUnroll][8];
#pragma unroll
      for (int u = 0; u < kPackUnroll; ++u)
        load8<SrcT>(t.src[e], s0 + (static_cast<int64_t>(u) * kThreads + threadIdx.x) * kPackVec, f[u]);
#pragma unroll
      for (int u = 0; u < kPackUnroll; ++u) {
#pragma unroll
        for (int k = 0; k < 8; ++k) f[u][k] = __fmul_rn(f[u][k], scale);
        reinterpret_cast<uint4*>(dst + a)[static_cast<int64_t>(u) * kThreads + threadIdx.x] = pack8(f[u]);
      }
    } else {
      // boundary / padding tile: element-wise with a per-thread entry cursor
      int ei = e;
      for (int64_t i = a + threadIdx.x; i < b; i += kThreads) {
        while (ei < t.n && t.off[ei] + t.numel[ei] <= i) ++ei;
        float x = 0.0f;
        if (ei < t.n && t.off[ei] <= i) x = __fmul_rn(load_src<SrcT>(t.src[ei], i - t.off[ei]), scale);
        dst[i] = (ei < t.n && t.off[ei] <= i) ? f32_to_bf16(x) : static_cast<uint16_t>(0);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1+K2 fused (d == 1, no collective between them): the update reads the
// gradient straight from the per-parameter tensors through the pack table,
// with the same scale-then-RNE-to-bf16 the bucket would have held, so the
// result is bit-identical to pack followed by AdamW while the 2+2 B/element
// bucket round trip disappears (28 B/element instead of 32).
// ---------------------------------------------------------------------------
template <typename SrcT, bool kClip, bool kFast>
__global__ void __launch_bounds__(kThreads) pack_adamw_kernel(
    const __grid_constant__ PackTable t, int64_t numel, float scale, float* __restrict__ p,
    float* __restrict__ m, float* __restrict__ v, uint16_t* __restrict__ out, const AdamWConsts c,
    const float* __restrict__ coef_ptr) {
  pdl_trigger();  // the next bucket's update touches disjoint memory
  const float coef = kClip ? __ldg(coef_ptr) : 1.0f;
  // warp-strided 256-element chunks (same mapping as adamw_vec_kernel); the
  // table lookup is warp-uniform and the cursor only moves forward
  const int lane = threadIdx.x & 31;
  const int64_t n_chunks = (numel + kChunk - 1) / kChunk;
  ChunkRange r = chunk_range(n_chunks);
  int e = 0;
  for (int64_t ch = r.first; ch < r.last; ch += r.step) {
    const int64_t a = ch * kChunk;
    const int64_t b = min(a + kChunk, numel);
    while (e < t.n && t.off[e] + t.numel[e] <= a) ++e;  // warp-uniform
    const bool inside = e < t.n && t.off[e] <= a && b <= t.off[e] + t.numel[e];
    if (inside && ((t.vec_ok >> e) & 1ull) && (b - a) == kChunk) {
      const int64_t e0 = a + lane * 4;
      float g[8], pf[8], mf[8], vf[8];
      if constexpr (sizeof(SrcT) == 2) ld_bf16_quads(static_cast<const uint16_t*>(t.src[e]), e0 - t.off[e], g);
      else ld_f32_quads(static_cast<const float*>(t.src[e]), e0 - t.off[e], g);
      ld_f32_quads(p, e0, pf);
      ld_f32_quads(m, e0, mf);
      ld_f32_quads(v, e0, vf);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        g[k] = bf16_to_f32(f32_to_bf16(__fmul_rn(g[k], scale)));
        if (kClip) g[k] = __fmul_rn(g[k], coef);
        adamw_elem<kFast>(pf[k], mf[k], vf[k], g[k], c);
      }
      st_f32_quads(p, e0, pf);
      st_f32_quads(m, e0, mf);
      st_f32_quads(v, e0, vf);
      st_bf16_quads<kFast>(out, e0, pf);
    } else {
      int ei = e;
      for (int64_t i = a + lane; i < b; i += 32) {
        while (ei < t.n && t.off[ei] + t.numel[ei] <= i) ++ei;
        float gi = 0.0f;
        if (ei < t.n && t.off[ei] <= i)
          gi = bf16_to_f32(f32_to_bf16(__fmul_rn(load_src<SrcT>(t.src[ei], i - t.off[ei]), scale)));
        if (kClip) gi = __fmul_rn(gi, coef);
        float pi = p[i], mi = m[i], vi = v[i];
        adamw_elem<kFast>(pi, mi, vi, gi, c);
        p[i] = pi; m[i] = mi; v[i] = vi;
        out[i] = f32_to_bf16(pi);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2: AdamW.  Eight elements per thread per iteration: one 16-byte load of
// bf16 grad, two 16-byte loads each of master/m/v; stores mirror them plus a
// 16-byte bf16 param store.  28 B/element algorithmic traffic.
// ---------------------------------------------------------------------------
template <typename GradT, bool kClip, bool kFast>
__global__ void __launch_bounds__(kThreads) adamw_vec_kernel(
    float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
    const GradT* __restrict__ g, uint16_t* __restrict__ out, int64_t n_chunks,
    const AdamWConsts c, const float* __restrict__ coef_ptr) {
  const float coef = kClip ? __ldg(coef_ptr) : 1.0f;
  const int lane = threadIdx.x & 31;
  ChunkRange r = chunk_range(n_chunks);
  for (int64_t ch = r.first; ch < r.last; ch += r.step) {
    const int64_t e0 = ch * kChunk + lane * 4;
    float gf[8], pf[8], mf[8], vf[8];
    if constexpr (sizeof(GradT) == 2) ld_bf16_quads(reinterpret_cast<const uint16_t*>(g), e0, gf);
    else ld_f32_quads(reinterpret_cast<const float*>(g), e0, gf);
    ld_f32_quads(p, e0, pf);
    ld_f32_quads(m, e0, mf);
    ld_f32_quads(v, e0, vf);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float gk = kClip ? __fmul_rn(gf[k], coef) : gf[k];
      adamw_elem<kFast>(pf[k], mf[k], vf[k], gk, c);
    }
    st_f32_quads(p, e0, pf);
    st_f32_quads(m, e0, mf);
    st_f32_quads(v, e0, vf);
    st_bf16_quads<kFast>(out, e0, pf);
  }
}

template <typename GradT, bool kClip, bool kFast>
__global__ void __launch_bounds__(kThreads) adamw_scalar_kernel(
    float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
    const GradT* __restrict__ g, uint16_t* __restrict__ out, int64_t begin, int64_t n,
    const AdamWConsts c, const float* __restrict__ coef_ptr) {
  const float coef = kClip ? __ldg(coef_ptr) : 1.0f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t i = begin + static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    float gi;
    if constexpr (sizeof(GradT) == 2) gi = bf16_to_f32(g[i]); else gi = g[i];
    if (kClip) gi = __fmul_rn(gi, coef);
    float pi = p[i], mi = m[i], vi = v[i];
    adamw_elem<kFast>(pi, mi, vi, gi, c);
    p[i] = pi; m[i] = mi; v[i] = vi;
    out[i] = f32_to_bf16(pi);
  }
}

template <typename GradT>
static int launch_adamw(float* master, float* exp_avg, float* exp_avg_sq, const GradT* grad,
                        uint16_t* param, int64_t n, const hod_adamw_params* hp,
                        const float* clip_coef, cudaStream_t s) {
  if (n < 0 || !hp) { set_error("hod_adamw: bad n/hp"); return HOD_EINVAL; }
  if (n == 0) return HOD_OK;
  if (!master || !exp_avg || !exp_avg_sq || !grad || !param) {
    set_error("hod_adamw: null buffer"); return HOD_EINVAL;
  }
  if (hp->step < 1) { set_error("hod_adamw: step must be >= 1"); return HOD_EINVAL; }
  const AdamWConsts c = fold_adamw(*hp);
  const bool vec = aligned16(master) && aligned16(exp_avg) && aligned16(exp_avg_sq) &&
                   aligned16(grad) && aligned16(param);
  int64_t done = 0;
  if (vec) {
    const int64_t n_vec = n / kChunk;   // whole 256-element warp chunks
    if (n_vec > 0) {
      // 2 CTAs/SM measured best (6.3 TB/s vs 5.9 TB/s at 4-8/SM; tools/sweep_grid.sh)
      const int grid = grid_for(n_vec * 32, kThreads, 2);
      count_launch(1);
#define HOD_AV(CLIP, FAST) \
      launch(adamw_vec_kernel<GradT, CLIP, FAST>, grid, kThreads, 0, s, master, exp_avg, exp_avg_sq, grad, param, n_vec, c, clip_coef)
      if (clip_coef) { if (c.fast) HOD_AV(true, true); else HOD_AV(true, false); }
      else { if (c.fast) HOD_AV(false, true); else HOD_AV(false, false); }
#undef HOD_AV
    }
    done = n_vec * kChunk;
  }
  if (done < n) {
    const int grid = grid_for(n - done, kThreads);
    count_launch(1);
#define HOD_AS(CLIP, FAST) \
    launch(adamw_scalar_kernel<GradT, CLIP, FAST>, grid, kThreads, 0, s, master, exp_avg, exp_avg_sq, grad, param, done, n, c, clip_coef)
    if (clip_coef) { if (c.fast) HOD_AS(true, true); else HOD_AS(true, false); }
    else { if (c.fast) HOD_AS(false, true); else HOD_AS(false, false); }
#undef HOD_AS
  }
  return cuda_status(cudaGetLastError(), "hod_adamw launch");
}

// ---------------------------------------------------------------------------
// K3: sum of squares with a FIXED grid of HOD_SUMSQ_PARTIALS CTAs so the
// per-CTA partials (and their fixed-order final sum) are reproducible.
// ---------------------------------------------------------------------------
// The partials grid is only HOD_SUMSQ_PARTIALS (2 per SM) CTAs, so these
// read-only streams use 1024-thread CTAs to fill the SM (2048 threads).
constexpr int kSumsqThreads = 1024;
constexpr int kSumsqUnroll = 2;

template <int NT>
__device__ __forceinline__ float block_sum(float x) {
  __shared__ float warp_part[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = x;
  __syncthreads();
  float s = 0.0f;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) s += warp_part[w];
  return s;  // valid on thread 0
}

__global__ void __launch_bounds__(kSumsqThreads) sumsq_kernel(const uint16_t* __restrict__ x, int64_t n,
                                                               bool vec, float* __restrict__ partials) {
  constexpr int kThreads = kSumsqThreads;
  float acc = 0.0f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t n_vec = n / 8;
    for (int64_t iv = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; iv < n_vec; iv += stride) {
      float f[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(x) + iv), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = __fadd_rn(acc, __fmul_rn(f[k], f[k]));
    }
    tail_begin = n_vec * 8;
  }
  for (int64_t i = tail_begin + static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    const float f = bf16_to_f32(x[i]);
    acc = __fadd_rn(acc, __fmul_rn(f, f));
  }
  const float s = block_sum<kSumsqThreads>(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  if (blockIdx.x == 0)
    for (int i = gridDim.x + threadIdx.x; i < HOD_SUMSQ_PARTIALS; i += blockDim.x) partials[i] = 0.0f;
}

// Sum of squares of the PACKED gradient, read straight from the tensors (the
// values bf16_rne(src*scale) the bucket would hold; 0 in gaps) — d == 1 with
// clipping needs the norm before the fused pack+AdamW, and this pass costs
// 2 B/element instead of the 4 + 2 of pack-then-sumsq.  Fixed grid, fixed
// per-thread order => reproducible partials.
// kT threads per CTA: 1024 for full-GPU launches; 256 for co-resident ones
// (a 1024-thread CTA needs 31.7 K registers, more than the 22.5 K a GEMM CTA
// leaves on its SM).
template <typename SrcT, int kT = kSumsqThreads>
__global__ void __launch_bounds__(kT) pack_sumsq_kernel(const __grid_constant__ PackTable t,
                                                         int64_t numel, float scale,
                                                         float* __restrict__ partials,
                                                         int accumulate) {
  constexpr int kThreads = kT;
  constexpr int kPackTile = kT * kPackVec * kSumsqUnroll;
  pdl_trigger();  // the next bucket's norm pass writes other partial slots
  // 8 independent accumulators (one per vector lane), folded in a fixed order
  // at the end: breaks the serial FADD chain, stays reproducible
  float acc8[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  // a bf16 source times 1.0 is already its own bf16 rounding
  const bool exact = sizeof(SrcT) == 2 && scale == 1.0f;
  const int64_t n_tiles = (numel + kPackTile - 1) / kPackTile;
  int e = 0;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t a = tile * kPackTile;
    const int64_t b = min(a + kPackTile, numel);
    while (e < t.n && t.off[e] + t.numel[e] <= a) ++e;
    const bool inside = e < t.n && t.off[e] <= a && b <= t.off[e] + t.numel[e];
    if (inside && ((t.vec_ok >> e) & 1ull) && (b - a) == kPackTile) {
      const int64_t s0 = a - t.off[e];
#pragma unroll
      for (int u = 0; u < kSumsqUnroll; ++u) {
        float f[8];
        load8<SrcT>(t.src[e], s0 + (static_cast<int64_t>(u) * kThreads + threadIdx.x) * kPackVec, f);
        if (!exact) {
          // g = bf16_rne(src * scale), two at a time on the converter
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const uint32_t r = cvt_bf16x2_rn(__fmul_rn(f[k], scale), __fmul_rn(f[k + 1], scale));
            f[k] = __uint_as_float(r << 16);
            f[k + 1] = __uint_as_float(r & 0xffff0000u);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc8[k] = __fadd_rn(acc8[k], __fmul_rn(f[k], f[k]));
      }
    } else {
      int ei = e;
      for (int64_t i = a + threadIdx.x; i < b; i += kThreads) {
        while (ei < t.n && t.off[ei] + t.numel[ei] <= i) ++ei;
        if (ei < t.n && t.off[ei] <= i) {
          const float g = bf16_to_f32(f32_to_bf16(__fmul_rn(load_src<SrcT>(t.src[ei], i - t.off[ei]), scale)));
          acc8[0] = __fadd_rn(acc8[0], __fmul_rn(g, g));
        }
      }
    }
  }
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc = __fadd_rn(acc, acc8[k]);
  const float sblk = block_sum<kT>(acc);
  // windows after the first of a > HOD_PACK_MAX_ENTRIES table add onto the
  // partials of the windows before them (fixed window order: reproducible)
  if (threadIdx.x == 0) partials[blockIdx.x] = accumulate ? __fadd_rn(partials[blockIdx.x], sblk) : sblk;
  if (blockIdx.x == 0 && !accumulate)
    for (int i = gridDim.x + threadIdx.x; i < HOD_SUMSQ_PARTIALS; i += blockDim.x) partials[i] = 0.0f;
}

__global__ void sum_partials_kernel(const float* __restrict__ partials, int64_t n, float* out) {
  // one warp; lane-strided fp64 accumulation then a fixed shuffle tree
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 32) acc += static_cast<double>(partials[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) *out = static_cast<float>(acc);
}

// scratch of hod_sumsq (module-static: no runtime allocation by the library)
__device__ float g_sumsq_scratch[HOD_SUMSQ_PARTIALS];

__global__ void accumulate_partials_kernel(const float* __restrict__ partials, int64_t n, float* out) {
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 32) acc += static_cast<double>(partials[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) *out = __fadd_rn(*out, static_cast<float>(acc));
}

__global__ void clip_coef_kernel(const float* sumsq, float max_norm, float* coef, float* norm) {
  const float nrm = __fsqrt_rn(*sumsq);
  const float c = __fdiv_rn(max_norm, __fadd_rn(nrm, 1e-6f));
  *coef = c < 1.0f ? c : 1.0f;
  if (norm) *norm = nrm;
}

// Validate a pack table once on the host and split it into windows of at
// most HOD_PACK_MAX_ENTRIES entries; each window covers the destination range
// [lo, hi) from its first entry to the next window's first entry (the first
// window starts at 0, the last ends at bucket_numel, so gaps/padding are
// always covered).  `fn(table, lo, span)` launches one kernel per window.
template <typename Fn>
static int for_each_window(const char* who, const hod_pack_entry* entries, int n_entries,
                           int64_t bucket_numel, int src_dtype, Fn&& fn) {
  if (bucket_numel < 0 || n_entries < 0 || (n_entries > 0 && !entries)) {
    set_error("%s: bad arguments", who); return HOD_EINVAL;
  }
  if (src_dtype != HOD_DTYPE_BF16 && src_dtype != HOD_DTYPE_F32) {
    set_error("%s: unknown src_dtype %d", who, src_dtype); return HOD_EINVAL;
  }
  if (bucket_numel == 0) return HOD_OK;
  int64_t prev_end = 0;
  for (int i = 0; i < n_entries; ++i) {
    const hod_pack_entry& e = entries[i];
    // zero-element tensors (torch gives them a null data pointer) are allowed
    if ((e.numel > 0 && !e.src) || e.numel < 0 || e.dst_offset < prev_end || e.dst_offset + e.numel > bucket_numel) {
      set_error("%s: entry %d out of order or out of bounds", who, i); return HOD_EINVAL;
    }
    prev_end = e.dst_offset + e.numel;
  }
  // drop empty entries: they own no element (their range is padding), and a
  // zero-length entry may share its offset with the next tensor
  std::vector<hod_pack_entry> kept;
  kept.reserve(n_entries);
  for (int i = 0; i < n_entries; ++i)
    if (entries[i].numel > 0) kept.push_back(entries[i]);
  entries = kept.data();
  n_entries = static_cast<int>(kept.size());
  int first = 0;
  do {
    const int cnt = (n_entries - first) < HOD_PACK_MAX_ENTRIES ? (n_entries - first) : HOD_PACK_MAX_ENTRIES;
    const int64_t lo = (first == 0) ? 0 : entries[first].dst_offset;
    const int64_t hi = (first + cnt < n_entries) ? entries[first + cnt].dst_offset : bucket_numel;
    PackTable t;
    memset(&t, 0, sizeof(t));
    t.n = cnt;
    for (int i = 0; i < cnt; ++i) {
      const hod_pack_entry& e = entries[first + i];
      t.off[i] = e.dst_offset - lo;
      t.numel[i] = e.numel;
      t.src[i] = e.src;
      // the vector paths read 8 elements at (tile_start - off): needs off % 8 == 0
      if (aligned16(e.src) && ((e.dst_offset - lo) % 8 == 0)) t.vec_ok |= (1ull << i);
    }
    if (hi - lo > 0) {
      if (lo % 8) { set_error("%s: window start %lld not a multiple of 8", who, (long long)lo); return HOD_EALIGN; }
      const int rc = fn(t, lo, hi - lo);
      if (rc) return rc;
    }
    first += cnt;
  } while (first < n_entries);
  return HOD_OK;
}

}  // namespace hod

using namespace hod;

extern "C" {

int hod_abi_version(void) { return HOD_ABI_VERSION; }

const char* hod_last_error(void) { return g_err; }

long long hod_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int hod_set_grid_limit(int max_ctas) {
  if (max_ctas < 0) { set_error("hod_set_grid_limit: negative limit"); return HOD_EINVAL; }
  g_grid_limit.store(max_ctas, std::memory_order_relaxed);
  return HOD_OK;
}

int hod_pack_bf16(const hod_pack_entry* entries, int n_entries, uint16_t* bucket,
                  int64_t bucket_numel, float scale, int src_dtype, void* stream) {
  if (!bucket) { set_error("hod_pack_bf16: bad arguments"); return HOD_EINVAL; }
  if (!aligned16(bucket)) { set_error("hod_pack_bf16: bucket not 16-byte aligned"); return HOD_EALIGN; }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return for_each_window("hod_pack_bf16", entries, n_entries, bucket_numel, src_dtype,
                         [&](const PackTable& t, int64_t lo, int64_t span) {
    if (!aligned16(bucket + lo)) {
      set_error("hod_pack_bf16: window start %lld not 16-byte aligned", (long long)lo); return HOD_EALIGN;
    }
    // measured best (unroll 8): 16 CTAs/SM cap for bf16 sources (6.2 TB/s), 3 for fp32 (6.6 TB/s)
    const int grid = grid_for((span + kPackTile - 1) / kPackTile, 1, src_dtype == HOD_DTYPE_BF16 ? 16 : 3);
    count_launch(1);
    const bool gentle = coresident() && pack_gentle();
    if (src_dtype == HOD_DTYPE_BF16) {
      if (gentle) launch_pdl(pack_kernel<uint16_t, 2>, grid, kThreads, s, t, bucket + lo, span, scale);
      else launch_pdl(pack_kernel<uint16_t>, grid, kThreads, s, t, bucket + lo, span, scale);
    } else {
      if (gentle) launch_pdl(pack_kernel<float, 2>, grid, kThreads, s, t, bucket + lo, span, scale);
      else launch_pdl(pack_kernel<float>, grid, kThreads, s, t, bucket + lo, span, scale);
    }
    return cuda_status(cudaGetLastError(), "hod_pack_bf16 launch");
  });
}

int hod_pack_adamw(const hod_pack_entry* entries, int n_entries, int64_t bucket_numel, float scale,
                   int src_dtype, float* master, float* exp_avg, float* exp_avg_sq, uint16_t* param,
                   const hod_adamw_params* hp, const float* clip_coef, void* stream) {
  if (!master || !exp_avg || !exp_avg_sq || !param || !hp) {
    set_error("hod_pack_adamw: bad arguments"); return HOD_EINVAL;
  }
  if (hp->step < 1) { set_error("hod_pack_adamw: step must be >= 1"); return HOD_EINVAL; }
  if (!aligned16(master) || !aligned16(exp_avg) || !aligned16(exp_avg_sq) || !aligned16(param)) {
    set_error("hod_pack_adamw: state/param buffers must be 16-byte aligned"); return HOD_EALIGN;
  }
  const AdamWConsts c = fold_adamw(*hp);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return for_each_window("hod_pack_adamw", entries, n_entries, bucket_numel, src_dtype,
                         [&](const PackTable& t, int64_t lo, int64_t span) {
    // 3 CTAs/SM measured best for this kernel (2: -9 %, 4: -9 %; tools/sweep_grid.sh)
    const int grid = grid_for((span + kChunk - 1) / kChunk * 32, kThreads, 3);
    count_launch(1);
    // PDL: may overlap the tail of the previous kernel in the stream only if
    // that kernel triggered early — our own bucket kernels (disjoint memory);
    // anything else (clip_coef_kernel writing the coefficient read here)
    // triggers at completion, so that dependency holds
    float* mp = master + lo;
    float* ep = exp_avg + lo;
    float* vp = exp_avg_sq + lo;
    uint16_t* pp = param + lo;
#define HOD_PA_LAUNCH(T, CLIP, FAST) \
    launch_pdl(pack_adamw_kernel<T, CLIP, FAST>, grid, kThreads, s, t, span, scale, mp, ep, vp, pp, c, clip_coef)
#define HOD_PA_FAST(T, CLIP) \
    do { if (c.fast) HOD_PA_LAUNCH(T, CLIP, true); else HOD_PA_LAUNCH(T, CLIP, false); } while (0)
    if (src_dtype == HOD_DTYPE_BF16) {
      if (clip_coef) HOD_PA_FAST(uint16_t, true); else HOD_PA_FAST(uint16_t, false);
    } else {
      if (clip_coef) HOD_PA_FAST(float, true); else HOD_PA_FAST(float, false);
    }
#undef HOD_PA_FAST
#undef HOD_PA_LAUNCH
    return cuda_status(cudaGetLastError(), "hod_pack_adamw launch");
  });
}

int hod_pack_sumsq(const hod_pack_entry* entries, int n_entries, int64_t bucket_numel, float scale,
                   int src_dtype, float* partials, void* stream) {
  if (!partials) { set_error("hod_pack_sumsq: null partials"); return HOD_EINVAL; }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bucket_numel == 0) return hod_sumsq_bf16(nullptr, 0, partials, stream);
  int window = 0;
  return for_each_window("hod_pack_sumsq", entries, n_entries, bucket_numel, src_dtype,
                         [&](const PackTable& t, int64_t lo, int64_t span) {
    count_launch(1);
    // window 0 writes the fixed-grid partials; later windows of a long table
    // accumulate onto them, so they must see window 0's result: full stream
    // dependency (no PDL) for them.  Every window triggers its own dependents
    // at entry: the next bucket's norm pass writes other partial slots.
    const int acc = window++ > 0;
    const int grid = partials_grid();
    if (coresident()) {
      if (src_dtype == HOD_DTYPE_BF16) {
        if (!acc) launch_pdl(pack_sumsq_kernel<uint16_t, 256>, grid, 256, s, t, span, scale, partials, 0);
        else launch(pack_sumsq_kernel<uint16_t, 256>, grid, 256, 0, s, t, span, scale, partials, 1);
      } else {
        if (!acc) launch_pdl(pack_sumsq_kernel<float, 256>, grid, 256, s, t, span, scale, partials, 0);
        else launch(pack_sumsq_kernel<float, 256>, grid, 256, 0, s, t, span, scale, partials, 1);
      }
    } else if (!acc) {
      if (src_dtype == HOD_DTYPE_BF16)
        launch_pdl(pack_sumsq_kernel<uint16_t>, grid, kSumsqThreads, s, t, span, scale, partials, 0);
      else
        launch_pdl(pack_sumsq_kernel<float>, grid, kSumsqThreads, s, t, span, scale, partials, 0);
    } else if (src_dtype == HOD_DTYPE_BF16) {
      launch(pack_sumsq_kernel<uint16_t>, grid, kSumsqThreads, 0, s, t, span, scale, partials, 1);
    } else {
      launch(pack_sumsq_kernel<float>, grid, kSumsqThreads, 0, s, t, span, scale, partials, 1);
    }
    (void)lo;
    return cuda_status(cudaGetLastError(), "hod_pack_sumsq launch");
  });
}

int hod_sumsq_bf16(const uint16_t* x, int64_t n, float* partials, void* stream) {
  if (!partials || n < 0 || (n > 0 && !x)) { set_error("hod_sumsq_bf16: bad arguments"); return HOD_EINVAL; }
  count_launch(1);
  launch(sumsq_kernel, partials_grid(), kSumsqThreads, 0, static_cast<cudaStream_t>(stream), x, n, aligned16(x), partials);
  return cuda_status(cudaGetLastError(), "hod_sumsq_bf16 launch");
}

int hod_sumsq(const uint16_t* x, int64_t n, float* out, void* stream) {
  if (!out || n < 0 || (n > 0 && !x)) { set_error("hod_sumsq: bad arguments"); return HOD_EINVAL; }
  float* scratch = nullptr;
  int rc = cuda_status(cudaGetSymbolAddress(reinterpret_cast<void**>(&scratch), g_sumsq_scratch),
                       "hod_sumsq scratch");
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  count_launch(2);
  launch(sumsq_kernel, partials_grid(), kSumsqThreads, 0, s, x, n, aligned16(x), scratch);
  launch(accumulate_partials_kernel, 1, 32, 0, s, scratch, HOD_SUMSQ_PARTIALS, out);
  return cuda_status(cudaGetLastError(), "hod_sumsq launch");
}

int hod_adamw(float* master, float* exp_avg, float* exp_avg_sq, const uint16_t* grad, uint16_t* param,
              int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay, int64_t step,
              const float* clip_coef, void* stream) {
  const hod_adamw_params hp{lr, beta1, beta2, eps, weight_decay, step};
  return hod_adamw_bf16(master, exp_avg, exp_avg_sq, grad, param, n, &hp, clip_coef, stream);
}

int hod_sum_partials(const float* partials, int64_t n_partials, float* out, void* stream) {
  if (!partials || !out || n_partials < 0) { set_error("hod_sum_partials: bad arguments"); return HOD_EINVAL; }
  count_launch(1);
  launch(sum_partials_kernel, 1, 32, 0, static_cast<cudaStream_t>(stream), partials, n_partials, out);
  return cuda_status(cudaGetLastError(), "hod_sum_partials launch");
}

int hod_clip_coef(const float* sumsq, float max_norm, float* coef, float* norm, void* stream) {
  if (!sumsq || !coef || !(max_norm > 0.0f)) { set_error("hod_clip_coef: bad arguments"); return HOD_EINVAL; }
  count_launch(1);
  launch(clip_coef_kernel, 1, 1, 0, static_cast<cudaStream_t>(stream), sumsq, max_norm, coef, norm);
  return cuda_status(cudaGetLastError(), "hod_clip_coef launch");
}

int hod_adamw_bf16(float* master, float* exp_avg, float* exp_avg_sq, const uint16_t* grad,
                   uint16_t* param, int64_t n, const hod_adamw_params* hp, const float* clip_coef,
                   void* stream) {
  return launch_adamw<uint16_t>(master, exp_avg, exp_avg_sq, grad, param, n, hp, clip_coef,
                                static_cast<cudaStream_t>(stream));
}

int hod_adamw_f32(float* master, float* exp_avg, float* exp_avg_sq, const float* grad,
                  uint16_t* param, int64_t n, const hod_adamw_params* hp, const float* clip_coef,
                  void* stream) {
  return launch_adamw<float>(master, exp_avg, exp_avg_sq, grad, param, n, hp, clip_coef,
                             static_cast<cudaStream_t>(stream));
}

}  // extern "C"
