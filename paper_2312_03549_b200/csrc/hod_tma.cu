// hod_tma.cu — SM-light, TMA-fed AdamW for overlap with compute (sm_100a).
//
// The register-streaming kernels (hod_kernels.cu) need the whole GPU to reach
// HBM peak: bytes in flight per SM are capped by registers.  Here one elected
// producer thread per CTA moves whole 2048-element chunks with the Tensor
// Memory Accelerator (cp.async.bulk, SASS UBLKCP) into a 6-stage shared-memory
// ring (mbarrier complete_tx), four consumer warps update them in shared
// memory, and the results leave with bulk stores (cp.async.bulk ...bulk_group)
// — ~170 KB in flight per SM from 160 threads, so a few dozen CTAs can stream
// at HBM speed while the rest of the SMs run the backward GEMMs.
//
// Arithmetic and element order are identical to adamw_vec_kernel (same
// adamw_elem, same rounding): results are bit-identical.
#include <stdint.h>
#include <string.h>

#include "hod_common.cuh"

namespace hod {

constexpr int kTmaChunk = 2048;                  // elements per stage
constexpr int kTmaStages = 5;
constexpr int kTmaConsumers = 256;               // 8 warps
constexpr int kTmaThreads = kTmaConsumers + 32;  // + 1 producer warp

struct TmaStage {
  float p[kTmaChunk];
  float m[kTmaChunk];
  float v[kTmaChunk];
  uint16_t g[kTmaChunk];
  uint16_t out[kTmaChunk];
};
constexpr int kTmaSmem = kTmaStages * sizeof(TmaStage) + 2 * kTmaStages * 8 + 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
}

template <bool kClip>
__global__ void __launch_bounds__(kTmaThreads, 1) tma_adamw_kernel(
    float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
    const uint16_t* __restrict__ g, uint16_t* __restrict__ out, int64_t n_chunks, const AdamWConsts c,
    const float* __restrict__ coef_ptr) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TmaStage* st = reinterpret_cast<TmaStage*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + kTmaStages * sizeof(TmaStage));
  uint64_t* empty = full + kTmaStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t my_chunks = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x >= kTmaConsumers) {
    // ---- producer warp: one elected lane streams chunks into the ring
    if (threadIdx.x == kTmaConsumers) {
      for (int64_t i = 0; i < my_chunks; ++i) {
        const int s = static_cast<int>(i % kTmaStages);
        if (i >= kTmaStages) mbar_wait(&empty[s], static_cast<uint32_t>(((i / kTmaStages) - 1) & 1));
        const int64_t base = (blockIdx.x + i * gridDim.x) * kTmaChunk;
        mbar_expect_tx(&full[s], 3 * kTmaChunk * 4 + kTmaChunk * 2);
        bulk_g2s(st[s].p, p + base, kTmaChunk * 4, &full[s]);
        bulk_g2s(st[s].m, m + base, kTmaChunk * 4, &full[s]);
        bulk_g2s(st[s].v, v + base, kTmaChunk * 4, &full[s]);
        bulk_g2s(st[s].g, g + base, kTmaChunk * 2, &full[s]);
      }
    }
    return;
  }
  // ---- consumers: update in shared memory, bulk-store the results
  const float coef = kClip ? __ldg(coef_ptr) : 1.0f;
  for (int64_t i = 0; i < my_chunks; ++i) {
    const int s = static_cast<int>(i % kTmaStages);
    mbar_wait(&full[s], static_cast<uint32_t>((i / kTmaStages) & 1));
    TmaStage& S = st[s];
#pragma unroll 4
    for (int k = threadIdx.x; k < kTmaChunk; k += kTmaConsumers) {
      float gk = bf16_to_f32(S.g[k]);
      if (kClip) gk = __fmul_rn(gk, coef);
      float pk = S.p[k], mk = S.m[k], vk = S.v[k];
      adamw_elem(pk, mk, vk, gk, c);
      S.p[k] = pk;
      S.m[k] = mk;
      S.v[k] = vk;
      S.out[k] = f32_to_bf16(pk);
    }
    fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk-copy engine
    consumers_sync();
    if (threadIdx.x == 0) {
      const int64_t base = (blockIdx.x + i * gridDim.x) * kTmaChunk;
      bulk_s2g(p + base, S.p, kTmaChunk * 4);
      bulk_s2g(m + base, S.m, kTmaChunk * 4);
      bulk_s2g(v + base, S.v, kTmaChunk * 4);
      bulk_s2g(out + base, S.out, kTmaChunk * 2);
      bulk_commit();
      // release the stage only once its stores have read it; keeping up to
      // kTmaStages-2 store groups in flight overlaps them with the next loads
      bulk_wait_read<kTmaStages - 2>();
      if (i >= kTmaStages - 2) mbar_arrive(&empty[(i - (kTmaStages - 2)) % kTmaStages]);
    }
  }
  if (threadIdx.x == 0) {
    bulk_wait_all();
    // (remaining stages need no release: the producer is done)
  }
}

}  // namespace hod

using namespace hod;

extern "C" {

int hod_adamw_tma(float* master, float* exp_avg, float* exp_avg_sq, const uint16_t* grad, uint16_t* param,
                  int64_t n, const hod_adamw_params* hp, const float* clip_coef, int max_ctas, void* stream) {
  if (!master || !exp_avg || !exp_avg_sq || !grad || !param || !hp || n < 0) {
    set_error("hod_adamw_tma: bad arguments"); return HOD_EINVAL;
  }
  if (hp->step < 1) { set_error("hod_adamw_tma: step must be >= 1"); return HOD_EINVAL; }
  if (!aligned16(master) || !aligned16(exp_avg) || !aligned16(exp_avg_sq) || !aligned16(grad) || !aligned16(param)) {
    set_error("hod_adamw_tma: buffers must be 16-byte aligned"); return HOD_EALIGN;
  }
  const AdamWConsts c = fold_adamw(*hp);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n_chunks = n / kTmaChunk;
  if (n_chunks > 0) {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(tma_adamw_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
      cudaFuncSetAttribute(tma_adamw_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
      configured = true;
    }
    int grid = max_ctas > 0 ? max_ctas : kSMs;
    if (grid_limit() > 0 && grid_limit() < grid) grid = grid_limit();
    if (grid > n_chunks) grid = static_cast<int>(n_chunks);
    count_launch(1);
    if (clip_coef)
      tma_adamw_kernel<true><<<grid, kTmaThreads, kTmaSmem, s>>>(master, exp_avg, exp_avg_sq, grad, param, n_chunks, c, clip_coef);
    else
      tma_adamw_kernel<false><<<grid, kTmaThreads, kTmaSmem, s>>>(master, exp_avg, exp_avg_sq, grad, param, n_chunks, c, nullptr);
    const int rc = cuda_status(cudaGetLastError(), "hod_adamw_tma launch");
    if (rc) return rc;
  }
  const int64_t done = n_chunks * kTmaChunk;
  if (done < n)
    return hod_adamw_bf16(master + done, exp_avg + done, exp_avg_sq + done, grad + done, param + done, n - done,
                          hp, clip_coef, stream);
  return HOD_OK;
}

}  // extern "C"
