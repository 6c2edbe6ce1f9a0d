// peer_bw.cu — SM-issued NVLink bandwidth ceiling (measurement tool, not product).
//
// Each thread pulls VEC bytes per peer per unrolled step from the d peer-mapped
// buffers (rank-r shard region, like the RS kernel) and folds them with XOR
// into a local output so the loads stay live.  Built by tools/peer_bw.py:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

struct Peers { const uint8_t* p[8]; };

template <int VEC, int U>
__global__ void __launch_bounds__(256) peer_read(Peers ps, int d, int64_t off, int64_t bytes, uint8_t* out) {
  using V = typename std::conditional<VEC == 16, uint4, uint2>::type;
  const int64_t n = bytes / VEC;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride * U) {
    V v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < d && i + u * stride < n)
          v[u][q] = reinterpret_cast<const V*>(ps.p[q] + off)[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < d && i + u * stride < n) {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[u][q]);
#pragma unroll
          for (int k = 0; k < VEC / 4; ++k) acc ^= w[k];
        }
  }
  if (acc == 0x12345678u) out[0] = 1;  // practically never; keeps loads live
}

// push: each thread stores VEC bytes to every peer (AG pattern)
template <int VEC>
__global__ void __launch_bounds__(256) peer_write(Peers ps, int d, int64_t off, int64_t bytes) {
  using V = typename std::conditional<VEC == 16, uint4, uint2>::type;
  const int64_t n = bytes / VEC;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  V z{};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < d) reinterpret_cast<V*>(const_cast<uint8_t*>(ps.p[q]) + off)[i] = z;
}

// both: each thread pulls VEC bytes of its shard from every peer (RS) and
// stores VEC bytes to every peer's second region (AG) — the fused p2p mix
template <int VEC>
__global__ void __launch_bounds__(256) peer_both(Peers ps, int d, int64_t off, int64_t off2, int64_t bytes,
                                                 uint8_t* out) {
  using V = typename std::conditional<VEC == 16, uint4, uint2>::type;
  const int64_t n = bytes / VEC;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    V v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < d) v[q] = reinterpret_cast<const V*>(ps.p[q] + off)[i];
    V s = v[0];
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < d) s.x ^= v[q].x;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < d) reinterpret_cast<V*>(const_cast<uint8_t*>(ps.p[q]) + off2)[i] = s;
    acc ^= s.y;
  }
  if (acc == 0x12345678u) out[0] = 1;
}

extern "C" int peer_bw_run(const void* const* ptrs, int d, int64_t off, int64_t bytes, void* out, int mode,
                           int vec, int unroll, int grid, void* stream) {
  Peers ps{};
  for (int q = 0; q < d && q < 8; ++q) ps.p[q] = static_cast<const uint8_t*>(ptrs[q]);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* o = static_cast<uint8_t*>(out);
  if (mode == 0) {
    if (vec == 16) {
      if (unroll == 1) peer_read<16, 1><<<grid, 256, 0, s>>>(ps, d, off, bytes, o);
      else if (unroll == 2) peer_read<16, 2><<<grid, 256, 0, s>>>(ps, d, off, bytes, o);
      else peer_read<16, 4><<<grid, 256, 0, s>>>(ps, d, off, bytes, o);
    } else {
      if (unroll == 1) peer_read<8, 1><<<grid, 256, 0, s>>>(ps, d, off, bytes, o);
      else if (unroll == 2) peer_read<8, 2><<<grid, 256, 0, s>>>(ps, d, off, bytes, o);
      else peer_read<8, 4><<<grid, 256, 0, s>>>(ps, d, off, bytes, o);
    }
  } else if (mode == 1) {
    if (vec == 16) peer_write<16><<<grid, 256, 0, s>>>(ps, d, off, bytes);
    else peer_write<8><<<grid, 256, 0, s>>>(ps, d, off, bytes);
  } else {
    // mode 5: both (second region at off + d * bytes)
    if (vec == 16) peer_both<16><<<grid, 256, 0, s>>>(ps, d, off, off + d * bytes, bytes, o);
    else peer_both<8><<<grid, 256, 0, s>>>(ps, d, off, off + d * bytes, bytes, o);
  }
  return static_cast<int>(cudaGetLastError());
}

// NVLS through the multicast address: ld_reduce (RS pattern: the switch reads
// every copy and returns the bf16 sum), multimem.st (AG pattern: one store,
// the switch replicates), or both per thread (the fused span kernel's mix).
template <int VEC>
__device__ __forceinline__ void mc_ld_reduce(const uint8_t* p, uint32_t* r) {
  if constexpr (VEC == 16) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p) : "memory");
  } else {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v2.bf16x2 {%0, %1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1]) : "l"(p) : "memory");
  }
}

template <int VEC>
__device__ __forceinline__ void mc_store(uint8_t* p, const uint32_t* r) {
  if constexpr (VEC == 16) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "f"(__uint_as_float(r[0])), "f"(__uint_as_float(r[1])), "f"(__uint_as_float(r[2])),
                 "f"(__uint_as_float(r[3])) : "memory");
  } else {
    asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(p),
                 "f"(__uint_as_float(r[0])), "f"(__uint_as_float(r[1])) : "memory");
  }
}

// what: 1 = ld_reduce, 2 = store, 3 = both (load from off, store to off2)
template <int VEC, int U, int WHAT>
__global__ void __launch_bounds__(256) nvls_kernel(uint8_t* mc, int64_t off, int64_t off2, int64_t bytes,
                                                   uint8_t* out) {
  const int64_t n = bytes / VEC;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride * U) {
    uint32_t r[U][4] = {};
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((WHAT & 1) && i + u * stride < n) mc_ld_reduce<VEC>(mc + off + (i + u * stride) * VEC, r[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) {
        if (WHAT & 2) mc_store<VEC>(mc + off2 + (i + u * stride) * VEC, r[u]);
        else acc ^= r[u][0] ^ r[u][1];
      }
  }
  if (acc == 0x12345678u) out[0] = 1;
}

template <int VEC, int WHAT>
static void nvls_launch(uint8_t* mc, int64_t off, int64_t off2, int64_t bytes, uint8_t* o, int unroll, int grid,
                        cudaStream_t s) {
  if (unroll == 1) nvls_kernel<VEC, 1, WHAT><<<grid, 256, 0, s>>>(mc, off, off2, bytes, o);
  else if (unroll == 2) nvls_kernel<VEC, 2, WHAT><<<grid, 256, 0, s>>>(mc, off, off2, bytes, o);
  else nvls_kernel<VEC, 4, WHAT><<<grid, 256, 0, s>>>(mc, off, off2, bytes, o);
}

// mode 2/3/4 = nvls ld_reduce / store / both; ptr = multicast base
extern "C" int nvls_bw_run(void* mc, int64_t off, int64_t off2, int64_t bytes, void* out, int mode, int vec,
                           int unroll, int grid, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* m = static_cast<uint8_t*>(mc);
  uint8_t* o = static_cast<uint8_t*>(out);
  const int what = mode - 1;
  if (vec == 16) {
    if (what == 1) nvls_launch<16, 1>(m, off, off2, bytes, o, unroll, grid, s);
    else if (what == 2) nvls_launch<16, 2>(m, off, off2, bytes, o, unroll, grid, s);
    else nvls_launch<16, 3>(m, off, off2, bytes, o, unroll, grid, s);
  } else {
    if (what == 1) nvls_launch<8, 1>(m, off, off2, bytes, o, unroll, grid, s);
    else if (what == 2) nvls_launch<8, 2>(m, off, off2, bytes, o, unroll, grid, s);
    else nvls_launch<8, 3>(m, off, off2, bytes, o, unroll, grid, s);
  }
  return static_cast<int>(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// TMA modes: one elected thread per CTA moves whole tiles with the bulk-copy
// engine (cp.async.bulk) from the d peers' buffers into a STAGES-deep
// shared-memory ring (mbarrier complete_tx); the CTA's threads XOR-fold the d
// tiles (the reduce-scatter's read pattern) and, for "both", bulk-store the
// folded tile to every peer's second region (the all-gather's write pattern).
// Bytes in flight per CTA = STAGES * d * tile, independent of registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred done;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n@!done bra W_%=;\n}\n"
               ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)), "r"(bytes)
               : "memory");
}

template <int STAGES, bool BOTH>
__global__ void __launch_bounds__(256) tma_kernel(Peers ps, int d, int64_t off, int64_t off2, int64_t bytes,
                                                  int tile, uint8_t* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* in = smem;                                        // [STAGES][d][tile]
  uint8_t* red = smem + static_cast<int64_t>(STAGES) * d * tile;   // [STAGES][tile] (BOTH)
  uint64_t* full = reinterpret_cast<uint64_t*>(red + (BOTH ? STAGES * tile : 0));
  const int64_t n_tiles = bytes / tile;
  const int64_t mine = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mb_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t i) {
    const int s = static_cast<int>(i % STAGES);
    const int64_t t = blockIdx.x + i * gridDim.x;
    mb_expect(&full[s], static_cast<uint32_t>(d * tile));
    for (int q = 0; q < d; ++q)
      g2s(in + (static_cast<int64_t>(s) * d + q) * tile, ps.p[q] + off + t * tile, tile, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < mine && i < STAGES; ++i) issue(i);
  uint32_t acc = 0;
  for (int64_t i = 0; i < mine; ++i) {
    const int s = static_cast<int>(i % STAGES);
    if (BOTH && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    mb_wait(&full[s], static_cast<uint32_t>((i / STAGES) & 1));
    const uint4* src = reinterpret_cast<const uint4*>(in + static_cast<int64_t>(s) * d * tile);
    const int words = tile / 16;
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
      uint4 x = src[w];
      for (int q = 1; q < d; ++q) {
        const uint4 y = src[q * words + w];
        x.x ^= y.x; x.y ^= y.y; x.z ^= y.z; x.w ^= y.w;
      }
      if (BOTH) reinterpret_cast<uint4*>(red + static_cast<int64_t>(s) * tile)[w] = x;
      else acc ^= x.x ^ x.w;
    }
    if (BOTH) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      if (BOTH) {
        const int64_t t = blockIdx.x + i * gridDim.x;
        for (int q = 0; q < d; ++q)
          s2g(const_cast<uint8_t*>(ps.p[q]) + off2 + t * tile, red + static_cast<int64_t>(s) * tile, tile);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (i + STAGES < mine) issue(i + STAGES);
    }
  }
  if (BOTH && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 0x12345678u) out[0] = 1;
}

// mode 6 = tma read, 7 = tma both; `vec` carries the tile bytes per peer, `unroll` the stages
extern "C" int tma_bw_run(const void* const* ptrs, int d, int64_t off, int64_t bytes, void* out, int mode,
                          int tile, int stages, int grid, void* stream) {
  Peers ps{};
  for (int q = 0; q < d && q < 8; ++q) ps.p[q] = static_cast<const uint8_t*>(ptrs[q]);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* o = static_cast<uint8_t*>(out);
  const bool both = mode == 7;
  const int smem = stages * d * tile + (both ? stages * tile : 0) + stages * 8;
#define TMA_L(ST, B)                                                                                  \
  do {                                                                                                \
    cudaFuncSetAttribute(tma_kernel<ST, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);      \
    tma_kernel<ST, B><<<grid, 256, smem, s>>>(ps, d, off, off + d * bytes, bytes, tile, o);           \
  } while (0)
  if (stages == 2) { if (both) TMA_L(2, true); else TMA_L(2, false); }
  else if (stages == 3) { if (both) TMA_L(3, true); else TMA_L(3, false); }
  else { if (both) TMA_L(4, true); else TMA_L(4, false); }
#undef TMA_L
  return static_cast<int>(cudaGetLastError());
}
