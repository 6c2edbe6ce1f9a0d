// peer_bw.cu — SM-issued NVLink bandwidth ceiling (measurement tool, not product).
//
// Each thread pulls VEC bytes per peer per unrolled step from the d peer-mapped
// buffers (rank-r shard region, like the RS kernel) and folds them with XOR
// into a local output so the loads stay live.  Built by tools/peer_bw.py:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <stdint.h>

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
