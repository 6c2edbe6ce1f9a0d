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
  } else {
    if (vec == 16) peer_write<16><<<grid, 256, 0, s>>>(ps, d, off, bytes);
    else peer_write<8><<<grid, 256, 0, s>>>(ps, d, off, bytes);
  }
  return static_cast<int>(cudaGetLastError());
}
