// Pooling kernels of the multi-device group (csrc/group.cpp): per-trajectory
// records summed over the ensemble into one contiguous u64 vector, the buffer
// the group's single NCCL all-reduce then sums over devices.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace pbn_b200 {

// out[f] = sum_t counts[t * 8 + f] for f < 8 (one thread per (trajectory,
// field) pair; warp-reduced, one atomic per warp and field).
__global__ void pbn_pool_counts_kernel(const std::uint64_t* __restrict__ counts, std::uint32_t n,
                                       unsigned long long* __restrict__ out) {
  const std::uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    unsigned long long v = t < n ? counts[static_cast<std::uint64_t>(t) * 8 + f] : 0ull;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + f, v);
  }
}

// out[c] += sum over rows r of nc[r * cols + c]: per-node one-counts of the
// ensemble (engine.hpp:378-379 summed over trajectories). A thread owns one
// column of a slab of rows, so each warp reads 32 consecutive u64 of a row.
__global__ void pbn_pool_node_counts_kernel(const std::uint64_t* __restrict__ nc,
                                            std::uint32_t rows, std::uint32_t cols,
                                            std::uint32_t rows_per_slab,
                                            unsigned long long* __restrict__ out) {
  const std::uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const std::uint32_t r0 = blockIdx.y * rows_per_slab;
  const std::uint32_t r1 = min(rows, r0 + rows_per_slab);
  unsigned long long s = 0;
  for (std::uint32_t r = r0; r < r1; ++r) s += nc[static_cast<std::uint64_t>(r) * cols + c];
  if (s) atomicAdd(out + c, s);
}

// d_out[0..8) = pooled counts, d_out[8..8+cols) = pooled node counts (when
// d_nc != nullptr). Zeroes d_out first; asynchronous on `stream`.
cudaError_t launch_pool(const std::uint64_t* d_counts, const std::uint64_t* d_nc, std::uint32_t n,
                        std::uint32_t cols, unsigned long long* d_out, cudaStream_t stream) {
  const std::size_t len = 8 + (d_nc ? cols : 0);
  cudaError_t e = cudaMemsetAsync(d_out, 0, len * sizeof(unsigned long long), stream);
  if (e != cudaSuccess || n == 0) return e;
  pbn_pool_counts_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_counts, n, d_out);
  if (d_nc && cols) {
    const std::uint32_t slab = std::max<std::uint32_t>(64, (n + 65534) / 65535);  // grid.y <= 65535
    const dim3 grid((cols + 255) / 256, (n + slab - 1) / slab);
    pbn_pool_node_counts_kernel<<<grid, 256, 0, stream>>>(d_nc, n, cols, slab, d_out + 8);
  }
  return cudaGetLastError();
}

}  // namespace pbn_b200
