// Measured ceilings for the trajectory kernels (VERDICT r01 "measure the two
// ceilings on the B200 instead of asserting them"):
//
//  1. philox  — a kernel that does nothing but generate the injected stream:
//     the product's own Philox4x32-10 (csrc/device/philox.cuh: per-step
//     hoisted rounds), one trajectory per warp like the headline kernel
//     (28 warps x 148 CTAs), each lane producing `blocks` blocks per step.
//     Reports blocks/s and issued warp-instructions per block (the kernel's
//     own SASS count / block, from clock64 and the issue rate), so the
//     stream-only ceiling of a workload = issue peak / (its blocks per step).
//  2. probe   — shared-memory random probes: every lane of 32 warps per SM
//     reads 4-byte entries of a 128 KiB table at pseudo-random indices
//     (8 pointer-chasing chains per thread). Two layouts: `random`
//     (any bank: the ~3.5-way expected max bank load of SURVEY §7 hard
//     part 6) and `column` (lane-private bank: conflict-free by
//     construction). Reports probes per clock per SM against the 32/clk
//     peak the lookup roofline assumes.
//
// Build: make -C tools ceilings  (nvcc, sm_100a) -> tools/bin/ceilings
// Run:   tools/bin/ceilings  -> one JSON line per measurement
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_1605_00854_b200/csrc/device/philox.cuh"

using namespace pbn_b200;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

__global__ void __launch_bounds__(28 * 32, 1)
    philox_only(std::uint32_t steps, std::uint32_t blocks, std::uint32_t seed,
                std::uint32_t* out) {
  std::uint32_t rk0[10], rk1[10];
  rk0[0] = seed;
  rk1[0] = seed * 0x9E3779B9u;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    rk0[r] = rk0[r - 1] + 0x9E3779B9u;
    rk1[r] = rk1[r - 1] + 0xBB67AE85u;
  }
  const std::uint32_t lane = threadIdx.x & 31;
  const std::uint32_t traj = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  std::uint32_t thi, tlo;
  mulhilo(kPhiloxM0, traj, thi, tlo);
  std::uint32_t acc = 0;
  for (std::uint32_t s = 0; s < steps; ++s) {
    const step_philox sp = make_step_philox(thi, tlo, s, rk0, rk1);
    for (std::uint32_t b = lane; b < blocks; b += 32) {
      const uint4 x = philox_block(sp, b, rk0, rk1);
      acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <bool COLUMN>
__global__ void __launch_bounds__(1024, 1)
    smem_probe(std::uint32_t iters, std::uint32_t* out, unsigned long long* clk) {
  // pointer chasing through the table: every entry holds the byte offset of
  // a pseudo-random entry (random: any word; column: the first word of a
  // random 128-byte row, which the lane offsets into its own bank), so a
  // probe is one LDS (+ one IADD for column) and 8 chains per thread keep
  // the shared-memory pipe, not latency or issue, the limit
  extern __shared__ std::uint32_t tab[];
  constexpr std::uint32_t kEntries = 32768;  // 128 KiB
  for (std::uint32_t i = threadIdx.x; i < kEntries; i += blockDim.x) {
    std::uint32_t h = i * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    tab[i] = COLUMN ? ((h & (kEntries - 1)) & ~31u) * 4u : (h & (kEntries - 1)) * 4u;
  }
  __syncthreads();
  const std::uint32_t lane4 = (threadIdx.x & 31) * 4;
  const char* base = reinterpret_cast<const char*>(tab);
  std::uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = ((threadIdx.x * 8 + c) * 131u & (kEntries - 1) & ~31u) * 4u;
  const unsigned long long t0 = clock64();
  for (std::uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      x[c] = *reinterpret_cast<const std::uint32_t*>(base + (COLUMN ? x[c] + lane4 : x[c]));
  }
  const unsigned long long t1 = clock64();
  std::uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, mhz_khz = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&mhz_khz, cudaDevAttrClockRate, dev));
  std::uint32_t* out = nullptr;
  unsigned long long* clk = nullptr;
  CK(cudaMalloc(&out, sizeof(std::uint32_t) * sms * 1024));
  CK(cudaMalloc(&clk, sizeof(unsigned long long) * sms));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // ---- 1. Philox-only, one trajectory per warp, 4144 warps (c2: 4096)
  const std::uint32_t grid = sms, threads = 28 * 32;
  const std::uint32_t traj = grid * (threads / 32);
  for (std::uint32_t blocks : {32u, 64u, 128u, 416u}) {
    const std::uint32_t steps = 400000u / blocks * 32u / 32u;
    philox_only<<<grid, threads>>>(16, blocks, 1, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    philox_only<<<grid, threads>>>(steps, blocks, 7, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double nblk = static_cast<double>(traj) * steps * blocks;
    const double bps = nblk / (ms / 1e3);
    // issue peak: 4 warp-instructions per clock per SM at the max clock
    const double issue_peak = static_cast<double>(sms) * 4 * 1965e6;
    std::printf(
        "{\"ceiling\": \"philox\", \"blocks_per_step\": %u, \"trajectories\": %u, \"steps\": %u, "
        "\"ms\": %.3f, \"blocks_per_s\": %.4e, \"warp_instr_per_block_at_issue_peak\": %.2f}\n",
        blocks, traj, steps, ms, bps, issue_peak / (bps / 32.0));
  }

  // ---- 2. shared-memory probes, 32 warps per SM, 128 KiB table
  const std::size_t smem = 32768 * 4;
  CK(cudaFuncSetAttribute(smem_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(smem_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int column = 0; column < 2; ++column) {
    const std::uint32_t iters = 20000;
    auto k = column ? smem_probe<true> : smem_probe<false>;
    k<<<sms, 1024, smem>>>(100, out, clk);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    k<<<sms, 1024, smem>>>(iters, out, clk);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long* hclk = new unsigned long long[sms];
    CK(cudaMemcpy(hclk, clk, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += static_cast<double>(hclk[i]);
    cyc /= sms;
    delete[] hclk;
    const double probes_per_sm = 1024.0 * iters * 8;
    const double probes = probes_per_sm * sms;
    std::printf(
        "{\"ceiling\": \"smem_probe\", \"layout\": \"%s\", \"probes_per_clk_per_sm\": %.3f, "
        "\"probes_per_s\": %.4e, \"ms\": %.3f, \"sm_clock_mhz_implied\": %.0f}\n",
        column ? "column" : "random", probes_per_sm / cyc, probes / (ms / 1e3), ms,
        cyc / (ms * 1e3));
  }
  (void)argc;
  (void)argv;
  return 0;
}
