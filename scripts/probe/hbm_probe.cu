// HBM traffic-mix probes (context for the gather roofline; not product code).
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_read(const int4* __restrict__ a, int64_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(a + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}
__global__ void k_write(int4* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = make_int4((int)i, 1, 2, 3);
}
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __ldg(a + i);
}
// 1 read : R writes (each source int4 stored to R destinations, like a k-stack gather)
__global__ void k_bcast(const int4* __restrict__ a, int4* __restrict__ b, int64_t n, int R) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(a + i);
    for (int r = 0; r < R; ++r) b[(int64_t)r * n + i] = v;
  }
}
// TMA bulk store only: each CTA stores its smem tile (bytes) to consecutive destinations
__global__ void k_bulk_write(uint8_t* __restrict__ dst, int64_t total, int tile) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < tile / 16; i += blockDim.x) reinterpret_cast<int4*>(sm)[i] = make_int4(i, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    int inflight = 0;
    for (int64_t off = (int64_t)blockIdx.x * tile; off + tile <= total; off += (int64_t)gridDim.x * tile) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(s), "r"(tile)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight > 8) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

extern "C" int probe_run(int which, void* a, void* b, int64_t bytes, int R, int grid, int block, int tile) {
  int64_t n = bytes / 16;
  switch (which) {
    case 0: k_read<<<grid, block>>>((const int4*)a, n, (int4*)b); break;
    case 1: k_write<<<grid, block>>>((int4*)a, n); break;
    case 2: k_copy<<<grid, block>>>((const int4*)a, (int4*)b, n); break;
    case 3: k_bcast<<<grid, block>>>((const int4*)a, (int4*)b, n, R); break;
    case 4:
      cudaFuncSetAttribute(k_bulk_write, cudaFuncAttributeMaxDynamicSharedMemorySize, tile);
      k_bulk_write<<<grid, 32, tile>>>((uint8_t*)a, bytes, tile);
      break;
  }
  return (int)cudaGetLastError();
}

// Strided bulk stores: CTA c stores `rows` tiles of `tile` bytes at dst + ((r * nsamp + c % nsamp) * tile)
// (time-major [L, n] output of the gather: consecutive rows are nsamp*tile apart), or contiguous
// (dst + (c * rows + r) * tile) when nsamp == 0.  G tiles in flight.
__global__ void k_bulk_rows(uint8_t* __restrict__ dst, int rows, int tile, int nsamp, int G) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < tile / 16; i += blockDim.x) reinterpret_cast<int4*>(sm)[i] = make_int4(i, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    for (int r = 0; r < rows; ++r) {
      int64_t off = nsamp ? ((int64_t)r * nsamp + (blockIdx.x % nsamp) + (int64_t)(blockIdx.x / nsamp) * rows * nsamp) * tile
                          : ((int64_t)blockIdx.x * rows + r) * tile;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(s), "r"(tile)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (G == 4) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 16;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
// LSU rows: each warp stores one tile; CTA of 8 warps handles 8 consecutive rows
__global__ void k_lsu_rows(int4* __restrict__ dst, int rows, int tile, int nsamp) {
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int c = blockIdx.x;
  for (int r = warp; r < rows; r += blockDim.x / 32) {
    int64_t off = nsamp ? ((int64_t)r * nsamp + (c % nsamp) + (int64_t)(c / nsamp) * rows * nsamp) * tile
                        : ((int64_t)c * rows + r) * tile;
    int4* d = dst + off / 16;
    for (int i = lane; i < tile / 16; i += 32) d[i] = make_int4(i, r, c, 0);
  }
}
extern "C" int probe_rows(int which, void* dst, int ctas, int rows, int tile, int nsamp, int G) {
  if (which == 0) {
    cudaFuncSetAttribute(k_bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, tile);
    k_bulk_rows<<<ctas, 32, tile>>>((uint8_t*)dst, rows, tile, nsamp, G);
  } else {
    k_lsu_rows<<<ctas, 256>>>((int4*)dst, rows, tile, nsamp);
  }
  return (int)cudaGetLastError();
}
