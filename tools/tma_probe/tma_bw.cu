// TMA streaming bandwidth probe: each block walks z-planes of a padded fp64 array, copying one
// (bx x by) box per plane into a kStages-deep shared ring (one elected thread issues,
// mbarrier completion), the block sums the box so the load is consumed. Reports GB/s of box
// bytes for several box shapes (x start offset 16 B like the blocked smoother's).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Map {
  CUtensorMap m;
};

template <int S>
__global__ void k_stream(const __grid_constant__ Map map, int bx, int by, int nx_blocks, int ny_blocks, int zc, int nz,
                         int xstart, double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int bytes = bx * by * 8, slot = (bytes + 127) / 128 * 128;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + S * slot);
  const int ox = blockIdx.x * (bx - 4) + xstart, oy = blockIdx.y * (by - 2);
  const int k0 = blockIdx.z * zc, k1 = min(k0 + zc, nz);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k, int s) {
    if (k >= k1) return;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + s)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su(sm + s * slot)),
        "l"(reinterpret_cast<unsigned long long>(&map.m)), "r"(ox), "r"(oy), "r"(k), "r"(su(bar + s))
        : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < S - 1; ++s) issue(k0 + s, s);
  double acc = 0.0;
  int s = 0;
  unsigned ph = 0;
  for (int k = k0; k < k1; ++k) {
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            su(bar + s)),
        "r"(ph)
        : "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      int is = s + S - 1;
      if (is >= S) is -= S;
      issue(k + S - 1, is);
    }
    const double* b = reinterpret_cast<const double*>(sm + s * slot);
    for (int e = threadIdx.x; e < bx * by; e += blockDim.x) acc += b[e];
    if (++s == S) s = 0, ph ^= 1;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const int N = 257, px = 264, py = N + 2, pz = N + 2;
  double *d, *o;
  cudaMalloc(&d, (size_t)px * py * pz * 8);
  cudaMemset(d, 0, (size_t)px * py * pz * 8);
  cudaMalloc(&o, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct C {
    int bx, by, threads, stages;
  } cs[] = {{34, 16, 256, 4}, {34, 18, 256, 4}, {66, 16, 256, 4}, {66, 16, 512, 4}, {130, 8, 256, 4},
            {34, 16, 256, 8}, {130, 16, 512, 4}, {258, 4, 256, 4}, {34, 34, 256, 4}};
  for (auto& c : cs) {
    Map map;
    const cuuint64_t dims[3] = {(cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)pz};
    const cuuint64_t strides[2] = {(cuuint64_t)px * 8, (cuuint64_t)px * py * 8};
    const cuuint32_t box[3] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    enc(&map.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int nxb = (N + c.bx - 5) / (c.bx - 4), nyb = (N + c.by - 3) / (c.by - 2), zc = 32;
    const dim3 gr(nxb, nyb, (N + zc - 1) / zc);
    const int slot = (c.bx * c.by * 8 + 127) / 128 * 128;
    const size_t smem = (size_t)c.stages * slot + 8 * c.stages;
    auto kern = c.stages == 4 ? k_stream<4> : k_stream<8>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) kern<<<gr, c.threads, smem>>>(map, c.bx, c.by, nxb, nyb, zc, N, 2, o);
    cudaEventRecord(e0);
    const int it = 10;
    for (int w = 0; w < it; ++w) kern<<<gr, c.threads, smem>>>(map, c.bx, c.by, nxb, nyb, zc, N, 2, o);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)gr.x * gr.y * N * c.bx * c.by * 8;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, c.threads, smem);
    printf("box %3dx%-3d thr %d stages %d: %7.1f us  %6.0f GB/s (box bytes)  useful %6.0f GB/s  blocks/SM %d  %s\n", c.bx,
           c.by, c.threads, c.stages, ms / it * 1e3, bytes / (ms / it * 1e-3) / 1e9,
           (double)N * N * N * 8 / (ms / it * 1e-3) / 1e9, per, cudaGetErrorString(e));
  }
  return 0;
}
