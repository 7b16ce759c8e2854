// Standalone probe: 3D fp64 TMA box loads (box larger / smaller than the tensor, negative
// coordinates) into shared memory with mbarrier completion; prints the CUDA error per case.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

struct Maps {
  CUtensorMap m;
};

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_probe(const __grid_constant__ Maps maps, int bx, int by, int c0, int c1, int c2, double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double* buf = reinterpret_cast<double*>(sm);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + 65536);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(bar)), "r"(bx * by * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            su(buf)),
        "l"(reinterpret_cast<unsigned long long>(&maps.m)), "r"(c0), "r"(c1), "r"(c2), "r"(su(bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          su(bar))
      : "memory");
  for (int e = threadIdx.x; e < bx * by; e += blockDim.x) out[e] = buf[e];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  printf("enc=%p q=%d\n", (void*)enc, (int)q);
  struct Case {
    int px, ny, nz, bx, by, c0, c1, c2;
  } cases[] = {{64, 40, 40, 32, 16, 4, 1, 1},   {64, 40, 40, 32, 16, -2, -1, 0}, {24, 19, 19, 32, 16, 3, 0, 0},
               {24, 19, 19, 16, 16, 3, 0, 0},   {264, 259, 259, 34, 18, 2, -1, 5}, {64, 40, 40, 32, 16, 40, 0, 0},
               {40, 35, 35, 34, 18, 32, 0, 0},  {40, 35, 35, 34, 18, 2, 0, -1},  {40, 35, 35, 34, 18, 100, 0, 0},
               {40, 35, 35, 34, 18, 2, 30, 34}, {24, 19, 19, 20, 10, 2, 0, 0},   {24, 19, 19, 20, 10, 20, 15, 0},
               {40, 35, 35, 32, 16, 3, 0, 0},   {40, 35, 35, 34, 18, 3, 0, 0}};
  int ci = -1;
  for (auto& c : cases) {
    ++ci;
    if (only >= 0 && ci != only) continue;
    std::vector<double> h((size_t)c.px * c.ny * c.nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 65536);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    Maps maps;
    const cuuint64_t dims[3] = {(cuuint64_t)c.px, (cuuint64_t)c.ny, (cuuint64_t)c.nz};
    const cuuint64_t strides[2] = {(cuuint64_t)c.px * 8, (cuuint64_t)c.px * c.ny * 8};
    const cuuint32_t box[3] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&maps.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
    k_probe<<<1, 128, 65536 + 64>>>(maps, c.bx, c.by, c.c0, c.c1, c.c2, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> ho(c.bx * c.by);
    if (e == cudaSuccess) cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < c.by; ++y)
      for (int x = 0; x < c.bx; ++x) {
        const int gx = c.c0 + x, gy = c.c1 + y, gz = c.c2;
        const bool in = gx >= 0 && gy >= 0 && gz >= 0 && gx < c.px && gy < c.ny && gz < c.nz;
        const double want = in ? (double)((size_t)gz * c.px * c.ny + (size_t)gy * c.px + gx) : 0.0;
        if (e == cudaSuccess && ho[y * c.bx + x] != want) ++bad;
      }
    printf("px=%d box=%dx%d at (%d,%d,%d): encode=%d kernel=%s bad=%d\n", c.px, c.bx, c.by, c.c0, c.c1, c.c2, (int)r,
           cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
    cudaFree(d);
    cudaFree(o);
  }
  return 0;
}
