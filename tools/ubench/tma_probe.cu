// Probe: which 2D tensor maps over the reference layout (odd row stride) the TMA accepts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_probe.cu ; ./tma_probe <mode>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap m; int pad; };
__global__ void probe(const __grid_constant__ Maps maps, int c0, int c1, double* out, int W, int R) {
  extern __shared__ __align__(128) double sm[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + 1024);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(W * R * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            s32(sm)),
        "l"(reinterpret_cast<unsigned long long>(&maps.m)), "r"(c0), "r"(c1), "r"(s32(bar))
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(s32(bar))
      : "memory");
  for (int i = threadIdx.x; i < W * R; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  Enc enc = (Enc)p;
  const int nz = 257, ny = 257, nx = 8;
  const long long total = (long long)nx * ny * nz;
  std::vector<double> h(total);
  for (long long i = 0; i < total; ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, total * 8 + 64);
  cudaMalloc(&o, 4096 * 8);
  cudaMemcpy(d, h.data(), total * 8, cudaMemcpyHostToDevice);
  Maps maps;
  int W = 22, R = 11;
  cuuint64_t dims[2], stride[1];
  cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)R}, es[2] = {1, 1};
  int c0 = 0, c1 = 0;
  if (mode == 0) { dims[0] = 256; dims[1] = 64; stride[0] = 257 * 16; c0 = 3; c1 = 2; }         // plain
  if (mode == 1) { dims[0] = total; dims[1] = 129; stride[0] = 257 * 16; c0 = 5 * ny * nz + 12 * nz + 7; c1 = 4; }  // overlapping
  if (mode == 2) { dims[0] = total; dims[1] = 129; stride[0] = 257 * 16; c0 = -6; c1 = -2; }    // negative coords
  if (mode == 3) { dims[0] = total; dims[1] = 9; stride[0] = 257 * 16; c0 = 40; c1 = 0; }       // fewer rows than the box
  if (mode == 4) { dims[0] = 2 * nz + W; dims[1] = 1000; stride[0] = 257 * 16; c0 = 300; c1 = 5; }  // slight overlap
  if (mode == 5) { dims[0] = 256; dims[1] = 64; stride[0] = 257 * 16; c0 = 4; c1 = 2; }         // plain, even start
  if (mode == 6) { dims[0] = total; dims[1] = 129; stride[0] = 257 * 16; c0 = (int)total - 10; c1 = 127; }  // dim0 overrun at the end
  CUresult r = enc(&maps.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("mode %d encode rc=%d\n", mode, (int)r);
  if (r) return 0;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  probe<<<1, 128, 16384>>>(maps, c0, c1, o, W, R);
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d run: %s\n", mode, cudaGetErrorString(e));
  if (e) return 0;
  std::vector<double> ho(W * R);
  cudaMemcpy(ho.data(), o, W * R * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int j = 0; j < R; ++j)
    for (int i = 0; i < W; ++i) {
      long long f = (long long)c0 + i + (long long)(c1 + j) * 2 * nz;
      bool in = (c0 + i) >= 0 && (unsigned long long)(c0 + i) < dims[0] && (c1 + j) >= 0 && (unsigned long long)(c1 + j) < dims[1];
      double want = in ? (double)f : 0.0;
      if (ho[j * W + i] != want) { if (bad < 5) printf("  mismatch (%d,%d): got %g want %g\n", i, j, ho[j * W + i], want); ++bad; }
    }
  printf("mode %d mismatches %d\n", mode, bad);
  return 0;
}
