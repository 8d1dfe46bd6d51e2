// fp64 pipe vs occupancy / ILP / instruction mix: how much DFMA throughput do 4 warps per
// scheduler (K1's occupancy: 16 warps / SM) reach, alone and with interleaved ALU / LDS work?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

// ILP independent DFMA chains; after every DFMA group of size G, NALU integer ops and NLDS LDS.128
template <int ILP, int NALU, int NLDS>
__global__ void mix_kernel(double* out, int iters, double a, double b) {
  __shared__ double2 sm[1024];
  double acc[ILP];
  unsigned x = threadIdx.x;
  double2 ld = make_double2(0.0, 0.0);
  sm[threadIdx.x] = make_double2(threadIdx.x, 1.0);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
#pragma unroll
      for (int j = 0; j < NALU; ++j) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(it), "r"(j + r));
#pragma unroll
      for (int j = 0; j < NLDS; ++j) {
        double2 t;
        asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(t.x), "=d"(t.y) : "r"((unsigned)__cvta_generic_to_shared(&sm[(threadIdx.x + j * 33 + r) & 1023])));
        ld.x += t.x;  // one DADD per load
      }
    }
  }
  double s = ld.x + ld.y + x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int ILP, int NALU, int NLDS>
void run(double* out, const char* name) {
  const int sms = 148, iters = 2048;
  printf("%-28s", name);
  for (int warps : {4, 8, 16, 32}) {
    const int threads = warps * 32;
    float ms = timeit([&] { mix_kernel<ILP, NALU, NLDS><<<sms, threads>>>(out, iters, 1.0000001, 1e-9); });
    double f = 2.0 * sms * threads * (double)iters * 8 * (ILP + NLDS);
    printf("  w%-2d %6.2f TF", warps, f / ms / 1e9);
  }
  printf("\n");
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  run<1, 0, 0>(out, "ILP1");
  run<2, 0, 0>(out, "ILP2");
  run<4, 0, 0>(out, "ILP4");
  run<8, 0, 0>(out, "ILP8");
  run<16, 0, 0>(out, "ILP16");
  run<8, 4, 0>(out, "ILP8 + 4 ALU / 8 DFMA");
  run<8, 8, 0>(out, "ILP8 + 8 ALU / 8 DFMA");
  run<8, 12, 0>(out, "ILP8 + 12 ALU / 8 DFMA");
  run<8, 0, 1>(out, "ILP8 + 1 LDS.128 / 8 DFMA");
  run<8, 0, 2>(out, "ILP8 + 2 LDS.128 / 8 DFMA");
  run<8, 8, 2>(out, "ILP8 + 8 ALU + 2 LDS / 8");
  run<4, 4, 1>(out, "ILP4 + 4 ALU + 1 LDS / 4");
  return 0;
}
