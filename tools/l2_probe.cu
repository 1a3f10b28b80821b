// l2_probe.cu — SM<->L2 bandwidth probe (replaces the torch-copy probe, whose
// small copies were launch-latency bound).  One launch per measurement, a
// persistent grid (148 x OCC CTAs), 16-byte ld/st.global.cg (L2 only, L1
// bypassed), REPS sweeps over a footprint of F bytes inside the launch.
//   read : every CTA streams its grid-stride share of the footprint REPS times
//   copy : dst[i] = src[i] over F/2 + F/2 bytes, REPS times (read + write bytes)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2_probe.cu -o tools/l2_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) rd(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    // rotate the start so no CTA re-reads what it read last sweep (no L1 reuse anyway: .cg)
    const size_t off = ((size_t)blockIdx.x * blockDim.x + threadIdx.x + (size_t)r * 4096u * 33u) % stride;
    for (size_t i = off; i < n4; i += stride) {
      float4 v;
      asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p + i));
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 1234.5f) *sink = acc;
}

__global__ void __launch_bounds__(512) cp(const float4* __restrict__ s, float4* __restrict__ d, size_t n4, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 v;
      asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(s + i));
      asm volatile("st.global.cg.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
  }
}

int main() {
  const size_t big = (size_t)4 << 30;
  char* buf;
  float* sink;
  cudaMalloc(&buf, big);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 0, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int occs[] = {2, 4};
  const size_t mibs[] = {4, 8, 16, 24, 32, 48, 64, 96, 128, 2048};
  for (int occ : occs) {
    const int grid = 148 * occ;
    for (size_t mib : mibs) {
      const size_t F = mib << 20;
      const int reps = mib >= 1024 ? 2 : (int)((size_t)(2048ull << 20) / F);
      for (int kind = 0; kind < 2; ++kind) {
        float best = 1e30f;
        for (int t = 0; t < 4; ++t) {
          cudaEventRecord(e0);
          if (kind == 0)
            rd<<<grid, 512>>>((const float4*)buf, F / 16, reps, sink);
          else
            cp<<<grid, 512>>>((const float4*)buf, (float4*)(buf + F / 2), F / 32, reps);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (t > 0 && ms < best) best = ms;
        }
        const double bytes = (double)F * reps;  // read: F per sweep; copy: F/2 read + F/2 write
        printf("occ %d  %-4s footprint %5zu MiB  reps %5d  %8.1f GB/s\n", occ, kind ? "copy" : "read", mib, reps,
               bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
