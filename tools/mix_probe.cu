// mix_probe.cu — memory-system ceiling for a single-HBM-pass long-row schedule
// (K9, cfg5).  No arithmetic: plain 16-byte loads/stores that reproduce the
// four byte streams such a schedule must move per element,
//     in  : HBM -> SM            (streaming read, touched once)
//     wsW : SM  -> L2 workspace  (64 MiB, rewritten every row)
//     wsR : L2 workspace -> SM
//     out : SM  -> HBM           (streaming write, touched once)
// and the reduced mixes that the K9 diagnostics time (A only = in + wsW,
// B only = wsR + out), next to a plain HBM copy (in + out).  Every mode reports
//   sm_l2  : bytes crossing the SM <-> L2 interface per second,
//   alg    : the HBM-roofline equivalent (in + out bytes only) per second.
// If `mix` tops out near the same sm_l2 rate as `copy`, a schedule that sends
// its intermediate through L2 is capped at about half the copy roofline no
// matter how its SM side is written.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mix_probe.cu -o tools/mix_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ld_cs(const float4* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_cg(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 ld_df(const float4* p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_df(float4* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void st_cg(float4* p, float4 v) {
  asm volatile("st.global.cg.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// role 0: big -> ws ring (A-like);  role 1: ws ring -> big (B-like);  role 2: big -> big (copy)
// Each CTA of a role streams a contiguous 64 KiB chunk per step (like a K9
// tile), chunks handed out round-robin over the role's CTAs.
constexpr int UNROLL = 8;
__global__ void __launch_bounds__(512) mix(const float4* __restrict__ in, float4* __restrict__ out,
                                           float4* __restrict__ ws, size_t n4, size_t ws4, int mode, int pol,
                                           size_t chunk) {
  // mode 0: copy (all CTAs role 2); 1: A only; 2: B only; 3: mix (even CTAs A, odd CTAs B)
  int role, nrole, idx;
  if (mode == 0) { role = 2; nrole = gridDim.x; idx = blockIdx.x; }
  else if (mode == 1) { role = 0; nrole = gridDim.x; idx = blockIdx.x; }
  else if (mode == 2) { role = 1; nrole = gridDim.x; idx = blockIdx.x; }
  else { role = blockIdx.x & 1; nrole = gridDim.x / 2; idx = blockIdx.x / 2; }
  const size_t nchunks = n4 / chunk;
  for (size_t c = idx; c < nchunks; c += nrole) {
    const size_t base = c * chunk;
    const size_t wbase = base % ws4;
    for (size_t i = threadIdx.x; i < chunk; i += 512 * UNROLL) {
      float4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const size_t j = i + u * 512;
        v[u] = role == 1 ? ld_cg(ws + wbase + j) : (pol ? ld_df(in + base + j) : ld_cs(in + base + j));
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const size_t j = i + u * 512;
        if (role == 0) st_cg(ws + wbase + j, v[u]);
        else if (pol) st_df(out + base + j, v[u]);
        else st_cs(out + base + j, v[u]);
      }
    }
  }
}

int main(int argc, char** argv) {
  const size_t N = (size_t)8 << 30;  // bytes per HBM stream per launch (in and out buffers)
  // workspace footprint in MiB (default 64 = one cfg5 row; 37 ~ K6's per-CTA rows for cfg4)
  const size_t WS = (size_t)(argc > 1 ? atoi(argv[1]) : 64) << 20;
  const int pol = argc > 2 ? atoi(argv[2]) : 0;            // 0: .cs streams, 1: default-policy streams
  // KiB per chunk -> float4 count (multiples of 64 KiB: one pass of 512 threads x UNROLL vectors)
  const size_t chunk = (size_t)((argc > 3 ? atoi(argv[3]) : 64) / 64 * 64 > 0 ? (argc > 3 ? atoi(argv[3]) : 64) / 64 * 64 : 64) << 6;
  printf("workspace footprint %zu MiB, stream policy %s, chunk %zu KiB\n", WS >> 20, pol ? "default" : ".cs", chunk >> 6);
  char *in, *out, *ws;
  cudaMalloc(&in, N);
  cudaMalloc(&out, N);
  cudaMalloc(&ws, WS);
  cudaMemset(in, 0, N);
  cudaMemset(out, 0, N);
  cudaMemset(ws, 0, WS);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"copy (in+out)", "A only (in+wsW)", "B only (wsR+out)", "mix (in+wsW | wsR+out)"};
  for (int occ : {2, 4}) {
    for (int mode = 0; mode < 4; ++mode) {
      float best = 1e30f;
      for (int t = 0; t < 4; ++t) {
        cudaEventRecord(e0);
        mix<<<148 * occ, 512>>>((const float4*)in, (float4*)out, (float4*)ws, N / 16, WS / 16, mode, pol, chunk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (t > 0 && ms < best) best = ms;
      }
      // bytes: every mode reads N and writes N across the SM<->L2 interface per
      // role pass; mix runs both roles over N each -> 4N.
      const double sm_l2 = (mode == 3 ? 4.0 : 2.0) * (double)N;
      const double alg = (mode == 0 || mode == 3) ? 2.0 * (double)N : (double)N;  // HBM bytes that count
      printf("occ %d  %-24s %7.3f ms   sm_l2 %7.1f GB/s   hbm-side %7.1f GB/s%s\n", occ, names[mode], best,
             sm_l2 / (best * 1e-3) / 1e9, alg / (best * 1e-3) / 1e9,
             mode == 3 ? "  <- ceiling of a single-pass schedule with an L2 intermediate" : "");
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
