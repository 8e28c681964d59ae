// Microbenchmark (diagnostics): the pair kernel's split-N tail sum (own partial in registers + partner
// rows from shared memory, bf16 SW128 staging) in isolation.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o sum_mb sum_mb.cu; results in profiles/r02/s5/sum_microbench.log.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
extern "C" __global__ void __launch_bounds__(256, 1) k(float* out, unsigned long long* cyc, int S, int reps) {
  extern __shared__ uint8_t sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int R = 128 / S, kChunks = 64;
  const int warp = threadIdx.x / 32, wq = warp & 3, row = wq * 32 + (threadIdx.x & 31);
  const int c_lo = warp < 4 ? 128 : 0;
  const int sp = 0;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += 256) reinterpret_cast<float*>(sm)[i] = i * 0.5f;
  __syncthreads();
  float ev[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) ev[i] = row * 0.25f + i;
  const uint32_t ebuf = base + S * R * kChunks * 16;
  const int slice = row / R;
  unsigned long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (slice == sp) {
      const int rr = row - sp * R;
      const uint32_t part = base + rr * 16 + (c_lo / 4) * (R * 16);
#pragma unroll
      for (int k = 0; k < 32; k += 8) {
#pragma unroll 1
        for (int j = 0; j < S; ++j) {
          if (j == sp) continue;
          float4 f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = ld_shared_f4(part + j * (R * kChunks * 16) + (k + i) * (R * 16));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ev[4 * (k + i)] += f[i].x; ev[4 * (k + i) + 1] += f[i].y; ev[4 * (k + i) + 2] += f[i].z; ev[4 * (k + i) + 3] += f[i].w;
          }
        }
        const int c0 = c_lo + 4 * k;
        const int ch = (c0 % 64) / 8;
        const uint32_t dst = ebuf + (c0 / 64) * (R * 128) + rr * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          st_shared_v4(dst + (((ch + i) ^ (rr & 7)) << 4), pack(ev[4 * k + 8 * i], ev[4 * k + 8 * i + 1]),
                       pack(ev[4 * k + 8 * i + 2], ev[4 * k + 8 * i + 3]), pack(ev[4 * k + 8 * i + 4], ev[4 * k + 8 * i + 5]),
                       pack(ev[4 * k + 8 * i + 6], ev[4 * k + 8 * i + 7]));
      }
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 128) cyc[blockIdx.x] = (t1 - t0) / reps;
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 128; ++i) acc += ev[i];
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}
extern "C" __global__ void __launch_bounds__(256, 1) kb(float* out, unsigned long long* cyc, int S, int reps) {
  extern __shared__ uint8_t sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int R = 128 / S, kChunks = 64;
  const int warp = threadIdx.x / 32, wq = warp & 3, row = wq * 32 + (threadIdx.x & 31);
  const int c_lo = warp < 4 ? 128 : 0;
  const int sp = 0;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += 256) reinterpret_cast<float*>(sm)[i] = i * 0.5f;
  __syncthreads();
  float ev[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) ev[i] = row * 0.25f + i;
  const uint32_t ebuf = base + S * R * kChunks * 16;
  const int slice = row / R;
  unsigned long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (slice == sp) {
      const int rr = row - sp * R;
      const uint32_t part = base + rr * 16 + (c_lo / 4) * (R * 16);
#pragma unroll
      for (int k = 0; k < 32; k += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= S || j == sp) continue;
          float4 f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = ld_shared_f4(part + j * (R * kChunks * 16) + (k + i) * (R * 16));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ev[4 * (k + i)] += f[i].x; ev[4 * (k + i) + 1] += f[i].y; ev[4 * (k + i) + 2] += f[i].z; ev[4 * (k + i) + 3] += f[i].w;
          }
        }
        const int c0 = c_lo + 4 * k;
        const int ch = (c0 % 64) / 8;
        const uint32_t dst = ebuf + (c0 / 64) * (R * 128) + rr * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          st_shared_v4(dst + (((ch + i) ^ (rr & 7)) << 4), pack(ev[4 * k + 8 * i], ev[4 * k + 8 * i + 1]),
                       pack(ev[4 * k + 8 * i + 2], ev[4 * k + 8 * i + 3]), pack(ev[4 * k + 8 * i + 4], ev[4 * k + 8 * i + 5]),
                       pack(ev[4 * k + 8 * i + 6], ev[4 * k + 8 * i + 7]));
      }
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 128) cyc[blockIdx.x] = (t1 - t0) / reps;
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 128; ++i) acc += ev[i];
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}
int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int var = 0; var < 2; ++var) for (int S : {2, 4, 8}) for (int reps : {1, 10}) {
    if (var == 0) k<<<148, 256, 220 * 1024>>>(out, cyc, S, reps); else kb<<<148, 256, 220 * 1024>>>(out, cyc, S, reps);
    cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
    printf("var %d S=%d reps=%d: %.0f cycles per pass (thread 128)\n", var, S, reps, m);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
