// Microbenchmark: 2.6M scattered 32-byte record stores vs 4 x 2.6M scattered
// int64 reductions (red.global.add.u64) into 800k owners x 4 (what a
// fixed-point owner accumulation inside K1 would issue), vs a v4 f32 red.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_store(int n, const int* slot, double4* out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double v = p * 1e-3;
    out[slot[p]] = make_double4(v, v + 1, v + 2, v + 3);
  }
}
__global__ void k_red(int n, const int* owner, unsigned long long* acc) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    unsigned long long v = (unsigned long long)p * 12345ull;
    unsigned long long* a = acc + 4 * (long long)owner[p];
    atomicAdd(a + 0, v); atomicAdd(a + 1, v + 1); atomicAdd(a + 2, v + 2); atomicAdd(a + 3, v + 3);
  }
}
__global__ void k_redf(int n, const int* owner, float* acc) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    float v = p * 1e-3f;
    float* a = acc + 4 * (long long)owner[p];
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(a), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
  }
}
int main() {
  const int P = 2635445, O = 800064;
  std::vector<int> owner(P), slot(P);
  std::mt19937 rng(1);
  for (int p = 0; p < P; ++p) owner[p] = rng() % O;
  std::vector<int> perm(P); for (int p = 0; p < P; ++p) perm[p] = p; std::shuffle(perm.begin(), perm.end(), rng);
  int *d_owner, *d_slot; double4* d_out; unsigned long long* d_acc; float* d_accf;
  cudaMalloc(&d_owner, P * 4); cudaMalloc(&d_slot, P * 4); cudaMalloc(&d_out, (size_t)P * 32);
  cudaMalloc(&d_acc, (size_t)O * 32); cudaMalloc(&d_accf, (size_t)O * 16);
  cudaMemcpy(d_owner, owner.data(), P * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_slot, perm.data(), P * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(a); k_store<<<148 * 8, 256>>>(P, d_slot, d_out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("scattered 32B stores: %.1f us\n", ms * 1e3);
    cudaEventRecord(a); k_red<<<148 * 8, 256>>>(P, d_owner, d_acc); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("4x red.add.u64: %.1f us\n", ms * 1e3);
    cudaEventRecord(a); k_redf<<<148 * 8, 256>>>(P, d_owner, d_accf); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("red.add.v4.f32: %.1f us\n", ms * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
