// Does a cooperative launch (grid-wide sync) capture into a CUDA graph and
// replay correctly on this driver?  Each block adds 1 before the grid sync;
// block 0 reads the total after it.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k(int* cnt, int* out) {
  cg::grid_group g = cg::this_grid();
  if (threadIdx.x == 0) atomicAdd(cnt, 1);
  g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) { *out = *cnt; *cnt = 0; }
  g.sync();
}

int main() {
  int *cnt, *out;
  cudaMalloc(&cnt, 4); cudaMalloc(&out, 4); cudaMemset(cnt, 0, 4); cudaMemset(out, 0, 4);
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
  dim3 grid(nsm * per), block(256);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = block; cfg.stream = s;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaError_t e0 = cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, cnt, out);
  cudaError_t e2 = cudaStreamEndCapture(s, &g);
  cudaError_t e3 = cudaGraphInstantiate(&ge, g, 0);
  printf("capture %s / launch %s / end %s / instantiate %s\n", cudaGetErrorString(e0),
         cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3));
  if (e3 == cudaSuccess) {
    for (int r = 0; r < 3; ++r) cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    int h = -1; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
    printf("blocks %d, counted %d, %s\n", grid.x, h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
