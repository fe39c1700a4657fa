// Cost of cooperative-groups grid barriers on this device (diagnostic micro-benchmark).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void syncs(int n, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = n;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int per : {1, 2, 4}) {
    for (int n : {0, 9, 90}) {
      int blocks = sms * per;
      void* args[] = {&n, &sink};
      for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel((void*)syncs, blocks, 256, args, 0, 0);
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) cudaLaunchCooperativeKernel((void*)syncs, blocks, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("blocks %d syncs %d: %.2f us per launch\n", blocks, n, ms * 1000 / 20);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
