__global__ void k(unsigned* a, unsigned* b) {
  unsigned x = a[threadIdx.x], y = b[threadIdx.x];
  a[threadIdx.x] = __vminu2(x, y);
  b[threadIdx.x] = __vmaxu2(x, y);
}
