// MUFU sin/cos accuracy vs |x| (radians) on sm_100a
#include <cstdio>
#include <cmath>
__global__ void k(const float* x, float* s, float* c, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { float a, b; __sincosf(x[i], &a, &b); s[i] = a; c[i] = b; }
}
int main() {
  const int n = 1 << 20;
  float *x, *s, *c;
  cudaMallocManaged(&x, n * 4); cudaMallocManaged(&s, n * 4); cudaMallocManaged(&c, n * 4);
  float ranges[] = {3.2f, 32.f, 320.f, 1000.f, 3200.f, 1e4f};
  for (float R : ranges) {
    for (int i = 0; i < n; ++i) x[i] = (float)((2.0 * i / n - 1.0) * R);
    k<<<(n + 255) / 256, 256>>>(x, s, c, n);
    cudaDeviceSynchronize();
    double es = 0, ec = 0;
    for (int i = 0; i < n; ++i) { es = fmax(es, fabs(s[i] - sin((double)x[i]))); ec = fmax(ec, fabs(c[i] - cos((double)x[i]))); }
    printf("|x|<=%g rad: max abs err sin %.3e cos %.3e\n", R, es, ec);
  }
  return 0;
}
