#include <cstdio>
#include <cmath>
__global__ void k(const double* x, double* e0, double* e1, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = x[i], y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  double r = s * y;
  double h = 0.5 * s, e = fma(-h * y, y, 0.5), y2 = fma(y, e, y);
  double r2 = s * y2;
  double t = sqrt(s);
  e0[i] = fabs(r - t) / t;
  e1[i] = fabs(r2 - t) / t;
}
int main() {
  const int n = 1 << 24;
  double *x, *e0, *e1;
  cudaMallocManaged(&x, n * 8); cudaMallocManaged(&e0, n * 8); cudaMallocManaged(&e1, n * 8);
  unsigned long long st = 88172645463325252ULL;
  for (int i = 0; i < n; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    double u = (st >> 11) * (1.0 / 9007199254740992.0);
    x[i] = ldexp(0.5 + u, (int)(st % 60) - 50);  // spread over exponents
  }
  k<<<n / 256, 256>>>(x, e0, e1, n);
  cudaDeviceSynchronize();
  double m0 = 0, m1 = 0;
  for (int i = 0; i < n; ++i) { m0 = fmax(m0, e0[i]); m1 = fmax(m1, e1[i]); }
  printf("rsqrt.approx.ftz.f64: max rel err of s*rsqrt %.3e (2^%.1f); after one Newton step %.3e\n", m0, log2(m0), m1);
}
