// Device check of the sqrt-free BFGS tests (bfgs_common.cuh gsq_max_for,
// zeus_common.cuh curvature_update) against the reference expressions, and
// of the one-polynomial cos_fast against sincos_fast (zeus_trig.cuh);
// built and run by tests/test_gpu_bfgs.py.
#include <cstdio>
#include <cmath>
#include <random>
#include "bfgs_common.cuh"
using namespace zeus;
__global__ void k(const double* c, const double* a, const double* b, int n, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ref = !(c[i] <= kCurvatureFloor * sqrt(a[i]) * sqrt(b[i]));
  if (ref != curvature_update(c[i], a[i], b[i])) atomicAdd(bad, 1);
  if (ref != curvature_update_sl(c[i], a[i], b[i])) atomicAdd(bad, 1);
}
// cos_fast(x) == sincos_fast(x).c bit for bit
__global__ void kc(const double* x, int n, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = cos_fast(x[i]), b = sincos_fast(x[i]).c;
  if (__double_as_longlong(a) != __double_as_longlong(b)) atomicAdd(bad, 1);
}

// |g| < theta <=> |g|^2 <= gsq_max_for(theta), checked with the device sqrt
__global__ void kt(const double* q, int n, double theta, double qmax, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if ((sqrt(q[i]) < theta) != (q[i] <= qmax)) atomicAdd(bad, 1);
}
int main() {
  const int n = 1 << 22;
  std::mt19937_64 rng(1);
  std::vector<double> c(n), a(n), b(n);
  std::uniform_real_distribution<double> u(-300, 300), m(0.5, 2);
  for (int i = 0; i < n; ++i) {
    a[i] = pow(10.0, u(rng) * 1.1) * m(rng);
    b[i] = pow(10.0, u(rng) * 1.1) * m(rng);
    double t = 1e-12 * sqrt(a[i]) * sqrt(b[i]);
    int mode = i % 6;
    if (mode == 0) c[i] = t;
    else if (mode == 1) c[i] = nextafter(t, 0.0);
    else if (mode == 2) c[i] = nextafter(t, 1e308);
    else if (mode == 3) c[i] = t * m(rng);
    else if (mode == 4) c[i] = -t;
    else c[i] = (i % 12 == 5) ? NAN : (i % 18 == 11 ? 0.0 : INFINITY);
    if (i % 97 == 0) a[i] = 0.0;
    if (i % 89 == 0) b[i] = INFINITY;
    if (i % 83 == 0) a[i] = NAN;
  }
  double *dc, *da, *db; int* bad;
  cudaMalloc(&dc, n * 8); cudaMalloc(&da, n * 8); cudaMalloc(&db, n * 8); cudaMalloc(&bad, 4);
  cudaMemcpy(dc, c.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(da, a.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0, 4);
  k<<<(n + 255) / 256, 256>>>(dc, da, db, n, bad);
  int h = -1; cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
  printf("guard mismatches: %d of %d\n", h, n);
  int h2 = 0;
  for (double theta : {1e-6, 1e-8, 0.1, 3.0, 1e-150, 1e150}) {
    const double qm = gsq_max_for(theta);
    std::vector<double> q;
    double lo = qm, hi = qm;
    for (int j = 0; j < 2000; ++j) { q.push_back(lo); q.push_back(hi); lo = nextafter(lo, 0.0); hi = nextafter(hi, 1e308); }
    q.push_back(theta * theta); q.push_back(0.0); q.push_back(INFINITY); q.push_back(NAN);
    cudaMemcpy(dc, q.data(), q.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(bad, 0, 4);
    kt<<<(int)(q.size() + 255) / 256, 256>>>(dc, (int)q.size(), theta, qm, bad);
    int hb = -1; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("theta %g: gsq_max %.17g, mismatches %d\n", theta, qm, hb);
    h2 += hb;
  }
  // cos_fast vs sincos_fast: uniform over the fast range, small arguments,
  // neighbourhoods of multiples of pi/4 (quadrant edges), tiny and signed zeros
  std::vector<double> xs(n);
  std::uniform_real_distribution<double> big(-1e5, 1e5), small(-10.0, 10.0), tiny(-1e-7, 1e-7);
  for (int i = 0; i < n; ++i) {
    const int m = i % 4;
    if (m == 0) xs[i] = big(rng);
    else if (m == 1) xs[i] = small(rng);
    else if (m == 2) xs[i] = (double)((i / 4) % 20001 - 10000) * 0.7853981633974483 + tiny(rng);
    else xs[i] = (i % 8 == 3) ? tiny(rng) : ((i % 16 == 7) ? -0.0 : 6.283185307179586 * small(rng));
  }
  cudaMemcpy(dc, xs.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0, 4);
  kc<<<(n + 255) / 256, 256>>>(dc, n, bad);
  int h3 = -1;
  cudaMemcpy(&h3, bad, 4, cudaMemcpyDeviceToHost);
  printf("cos_fast vs sincos_fast: %d mismatches of %d\n", h3, n);
  return (h != 0 || h2 != 0 || h3 != 0);
}
