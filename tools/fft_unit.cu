// Developer tool: unit check of the K2F device FFT (fft_fwd / fft_inv of kernels_fft.cu) against a direct
// DFT on the host.  One warp: forward transform of a digit polynomial, pointwise product with a key given in
// the lane layout, inverse transform; prints the max error of the forward points and of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2506_12761_b200/csrc \
//        -o tools/fft_unit tools/fft_unit.cu && tools/fft_unit
#include "../paper_2506_12761_b200/csrc/kernels_fft.cu"

#include <cmath>
#include <complex>
#include <cstdio>
#include <random>
#include <vector>

namespace vlp {
__global__ void fft_unit_kernel(const int* x, const double2* key, const double2* psi, double2* Xout, double* out) {
  __shared__ double2 trb[2 * 16 * kTrStride];
  const uint32_t lane = threadIdx.x, h = lane >> 4;
  Lane lc;
  for (int r = 0; r < 16; r++) {
    const double2 t = psi[(lane * (1u + 4u * (static_cast<uint32_t>(mrev(r)) ^ (8u * h)))) & 2047u];
    lc.tw[r] = {t.x, t.y};
  }
  const double2 w32 = psi[(64u * (lane & 15u)) & 2047u];
  lc.sgn = h ? -1.0 : 1.0;
  lc.tau = {lc.sgn * w32.x, lc.sgn * w32.y};
  lc.off = -lc.sgn * 4503599627370560.0;
  lc.lane = lane;
  lc.tbase = 8u * h * kTrStride + (lane & 15u);
  uint32_t wv[32];
  for (int q = 0; q < 32; q++) wv[q] = static_cast<uint32_t>(x[32 * q + lane] + 64) << 25;
  cd X[16];
  fft_fwd(X, wv, 25u, lc, trb);
  for (int r = 0; r < 16; r++) {
    Xout[lane * 16 + r] = make_double2(X[r].x, X[r].y);
    const double2 k = key[lane * 16 + r];
    X[r] = cmul(X[r], cd{k.x, k.y});
  }
  fft_inv(X, lc, trb);
  for (int a = 0; a < 16; a++) {
    const double sg = (a & 1) ? lc.sgn : 1.0;
    out[32 * a + lane] = sg * X[a].x;
    out[32 * a + lane + 512] = sg * X[a].y;
  }
}
}  // namespace vlp

int main() {
  using namespace vlp;
  typedef std::complex<double> C;
  std::vector<double2> psi(2048);
  for (int k = 0; k < 2048; k++) psi[k] = make_double2(cos(M_PI * k / 1024.0), sin(M_PI * k / 1024.0));
  set_fft_constants(psi.data());
  std::mt19937_64 rng(3);
  std::vector<int> x(1024), p(1024);
  for (auto& v : x) v = static_cast<int>(rng() % 128) - 64;
  for (auto& v : p) v = static_cast<int>(rng() % 65536) - 32768;
  // host: A_k = sum_j z_j psi^{j(1+4k)}, z_j = x_j + i x_{j+512}; same for the key, scaled 1/512
  auto dft = [&](const std::vector<int>& a, std::vector<C>& A) {
    A.assign(512, 0);
    for (int k = 0; k < 512; k++)
      for (int j = 0; j < 512; j++) {
        const double2 t = psi[(j * (1 + 4 * k)) & 2047];
        A[k] += C(a[j], a[j + 512]) * C(t.x, t.y);
      }
  };
  std::vector<C> XA, PA;
  dft(x, XA);
  dft(p, PA);
  std::vector<double2> key(512);
  for (int L = 0; L < 32; L++)
    for (int r = 0; r < 16; r++) {
      const C v = PA[L + 32 * mrev(r)] / 512.0;
      key[L * 16 + r] = make_double2(v.real(), v.imag());
    }
  int* dx;
  double2 *dk, *dp, *dX;
  double* dout;
  cudaMalloc(&dx, 4096);
  cudaMalloc(&dk, 512 * 16);
  cudaMalloc(&dp, 2048 * 16);
  cudaMalloc(&dX, 512 * 16);
  cudaMalloc(&dout, 1024 * 8);
  cudaMemcpy(dx, x.data(), 4096, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, key.data(), 512 * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, psi.data(), 2048 * 16, cudaMemcpyHostToDevice);
  fft_unit_kernel<<<1, 32>>>(dx, dk, dp, dX, dout);
  std::vector<double2> Xg(512);
  std::vector<double> out(1024);
  cudaMemcpy(Xg.data(), dX, 512 * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(out.data(), dout, 1024 * 8, cudaMemcpyDeviceToHost);
  printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
  double ef = 0;
  int worst = -1;
  for (int L = 0; L < 32; L++)
    for (int r = 0; r < 16; r++) {
      const C want = XA[L + 32 * mrev(r)];
      const double e = std::abs(C(Xg[L * 16 + r].x, Xg[L * 16 + r].y) - want);
      if (e > ef) { ef = e; worst = L * 16 + r; }
    }
  printf("forward max |err| = %.3g (lane %d reg %d)\n", ef, worst / 16, worst % 16);
  for (int L = 0; L < 2; L++)
    for (int r = 0; r < 4; r++) {
      const C want = XA[L + 32 * mrev(r)];
      printf("  L%d r%d got (%.4f, %.4f) want (%.4f, %.4f)\n", L, r, Xg[L * 16 + r].x, Xg[L * 16 + r].y, want.real(),
             want.imag());
    }
  // exact negacyclic product
  double ep = 0;
  for (int k = 0; k < 1024; k++) {
    long long s = 0;
    for (int i = 0; i < 1024; i++) {
      const int j = k - i;
      if (j >= 0) s += static_cast<long long>(x[i]) * p[j];
      else s -= static_cast<long long>(x[i]) * p[j + 1024];
    }
    ep = std::max(ep, std::fabs(out[k] - static_cast<double>(s)));
  }
  printf("product max |err| = %.3g\n", ep);
  // K4F on one (i, r) key row pair: raw[2][1024] u32 -> 2 chunks of [rho' 8][o*2 + l][32] complex
  std::vector<uint32_t> raw(6 * 2 * 1024);
  for (auto& v : raw) v = static_cast<uint32_t>(rng());
  uint32_t* draw;
  double2* dkf;
  cudaMalloc(&draw, raw.size() * 4);
  cudaMalloc(&dkf, 12 * 16384);
  cudaMemcpy(draw, raw.data(), raw.size() * 4, cudaMemcpyHostToDevice);
  vlp_bsk_fft_kernel<<<6, 512>>>(draw, dkf, dp);
  std::vector<double2> kf(12 * 1024);
  cudaMemcpy(kf.data(), dkf, 12 * 16384, cudaMemcpyDeviceToHost);
  printf("k4f: %s\n", cudaGetErrorString(cudaGetLastError()));
  double ek = 0;
  for (int r = 0; r < 6; r++)
    for (int o = 0; o < 2; o++) {
      std::vector<int> lo(1024), hi(1024);
      for (int j = 0; j < 1024; j++) {
        const long long sv = static_cast<int32_t>(raw[(r * 2 + o) * 1024 + j]);
        lo[j] = static_cast<int>(((sv + 32768) & 65535) - 32768);
        hi[j] = static_cast<int>((sv - lo[j]) >> 16);
      }
      std::vector<C> A0, A1;
      dft(lo, A0);
      dft(hi, A1);
      for (int k = 0; k < 512; k++) {
        const int L = k & 31, rho = mrev(k >> 5), h = rho >> 3, rp = rho & 7;
        for (int l = 0; l < 2; l++) {
          const double2 g = kf[(r * 2 + h) * 1024 + (rp * 4 + o * 2 + l) * 32 + L];
          const C want = (l ? A1[k] : A0[k]) / 512.0;
          ek = std::max(ek, std::abs(C(g.x, g.y) - want));
        }
      }
    }
  printf("k4f max |err| = %.3g\n", ek);
  return 0;
}
