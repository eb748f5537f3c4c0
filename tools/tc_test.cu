// Standalone check of tgemm_tc2_kernel / tgemm_tc3_kernel (tcgen05 tf32x3 translation GEMM)
// against a float64 host reference.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o /tmp/tc_test tools/tc_test.cu && /tmp/tc_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../paper_1801_03589_b200/csrc/nesa_kernels.cuh"
using namespace nesa;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

static float tf32h(float x) {  // host round-to-nearest-away tf32
  uint32_t u; memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float y; memcpy(&y, &u, 4); return y;
}

template <int R, int V>
int run() {
  const int Q = 64, QR = Q * R, EPT = 128 / R;
  const int ndt = 3, G = 300, nunits = 7;
  std::mt19937 rng(1);
  std::normal_distribution<double> nd(0, 1);
  std::vector<double> D(size_t(ndt) * Q * Q), S(size_t(G) * QR);
  for (auto& v : D) v = nd(rng);
  for (auto& v : S) v = nd(rng);
  // canonical hi / lo tables
  std::vector<float> DTC(size_t(ndt) * 2 * 4096);
  for (int t = 0; t < ndt; ++t)
    for (int nn = 0; nn < Q; ++nn)
      for (int k = 0; k < Q; ++k) {
        const float x = float(D[(size_t(t) * Q + nn) * Q + k]);
        const float hi = tf32h(x), lo = tf32h(x - hi);
        const size_t off = (nn / 8) * 512 + (k / 4) * 32 + (nn % 8) * 4 + (k % 4);
        DTC[size_t(t) * 8192 + off] = hi;
        DTC[size_t(t) * 8192 + 4096 + off] = lo;
      }
  std::vector<TUnit> units;
  std::vector<TEnt> ents;
  int eidx = 0;
  for (int u = 0; u < nunits; ++u) {
    const int n = u == nunits - 1 ? EPT / 3 : (u % 2 ? 128 : EPT);   // multi-tile units too
    units.push_back(TUnit{u % ndt, int(ents.size()), int(ents.size()) + n, 0});
    for (int i = 0; i < n; ++i) ents.push_back(TEnt{int(rng() % G), eidx++});
  }
  std::vector<float> Sf(S.begin(), S.end());
  float *dD, *dS, *dY; TUnit* dU; TEnt* dE;
  CK(cudaMalloc(&dD, DTC.size() * 4)); CK(cudaMalloc(&dS, Sf.size() * 4));
  CK(cudaMalloc(&dY, size_t(eidx) * QR * 4)); CK(cudaMalloc(&dU, units.size() * sizeof(TUnit)));
  CK(cudaMalloc(&dE, ents.size() * sizeof(TEnt)));
  CK(cudaMemcpy(dD, DTC.data(), DTC.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dS, Sf.data(), Sf.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dU, units.data(), units.size() * sizeof(TUnit), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dE, ents.data(), ents.size() * sizeof(TEnt), cudaMemcpyHostToDevice));
  CK(cudaMemset(dY, 0, size_t(eidx) * QR * 4));
  if (V == 2) {
    CK(cudaFuncSetAttribute(tgemm_tc2_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(tc2_smem_bytes<R>())));
    tgemm_tc2_kernel<R><<<nunits, 128, tc2_smem_bytes<R>()>>>(dU, dE, dD, dS, dY);
  } else {
    CK(cudaFuncSetAttribute(tgemm_tc3_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(tc2_smem_bytes<R>())));
    tgemm_tc3_kernel<R><<<3, 128, tc2_smem_bytes<R>()>>>(dU, nunits, dE, dD, dS, dY, 44);  // persistent
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> Y(size_t(eidx) * QR);
  CK(cudaMemcpy(Y.data(), dY, Y.size() * 4, cudaMemcpyDeviceToHost));
  double emax = 0, rmax = 0;
  for (auto& u : units)
    for (int i = u.ent_begin; i < u.ent_end; ++i) {
      const TEnt te = ents[i];
      for (int nn = 0; nn < Q; ++nn)
        for (int rr = 0; rr < R; ++rr) {
          double ref = 0;
          for (int k = 0; k < Q; ++k) ref += D[(size_t(u.dtab) * Q + nn) * Q + k] * S[size_t(te.src) * QR + k * R + rr];
          const double got = Y[size_t(te.e) * QR + nn * R + rr];
          emax = std::max(emax, std::fabs(got - ref));
          rmax = std::max(rmax, std::fabs(ref));
        }
    }
  printf("kernel %s R=%d max abs err %.3e (max |ref| %.3e, rel %.3e)\n", V == 2 ? "tc2 (A in TMEM)" : "tc3 (persistent)", R, emax, rmax, emax / rmax);
  return emax / rmax < 1e-5 ? 0 : 2;
}

int main() {
  int rc = 0;
  rc |= run<2, 2>();
  rc |= run<1, 2>();
  rc |= run<4, 2>();
  rc |= run<2, 3>();
  rc |= run<1, 3>();
  rc |= run<4, 3>();
  printf(rc ? "FAIL\n" : "PASS\n");
  return rc;
}
