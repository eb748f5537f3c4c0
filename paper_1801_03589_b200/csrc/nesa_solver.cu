// nesa_solver.cu -- the Gram-Schmidt steps of the GMRES solver around the
// product (the reference has no solver; the
// paper names the product as the inner kernel of one).
//
// One Arnoldi step orthogonalises w = A v_k against the basis v_0..v_k by
// classical Gram-Schmidt applied twice (CGS2).  Done with library GEMVs that
// is four passes over the basis and two host round trips; here it is three
// passes and none:
//   pass 1  (w += shift v_k,) h1 = V^H w             (partial dots per CTA)
//   pass 2  w' = w - V h1,  h2 = V^H w'
//   pass 3  w'' = w' - V h2, |w''|^2
// (each pass's last CTA reduces its partials for the next one)
//   scale   v_{k+1} = w'' / |w''|, H[:, k] = h1 + h2, H[k+1, k] = |w''|
// Vectors are complex (interleaved re, im) of one column, float32 or float64;
// the basis is V[j] = basis + j * stride.  Per-CTA partial sums are reduced
// in a fixed order (float64), so the step is bitwise reproducible.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <type_traits>

#include "../../include/nesa_b200.h"

namespace {

constexpr int kGsThreads = 256;
constexpr int kGsMaxK = 128;      // basis vectors per step (restart length + 1)
constexpr int kGsBlocks = 4 * 148;  // CTAs per pass (four per SM) = partial sums per pass

thread_local std::string g_solver_error;

template <typename T>
struct C2 {
  T x, y;
};

// block-wide sum of (re, im) into red[0] (fixed order)
template <typename T>
__device__ C2<T> block_sum(C2<T> v, C2<T>* red) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  C2<T> s{T(0), T(0)};
  if (threadIdx.x == 0)
    for (int w = 0; w < kGsThreads / 32; ++w) {
      s.x += red[w].x;
      s.y += red[w].y;
    }
  return s;
}

// Work buffer: per-CTA partial sums of the three passes, the reduced
// h1 / h2 / |w|^2 (float64 pairs) and one arrival counter per pass.
struct GsWork {
  double part[3][kGsBlocks][kGsMaxK][2];
  double h[3][kGsMaxK][2];
  unsigned int cnt[4];
};

// The last CTA of a pass to arrive reduces the per-CTA partials in a fixed
// order (ascending CTA per column: bitwise reproducible whichever CTA is
// last) and resets the counter for the next pass; the next kernel reads the
// nj reduced values instead of every CTA re-reducing 148 x nj partials.
__device__ void finish_pass(GsWork* wk, int pass, int nj) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&wk->cnt[pass], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < nj; j += kGsThreads / 32) {
    // lane l sums CTAs l, l + 32, ... (fixed), then a fixed shuffle tree
    double re = 0, im = 0;
    for (int b = lane; b < kGsBlocks; b += 32) {
      re += __ldcg(&wk->part[pass][b][j][0]);
      im += __ldcg(&wk->part[pass][b][j][1]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) {
      wk->h[pass][j][0] = re;
      wk->h[pass][j][1] = im;
    }
  }
  if (threadIdx.x == 0) wk->cnt[pass] = 0;
}

// One pass = streaming sweeps over this CTA's contiguous element range,
// kGsJB basis vectors per sweep: every sweep reads its V rows from HBM and w
// from L2 (16 MB at C4, L2-resident across the sweeps), kGsU complex
// elements per thread per step with all (kGsJB + 1) kGsU loads issued
// before the math, so each SM keeps enough bytes in flight to stream at HBM
// speed.
//   mode 0: (w += shift v_{kk-1};) part[j] = v_j^H w
//   mode 1: w -= sum_j v_j h1_j; part[j] = v_j^H w
//   mode 2: w -= sum_j v_j h2_j; part[0] = |w|^2
constexpr int kGsU = 2;   // complex elements per thread per sweep step
constexpr int kGsJB = 4;  // basis vectors per sweep

template <typename T, int MODE>
__global__ void __launch_bounds__(kGsThreads) gs_pass_kernel(const T* __restrict__ V, int64_t stride, int kk,
                                                             T* __restrict__ w, int64_t n, double shift,
                                                             GsWork* __restrict__ wk) {
  using V2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
  __shared__ C2<T> red[kGsThreads / 32];
  __shared__ double hs[2 * kGsMaxK];
  if constexpr (MODE >= 1) {
    for (int j = threadIdx.x; j < kk; j += blockDim.x) {
      hs[2 * j] = __ldcg(&wk->h[MODE - 1][j][0]);
      hs[2 * j + 1] = __ldcg(&wk->h[MODE - 1][j][1]);
    }
    __syncthreads();
  }
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = int64_t(blockIdx.x) * per, e1 = e0 + per < n ? e0 + per : n;
  V2* wv = reinterpret_cast<V2*>(w);
  constexpr int64_t kStep = int64_t(kGsThreads) * kGsU;
  // w += sum_{j in [j0, j0 + nb)} c_j v_j over the range (nb <= kGsJB basis
  // vectors per sweep, c_j = -h_j, or the shift); returns |w|^2
  auto axpy = [&](int j0, int nb, const T* cr, const T* ci) {
    T nn = T(0);
    for (int64_t b = e0; b < e1; b += kStep) {
      V2 x[kGsJB][kGsU], y[kGsU];
#pragma unroll
      for (int u = 0; u < kGsU; ++u) {
        const int64_t e = b + u * kGsThreads + threadIdx.x;
        const bool in = e < e1;
        y[u] = in ? __ldcg(wv + e) : V2{T(0), T(0)};
#pragma unroll
        for (int q = 0; q < kGsJB; ++q)
          x[q][u] = (in && q < nb) ? __ldcs(reinterpret_cast<const V2*>(V + (j0 + q) * stride) + e)
                                   : V2{T(0), T(0)};
      }
#pragma unroll
      for (int u = 0; u < kGsU; ++u) {
        const int64_t e = b + u * kGsThreads + threadIdx.x;
#pragma unroll
        for (int q = 0; q < kGsJB; ++q) {
          y[u].x += cr[q] * x[q][u].x - ci[q] * x[q][u].y;
          y[u].y += cr[q] * x[q][u].y + ci[q] * x[q][u].x;
        }
        if (e < e1) {
          __stcg(wv + e, y[u]);
          nn += y[u].x * y[u].x + y[u].y * y[u].y;
        }
      }
    }
    return nn;
  };
  // part[j] = v_j^H w for j in [j0, j0 + nb) over the range
  auto dots = [&](int j0, int nb) {
    C2<T> acc[kGsJB];
#pragma unroll
    for (int q = 0; q < kGsJB; ++q) acc[q] = C2<T>{T(0), T(0)};
    for (int64_t b = e0; b < e1; b += kStep) {
      V2 x[kGsJB][kGsU], y[kGsU];
#pragma unroll
      for (int u = 0; u < kGsU; ++u) {
        const int64_t e = b + u * kGsThreads + threadIdx.x;
        const bool in = e < e1;
        y[u] = in ? __ldcg(wv + e) : V2{T(0), T(0)};
#pragma unroll
        for (int q = 0; q < kGsJB; ++q)
          x[q][u] = (in && q < nb) ? __ldcs(reinterpret_cast<const V2*>(V + (j0 + q) * stride) + e)
                                   : V2{T(0), T(0)};
      }
#pragma unroll
      for (int u = 0; u < kGsU; ++u)
#pragma unroll
        for (int q = 0; q < kGsJB; ++q) {
          acc[q].x += x[q][u].x * y[u].x + x[q][u].y * y[u].y;   // conj(v) w
          acc[q].y += x[q][u].x * y[u].y - x[q][u].y * y[u].x;
        }
    }
#pragma unroll
    for (int q = 0; q < kGsJB; ++q)
      if (q < nb) {
        const C2<T> sm = block_sum(acc[q], red);
        if (threadIdx.x == 0) {
          wk->part[MODE][blockIdx.x][j0 + q][0] = double(sm.x);
          wk->part[MODE][blockIdx.x][j0 + q][1] = double(sm.y);
        }
      }
  };
  auto put = [&](int j, C2<T> v) {
    const C2<T> sm = block_sum(v, red);
    if (threadIdx.x == 0) {
      wk->part[MODE][blockIdx.x][j][0] = double(sm.x);
      wk->part[MODE][blockIdx.x][j][1] = double(sm.y);
    }
  };
  if constexpr (MODE == 0) {
    if (shift != 0.0) {
      T cr[kGsJB] = {}, ci[kGsJB] = {};
      cr[0] = T(shift);
      axpy(kk - 1, 1, cr, ci);
    }
  } else {
    T nn = T(0);
    for (int j0 = 0; j0 < kk; j0 += kGsJB) {
      const int nb = kk - j0 < kGsJB ? kk - j0 : kGsJB;
      T cr[kGsJB], ci[kGsJB];
#pragma unroll
      for (int q = 0; q < kGsJB; ++q) {
        cr[q] = q < nb ? -T(hs[2 * (j0 + q)]) : T(0);
        ci[q] = q < nb ? -T(hs[2 * (j0 + q) + 1]) : T(0);
      }
      nn = axpy(j0, nb, cr, ci);
    }
    if constexpr (MODE == 2) {
      put(0, C2<T>{nn, T(0)});
      finish_pass(wk, 2, 1);
    }
  }
  if constexpr (MODE <= 1) {
    // (each thread reads back only the w elements it wrote itself)
    for (int j0 = 0; j0 < kk; j0 += kGsJB) dots(j0, kk - j0 < kGsJB ? kk - j0 : kGsJB);
    finish_pass(wk, MODE, kk);
  }
}

// v_out = w / |w|; hcol[0..kk) = h1 + h2, hcol[kk] = |w| (float64 pairs,
// the Hessenberg column), from the passes' reduced values
template <typename T>
__global__ void __launch_bounds__(kGsThreads) gs_scale_kernel(const T* __restrict__ w, T* __restrict__ v_out,
                                                              int64_t n, int kk, const GsWork* __restrict__ wk,
                                                              double* __restrict__ hcol) {
  const double nrm = sqrt(__ldcg(&wk->h[2][0][0]));
  if (blockIdx.x == 0) {
    for (int j = threadIdx.x; j < kk; j += blockDim.x) {
      hcol[2 * j] = __ldcg(&wk->h[0][j][0]) + __ldcg(&wk->h[1][j][0]);
      hcol[2 * j + 1] = __ldcg(&wk->h[0][j][1]) + __ldcg(&wk->h[1][j][1]);
    }
    if (threadIdx.x == 0) {
      hcol[2 * kk] = nrm;
      hcol[2 * kk + 1] = 0.0;
    }
  }
  const T inv = nrm > 0 ? T(1.0 / nrm) : T(0);
  const int64_t m = 2 * n;
  if constexpr (sizeof(T) == 4) {
    if ((reinterpret_cast<uintptr_t>(w) & 15) == 0 && (reinterpret_cast<uintptr_t>(v_out) & 15) == 0) {
      const int64_t m4 = m / 4;
      const float4* w4 = reinterpret_cast<const float4*>(w);
      float4* v4 = reinterpret_cast<float4*>(v_out);
      for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m4; e += int64_t(gridDim.x) * blockDim.x) {
        float4 x = w4[e];
        x.x *= inv; x.y *= inv; x.z *= inv; x.w *= inv;
        v4[e] = x;
      }
      for (int64_t e = 4 * m4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
           e += int64_t(gridDim.x) * blockDim.x)
        v_out[e] = w[e] * inv;
      return;
    }
  }
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x)
    v_out[e] = w[e] * inv;
}

template <typename T>
int gs_step(const T* V, int64_t stride, int kk, T* w, T* v_out, int64_t n, double shift, void* work,
            double* hcol, cudaStream_t st) {
  GsWork* wk = static_cast<GsWork*>(work);
  gs_pass_kernel<T, 0><<<kGsBlocks, kGsThreads, 0, st>>>(V, stride, kk, w, n, shift, wk);
  gs_pass_kernel<T, 1><<<kGsBlocks, kGsThreads, 0, st>>>(V, stride, kk, w, n, 0.0, wk);
  gs_pass_kernel<T, 2><<<kGsBlocks, kGsThreads, 0, st>>>(V, stride, kk, w, n, 0.0, wk);
  gs_scale_kernel<T><<<4 * kGsBlocks, kGsThreads, 0, st>>>(w, v_out, n, kk, wk, hcol);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_solver_error = cudaGetErrorString(e);
    return NESA_ERR_CUDA;
  }
  return NESA_OK;
}

}  // namespace

#define NESA_SOLVER_API extern "C" __attribute__((visibility("default")))

// Work buffer size (bytes) for nesa_gs_step; zero-filled before first use.
NESA_SOLVER_API int64_t nesa_gs_work_bytes(void) { return int64_t(sizeof(GsWork)); }

NESA_SOLVER_API int nesa_gs_step_shifted(const void* basis, int64_t stride, int32_t kk, void* w, void* v_out,
                                         int64_t n, int32_t is_f64, double shift, void* work, void* hcol,
                                         void* stream) {
  if (!basis || !w || !v_out || !work || !hcol || kk < 1 || kk > kGsMaxK || n < 1) {
    g_solver_error = "bad nesa_gs_step arguments (1 <= kk <= 128)";
    return NESA_ERR_INVALID;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (is_f64)
    return gs_step<double>(static_cast<const double*>(basis), stride, kk, static_cast<double*>(w),
                           static_cast<double*>(v_out), n, shift, work, static_cast<double*>(hcol), st);
  return gs_step<float>(static_cast<const float*>(basis), stride, kk, static_cast<float*>(w),
                        static_cast<float*>(v_out), n, shift, work, static_cast<double*>(hcol), st);
}

NESA_SOLVER_API int nesa_gs_step(const void* basis, int64_t stride, int32_t kk, void* w, void* v_out,
                                 int64_t n, int32_t is_f64, void* work, void* hcol, void* stream) {
  return nesa_gs_step_shifted(basis, stride, kk, w, v_out, n, is_f64, 0.0, work, hcol, stream);
}

NESA_SOLVER_API const char* nesa_gs_last_error(void) { return g_solver_error.c_str(); }
