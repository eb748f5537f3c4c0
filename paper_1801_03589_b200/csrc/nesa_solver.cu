// nesa_solver.cu -- the Gram-Schmidt steps of the GMRES solver around the
// product (the reference has no solver; the
// paper names the product as the inner kernel of one).
//
// One Arnoldi step orthogonalises w = A v_k against the basis v_0..v_k by
// classical Gram-Schmidt applied twice (CGS2).  Done with library GEMVs that
// is four passes over the basis and two host round trips; here it is three
// passes and none:
//   pass 1  h1 = V^H w                               (partial dots per CTA)
//   pass 2  w' = w - V h1,  h2 = V^H w'               (h1 reduced on entry)
//   pass 3  w'' = w' - V h2, |w''|^2                  (h2 reduced on entry)
//   scale   v_{k+1} = w'' / |w''|, H[:, k] = h1 + h2, H[k+1, k] = |w''|
// Vectors are complex (interleaved re, im) of one column, float32 or float64;
// the basis is V[j] = basis + j * stride.  Per-CTA partial sums are reduced
// in a fixed order (float64), so the step is bitwise reproducible.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/nesa_b200.h"

namespace {

constexpr int kGsThreads = 256;
constexpr int kGsMaxK = 128;      // basis vectors per step (restart length + 1)
constexpr int kGsBlocks = 148;    // partial sums per pass (one CTA per SM)

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

// h[j] (float64 pairs) = sum over CTAs of part[cta][j]
__device__ void reduce_partials(const double* part, int kk, double* h) {
  for (int j = threadIdx.x; j < kk; j += blockDim.x) {
    double re = 0, im = 0;
    for (int b = 0; b < kGsBlocks; ++b) {
      re += part[(size_t(b) * kGsMaxK + j) * 2];
      im += part[(size_t(b) * kGsMaxK + j) * 2 + 1];
    }
    h[2 * j] = re;
    h[2 * j + 1] = im;
  }
}

// mode 0: part = V^H w; mode 1: w -= V h (h = reduced part_in), part = V^H w;
// mode 2: w -= V h, part[0] = |w|^2.  With kk <= KR the basis values of an
// element stay in registers between the update and the dots (one read of V
// per pass); larger kk reads V twice in mode 1.
template <typename T>
constexpr int kRegK = sizeof(T) == 4 ? 32 : 16;

template <typename T, int MODE>
__global__ void __launch_bounds__(kGsThreads, 1) gs_pass_kernel(const T* __restrict__ V, int64_t stride, int kk,
                                                             T* __restrict__ w, int64_t n,
                                                             const double* __restrict__ part_in,
                                                             double* __restrict__ part_out) {
  __shared__ C2<T> red[kGsThreads / 32];
  __shared__ double hs[2 * kGsMaxK];
  if constexpr (MODE >= 1) {
    reduce_partials(part_in, kk, hs);
    __syncthreads();
  }
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = int64_t(blockIdx.x) * per, e1 = e0 + per < n ? e0 + per : n;
  constexpr int KR = kRegK<T>;
  if (kk <= KR) {
    C2<T> acc[KR];
#pragma unroll
    for (int j = 0; j < KR; ++j) acc[j] = C2<T>{T(0), T(0)};
    for (int64_t e = e0 + threadIdx.x; e < e1; e += kGsThreads) {
      T wr = w[2 * e], wi = w[2 * e + 1];
      C2<T> v[KR];
      const T* vp = V + 2 * e;
#pragma unroll
      for (int j = 0; j < KR; ++j) {
        v[j] = j < kk ? C2<T>{vp[0], vp[1]} : C2<T>{T(0), T(0)};
        vp += stride;
      }
      if constexpr (MODE >= 1) {
#pragma unroll
        for (int j = 0; j < KR; ++j)
          if (j < kk) {
            const T hr = T(hs[2 * j]), hi = T(hs[2 * j + 1]);
            wr -= v[j].x * hr - v[j].y * hi;
            wi -= v[j].x * hi + v[j].y * hr;
          }
        w[2 * e] = wr;
        w[2 * e + 1] = wi;
      }
      if constexpr (MODE <= 1) {
#pragma unroll
        for (int j = 0; j < KR; ++j)
          if (j < kk) {
            acc[j].x += v[j].x * wr + v[j].y * wi;   // conj(v) w
            acc[j].y += v[j].x * wi - v[j].y * wr;
          }
      } else {
        acc[0].x += wr * wr + wi * wi;
      }
    }
    const int nj = MODE <= 1 ? kk : 1;
#pragma unroll
    for (int j = 0; j < KR; ++j) {
      if (j >= nj) break;
      const C2<T> s = block_sum(acc[j], red);
      if (threadIdx.x == 0) {
        part_out[(size_t(blockIdx.x) * kGsMaxK + j) * 2] = double(s.x);
        part_out[(size_t(blockIdx.x) * kGsMaxK + j) * 2 + 1] = double(s.y);
      }
    }
    return;
  }
  if constexpr (MODE >= 1) {
    for (int64_t e = e0 + threadIdx.x; e < e1; e += kGsThreads) {
      T re = w[2 * e], im = w[2 * e + 1];
      for (int j = 0; j < kk; ++j) {
        const T vr = V[j * stride + 2 * e], vi = V[j * stride + 2 * e + 1];
        const T hr = T(hs[2 * j]), hi = T(hs[2 * j + 1]);
        re -= vr * hr - vi * hi;
        im -= vr * hi + vi * hr;
      }
      w[2 * e] = re;
      w[2 * e + 1] = im;
    }
    __syncthreads();
  }
  if constexpr (MODE <= 1) {
    for (int j = 0; j < kk; ++j) {
      C2<T> acc{T(0), T(0)};
      for (int64_t e = e0 + threadIdx.x; e < e1; e += kGsThreads) {
        const T vr = V[j * stride + 2 * e], vi = V[j * stride + 2 * e + 1];
        const T wr = w[2 * e], wi = w[2 * e + 1];
        acc.x += vr * wr + vi * wi;   // conj(v) w
        acc.y += vr * wi - vi * wr;
      }
      const C2<T> s = block_sum(acc, red);
      if (threadIdx.x == 0) {
        part_out[(size_t(blockIdx.x) * kGsMaxK + j) * 2] = double(s.x);
        part_out[(size_t(blockIdx.x) * kGsMaxK + j) * 2 + 1] = double(s.y);
      }
    }
  } else {
    C2<T> acc{T(0), T(0)};
    for (int64_t e = e0 + threadIdx.x; e < e1; e += kGsThreads) {
      const T wr = w[2 * e], wi = w[2 * e + 1];
      acc.x += wr * wr + wi * wi;
    }
    const C2<T> s = block_sum(acc, red);
    if (threadIdx.x == 0) {
      part_out[(size_t(blockIdx.x) * kGsMaxK) * 2] = double(s.x);
      part_out[(size_t(blockIdx.x) * kGsMaxK) * 2 + 1] = 0.0;
    }
  }
}

// v_out = w / |w| (norm from the pass-3 partials); hcol[0..kk) = h1 + h2,
// hcol[kk] = |w| (float64 pairs, the Hessenberg column)
template <typename T>
__global__ void __launch_bounds__(kGsThreads) gs_scale_kernel(const T* __restrict__ w, T* __restrict__ v_out,
                                                              int64_t n, int kk, const double* __restrict__ p1,
                                                              const double* __restrict__ p2,
                                                              const double* __restrict__ p3,
                                                              double* __restrict__ hcol) {
  __shared__ double nrm;
  if (threadIdx.x == 0) {
    double s = 0;
    for (int b = 0; b < kGsBlocks; ++b) s += p3[size_t(b) * kGsMaxK * 2];
    nrm = sqrt(s);
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int j = threadIdx.x; j < kk; j += blockDim.x) {
      double re = 0, im = 0;
      for (int b = 0; b < kGsBlocks; ++b) {
        re += p1[(size_t(b) * kGsMaxK + j) * 2] + p2[(size_t(b) * kGsMaxK + j) * 2];
        im += p1[(size_t(b) * kGsMaxK + j) * 2 + 1] + p2[(size_t(b) * kGsMaxK + j) * 2 + 1];
      }
      hcol[2 * j] = re;
      hcol[2 * j + 1] = im;
    }
    if (threadIdx.x == 0) {
      hcol[2 * kk] = nrm;
      hcol[2 * kk + 1] = 0.0;
    }
  }
  const T inv = nrm > 0 ? T(1.0 / nrm) : T(0);
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < 2 * n;
       e += int64_t(gridDim.x) * blockDim.x)
    v_out[e] = w[e] * inv;
}

template <typename T>
int gs_step(const T* V, int64_t stride, int kk, T* w, T* v_out, int64_t n, double* work, double* hcol,
            cudaStream_t st) {
  double* p1 = work;
  double* p2 = p1 + size_t(kGsBlocks) * kGsMaxK * 2;
  double* p3 = p2 + size_t(kGsBlocks) * kGsMaxK * 2;
  gs_pass_kernel<T, 0><<<kGsBlocks, kGsThreads, 0, st>>>(V, stride, kk, w, n, nullptr, p1);
  gs_pass_kernel<T, 1><<<kGsBlocks, kGsThreads, 0, st>>>(V, stride, kk, w, n, p1, p2);
  gs_pass_kernel<T, 2><<<kGsBlocks, kGsThreads, 0, st>>>(V, stride, kk, w, n, p2, p3);
  gs_scale_kernel<T><<<kGsBlocks, kGsThreads, 0, st>>>(w, v_out, n, kk, p1, p2, p3, hcol);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_solver_error = cudaGetErrorString(e);
    return NESA_ERR_CUDA;
  }
  return NESA_OK;
}

}  // namespace

#define NESA_SOLVER_API extern "C" __attribute__((visibility("default")))

// Work buffer size (bytes) for nesa_gs_step.
NESA_SOLVER_API int64_t nesa_gs_work_bytes(void) { return int64_t(3) * kGsBlocks * kGsMaxK * 2 * 8; }

NESA_SOLVER_API int nesa_gs_step(const void* basis, int64_t stride, int32_t kk, void* w, void* v_out,
                                 int64_t n, int32_t is_f64, void* work, void* hcol, void* stream) {
  if (!basis || !w || !v_out || !work || !hcol || kk < 1 || kk > kGsMaxK || n < 1) {
    g_solver_error = "bad nesa_gs_step arguments (1 <= kk <= 128)";
    return NESA_ERR_INVALID;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (is_f64)
    return gs_step<double>(static_cast<const double*>(basis), stride, kk, static_cast<double*>(w),
                           static_cast<double*>(v_out), n, static_cast<double*>(work),
                           static_cast<double*>(hcol), st);
  return gs_step<float>(static_cast<const float*>(basis), stride, kk, static_cast<float*>(w),
                        static_cast<float*>(v_out), n, static_cast<double*>(work), static_cast<double*>(hcol),
                        st);
}

NESA_SOLVER_API const char* nesa_gs_last_error(void) { return g_solver_error.c_str(); }
