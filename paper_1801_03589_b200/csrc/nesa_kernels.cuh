// nesa_kernels.cuh -- sm_100a kernels of the NESA matvec.
//
// One product (reference: fastmvp.py:142-172, mvp_serial) is
//   gather      qt = q[perm]                               (fastmvp.py:148)
//   near        phi_a = sum_b K_ab qt_b     per target leaf (152-156)
//   radiation   s_b = V_b qt_b              per leaf        (158-159)
//   upward      s_p = sum_c C_c s_c         per level L..l0+1 (160-162)
//   translation o_a = sum_b D_ab s_b        all levels      (163-166)
//   downward    o_c += B_c o_parent         per level l0+1..L (167-169)
//   reception   phi[perm] = phi_a + U_a o_a per leaf        (170-172)
//
// Every output slice has exactly one writer per launch (the ADD-exclusive
// handles of runtime.py:235-254 become single ownership): no atomics, and
// bitwise run-to-run determinism.  Vectors hold R interleaved real columns
// per row (R = 2 for one complex right-hand side).
#pragma once
#include <cstdint>

#include "nesa_ptx.cuh"

namespace nesa {

// ----------------------------------------------------------------------------
// Kernel timeline (diagnostics, NESA_KTRACE): when g_kt_buf is set, thread 0
// of every CTA of an instrumented kernel appends {tag, grid, start, end}
// (%globaltimer, ns) -- a non-perturbing view of the concurrent schedule that
// graph event nodes cannot give.  One global load + branch per CTA when off.
// ----------------------------------------------------------------------------
__device__ unsigned long long* g_kt_buf = nullptr;
__device__ unsigned int* g_kt_cnt = nullptr;
__device__ unsigned int g_kt_cap = 0;

__device__ __forceinline__ unsigned long long kt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// complex multiply on float2 (re, im)
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

struct KtScope {
  unsigned long long t0;
  unsigned long long* buf;  // the log, read once per CTA (thread 0)
  int tag;
  __device__ __forceinline__ explicit KtScope(int t) : t0(0), buf(nullptr), tag(t) {
    if (threadIdx.x == 0) {  // the load is consumed only at the end: no stall here
      buf = g_kt_buf;
      t0 = kt_now();
    }
  }
  __device__ __forceinline__ ~KtScope() {
    if (threadIdx.x == 0 && buf) {
      const unsigned int i = atomicAdd(g_kt_cnt, 1u);
      if (i < g_kt_cap) {
        unsigned long long* r = buf + 4ull * i;
        r[0] = (unsigned long long)tag;
        r[1] = gridDim.x;
        r[2] = t0;
        r[3] = kt_now();
      }
    }
  }
};

// ----------------------------------------------------------------------------
// Block GEMV engine (near field, radiation V, reception U)
// ----------------------------------------------------------------------------
// A work item is a dense m x n block stored column-major at blob[a_off]; its
// x vector is the concatenation of `seg_count` row ranges of x; its result
// goes to rows y_row0 .. y_row0+m-1.  Items are split into column chunks of
// at most kABytes so each chunk is ONE contiguous bulk copy (cp.async.bulk,
// the TMA bulk engine) into a kStages-deep shared-memory ring.  One producer
// warp issues the bulk copies plus cp.async gathers of x, both completing on
// the stage's mbarrier; eight consumer warps run the row dot products from
// shared memory.  Rows are owned by threads (r = t % m) with column lanes
// (cl = t / m) reduced in a fixed order at the end of the item.

template <typename T>
__device__ __forceinline__ void ld4(const T* p, T v[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

struct BlockItem {
  int64_t a_off;     // element offset of the column-major block in blob (multiple of 4)
  int32_t m, n;      // rows, columns
  int32_t ld;        // leading dimension: m rounded up to 4 (pad rows are zero)
  int32_t y_row0;    // first output row
  int32_t seg_begin; // segments [seg_begin, seg_begin + seg_count)
  int32_t seg_count;
  int32_t x0;        // radiation items: first point of the leaf (device assembly)
  int32_t pad;
};
struct BlockSeg {
  int32_t x_row0;  // first x row of the segment
  int32_t col0;    // first column (within the item) of the segment
};

// One bulk-copy chunk, self-contained in 128 bytes so the producer warp
// fetches it with ONE coalesced load (lane l <- word l) and prefetches the
// next one while the current is in flight: no dependent metadata loads on
// the streaming path.
constexpr int kRecSegs = 11;
struct __align__(128) ChunkRec {
  int64_t src_off;   // element offset of the chunk's first element in blob
  int32_t m;         // rows of the item
  int32_t ncols;     // columns in this chunk
  int32_t y_row0;    // first output row of the item
  int32_t flags;     // bit0 first chunk of its item, bit1 last chunk
  int32_t nseg;      // x segments of this chunk (<= kRecSegs)
  int32_t ld;        // leading dimension (multiple of 4)
  uint32_t magic;    // ceil(2^32 / (ld/4)): thread -> (row quad, column lane) without division
  int32_t CL;        // column lanes = consumer threads / (ld/4)
  int32_t seg[2 * kRecSegs];  // (x_row0, first column within the chunk) pairs
};
static_assert(sizeof(ChunkRec) == 128, "ChunkRec must be 128 bytes");

constexpr int kStages = 3;                 // default ring depth (2 CTAs / SM)
constexpr int kABytes = 16 * 1024;         // payload per stage
constexpr int kMaxC = 256;                 // columns per chunk
constexpr int kNCW = 8;                    // consumer warps
constexpr int kNCT = kNCW * 32;            // consumer threads
constexpr int kBGThreads = kNCT + 32;      // + producer warp
constexpr int kMaxRows = 2 * kNCT;         // rows per item (taller blocks are paneled)
constexpr int kBGPerSM = 2;                // resident CTAs per SM
// near-field geometry (measured in the full C4 product: 4 warps x 24 KB x 2
// stages 555 us, 4 x 16 KB x 3 556, 4 x 32 KB x 2 580, 8 x 16 KB x 3 633;
// fewer consumer threads and larger stages amortise the per-chunk consumer
// overhead that bounds an SM's share)
constexpr int kNearNCW = 4;
constexpr int kNearABytes = 24 * 1024;
constexpr int kNearStages = 2;

// kModeStoreCplx: store mode for a complex operator held row-split (rows
// 2r / 2r+1 = Re / Im of operator row r, R = 2: one complex column), the
// epilogue combines each row pair into y_r = (Re K) x + i (Im K) x
// kModeScatterCplx: the scatter mode for a row-split complex operator (the
// reception U of Track B): row pairs combine into one complex value, written
// to the original-order position of its real part (perm of the embedded
// vector) and the next element, plus the base (near-field) value.
enum { kModeStore = 0, kModeScatter = 1, kModeStoreCplx = 2, kModeScatterCplx = 3 };

template <typename T>
struct BlockGemvArgs {
  const T* blob;
  const ChunkRec* recs;
  const int32_t* cta_chunk_ptr;  // [grid + 1]
  const T* x;                    // x rows (R values each)
  T* y;                          // store: y rows; scatter: output in original order
  const T* base;                 // scatter: added per tree row (may be null)
  const int64_t* perm;           // scatter: tree row -> original row
  int ldy;                       // scatter: row stride of y (elements)
};

struct StageHdr {
  int32_t m, ncols, ld, flags, y_row0, CL;
  uint32_t magic;
  int32_t pad;
};

// Per-stage shared memory: [A | X | header | (scatter) perm | base]
template <typename T, int R, int MODE, int NST = kStages, int NCW = kNCW, int AB = kABytes>
struct BGLayout {
  static constexpr int kNCT = NCW * 32;
  static constexpr int kMaxC = AB / 64;  // columns per chunk
  static constexpr size_t kA = AB;
  static constexpr size_t kX = size_t(kMaxC) * R * sizeof(T);
  static constexpr bool kScat = MODE == kModeScatter || MODE == kModeScatterCplx;
  static constexpr size_t kFinPerm = kScat ? size_t(kMaxRows) * 8 : 0;
  static constexpr size_t kFinBase = kScat ? size_t(kMaxRows) * R * sizeof(T) : 0;
  static constexpr size_t kStage =
      ((kA + kX + sizeof(StageHdr) + kFinPerm + kFinBase) + 127) & ~size_t(127);
  // the end-of-item column-lane reduction reuses the finished chunk's A
  // buffer when it fits (keeps 2 CTAs/SM at ~57 KB, leaving room for the
  // concurrent far-field kernels); otherwise it gets its own area
  static constexpr size_t kRedNeed = size_t(4) * kNCT * R * sizeof(T);
  static constexpr bool kRedInA = kRedNeed <= kA;
  static constexpr size_t kRed = kRedInA ? 0 : kRedNeed;
  static constexpr size_t kBytes = NST * kStage + kRed + 2 * NST * sizeof(uint64_t) + 16;
  static constexpr size_t offX = kA;
  static constexpr size_t offHdr = kA + kX;
  static constexpr size_t offPerm = offHdr + sizeof(StageHdr);
  static constexpr size_t offBase = offPerm + kFinPerm;
};

template <typename T, int R, int MODE, int NST = kStages, int NCW = kNCW, int AB = kABytes>
constexpr size_t blockgemv_smem_bytes() {
  return BGLayout<T, R, MODE, NST, NCW, AB>::kBytes;
}

template <typename T, int R>
__device__ __forceinline__ void ldx(const T* p, T v[R]) {
  if constexpr (R * sizeof(T) == 8) {
    if constexpr (sizeof(T) == 4) {
      const float2 t = *reinterpret_cast<const float2*>(p);
      v[0] = t.x;
      v[1] = t.y;
    } else {
      v[0] = p[0];
    }
  } else if constexpr (R * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      const float4 t = *reinterpret_cast<const float4*>(p);
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
      const double2 t = *reinterpret_cast<const double2*>(p);
      v[0] = t.x;
      v[1] = t.y;
    }
  } else {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) v[rr] = p[rr];
  }
}


template <typename T, int R, int MODE, int NST = kStages, int NCW = kNCW, int AB = kABytes>
__global__ void __launch_bounds__(NCW * 32 + 32, NST * AB <= 3 * 16384 ? 2 : 1)
    blockgemv_kernel(const BlockGemvArgs<T> a) {
  KtScope kt_(10 + MODE);
  using Lay = BGLayout<T, R, MODE, NST, NCW, AB>;
  constexpr int kNCW = NCW;
  constexpr int kNCT = NCW * 32;
  constexpr int kStages = NST;
  extern __shared__ __align__(128) unsigned char smem[];
  T* const sRedOwn = reinterpret_cast<T*>(smem + kStages * Lay::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(smem + kStages * Lay::kStage + Lay::kRed) + 15) & ~uintptr_t(15));
  uint64_t* empty = full + kStages;

  const int c0 = a.cta_chunk_ptr[blockIdx.x];
  const int c1 = a.cta_chunk_ptr[blockIdx.x + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 33);  // 1 expect_tx arrival + 32 cp.async arrivals
      mbar_init(&empty[s], kNCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kNCW) {
    // ------------------------------ producer ------------------------------
    const int32_t* recw = reinterpret_cast<const int32_t*>(a.recs);
    const uint64_t pol = l2_evict_first_policy();
    int i0 = c0;
    const int i1 = c1;
    int k = 0;
    int32_t w_next = i0 < i1 ? __ldg(recw + int64_t(i0) * 32 + lane) : 0;
    while (i0 < i1) {
      const int i = i0++;
      const int32_t w = w_next;
      if (i + 1 < i1) w_next = __ldg(recw + int64_t(i + 1) * 32 + lane);
      const int st = k % kStages;
      const uint32_t round = uint32_t(k / kStages);
      ++k;
      unsigned char* stg = smem + size_t(st) * Lay::kStage;
      const uint32_t lo = uint32_t(__shfl_sync(0xffffffffu, w, 0));
      const uint32_t hi = uint32_t(__shfl_sync(0xffffffffu, w, 1));
      const int64_t src_off = int64_t((uint64_t(hi) << 32) | lo);
      const int m = __shfl_sync(0xffffffffu, w, 2);
      const int ncols = __shfl_sync(0xffffffffu, w, 3);
      const int y_row0 = __shfl_sync(0xffffffffu, w, 4);
      const int flags = __shfl_sync(0xffffffffu, w, 5);
      const int nseg = __shfl_sync(0xffffffffu, w, 6);
      const int ld = __shfl_sync(0xffffffffu, w, 7);
      const uint32_t magic = uint32_t(__shfl_sync(0xffffffffu, w, 8));
      const int CLv = __shfl_sync(0xffffffffu, w, 9);
      const uint32_t bytes = uint32_t(ncols) * uint32_t(ld) * uint32_t(sizeof(T));
      mbar_wait(&empty[st], (round & 1u) ^ 1u);
      if (lane == 0) {
        StageHdr* h = reinterpret_cast<StageHdr*>(stg + Lay::offHdr);
        h->m = m;
        h->ncols = ncols;
        h->ld = ld;
        h->flags = flags;
        h->y_row0 = y_row0;
        h->magic = magic;
        h->CL = CLv;
        mbar_arrive_expect_tx(&full[st], bytes);
        bulk_g2s_hint(stg, a.blob + src_off, bytes, &full[st], pol);
      }
      T* xs = reinterpret_cast<T*>(stg + Lay::offX);
      for (int sg = 0; sg < nseg; ++sg) {
        const int xr = __shfl_sync(0xffffffffu, w, 10 + 2 * sg);
        const int cs = __shfl_sync(0xffffffffu, w, 11 + 2 * sg);
        const int ce = sg + 1 < nseg ? __shfl_sync(0xffffffffu, w, 13 + 2 * sg) : ncols;
        for (int c = cs + lane; c < ce; c += 32)
          cp_async_n<R * sizeof(T)>(xs + c * R, a.x + int64_t(xr + (c - cs)) * R);
      }
      if constexpr (MODE == kModeScatter) {
        if (flags & 2) {
          int64_t* sp = reinterpret_cast<int64_t*>(stg + Lay::offPerm);
          T* sb = reinterpret_cast<T*>(stg + Lay::offBase);
          for (int r = lane; r < m; r += 32) {
            cp_async<8>(sp + r, a.perm + y_row0 + r);
            if (a.base) cp_async_n<R * sizeof(T)>(sb + r * R, a.base + int64_t(y_row0 + r) * R);
          }
        }
      } else if constexpr (MODE == kModeScatterCplx) {
        // complex rows: y_row0 and the rows below count complex points; perm
        // and base are those of the embedded (real, one column) vector
        if (flags & 2) {
          int64_t* sp = reinterpret_cast<int64_t*>(stg + Lay::offPerm);
          T* sb = reinterpret_cast<T*>(stg + Lay::offBase);
          for (int r = lane; r < (m >> 1); r += 32) {
            cp_async<8>(sp + r, a.perm + 2 * int64_t(y_row0 + r));
            if (a.base) cp_async_n<2 * sizeof(T)>(sb + 2 * r, a.base + 2 * int64_t(y_row0 + r));
          }
        }
      }
      cp_async_mbar_arrive_noinc(&full[st]);
    }
  } else {
    // ------------------------------ consumers -----------------------------
    // Thread (rq, cl): rows 4rq..4rq+3 of the item, columns cl, cl+CL, ...;
    // one 16-byte shared load of A per column; column lanes are reduced in
    // a fixed order at the end of the item.
    const int tid = threadIdx.x;
    T acc[4][R];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[i][rr] = T(0);
    for (int k = 0; k < c1 - c0; ++k) {
      const int st = k % kStages;
      const uint32_t round = uint32_t(k / kStages);
      const unsigned char* stg = smem + size_t(st) * Lay::kStage;
      mbar_wait(&full[st], round & 1u);
      const StageHdr h = *reinterpret_cast<const StageHdr*>(stg + Lay::offHdr);
      const int m = h.m, nc = h.ncols, ld = h.ld, CL = h.CL;
      const int RQ = ld >> 2;
      const int cl = RQ == 1 ? tid : int(__umulhi(uint32_t(tid), h.magic));
      const int rq = tid - cl * RQ;
      const T* A = reinterpret_cast<const T*>(stg);
      const T* X = reinterpret_cast<const T*>(stg + Lay::offX);
      if (h.flags & 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc[q][rr] = T(0);
      }
      if (cl < CL) {
        const T* Ap = A + 4 * rq;
#pragma unroll 4
        for (int c = cl; c < nc; c += CL) {
          T a4[4], xv[R];
          ld4(Ap + c * ld, a4);
          ldx<T, R>(X + c * R, xv);
#pragma unroll
          for (int q = 0; q < 4; ++q) fma_row<T, R>(acc[q], a4[q], xv);
        }
      }

      if (h.flags & 2) {  // last chunk of the item: reduce column lanes + write
        const int64_t* sperm = reinterpret_cast<const int64_t*>(stg + Lay::offPerm);
        const T* sbase = reinterpret_cast<const T*>(stg + Lay::offBase);
        T* sRed = sRedOwn;
        if constexpr (Lay::kRedInA) {
          sRed = reinterpret_cast<T*>(const_cast<unsigned char*>(stg));
          named_bar_sync(1, kNCT);  // every consumer is done reading this chunk's A
        }
        if (cl < CL) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int rr = 0; rr < R; ++rr) sRed[(cl * ld + 4 * rq + q) * R + rr] = acc[q][rr];
        }
        named_bar_sync(1, kNCT);
        if constexpr (MODE == kModeStoreCplx || MODE == kModeScatterCplx) {
          // rows 2cr, 2cr+1 of the item hold (Re K_cr) x and (Im K_cr) x,
          // each a complex value: y_cr = first + i * second
          static_assert(R == 2, "complex near: one complex column");
          for (int cr = tid; cr < (m >> 1); cr += kNCT) {
            T u0 = sRed[(2 * cr) * 2], u1 = sRed[(2 * cr) * 2 + 1];
            T w0 = sRed[(2 * cr + 1) * 2], w1 = sRed[(2 * cr + 1) * 2 + 1];
            for (int l = 1; l < CL; ++l) {
              u0 += sRed[(l * ld + 2 * cr) * 2];
              u1 += sRed[(l * ld + 2 * cr) * 2 + 1];
              w0 += sRed[(l * ld + 2 * cr + 1) * 2];
              w1 += sRed[(l * ld + 2 * cr + 1) * 2 + 1];
            }
            if constexpr (MODE == kModeStoreCplx) {
              const int64_t o = (int64_t(h.y_row0) + cr) * 2;
              a.y[o] = u0 - w1;
              a.y[o + 1] = u1 + w0;
            } else {
              const int64_t* sperm = reinterpret_cast<const int64_t*>(stg + Lay::offPerm);
              const T* sbase = reinterpret_cast<const T*>(stg + Lay::offBase);
              const int64_t dst = sperm[cr];
              a.y[dst * a.ldy] = (a.base ? sbase[2 * cr] : T(0)) + (u0 - w1);
              a.y[(dst + 1) * a.ldy] = (a.base ? sbase[2 * cr + 1] : T(0)) + (u1 + w0);
            }
          }
        }
        for (int row = tid; MODE != kModeStoreCplx && MODE != kModeScatterCplx && row < m; row += kNCT) {
          T v[R];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) v[rr] = sRed[row * R + rr];
          for (int l = 1; l < CL; ++l) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) v[rr] += sRed[(l * ld + row) * R + rr];
          }
          if constexpr (MODE == kModeStore || MODE == kModeStoreCplx) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) a.y[int64_t(h.y_row0 + row) * R + rr] = v[rr];
          } else {
            const int64_t dst = sperm[row];
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
              a.y[dst * a.ldy + rr] = (a.base ? sbase[row * R + rr] : T(0)) + v[rr];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        named_bar_sync(1, kNCT);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    }
  }
}

// ----------------------------------------------------------------------------
// gather qt[i] = q[perm[i]]; scatter phi[perm[i]] = phin[i]
// ----------------------------------------------------------------------------
// qt[iperm[j]] = q[j]: the gather walked in the original order --
// coalesced reads of q and iperm, scattered 8-byte writes that merge in L2
// (random 8-byte reads would each fetch a whole sector from DRAM)
template <typename T, int R>
__global__ void gather_inv_kernel(const T* __restrict__ q, const int32_t* __restrict__ iperm,
                                  T* __restrict__ qt, int64_t n, int ldq) {
  KtScope kt_(3);
  // four consecutive points per thread, every load of the group issued before
  // the first store (one memory round trip per group instead of per point)
  constexpr int U = 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * U;
  for (int64_t j0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * U; j0 < n; j0 += stride) {
    int32_t ii[U];
    T v[U][R];
    if (j0 + U <= n && (j0 & 3) == 0) {
      const int4 t = *reinterpret_cast<const int4*>(iperm + j0);
      ii[0] = t.x;
      ii[1] = t.y;
      ii[2] = t.z;
      ii[3] = t.w;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) ii[u] = j0 + u < n ? iperm[j0 + u] : -1;
    }
    if constexpr (R == 2 && sizeof(T) == 4) {
      if (ldq == 2 && j0 + U <= n && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
        const float4 a = *reinterpret_cast<const float4*>(q + j0 * 2);
        const float4 b = *reinterpret_cast<const float4*>(q + j0 * 2 + 4);
        v[0][0] = a.x; v[0][1] = a.y; v[1][0] = a.z; v[1][1] = a.w;
        v[2][0] = b.x; v[2][1] = b.y; v[3][0] = b.z; v[3][1] = b.w;
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int rr = 0; rr < R; ++rr) v[u][rr] = j0 + u < n ? q[(j0 + u) * ldq + rr] : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < n) *reinterpret_cast<float2*>(qt + int64_t(ii[u]) * 2) = make_float2(v[u][0], v[u][1]);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) v[u][rr] = j0 + u < n ? q[(j0 + u) * ldq + rr] : T(0);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < n)
#pragma unroll
          for (int rr = 0; rr < R; ++rr) qt[int64_t(ii[u]) * R + rr] = v[u][rr];
    }
  }
}

// phi[perm[i]] = phin[i] + phif[i] (a null term is zero), phi rows of stride ldp
template <typename T, int R>
__global__ void scatter_kernel(const T* __restrict__ phin, const T* __restrict__ phif,
                               const int64_t* __restrict__ perm, T* __restrict__ phi, int64_t row0,
                               int64_t n, int ldp) {
  KtScope kt_(2);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = perm[row0 + i];
    const int64_t k = (row0 + i) * R;
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
      phi[j * ldp + rr] = (phin ? phin[k + rr] : T(0)) + (phif ? phif[k + rr] : T(0));
  }
}

// ----------------------------------------------------------------------------
// Far-field micro-kernel.  All Q x Q operators (C, B, D) are stored
// transposed with the output index padded to Qp = ceil(Q/4)*4:
// MT[j * Qp + k] = M[k][j] (zero for k >= Q).  Amplitude vectors are staged
// in shared memory as X[j * NC + col], one column per (group, rhs).  Thread
// (rg, cg) owns a 4 x 4 register tile: rows 4rg.., columns 4cg.. and per j
// does two 16-byte shared loads for 16 FMAs.
// ----------------------------------------------------------------------------
constexpr int kFarThreads = 256;

struct FarGeom {
  int Q, Qp, RG, CG, NC;  // rows, padded rows, row groups, column groups, columns
};

__host__ __device__ inline FarGeom far_geom(int Q) {
  FarGeom g;
  g.Q = Q;
  g.Qp = (Q + 3) / 4 * 4;
  g.RG = g.Qp / 4;
  g.CG = kFarThreads / g.RG;
  g.NC = g.CG * 4;
  return g;
}

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  using type = float4;
};
template <>
struct Vec4<double> {
  using type = double4;
};

// acc[r][c] += sum_{j in [jb, je)} MT[j*Qp + k0 + r] * X[j*NC + c0 + c]
template <typename T>
__device__ __forceinline__ void mm4x4(const T* __restrict__ MT, const T* __restrict__ X,
                                      const FarGeom& G, int k0, int c0, T acc[4][4], int jb = 0,
                                      int je = -1) {
  if (je < 0) je = G.Q;
#pragma unroll 4
  for (int j = jb; j < je; ++j) {
    T m[4], x[4];
    ld4(MT + j * G.Qp + k0, m);
    ld4(X + j * G.NC + c0, x);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = fma(m[r], x[c], acc[r][c]);
  }
}

template <typename T>
__device__ __forceinline__ void zero4x4(T acc[4][4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
}

// bytes of one padded Q x Qp matrix, rounded to 16 B
__host__ __device__ inline size_t mat_bytes(int Q, size_t es) {
  return ((size_t(Q) * ((Q + 3) / 4 * 4) * es) + 15) & ~size_t(15);
}

// ----------------------------------------------------------------------------
// Level transfer kernels (one launch per level).  The level's groups are
// visited in `order` (sorted by child quadrant, then id), NC/R per CTA, so a
// CTA needs one quadrant matrix (two at a boundary).  Children-major form:
//   kLvlUpLeaf  T[c] = C_{quad c} s[c]                 (leaf level, s from V)
//   kLvlUpSum   s[c] = sum_k T[first child of c + k];  T[c] = C_{quad c} s[c]
//   kLvlDown    o[c] += B_{quad c} o[parent c]
// The parent's s is the ordered sum of its children's T (fastmvp.py:160-162
// accumulates s[parent] += C s[child] in child-id order); o[c] already holds
// its translation sum (reduce_kernel) when the downward kernel runs, matching
// fastmvp.py:163-169 (translations first, then potential transfer).
// Matrices arrive by bulk copy; amplitudes by cp.async or summed in staging.
// ----------------------------------------------------------------------------
//   kLvlDownBeta  (leaf level, float32 expansion plans) kLvlDown plus the
//                 reception coefficients beta^ = E^ o of the leaves
enum { kLvlUpLeaf = 0, kLvlUpSum = 1, kLvlDown = 2, kLvlDownBeta = 4 };

struct RecvArgs {
  const float* ET;          // [64][64]: ET[j * 64 + row] = E^[row][j] (row 0 = 1, 2m-1 / 2m = Re / Im (1/m) e^{-i m theta_j})
  float* beta;              // kLvlDownBeta: [NL][64][R] reception coefficients out
};

template <typename T, int R>
struct LevelArgs {
  const T* MT4;               // this level's four quadrant matrices (padded, transposed)
  const int32_t* quad;        // [G]
  const int32_t* order;       // level ids sorted by quadrant
  const int32_t* opar;        // kLvlDown: parent of order[i]
  const int2* ochild;         // kLvlUpSum: (first local child, count) of order[i]
  const T* Tin;               // kLvlUpSum: finer level's transfers
  T* s;                       // up: amplitudes (read leaf / written sum)
  T* Tout;                    // up: transfers out
  T* o;                       // down: incoming amplitudes
  int64_t count;
  int Q;
};

// ----------------------------------------------------------------------------
// Fused coarse levels.  The levels l0+1 .. lf (too small to fill the GPU) run
// as ONE kernel per pass instead of one launch per level:
//
//  fused_up_kernel    one CTA per level-lf group.  A CTA computes
//                     s[g] = sum of its children's T (fixed child order) and
//                     T[g] = C_{lv, quad g} s[g], then counts itself in at its
//                     parent; the LAST child to arrive continues with the
//                     parent (fence + atomic: the parent's sum is formed once,
//                     by one CTA, in child order -> deterministic).  At level
//                     l0 only s is formed (the old top-level sum).  No CTA
//                     ever waits, so residency does not matter.
//  fused_down_kernel  one CTA per level-lf group g.  Every coarse group is
//                     OWNED by the CTA of its first level-lf descendant (a
//                     host table), which computes o[a] += B_{lv, quad a}
//                     o[parent a] and publishes it (state 2).  A CTA waits
//                     once (for the parent of its top owned group), then runs
//                     its chain down to g.  CTAs take their group in start
//                     order (an atomic ticket, as decoupled look-back scans
//                     do), and an owner always precedes the groups below it,
//                     so a waited-for CTA has started: no deadlock without
//                     co-residency.
//
// The up kernel also resets the down-claim state of every group it passes
// and the last arriver resets the parent's counter, so no memset is needed
// between products.
// ----------------------------------------------------------------------------
template <typename T>
struct FusedArgs {
  const T* MT;            // C (up) / B (down) tables, padded + transposed
  size_t mstride;         // elements per matrix; level ci = lv - l0 >= 1: ((ci-1)*nkind + quad)
  const int32_t* quad;    // [G] child kind: quadrant (quadtree) or octant (octree)
  const int64_t* parent;  // [G]
  const int2* uchild;     // [G] local children (first id, count)
  const int32_t* anc;     // down: [count][D] ancestors of the level-lf groups (level lf-1 first)
  const int32_t* own;     // down: [count] ancestors each level-lf group's CTA owns (computes)
  const int4* chain_up;   // up: [count][D + 2] (group, first child, children, quad) from level lf to l0
  const int4* chain_down; // down: [count][D + 1] (x, parent x, quad x, own) top owned group first
  int* cnt;               // up: arrivals per group
  int* state;             // down: 0 pending, 2 done (reset by the up kernel)
  int* ticket;            // down: [2] start-order counter, finished CTAs
  T* Tup;
  T* s;
  T* o;
  int64_t first, count;   // level-lf groups (local)
  int lf, l0, L, Q, D;
  int nkind;              // child kinds per level: 4 (quadtree) or 8 (octree)
};

__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// acquire-release fence at GPU scope: publishes the CTA's prior writes
// (ordered before by bar.sync) / makes other CTAs' published writes visible;
// lighter than the sequentially consistent __threadfence()
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release_s32(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kFusedThreads = 128;

template <typename T>
// dynamic shared memory of the fused kernels: matrix, nvec vectors (up: 1,
// down: 2), 16 bytes of mbarrier + ticket / next, the chain constants
// (nchain = lf - l0 + 1 steps: group, quad; up also the children).  Kept
// tight: the float64 Q = 48 downward kernel fits 11 CTAs per SM only up to
// 20096 bytes per CTA (10 CTAs cost a third wave at C3: 56 -> 68 us).
__host__ __device__ inline size_t fused_smem_bytes(int Q, int R, int nvec, int nchain) {
  const size_t chain = size_t(nchain) * (nvec == 1 ? 13 : 5);
  return mat_bytes(Q, sizeof(T)) + nvec * ((size_t(Q) * R * sizeof(T) + 15) & ~size_t(15)) + 16 +
         ((chain + 15) & ~size_t(15));
}

template <typename T, int R>
__global__ void __launch_bounds__(kFusedThreads) fused_up_kernel(const FusedArgs<T> a) {
  KtScope kt_(30);
  extern __shared__ __align__(128) unsigned char smem[];
  const int Q = a.Q, Qp = (Q + 3) / 4 * 4, QR = Q * R, tid = threadIdx.x;
  const size_t mb = mat_bytes(Q, sizeof(T));
  T* M = reinterpret_cast<T*>(smem);
  T* X = reinterpret_cast<T*>(smem + mb);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + mb + ((size_t(QR) * sizeof(T) + 15) & ~size_t(15)));
  int64_t* nxt = reinterpret_cast<int64_t*>(bar + 1);
  int64_t g = a.first + blockIdx.x;
  int lv = a.lf;
  // plan constants of the CTA's whole ancestor chain (group, children,
  // quadrant per step): one packed 16-byte record per step, fetched in one
  // round trip ahead of the dependency wait, so the climb pays no index
  // round trips between its levels
  const int nstep = a.lf - a.l0 + 1;  // groups on the chain, level lf down to l0 (= D + 2)
  int2* ch_uc = reinterpret_cast<int2*>(nxt + 1);
  int32_t* ch_x = reinterpret_cast<int32_t*>(ch_uc + nstep);
  uint8_t* ch_quad = reinterpret_cast<uint8_t*>(ch_x + nstep);
  if (tid < nstep) {
    const int4 c = a.chain_up[int64_t(blockIdx.x) * nstep + tid];
    ch_x[tid] = c.x;
    ch_uc[tid] = make_int2(c.y, c.z);
    ch_quad[tid] = uint8_t(c.w);
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      if (lv > a.l0) {  // constant data: before the dependency wait
        mbar_arrive_expect_tx(bar, uint32_t(mb));
        bulk_g2s(M, a.MT + (size_t(lv - a.l0 - 1) * a.nkind + c.w) * a.mstride, uint32_t(mb), bar);
      }
    }
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  uint32_t phase = 0;
  int step = 0;
  while (true) {
    if (tid == 0) a.state[g] = 0;
    const int2 uc = ch_uc[step];
    for (int w = tid; w < QR; w += kFusedThreads) {
      T v;
      if (lv == a.L) {
        v = __ldcg(a.s + g * QR + w);
      } else {
        v = T(0);
        for (int k = 0; k < uc.y; ++k) v += __ldcg(a.Tup + (int64_t(uc.x) + k) * QR + w);
        a.s[g * QR + w] = v;
      }
      X[w] = v;
    }
    if (lv == a.l0) break;
    __syncthreads();
    mbar_wait(bar, phase);
    phase ^= 1u;
    for (int w = tid; w < QR; w += kFusedThreads) {
      const int k = w / R, rr = w - (w / R) * R;
      T acc = T(0);
#pragma unroll 8
      for (int j = 0; j < Q; ++j) acc = fma(M[j * Qp + k], X[j * R + rr], acc);
      a.Tup[g * QR + w] = acc;
    }
    __syncthreads();  // T[g] written, M and X consumed
    if (tid == 0) {
      const int64_t p = ch_x[step + 1];
      const int p_nch = ch_uc[step + 1].y, p_quad = ch_quad[step + 1];
      fence_acq_rel_gpu();  // release T[g] (and s[g]) to the parent's CTA
      const int old = atomicAdd(a.cnt + p, 1);
      const bool last = old == p_nch - 1;
      if (last) {
        fence_acq_rel_gpu();  // acquire the siblings' T
        a.cnt[p] = 0;         // (visible to the next launch at the kernel boundary)
        if (lv - 1 > a.l0) {
          mbar_arrive_expect_tx(bar, uint32_t(mb));
          bulk_g2s(M, a.MT + (size_t(lv - 1 - a.l0 - 1) * a.nkind + p_quad) * a.mstride, uint32_t(mb), bar);
        }
      }
      *nxt = last ? p : -1;
    }
    __syncthreads();
    const int64_t p = *nxt;
    if (p < 0) break;
    g = p;
    --lv;
    ++step;
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(kFusedThreads) fused_down_kernel(const FusedArgs<T> a) {
  KtScope kt_(31);
  extern __shared__ __align__(128) unsigned char smem[];
  const int Q = a.Q, Qp = (Q + 3) / 4 * 4, QR = Q * R, tid = threadIdx.x;
  const size_t mb = mat_bytes(Q, sizeof(T));
  const size_t vb = (size_t(QR) * sizeof(T) + 15) & ~size_t(15);
  T* M = reinterpret_cast<T*>(smem);
  T* X = reinterpret_cast<T*>(smem + mb);        // o[parent]
  T* Xo = reinterpret_cast<T*>(smem + mb + vb);  // o[x], the next step's parent vector
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + mb + 2 * vb);
  int* ticket = reinterpret_cast<int*>(bar + 1);
  int* s_own = ticket + 1;               // owned steps
  int32_t* ch_x = s_own + 1;             // [D + 2]: x per step, then the parent of the top owned group
  uint8_t* ch_quad = reinterpret_cast<uint8_t*>(ch_x + a.D + 2);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    *ticket = atomicAdd(a.ticket, 1);  // start-order index
  }
  __syncthreads();
  const int vid = *ticket;
  // This CTA owns the ancestors whose first level-lf descendant is g = first
  // + vid (its chain up to own[cta] levels; every coarse group has exactly
  // one owner).  It waits once -- for the parent of its top owned group,
  // published by that group's owner -- then computes its chain top down
  // without further waits, publishing each owned group for the CTAs below.
  // Step st handles x = anc[own - 1 - st] (st = own: g itself).  The chain's
  // plan constants (one packed record per step, one round trip) and the first
  // matrix are fetched ahead of the dependency wait; from the second step on
  // the parent's vector is the previous step's result (kept in shared
  // memory), so a step costs one matrix copy, overlapped with the release of
  // the previous group.
  if (tid <= a.D) {
    const int4 c = a.chain_down[vid * int64_t(a.D + 1) + tid];  // (entries past own are zero-filled)
    ch_x[tid] = c.x;
    ch_quad[tid] = uint8_t(c.z);
    if (tid == 0) {
      *s_own = c.w;
      ch_x[a.D + 1] = c.y;
    }
  }
  __syncthreads();
  const int own = *s_own;
  auto load_mat = [&](int st) {
    const int lvx = a.lf - own + st;  // level of step st's group
    mbar_arrive_expect_tx(bar, uint32_t(mb));
    bulk_g2s(M, a.MT + (size_t(lvx - a.l0 - 1) * a.nkind + ch_quad[st]) * a.mstride, uint32_t(mb), bar);
  };
  if (tid == 0) load_mat(0);  // constant data: before the dependency wait
  pdl_trigger();
  pdl_wait();  // o holds the translation sums
  uint32_t phase = 0;
  for (int st = 0; st <= own; ++st) {
    const int64_t x = ch_x[st];
    if (st == 0) {
      const int64_t px = ch_x[a.D + 1];
      if (a.lf - own - 1 > a.l0) {
        // the parent of the top owned group belongs to another CTA
        if (tid == 0) {
          unsigned ns = 64;
          while (ld_acquire_s32(a.state + px) != 2) {
            __nanosleep(ns);
            if (ns < 512) ns *= 2;
          }
        }
        __syncthreads();
      }
      for (int w = tid; w < QR; w += kFusedThreads) X[w] = __ldcg(a.o + px * QR + w);
    }
    __syncthreads();
    mbar_wait(bar, phase);
    phase ^= 1u;
    // o[x] += B_{lvx, quad x} o[parent x]
    for (int w = tid; w < QR; w += kFusedThreads) {
      const int k = w / R, rr = w - (w / R) * R;
      T acc = T(0);
#pragma unroll 8
      for (int j = 0; j < Q; ++j) acc = fma(M[j * Qp + k], X[j * R + rr], acc);
      // (x's own translation sum: an independent load, overlapped with the FMAs)
      const T val = __ldcg(a.o + x * QR + w) + acc;
      a.o[x * QR + w] = val;
      Xo[w] = val;
    }
    __syncthreads();  // o[x] written, M and X consumed
    if (tid == 0 && st < own) {
      load_mat(st + 1);  // overlaps the release below
      fence_acq_rel_gpu();
      st_release_s32(a.state + x, 2);
    }
    T* t = X;  // the next step's parent vector is this step's result
    X = Xo;
    Xo = t;
  }
  // the last CTA to finish resets the ticket counter for the next launch
  if (tid == 0 && atomicAdd(a.ticket + 1, 1) == int(gridDim.x) - 1) {
    a.ticket[0] = 0;
    a.ticket[1] = 0;
  }
}


// o[g] = sum_{e in interaction entries of g} Y[e] (entry order) for the
// listed groups: the translation sums of every level, one warp per group.
template <typename T, int R>
__global__ void reduce_kernel(const int32_t* __restrict__ ids, int64_t n_ids,
                              const int64_t* __restrict__ int_ptr, const T* __restrict__ Y, T* o,
                              int Q) {
  KtScope kt_(33);
  pdl_wait();
  const int QR = Q * R;
  const int lane = threadIdx.x & 31;
  const bool vec = (QR % 4) == 0;
  const uint64_t drop = l2_evict_first_policy();  // last use of Y
  for (int64_t wg = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; wg < n_ids;
       wg += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t g = ids[wg];
    const int64_t e0 = int_ptr[g], e1 = int_ptr[g + 1];
    if (vec) {
      for (int w = 4 * lane; w < QR; w += 128) {
        T v[4] = {T(0), T(0), T(0), T(0)};
        int64_t e = e0;
        for (; e + 2 <= e1; e += 2) {
          T a[4], b[4];
          if constexpr (sizeof(T) == 4) {
            const float4 fa = ld16_hint(Y + e * QR + w, drop), fb = ld16_hint(Y + (e + 1) * QR + w, drop);
            a[0] = fa.x; a[1] = fa.y; a[2] = fa.z; a[3] = fa.w;
            b[0] = fb.x; b[1] = fb.y; b[2] = fb.z; b[3] = fb.w;
          } else {
            ld4(Y + e * QR + w, a);
            ld4(Y + (e + 1) * QR + w, b);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = (v[i] + a[i]) + b[i];
        }
        if (e < e1) {
          T a[4];
          ld4(Y + e * QR + w, a);
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] += a[i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) o[g * QR + w + i] = v[i];
      }
    } else {
      for (int w = lane; w < QR; w += 32) {
        T v = T(0);
        for (int64_t e = e0; e < e1; ++e) v += Y[e * QR + w];
        o[g * QR + w] = v;
      }
    }
  }
  // (dependents start their prologue once this CTA's sums are done: the fused
  // downward kernel's 770 CTAs otherwise sit resident through the whole pass)
  pdl_trigger();
}

// ----------------------------------------------------------------------------
// Translation as a pair-major GEMM: Y[e] = D_{dtab} s[src(e)] for every
// interaction entry e.  Entries are grouped by unique D (operators.py:225-239
// caches D per (level, offset)); a unit = one D and up to kTUnitPasses x
// NC/R entries.  D arrives by bulk copy, sources by cp.async (double-
// buffered across passes); results go straight to Y (the per-target sums
// happen in the fused downward kernel, in reference order).
// ----------------------------------------------------------------------------
constexpr int kTUnitPasses = 8;

struct TUnit {
  int32_t dtab;
  int32_t ent_begin;  // into the dtab-sorted entry list
  int32_t ent_end;
  int32_t pad;
};
struct TEnt {
  int32_t src;  // source group
  int32_t e;    // interaction entry (Y row)
};

// Translation GEMM geometry: 128 threads, 8 x 4 register tile per thread
// (rows 8rg.., columns 4cg..): per j two 16-byte loads of D and one of the
// sources feed 32 FMAs.
constexpr int kTGThreads = 128;

struct TGGeom {
  int Q, Qp, RG, CG, NC;
};
__host__ __device__ inline TGGeom tg_geom(int Q) {
  TGGeom g;
  g.Q = Q;
  g.Qp = (Q + 3) / 4 * 4;               // table row stride
  g.RG = (Q + 7) / 8;                   // 8-row groups (rows >= Q are discarded)
  g.CG = kTGThreads / g.RG;
  g.NC = g.CG * 4;
  return g;
}

// Entry-major staging: source vector p lives at X + p * XS (XS = QR padded to
// 16 bytes plus 16 bytes, so column groups of one warp hit distinct banks);
// each vector arrives as ONE bulk copy when QR * sizeof(T) is a multiple of
// 16 (the usual case), else by 4/8-byte cp.async.
template <typename T>
__host__ __device__ inline int tg_xstride(int QR) {
  const int per16 = 16 / int(sizeof(T));
  return (QR + per16 - 1) / per16 * per16 + per16;
}

template <typename T, int R>
size_t tgemm_smem_bytes(int Q) {
  const TGGeom G = tg_geom(Q);
  const size_t xb = (size_t(G.NC / R) * tg_xstride<T>(Q * R) * sizeof(T) + 127) & ~size_t(127);
  return mat_bytes(Q, sizeof(T)) + 64 /* row overrun pad */ + 2 * xb + 2 * 4 * size_t(G.NC) + 64;
}

template <typename T, int R>
__device__ __forceinline__ void tgemm_stage(const TEnt* ents, int eb, int n, const T* s,
                                            const TGGeom& G, T* X, int XS, int32_t* eid,
                                            uint64_t* bar, int tid) {
  const int QR = G.Q * R;
  const uint32_t vb = uint32_t(QR * sizeof(T));
  if ((vb & 15u) == 0) {
    if (tid < 32) {
      if (tid == 0) mbar_arrive_expect_tx(bar, vb * uint32_t(n));
      __syncwarp();
      for (int p = tid; p < n; p += 32) {
        const TEnt te = ents[eb + p];
        eid[p] = te.e;
        bulk_g2s(X + p * XS, s + int64_t(te.src) * QR, vb, bar);
      }
    }
  } else {
    for (int p = tid >> 5; p < n; p += kTGThreads / 32) {
      const TEnt te = ents[eb + p];
      if ((tid & 31) == 0) eid[p] = te.e;
      const T* src = s + int64_t(te.src) * QR;
      for (int w = tid & 31; w < QR; w += 32) cp_async<sizeof(T)>(X + p * XS + w, src + w);
    }
    cp_async_commit();
    if (tid == 0) mbar_arrive(bar);
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(kTGThreads) tgemm_kernel(const TUnit* __restrict__ units,
                                                           const TEnt* __restrict__ ents,
                                                           const T* __restrict__ DT,
                                                           const T* __restrict__ s, T* Y, int Q) {
  KtScope kt_(40);
  extern __shared__ __align__(128) unsigned char smem[];
  const TGGeom G = tg_geom(Q);
  const int QR = Q * R, per = G.NC / R;
  const int XS = tg_xstride<T>(QR);
  const size_t mb = mat_bytes(Q, sizeof(T));
  const size_t xb = (size_t(per) * XS * sizeof(T) + 127) & ~size_t(127);
  T* Dm = reinterpret_cast<T*>(smem);
  T* Xb[2] = {reinterpret_cast<T*>(smem + mb + 64), reinterpret_cast<T*>(smem + mb + 64 + xb)};
  int32_t* Eb[2] = {reinterpret_cast<int32_t*>(smem + mb + 64 + 2 * xb), nullptr};
  Eb[1] = Eb[0] + G.NC;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Eb[1] + G.NC);  // [0] D, [1] X0, [2] X1
  const TUnit u = units[blockIdx.x];
  const int tid = threadIdx.x;
  const int rg = tid % G.RG, cg = tid / G.RG;
  const bool bulk = ((QR * sizeof(T)) & 15) == 0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar[0], uint32_t(mb));
    bulk_g2s(Dm, reinterpret_cast<const unsigned char*>(DT) + size_t(u.dtab) * mb, uint32_t(mb),
             &bar[0]);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  const int n_all = u.ent_end - u.ent_begin;
  const int npass = (n_all + per - 1) / per;
  tgemm_stage<T, R>(ents, u.ent_begin, min(per, n_all), s, G, Xb[0], XS, Eb[0], &bar[1], tid);
  mbar_wait(&bar[0], 0);
  for (int ps = 0; ps < npass; ++ps) {
    const int b = ps & 1;
    const T* X = b ? Xb[1] : Xb[0];
    const int32_t* eid = b ? Eb[1] : Eb[0];
    const int eb = u.ent_begin + ps * per;
    const int n = min(per, u.ent_end - eb);
    if (ps + 1 < npass) {
      const int eb2 = eb + per;
      tgemm_stage<T, R>(ents, eb2, min(per, u.ent_end - eb2), s, G, b ? Xb[0] : Xb[1], XS,
                        b ? Eb[0] : Eb[1], &bar[1 + (b ^ 1)], tid);
    }
    if (!bulk) {
      if (ps + 1 < npass)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      else
        cp_async_wait_all();
    }
    mbar_wait(&bar[1 + b], uint32_t(ps >> 1) & 1u);
    __syncthreads();
    if (cg < G.CG && 4 * cg < n * R) {
      T acc[8][4];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
      const T* mp = Dm + 8 * rg;
      // column c of this thread = entry (4cg + c) / R, component (4cg + c) % R
      const T* xq[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = 4 * cg + c;
        xq[c] = X + (col / R) * XS + (col % R);
      }
#pragma unroll 2
      for (int j = 0; j < G.Q; ++j) {
        T m0[4], m1[4], x[4];
        ld4(mp + j * G.Qp, m0);
        ld4(mp + j * G.Qp + 4, m1);
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c] = xq[c][j * R];
        tile_fma8x4<T>(acc, m0, m1, x);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = 4 * cg + c, p = col / R, rr = col % R;
        if (p >= n) continue;
        T* dst = Y + int64_t(eid[p]) * QR + rr;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (8 * rg + r < Q) dst[(8 * rg + r) * R] = acc[r][c];
      }
    }
    __syncthreads();  // X buffer reuse
  }
}

// ----------------------------------------------------------------------------
// Warp-tiled translation GEMM for Q in {32, 64, 128} (the benchmark uses 64).
// 128 threads = RW row-warps x CW column-warps, each warp a 32 x 32 tile of
// Y = D S: lane (tr = lane / 8, tc = lane % 8) owns rows 8tr..8tr+7 and
// columns 4tc..4tc+3.  Per j the 8 lanes of a row group read the same D
// words (broadcast) and the four row groups one contiguous 128-byte line, so
// a warp issues ~4 shared wavefronts per 32 FMAs.
// ----------------------------------------------------------------------------
// QT output rows; KT input length (KT = QT for the square far-field
// operators; the radiation's moment map uses KT > QT).
template <typename T, int R, int QT, int KT = QT>
struct TGW {
  static constexpr int RW = QT / 32;
  static constexpr int CW = 4 / RW;
  static constexpr int NC = 32 * CW;       // real columns per pass
  static constexpr int PER = NC / R;       // entries per pass
  static constexpr int QR = QT * R;        // output values per entry
  static constexpr int KR = KT * R;        // input values per entry
  static constexpr int XS = ((KR > QR ? KR : QR) + 16 / int(sizeof(T)) - 1) / (16 / int(sizeof(T))) *
                                (16 / int(sizeof(T))) + 16 / int(sizeof(T));
  static constexpr size_t MB = size_t(KT) * QT * sizeof(T);
  static constexpr size_t XB = (size_t(PER) * XS * sizeof(T) + 127) & ~size_t(127);
  static constexpr size_t SMEM = MB + 2 * XB + 2 * 4 * PER + 64;
};

template <typename T, int R, int QT, int KT = QT>
__global__ void __launch_bounds__(128) tgemm_wt_kernel(const TUnit* __restrict__ units,
                                                       const TEnt* __restrict__ ents,
                                                       const T* __restrict__ DT,
                                                       const T* __restrict__ s, T* Y) {
  KtScope kt_(41);
  using W = TGW<T, R, QT, KT>;
  extern __shared__ __align__(128) unsigned char smem[];
  T* Dm = reinterpret_cast<T*>(smem);
  T* Xb0 = reinterpret_cast<T*>(smem + W::MB);
  T* Xb1 = reinterpret_cast<T*>(smem + W::MB + W::XB);
  int32_t* Eb0 = reinterpret_cast<int32_t*>(smem + W::MB + 2 * W::XB);
  int32_t* Eb1 = Eb0 + W::PER;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Eb1 + W::PER);  // [0] D, [1] X0, [2] X1
  const TUnit u = units[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp % W::RW, wc = warp / W::RW;
  const int tr = lane >> 3, tc = lane & 7;
  const int row0 = 32 * wr + 8 * tr;   // first output row of this thread
  // this thread's entries: e_i = E0 + tc + 8 i (i < 4/R), components rr < R;
  // the 8 lanes of a row group read 8 consecutive entries (conflict-free)
  constexpr int NE = 4 / R;
  const int E0 = 32 * wc / R;
  constexpr uint32_t kVB = uint32_t(W::KR * sizeof(T));
  const size_t mb = W::MB;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar[0], uint32_t(mb));
    bulk_g2s(Dm, reinterpret_cast<const unsigned char*>(DT) + size_t(u.dtab) * mb, uint32_t(mb),
             &bar[0]);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // s comes from the upward pass
  auto stage = [&](int eb, int n, T* X, int32_t* eid, uint64_t* b) {
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(b, kVB * uint32_t(n));
      __syncwarp();
      for (int p = lane; p < n; p += 32) {
        const TEnt te = ents[eb + p];
        eid[p] = te.e;
        bulk_g2s(X + p * W::XS, s + int64_t(te.src) * W::KR, kVB, b);
      }
    }
  };
  const int n_all = u.ent_end - u.ent_begin;
  const int npass = (n_all + W::PER - 1) / W::PER;
  stage(u.ent_begin, min(W::PER, n_all), Xb0, Eb0, &bar[1]);
  mbar_wait(&bar[0], 0);
  for (int ps = 0; ps < npass; ++ps) {
    const int b = ps & 1;
    const T* X = b ? Xb1 : Xb0;
    const int32_t* eid = b ? Eb1 : Eb0;
    const int eb = u.ent_begin + ps * W::PER;
    const int n = min(W::PER, u.ent_end - eb);
    if (ps + 1 < npass)
      stage(eb + W::PER, min(W::PER, u.ent_end - eb - W::PER), b ? Xb0 : Xb1, b ? Eb0 : Eb1,
            &bar[1 + (b ^ 1)]);
    mbar_wait(&bar[1 + b], uint32_t(ps >> 1) & 1u);
    __syncthreads();  // eid visible
    const bool active = E0 + tc < n;
    T acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
    if (active) {
      const T* mp = Dm + row0;
      const T* xp = X + (E0 + tc) * W::XS;
#pragma unroll 4
      for (int j = 0; j < KT; ++j) {
        T m0[4], m1[4], x[4];
        ld4(mp + j * QT, m0);
        ld4(mp + j * QT + 4, m1);
#pragma unroll
        for (int i = 0; i < NE; ++i) ldx<T, R>(xp + i * 8 * W::XS + j * R, x + i * R);
        tile_fma8x4<T>(acc, m0, m1, x);
      }
    }
    // stage the tile entry-major in the consumed X buffer, then write each
    // entry's contiguous QR block with 16-byte stores (no partial sectors)
    __syncthreads();
    T* O = (b ? Xb1 : Xb0);
    if (active) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int p = E0 + tc + 8 * (c / R), rr = c % R;
#pragma unroll
        for (int r = 0; r < 8; ++r) O[p * W::XS + (row0 + r) * R + rr] = acc[r][c];
      }
    }
    __syncthreads();
    {
      constexpr int V = 16 / int(sizeof(T));  // elements per 16-byte store
      constexpr int NV = W::QR / V;
      const uint64_t keep = l2_evict_last_policy();  // Y is re-read by reduce_kernel
      for (int i = tid; i < n * NV; i += 128) {
        const int p = i / NV, v = i - p * NV;
        const float4 val = *reinterpret_cast<const float4*>(O + p * W::XS + v * V);
        st16_hint(Y + int64_t(eid[p]) * W::QR + v * V, val, keep);
      }
    }
    __syncthreads();  // X buffer reuse
  }
}

// ----------------------------------------------------------------------------
// Translation GEMM on the 5th-generation tensor cores (float32 plans, Q = 64).
//   Y_e = D_{dtab} s_src(e) for the <= 128 / R entries of a unit, as ONE
//   M = 128 tile: A = the unit's sources, one row per (entry, component)
//   (K = 64 = source coefficients), B = D (N = 64 output rows, K-major =
//   D row-major), accumulator 128 lanes x 64 columns fp32 in TMEM.
// float32 accuracy from TF32 operands by the 3-term split
//   D s ~= D_hi s_hi + D_hi s_lo + D_lo s_hi   (x_hi = tf32(x), x_lo = tf32(x - x_hi))
// (the dropped D_lo s_lo term is ~2^-22 relative): 3 x 8 tcgen05.mma (K = 8
// each) issued by one thread.  D_hi / D_lo arrive pre-split in the canonical
// no-swizzle K-major layout (core matrices of 8 rows x 16 bytes; the two K
// chunks of a core-matrix pair 128 B apart (LBO), 8-row groups 2048 B apart
// (SBO)) by one bulk copy; the sources are split while being staged.  The
// epilogue moves TMEM -> registers (tcgen05.ld 32x32b: thread = lane = row)
// -> smem -> coalesced 16-byte stores of Y.
// ----------------------------------------------------------------------------
constexpr int kTcLBO = 128;                  // bytes between the K-adjacent core matrices
constexpr int kTcSBO = 2048;                 // bytes between 8-row groups (16 K chunks)
constexpr uint32_t kTcBBytes = 64 * 64 * 4;  // one 64 x 64 tf32 operand (16 KB)

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}

__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((kTcLBO >> 4) & 0x3FFF) << 16;
  d |= uint64_t((kTcSBO >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // sm100 descriptor version; base offset 0, no swizzle
  return d;
}

// kind::tf32, D = F32, A = B = TF32, both K-major, N = 64, M = 128
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kTcIdesc), "r"(accumulate));
}


// Variant with the A operand (sources, split hi / lo) in TMEM instead of
// shared memory (tcgen05.mma ... [d], [a_tmem], b_desc): thread m = TMEM
// lane m writes its row with tcgen05.st, and the epilogue stages half a
// tile at a time, so the kernel needs ~50 KB of shared memory and two CTAs
// fit beside the near field's two on an SM.  TMEM: 256 columns =
// accumulator [0, 64) | A_hi [64, 128) | A_lo [128, 192).
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(accumulate), "r"(kTcIdesc), "r"(0u));
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, float4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
               "r"(__float_as_uint(v.w))
               : "memory");
}

template <int R>
__global__ void __launch_bounds__(128) tgemm_tc2_kernel(const TUnit* __restrict__ units,
                                                        const TEnt* __restrict__ ents,
                                                        const float* __restrict__ DTC,
                                                        const float* __restrict__ s, float* Y) {
  KtScope kt_(43);
  constexpr int QT = 64, QR = QT * R;
  constexpr int EPT = 128 / R;   // entries per M = 128 tile
  constexpr int HALF = EPT / 2;  // entries staged per epilogue round
  constexpr int OS = QR + 4;
  extern __shared__ __align__(128) unsigned char smem[];
  float* Bhi = reinterpret_cast<float*>(smem);        // 16 KB
  float* Blo = Bhi + 4096;                             // 16 KB
  float* stage = Blo + 4096;                           // HALF x OS floats
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + ((HALF * OS + 3) & ~3));  // [0] D, [1] MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  int32_t* eids = reinterpret_cast<int32_t*>(tslot + 4);
  const TUnit u = units[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar[0], 2 * kTcBBytes);
    bulk_g2s(Bhi, DTC + size_t(u.dtab) * (2 * 4096), 2 * kTcBBytes, &bar[0]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  const uint32_t t_acc = tmem + lane_base, t_hi = tmem + lane_base + 64, t_lo = tmem + lane_base + 128;
  pdl_trigger();
  pdl_wait();  // s comes from the upward pass
  const int n_all = u.ent_end - u.ent_begin;
  const int m = tid, e = m / R, rr = m - (m / R) * R;
  float4 c[16];
  int32_t eid = -1;
  auto load = [&](int t0) {
    const bool live = t0 + e < n_all;
    eid = -1;
    int64_t srcg = 0;
    if (live) {
      const TEnt te = ents[u.ent_begin + t0 + e];
      eid = te.e;
      srcg = te.src;
    }
    if constexpr (R == 1 || R == 2) {
      const float4* src4 = reinterpret_cast<const float4*>(s + srcg * QR) + rr * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = live ? src4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const float* src = s + srcg * QR + rr;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        c[i] = live ? make_float4(src[(4 * i) * R], src[(4 * i + 1) * R], src[(4 * i + 2) * R],
                                  src[(4 * i + 3) * R])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto put = [&](int kb, float4 v) {  // columns 4kb..4kb+3 of this thread's row
    float4 h, l;
    h.x = tf32_rna(v.x);
    h.y = tf32_rna(v.y);
    h.z = tf32_rna(v.z);
    h.w = tf32_rna(v.w);
    l.x = tf32_rna(v.x - h.x);
    l.y = tf32_rna(v.y - h.y);
    l.z = tf32_rna(v.z - h.z);
    l.w = tf32_rna(v.w - h.w);
    tmem_st4(t_hi + 4 * kb, h);
    tmem_st4(t_lo + 4 * kb, l);
  };
  uint32_t phase = 0;
  load(0);
  for (int t0 = 0; t0 < n_all; t0 += EPT) {
    const int eid_t = eid;
    if constexpr (R == 1 || R == 4) {
      // R = 1: c[i] = k 4i..4i+3 of this row; R = 4: the loader fetched the
      // component rr strided (one float4 = 4 consecutive k)
#pragma unroll
      for (int kb = 0; kb < 16; ++kb) put(kb, c[kb]);
    } else {
      float mine[32], other[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        mine[2 * i] = rr ? c[i].y : c[i].x;
        mine[2 * i + 1] = rr ? c[i].w : c[i].z;
        other[2 * i] = rr ? c[i].x : c[i].y;
        other[2 * i + 1] = rr ? c[i].z : c[i].w;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) other[i] = __shfl_xor_sync(0xffffffffu, other[i], 1);
      // tcgen05.st is warp-collective (one column address per warp): lane rr
      // owns k in [32 rr, 32 rr + 32) as `mine`, the rest as `other`
#pragma unroll
      for (int kb = 0; kb < 8; ++kb) {
        const float4 a = make_float4(mine[4 * kb], mine[4 * kb + 1], mine[4 * kb + 2], mine[4 * kb + 3]);
        const float4 b = make_float4(other[4 * kb], other[4 * kb + 1], other[4 * kb + 2], other[4 * kb + 3]);
        put(kb, rr ? b : a);       // k in [0, 32)
        put(8 + kb, rr ? a : b);   // k in [32, 64)
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      if (t0 == 0) mbar_wait(&bar[0], 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t bh = smem_u32(Bhi), bl = smem_u32(Blo);
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        const uint32_t a0 = tmem + (cc == 2 ? 128u : 64u), b0 = cc == 1 ? bl : bh;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_tf32_ts(tmem, a0 + ks * 8, umma_desc_kmajor(b0 + ks * 2 * kTcLBO), (cc | ks) != 0);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar[1]))
                   : "memory");
    }
    if (t0 + EPT < n_all) load(t0 + EPT);  // overlaps the tensor core
    mbar_wait(&bar[1], phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]),
          "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]),
          "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
          "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]),
          "=r"(r[63])
        : "r"(t_acc));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (rr == 0) eids[e] = eid_t;
    const int n = min(EPT, n_all - t0);
    const uint64_t keep = l2_evict_last_policy();  // Y is re-read by reduce_kernel
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e0 = h * HALF;
      if (e >= e0 && e < e0 + HALF && eid_t >= 0)
#pragma unroll
        for (int k = 0; k < 64; ++k) stage[(e - e0) * OS + k * R + rr] = __uint_as_float(r[k]);
      __syncthreads();
      constexpr int NV = QR / 4;
      const int nh = max(0, min(HALF, n - e0));
      for (int i = tid; i < nh * NV; i += 128) {
        const int ee = i / NV, v = i - (i / NV) * NV;
        const float4 val = *reinterpret_cast<const float4*>(stage + ee * OS + 4 * v);
        st16_hint(Y + int64_t(eids[e0 + ee]) * QR + 4 * v, val, keep);
      }
      __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

constexpr int kTc3CtasPerSM = 1;  // persistent translation CTAs per SM (A/B: 1 per SM 0.6 us faster
                                   // than 2: TMEM left to the concurrent level kernels)

// Persistent form of tgemm_tc2_kernel: a CTA loops over units (grid-stride),
// allocates TMEM once, and fetches the next unit's D as soon as the last MMA
// of the current one has consumed the D buffer, so the D copy, the next
// sources and the epilogue overlap instead of paying one CTA start per unit.
// Register budget of the tensor-core far-field kernels (128 threads, one warp
// per SM sub-partition).  A sub-partition's 16384 registers hold up to 3 of the
// near field's 10 warps (2 CTAs x 5 warps x 64 registers x 32 = 6144), which
// leaves 10240 for one translation warp AND one level-kernel warp: 160 + 160
// registers per thread.  At the natural 240 + 168 the upward level kernels
// could not become resident beside the persistent translation and waited
// ~40 us for its CTAs to exit (ktrace, profiles/r2_ktrace_sched.txt).  Only
// the complex64 bench path (R = 2) is capped; R = 1 / 4 would spill.
constexpr int kTcFarMaxReg = 160;
template <int R>
__global__ void __maxnreg__(R == 2 ? kTcFarMaxReg : 255) tgemm_tc3_kernel(const TUnit* __restrict__ units, int n_units,
                                                        const TEnt* __restrict__ ents,
                                                        const float* __restrict__ DTC,
                                                        const float* __restrict__ s, float* Y, int tag = 44) {
  KtScope kt_(tag);
  constexpr int QT = 64, QR = QT * R;
  constexpr int EPT = 128 / R;
  constexpr int HALF = EPT / 2;
  constexpr int OS = QR + 4;
  extern __shared__ __align__(128) unsigned char smem[];
  float* Bhi = reinterpret_cast<float*>(smem);
  float* Blo = Bhi + 4096;
  float* stage = Blo + 4096;
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + ((HALF * OS + 3) & ~3));  // [0] D, [1] MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  int32_t* eids = reinterpret_cast<int32_t*>(tslot + 4);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  int ui = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    if (ui < n_units) {
      mbar_arrive_expect_tx(&bar[0], 2 * kTcBBytes);
      bulk_g2s(Bhi, DTC + size_t(units[ui].dtab) * (2 * 4096), 2 * kTcBBytes, &bar[0]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  const uint32_t t_acc = tmem + lane_base, t_hi = tmem + lane_base + 64, t_lo = tmem + lane_base + 128;
  pdl_trigger();
  pdl_wait();  // s comes from the upward pass
  const int m = tid, e = m / R, rr = m - (m / R) * R;
  float4 c[16];
  int32_t eid = -1;
  auto load = [&](const TUnit& uu, int t0) {
    const int na = uu.ent_end - uu.ent_begin;
    const bool live = t0 + e < na;
    eid = -1;
    int64_t srcg = 0;
    if (live) {
      const TEnt te = ents[uu.ent_begin + t0 + e];
      eid = te.e;
      srcg = te.src;
    }
    if constexpr (R == 1 || R == 2) {
      const float4* src4 = reinterpret_cast<const float4*>(s + srcg * QR) + rr * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = live ? src4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const float* src = s + srcg * QR + rr;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        c[i] = live ? make_float4(src[(4 * i) * R], src[(4 * i + 1) * R], src[(4 * i + 2) * R],
                                  src[(4 * i + 3) * R])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto put = [&](int kb, float4 v) {
    float4 h, l;
    h.x = tf32_rna(v.x);
    h.y = tf32_rna(v.y);
    h.z = tf32_rna(v.z);
    h.w = tf32_rna(v.w);
    l.x = tf32_rna(v.x - h.x);
    l.y = tf32_rna(v.y - h.y);
    l.z = tf32_rna(v.z - h.z);
    l.w = tf32_rna(v.w - h.w);
    tmem_st4(t_hi + 4 * kb, h);
    tmem_st4(t_lo + 4 * kb, l);
  };
  const uint64_t keep = l2_evict_last_policy();  // Y is re-read by reduce_kernel
  uint32_t phase = 0, dphase = 0;
  TUnit u = ui < n_units ? units[ui] : TUnit{0, 0, 0, 0};
  if (ui < n_units) load(u, 0);
  while (ui < n_units) {
    const int n_all = u.ent_end - u.ent_begin;
    const int next = ui + int(gridDim.x);
    const TUnit un = next < n_units ? units[next] : TUnit{0, 0, 0, 0};
    for (int t0 = 0; t0 < n_all; t0 += EPT) {
      const bool last_tile = t0 + EPT >= n_all;
      const int eid_t = eid;
      if constexpr (R == 1 || R == 4) {
#pragma unroll
        for (int kb = 0; kb < 16; ++kb) put(kb, c[kb]);
      } else {
        float mine[32], other[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          mine[2 * i] = rr ? c[i].y : c[i].x;
          mine[2 * i + 1] = rr ? c[i].w : c[i].z;
          other[2 * i] = rr ? c[i].x : c[i].y;
          other[2 * i + 1] = rr ? c[i].z : c[i].w;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) other[i] = __shfl_xor_sync(0xffffffffu, other[i], 1);
#pragma unroll
        for (int kb = 0; kb < 8; ++kb) {
          const float4 a = make_float4(mine[4 * kb], mine[4 * kb + 1], mine[4 * kb + 2], mine[4 * kb + 3]);
          const float4 b = make_float4(other[4 * kb], other[4 * kb + 1], other[4 * kb + 2], other[4 * kb + 3]);
          put(kb, rr ? b : a);
          put(8 + kb, rr ? a : b);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        if (t0 == 0) {
          mbar_wait(&bar[0], dphase);
          dphase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bh = smem_u32(Bhi), bl = smem_u32(Blo);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          const uint32_t a0 = tmem + (cc == 2 ? 128u : 64u), b0 = cc == 1 ? bl : bh;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            umma_tf32_ts(tmem, a0 + ks * 8, umma_desc_kmajor(b0 + ks * 2 * kTcLBO), (cc | ks) != 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar[1]))
                     : "memory");
      }
      // prefetch the next tile's sources (this unit's or the next unit's first)
      if (!last_tile)
        load(u, t0 + EPT);
      else if (next < n_units)
        load(un, 0);
      mbar_wait(&bar[1], phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // D consumed: fetch the next unit's D while the epilogue runs
      if (last_tile && tid == 0 && next < n_units) {
        mbar_arrive_expect_tx(&bar[0], 2 * kTcBBytes);
        bulk_g2s(Bhi, DTC + size_t(un.dtab) * (2 * 4096), 2 * kTcBBytes, &bar[0]);
      }
      uint32_t r[64];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
          "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
          "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
            "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
            "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]),
            "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]),
            "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
            "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
            "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]),
            "=r"(r[63])
          : "r"(t_acc));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (rr == 0) eids[e] = eid_t;
      const int n = min(EPT, n_all - t0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e0 = h * HALF;
        if (e >= e0 && e < e0 + HALF && eid_t >= 0)
#pragma unroll
          for (int k = 0; k < 64; ++k) stage[(e - e0) * OS + k * R + rr] = __uint_as_float(r[k]);
        __syncthreads();
        constexpr int NV = QR / 4;
        const int nh = max(0, min(HALF, n - e0));
        for (int i = tid; i < nh * NV; i += 128) {
          const int ee = i / NV, v = i - (i / NV) * NV;
          const float4 val = *reinterpret_cast<const float4*>(stage + ee * OS + 4 * v);
          st16_hint(Y + int64_t(eids[e0 + ee]) * QR + 4 * v, val, keep);
        }
        __syncthreads();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    ui = next;
    u = un;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int R>
constexpr size_t tc2_smem_bytes() {
  constexpr int HALF = 64 / R, OS = 64 * R + 4;
  return 2 * size_t(kTcBBytes) + size_t((HALF * OS + 3) & ~3) * 4 + 64 + 4 * 128 + 256;
}


// ----------------------------------------------------------------------------
// Level transfers on the tensor cores (float32 plans, Q = 64): the same
// M = 128 row tiles as the translation (row m = component m % R of group
// m / R, A in TMEM split hi / lo, tf32x3), with the tile's quadrant matrix
// C_{lv,q} / B_{lv,q} as the B operand.  Tiles are quadrant-pure (the host
// cuts each level's quadrant-sorted order at quadrant changes), so a tile
// needs one matrix and one 3 x 8 MMA group:
//   kLvlUpLeaf    T[g] = C s[g]                       (leaf level)
//   kLvlUpSum     s[g] = sum of its children's T; T[g] = C s[g]
//   kLvlDown      o[c] = o[c] + B o[parent c]         (o[c] = its translation sum)
//   kLvlDownBeta  the leaf level's o, then beta^ = E^ o (a second MMA with
//                 the same A slots; the leaf o itself is never stored)
// One MMA per tile instead of the warp-tiled FFMA loop: the level kernels
// were latency-bound (0.1-0.3 issued warps per scheduler, ~2300 dependent
// instructions per warp) and competed with the near field for FP32 issue.
// ----------------------------------------------------------------------------
struct LevelTcArgs {
  const float* MTC;       // this level's canonical tf32 tables: [4 quadrants][hi | lo][4096]
  const float* ETC;       // kLvlDownBeta: E^ hi | lo
  const int4* tiles;      // (first index into order, groups, quadrant, -)
  const int32_t* order;   // level ids sorted by quadrant
  const int32_t* opar;    // down: parent of order[i]
  const int2* ochild;     // up-sum: (first child id, count) of order[i]
  const float* Tin;       // up-sum: finer level's transfers
  float* s;               // up: amplitudes (leaf level: read; else written)
  float* Tout;            // up: transfers out
  float* o;               // down: translation sums in, o out
  float* beta;            // kLvlDownBeta: [NL][64][R] reception coefficients
};

template <int R>
constexpr size_t level_tc_smem_bytes(int mode) {
  constexpr int HALF = 64 / R, OS = 64 * R + 4;
  return size_t(mode == kLvlDownBeta ? 4 : 2) * kTcBBytes + size_t((HALF * OS + 3) & ~3) * 4 + 64 + 4 * 128 +
         256;
}

// the 64 values of tile row (group vector src, component rr) as 16 float4,
// in the per-R arrangement tc_put_row expects (R = 1, 2: the rr-th contiguous
// 1/R of the vector; R = 4: component rr strided)
template <int R>
__device__ __forceinline__ void tc_load_row(const float* src, int rr, float4 (&c)[16]) {
  if constexpr (R == 1 || R == 2) {
    const float4* src4 = reinterpret_cast<const float4*>(src) + rr * 16;
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = src4[i];
  } else {
    const float* p = src + rr;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      c[i] = make_float4(p[(4 * i) * R], p[(4 * i + 1) * R], p[(4 * i + 2) * R], p[(4 * i + 3) * R]);
  }
}
template <int R>
__device__ __forceinline__ void tc_store_row(float* dst, int rr, const float4 (&c)[16]) {
  if constexpr (R == 1 || R == 2) {
    float4* d4 = reinterpret_cast<float4*>(dst) + rr * 16;
#pragma unroll
    for (int i = 0; i < 16; ++i) d4[i] = c[i];
  } else {
    float* p = dst + rr;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      p[(4 * i) * R] = c[i].x;
      p[(4 * i + 1) * R] = c[i].y;
      p[(4 * i + 2) * R] = c[i].z;
      p[(4 * i + 3) * R] = c[i].w;
    }
  }
}

// split v = hi + lo (tf32) and store columns 4kb.. of this thread's TMEM lane
__device__ __forceinline__ void tc_put4(uint32_t t_hi, uint32_t t_lo, int kb, float4 v) {
  float4 h, l;
  h.x = tf32_rna(v.x);
  h.y = tf32_rna(v.y);
  h.z = tf32_rna(v.z);
  h.w = tf32_rna(v.w);
  l.x = tf32_rna(v.x - h.x);
  l.y = tf32_rna(v.y - h.y);
  l.z = tf32_rna(v.z - h.z);
  l.w = tf32_rna(v.w - h.w);
  tmem_st4(t_hi + 4 * kb, h);
  tmem_st4(t_lo + 4 * kb, l);
}

// A row (k = 0..63 of this thread's component) from tc_load_row's arrangement
// into TMEM (warp-collective: every lane of the warp must call it)
template <int R>
__device__ __forceinline__ void tc_put_row(uint32_t t_hi, uint32_t t_lo, int rr, const float4 (&c)[16]) {
  if constexpr (R == 1 || R == 4) {
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) tc_put4(t_hi, t_lo, kb, c[kb]);
  } else {
    // chunk i holds (k, 0), (k, 1), (k+1, 0), (k+1, 1) for k = 2i + 32 rr:
    // swap the partner's component with the partner lane
    float mine[32], other[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      mine[2 * i] = rr ? c[i].y : c[i].x;
      mine[2 * i + 1] = rr ? c[i].w : c[i].z;
      other[2 * i] = rr ? c[i].x : c[i].y;
      other[2 * i + 1] = rr ? c[i].z : c[i].w;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) other[i] = __shfl_xor_sync(0xffffffffu, other[i], 1);
#pragma unroll
    for (int kb = 0; kb < 8; ++kb) {
      const float4 x = make_float4(mine[4 * kb], mine[4 * kb + 1], mine[4 * kb + 2], mine[4 * kb + 3]);
      const float4 y = make_float4(other[4 * kb], other[4 * kb + 1], other[4 * kb + 2], other[4 * kb + 3]);
      tc_put4(t_hi, t_lo, kb, rr ? y : x);       // k in [0, 32)
      tc_put4(t_hi, t_lo, 8 + kb, rr ? x : y);   // k in [32, 64)
    }
  }
}

// D[acc] = A B^T (tf32x3) with B = the canonical hi | lo pair at bsm; one thread
__device__ __forceinline__ void tc_mma3(uint32_t tmem, const float* bsm, uint64_t* done) {
  const uint32_t bh = smem_u32(bsm), bl = smem_u32(bsm + 4096);
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    const uint32_t a0 = tmem + (cc == 2 ? 128u : 64u), b0 = cc == 1 ? bl : bh;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      umma_tf32_ts(tmem, a0 + ks * 8, umma_desc_kmajor(b0 + ks * 2 * kTcLBO), (cc | ks) != 0);
  }
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(done))
               : "memory");
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]),
        "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),
        "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
        "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int R, int MODE>
__global__ void __maxnreg__(R == 2 ? kTcFarMaxReg : 255) level_tc_kernel(const LevelTcArgs a) {
  KtScope kt_(80 + MODE);
  constexpr int QR = 64 * R, EPT = 128 / R, HALF = EPT / 2, OS = QR + 4, NV = QR / 4;
  constexpr bool kDown = MODE == kLvlDown || MODE == kLvlDownBeta;
  static_assert(HALF * NV == 1024, "epilogue: 8 float4 per thread and half");
  extern __shared__ __align__(128) unsigned char smem[];
  float* Bm = reinterpret_cast<float*>(smem);                          // hi | lo (32 KB)
  float* Em = Bm + 8192;                                                // kLvlDownBeta: E^ hi | lo
  float* stage = Bm + (MODE == kLvlDownBeta ? 16384 : 8192);            // HALF x OS
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + ((HALF * OS + 3) & ~3));  // [0] B, [1] MMA, [2] E
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  int32_t* gid = reinterpret_cast<int32_t*>(tslot + 4);                 // [EPT] group of each tile entry
  const int tid = threadIdx.x, warp = tid >> 5;
  const int4 tl = a.tiles[blockIdx.x];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
    // constant data ahead of the dependency wait (overlaps the predecessor)
    mbar_arrive_expect_tx(&bar[0], 2 * kTcBBytes);
    bulk_g2s(Bm, a.MTC + size_t(tl.z) * 8192, 2 * kTcBBytes, &bar[0]);
    if constexpr (MODE == kLvlDownBeta) {
      mbar_arrive_expect_tx(&bar[2], 2 * kTcBBytes);
      bulk_g2s(Em, a.ETC, 2 * kTcBBytes, &bar[2]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  const uint32_t t_acc = tmem + lane_base, t_hi = tmem + lane_base + 64, t_lo = tmem + lane_base + 128;
  // plan constants (tile rows, children, parents) before the dependency
  // wait: they overlap the predecessor instead of adding a round trip
  const int n = tl.y;
  const int e = tid / R, rr = tid - (tid / R) * R;
  const bool live = e < n;
  const int64_t g = live ? int64_t(a.order[tl.x + e]) : 0;
  int2 kr = make_int2(0, 0);
  int64_t par = 0;
  if (live) {
    if constexpr (MODE == kLvlUpSum) kr = a.ochild[tl.x + e];
    if constexpr (kDown) par = a.opar[tl.x + e];
  }
  if (rr == 0 && live) gid[e] = int32_t(g);
  pdl_wait();  // amplitudes come from the previous kernel in the chain
  float4 c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (live) {
    if constexpr (MODE == kLvlUpLeaf) {
      tc_load_row<R>(a.s + g * QR, rr, c);
    } else if constexpr (MODE == kLvlUpSum) {
      // s[g] = ordered sum of its children's T (fastmvp.py:160-162 child
      // order), two children's loads in flight at a time
      for (int k = 0; k < kr.y; k += 2) {
        float4 t0[16], t1[16];
        tc_load_row<R>(a.Tin + (int64_t(kr.x) + k) * QR, rr, t0);
        const bool two = k + 1 < kr.y;
        if (two) tc_load_row<R>(a.Tin + (int64_t(kr.x) + k + 1) * QR, rr, t1);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          c[i].x += t0[i].x;
          c[i].y += t0[i].y;
          c[i].z += t0[i].z;
          c[i].w += t0[i].w;
          if (two) {
            c[i].x += t1[i].x;
            c[i].y += t1[i].y;
            c[i].z += t1[i].z;
            c[i].w += t1[i].w;
          }
        }
      }
      tc_store_row<R>(a.s + g * QR, rr, c);
    } else {
      tc_load_row<R>(a.o + par * QR, rr, c);
    }
  }
  tc_put_row<R>(t_hi, t_lo, rr, c);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    mbar_wait(&bar[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tc_mma3(tmem, Bm, &bar[1]);
  }
  // down: this thread's share of the translation sums (o[c] before the
  // transfer), loaded while the tensor core runs: <= 8 float4 per half
  float4 oc[2][8];
  if constexpr (kDown) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int nh = max(0, min(HALF, n - h * HALF));
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = tid + 128 * j, ee = i / NV, v = i - (i / NV) * NV;
        oc[h][j] = ee < nh ? __ldcg(reinterpret_cast<const float4*>(a.o + int64_t(gid[h * HALF + ee]) * QR) + v)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  mbar_wait(&bar[1], 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // the dependent kernel may start its prologue now, one epilogue ahead of
  // its inputs: triggered at the top of the kernel, the next kernel's CTAs
  // (770 fused-chain CTAs after the last upward level) sat resident for the
  // whole level and kept the side stream's translation out (ktrace: 31 us)
  pdl_trigger();
  uint32_t r[64];
  tmem_ld64(t_acc, r);
  float* out = kDown ? a.o : a.Tout;
  // rows -> smem half a tile at a time -> coalesced 16-byte rows of the
  // groups' vectors (down: + the translation sums already in o)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e0 = h * HALF;
    const bool mine = e >= e0 && e < e0 + HALF;
    if (mine && live)
#pragma unroll
      for (int k = 0; k < 64; ++k) stage[(e - e0) * OS + k * R + rr] = __uint_as_float(r[k]);
    __syncthreads();
    const int nh = max(0, min(HALF, n - e0));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = tid + 128 * j;
      if (i >= nh * NV) break;
      const int ee = i / NV, v = i - (i / NV) * NV;
      float4* sp = reinterpret_cast<float4*>(stage + ee * OS + 4 * v);
      float* dst = out + int64_t(gid[e0 + ee]) * QR + 4 * v;
      float4 val = *sp;
      if constexpr (kDown) {
        const float4 t = oc[h][j];
        val.x += t.x;
        val.y += t.y;
        val.z += t.z;
        val.w += t.w;
      }
      if constexpr (MODE == kLvlDownBeta) {
        *sp = val;  // the leaf o stays on chip: it only feeds beta^
      } else {
        *reinterpret_cast<float4*>(dst) = val;
      }
    }
    if constexpr (MODE == kLvlDownBeta) {
      __syncthreads();
      if (mine && live)
#pragma unroll
        for (int k = 0; k < 64; ++k) r[k] = __float_as_uint(stage[(e - e0) * OS + k * R + rr]);
    }
    __syncthreads();
  }
  if constexpr (MODE == kLvlDownBeta) {
    // beta^ = E^ o: the leaf o rows back into the A slots, second MMA
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) {
      const float4 v = live ? make_float4(__uint_as_float(r[4 * kb]), __uint_as_float(r[4 * kb + 1]),
                                          __uint_as_float(r[4 * kb + 2]), __uint_as_float(r[4 * kb + 3]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      tc_put4(t_hi, t_lo, kb, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&bar[2], 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      tc_mma3(tmem, Em, &bar[1]);
    }
    mbar_wait(&bar[1], 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmem_ld64(t_acc, r);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e0 = h * HALF;
      if (e >= e0 && e < e0 + HALF && live)
#pragma unroll
        for (int k = 0; k < 64; ++k) stage[(e - e0) * OS + k * R + rr] = __uint_as_float(r[k]);
      __syncthreads();
      const int nh = max(0, min(HALF, n - e0));
      for (int i = tid; i < nh * NV; i += 128) {
        const int ee = i / NV, v = i - (i / NV) * NV;
        *reinterpret_cast<float4*>(a.beta + int64_t(gid[e0 + ee]) * QR + 4 * v) =
            *reinterpret_cast<const float4*>(stage + ee * OS + 4 * v);
      }
      __syncthreads();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// ----------------------------------------------------------------------------
// Warp-tiled level transfer for Q in {32, 64} on the large levels (same
// roles as level_kernel).  The tile's groups (sorted by quadrant, so one or
// two quadrant matrices) are staged group-major by bulk copy (UpLeaf, Down)
// or summed from the children (UpSum); each warp computes a 32 x 32 block
// with the conflict-free lane layout of tgemm_wt_kernel.
// ----------------------------------------------------------------------------
template <typename T, int R, int QT, int MODE>
struct LVW {
  using W = TGW<T, R, QT>;
  // quadrant matrices per round: tiles are quadrant-sorted, so only the (at
  // most 3) boundary tiles of a level need a second round; one slot keeps the
  // kernel small enough to run 2-3 CTAs per SM beside the near field
  static constexpr int kSlots = 1;
  static constexpr bool kDown = MODE == kLvlDown || MODE == kLvlDownBeta;
  static constexpr int kXBufs = kDown ? 2 : 1;      // the downward modes also stage o[c]
  static constexpr int kEMat = MODE == kLvlDownBeta ? 1 : 0;  // the E^ matrix
  static constexpr size_t SMEM = (kSlots + kEMat) * W::MB + kXBufs * W::XB + 3 * 64;
};

template <typename T, int R, int QT, int MODE>
__global__ void __launch_bounds__(128) level_wt_kernel(const LevelArgs<T, R> a, const RecvArgs rv) {
  KtScope kt_(50 + MODE);
  using W = TGW<T, R, QT>;
  using LV = LVW<T, R, QT, MODE>;
  constexpr bool kDown = LV::kDown;
  extern __shared__ __align__(128) unsigned char smem[];
  T* M = reinterpret_cast<T*>(smem);                                  // kSlots matrices
  T* X = reinterpret_cast<T*>(smem + LV::kSlots * W::MB);             // inputs / outputs
  T* Oc = reinterpret_cast<T*>(smem + LV::kSlots * W::MB + W::XB);    // down: o[c] (reduce output)
  T* Em = reinterpret_cast<T*>(smem + LV::kSlots * W::MB + LV::kXBufs * W::XB);  // kLvlDownBeta: E^
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (LV::kSlots + LV::kEMat) * W::MB +
                                               LV::kXBufs * W::XB);  // M, X
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t t0 = int64_t(blockIdx.x) * W::PER;
  const int n = int(a.count - t0 < W::PER ? a.count - t0 : W::PER);
  const int q_lo = a.quad[a.order[t0]], q_hi = a.quad[a.order[t0 + n - 1]];
  constexpr uint32_t kVB = uint32_t(W::QR * sizeof(T));
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    const int nq = min(LV::kSlots, q_hi - q_lo + 1);
    mbar_arrive_expect_tx(&bar[0], uint32_t(nq * W::MB));
    bulk_g2s(M, reinterpret_cast<const unsigned char*>(a.MT4) + q_lo * W::MB, uint32_t(nq * W::MB),
             &bar[0]);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // amplitudes come from the previous kernel in the chain
  if constexpr (MODE == kLvlUpSum) {
    // X[p] = s[order p] = ordered sum of its children's T (also stored to s).
    // Warp w sums groups w, w+4, ...: in batches of GB groups, every child
    // load of the batch is issued before any sum (one memory round trip per
    // batch instead of one per group).
    constexpr int GB = 4;
    constexpr int NW = W::QR / 128 > 0 ? W::QR / 128 : 1;  // 4-element slices per lane
    for (int p0 = warp; p0 < n; p0 += 4 * GB) {
      int64_t cid[GB];
      int2 kr[GB];
#pragma unroll
      for (int b = 0; b < GB; ++b) {
        const int p = p0 + 4 * b;
        cid[b] = p < n ? int64_t(a.order[t0 + p]) : 0;
        kr[b] = p < n ? a.ochild[t0 + p] : make_int2(0, 0);
      }
#pragma unroll
      for (int sl = 0; sl < NW; ++sl) {
        const int w = 4 * lane + 128 * sl;
        if (w >= W::QR) break;
        T t[GB][4][4];
#pragma unroll
        for (int b = 0; b < GB; ++b)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < kr[b].y) ld4(a.Tin + (int64_t(kr[b].x) + k) * W::QR + w, t[b][k]);
#pragma unroll
        for (int b = 0; b < GB; ++b) {
          const int p = p0 + 4 * b;
          if (p >= n) break;
          T v[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < kr[b].y)
#pragma unroll
              for (int i = 0; i < 4; ++i) v[i] += t[b][k][i];
          // octree parents: children 5..8, in order after the preloaded four
          for (int k = 4; k < kr[b].y; ++k) {
            T u[4];
            ld4(a.Tin + (int64_t(kr[b].x) + k) * W::QR + w, u);
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] += u[i];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            a.s[cid[b] * W::QR + w + i] = v[i];
            X[p * W::XS + w + i] = v[i];
          }
        }
      }
    }
  } else {
    if (warp == 0) {
      const uint32_t nb = (kDown ? 2u : 1u) * kVB * uint32_t(n) + (LV::kEMat ? uint32_t(W::MB) : 0u);
      if (lane == 0) {
        mbar_arrive_expect_tx(&bar[1], nb);
        if constexpr (LV::kEMat)
          if constexpr (sizeof(T) == 4) bulk_g2s(Em, rv.ET, uint32_t(W::MB), &bar[1]);
      }
      __syncwarp();
      for (int p = lane; p < n; p += 32) {
        const int64_t g = kDown ? a.opar[t0 + p] : a.order[t0 + p];
        bulk_g2s(X + p * W::XS, (kDown ? a.o : a.s) + g * W::QR, kVB, &bar[1]);
        if constexpr (kDown)
          bulk_g2s(Oc + p * W::XS, a.o + int64_t(a.order[t0 + p]) * W::QR, kVB, &bar[1]);
      }
    }
    mbar_wait(&bar[1], 0);
  }

  const int wr = warp % W::RW, wc = warp / W::RW;
  const int tr = lane >> 3, tc = lane & 7;
  const int row0 = 32 * wr + 8 * tr;
  constexpr int NE = 4 / R;
  const int E0 = 32 * wc / R;
  int eq[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = E0 + tc + 8 * i;
    eq[i] = e < n ? a.quad[a.order[t0 + e]] : -1;
  }
  T acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
  int round = 0;
  for (int q0 = q_lo; q0 <= q_hi; q0 += LV::kSlots, ++round) {
    const int nq = min(LV::kSlots, q_hi - q0 + 1);
    if (round) {
      __syncthreads();  // previous slots consumed
      if (tid == 0) {
        mbar_arrive_expect_tx(&bar[0], uint32_t(nq * W::MB));
        bulk_g2s(M, reinterpret_cast<const unsigned char*>(a.MT4) + q0 * W::MB,
                 uint32_t(nq * W::MB), &bar[0]);
      }
    }
    mbar_wait(&bar[0], uint32_t(round) & 1u);
    __syncthreads();  // staged inputs visible (first round)
    if (E0 + tc < n) {
      const T* xp = X + (E0 + tc) * W::XS;
      for (int qq = 0; qq < nq; ++qq) {
        const int qd = q0 + qq;
        bool any = false;
#pragma unroll
        for (int i = 0; i < NE; ++i) any |= eq[i] == qd;
        if (!any) continue;
        const T* mp = M + qq * (W::MB / sizeof(T)) + row0;
        T part[8][4];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) part[r][c] = T(0);
#pragma unroll 4
        for (int j = 0; j < QT; ++j) {
          T m0[4], m1[4], x[4];
          ld4(mp + j * QT, m0);
          ld4(mp + j * QT + 4, m1);
#pragma unroll
          for (int i = 0; i < NE; ++i) ldx<T, R>(xp + i * 8 * W::XS + j * R, x + i * R);
          tile_fma8x4<T>(part, m0, m1, x);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (eq[c / R] == qd)
#pragma unroll
            for (int r = 0; r < 8; ++r) acc[r][c] = part[r][c];
      }
    }
  }
  __syncthreads();  // inputs consumed
  if (E0 + tc < n) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int p = E0 + tc + 8 * (c / R), rr = c % R;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int idx = p * W::XS + (row0 + r) * R + rr;
        if constexpr (kDown)
          X[idx] = Oc[idx] + acc[r][c];  // translation sum + potential transfer
        else
          X[idx] = acc[r][c];
      }
    }
  }
  __syncthreads();
  if constexpr (MODE == kLvlDownBeta) {
    if constexpr (sizeof(T) == 4 && QT == 64) {
      // ---- reception coefficients of the tile's leaves: beta^ = E^ o (same
      // warp tiling; E^ is one matrix for every column), into the Oc buffer
      if (E0 + tc < n) {
        const T* xp = X + (E0 + tc) * W::XS;
        const T* mp = Em + row0;
        T part[8][4];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) part[r][c] = T(0);
#pragma unroll 4
        for (int j = 0; j < QT; ++j) {
          T m0[4], m1[4], x[4];
          ld4(mp + j * QT, m0);
          ld4(mp + j * QT + 4, m1);
#pragma unroll
          for (int i = 0; i < NE; ++i) ldx<T, R>(xp + i * 8 * W::XS + j * R, x + i * R);
          tile_fma8x4<T>(part, m0, m1, x);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int p = E0 + tc + 8 * (c / R), rr = c % R;
#pragma unroll
          for (int r = 0; r < 8; ++r) Oc[p * W::XS + (row0 + r) * R + rr] = part[r][c];
        }
      }
      __syncthreads();
      {
        // beta^ rows of the tile's leaves -> global, coalesced (the leaf
        // level's o is only ever read through beta^, so it is not stored)
        constexpr int V = 4;
        constexpr int NV = W::QR / V;
        for (int i = tid; i < n * NV; i += 128) {
          const int p = i / NV, v = i - p * NV;
          *reinterpret_cast<float4*>(rv.beta + int64_t(a.order[t0 + p]) * W::QR + v * V) =
              *reinterpret_cast<const float4*>(Oc + p * W::XS + v * V);
        }
      }
    }
    return;
  }
  T* outb = kDown ? a.o : a.Tout;
  constexpr int V = 16 / int(sizeof(T));
  constexpr int NV = W::QR / V;
  for (int i = tid; i < n * NV; i += 128) {
    const int p = i / NV, v = i - p * NV;
    T* dst = outb + int64_t(a.order[t0 + p]) * W::QR + v * V;
    if constexpr (sizeof(T) == 4)
      *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(X + p * W::XS + v * V);
    else
      *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(X + p * W::XS + v * V);
  }
}

// ----------------------------------------------------------------------------
// Radiation and reception through circle expansions (float32 plans built
// from geometry).  With w = (p - c) / r for a point p of a leaf with center
// c and a circle of radius r > |p - c| through x_l = c + r e^{i phi_l}:
//   -0.5 log|x_l - p|^2 = -log r + Re sum_{m>=1} (1/m) w^m e^{-i m phi_l}
// (|w| <= sqrt2 h / r: 0.57 for the outgoing check circle, 0.51 for the
// incoming aux circle, so the series converges geometrically).
//
// Radiation V = fit K(out_check, pts) (operators.py:107-112):
//   s_k = -log(r) F_k mu_0 + sum_{m>=1} Re(A_km mu_m),
//   mu_m = sum_j w_j^m q_j,  A_km = sum_l fit_kl (1/m) e^{-i m phi_l},
//   F_k = sum_l fit_kl   (A, F formed once per plan in float64).
// Reception U = K(pts, in_aux) (operators.py:147-149):
//   phi_j = -log(r) sum_k o_k + Re sum_{m>=1} beta_m w_j^m,
//   beta_m = sum_k (1/m) e^{-i m theta_k} o_k.
// Both replace a streamed Q x n operator (4Q bytes per point each way) by
// ~8 FP32 instructions per point and term; the plan picks the number of
// terms from the largest |w| of its points (truncation below float32
// rounding).  One warp per leaf; moment sums over the leaf's points use a
// fixed transpose-reduction tree (deterministic).
// ----------------------------------------------------------------------------

// Sum 32 per-lane values over the warp: afterwards lane l returns the sum of
// value l (31 shuffles; fixed pairing, so bitwise reproducible).
__device__ __forceinline__ float warp_transpose_sum32(float (&v)[32], int lane) {
#pragma unroll
  for (int sft = 16; sft >= 1; sft >>= 1) {
    const bool up = lane & sft;
#pragma unroll
    for (int j = 0; j < sft; ++j) {
      const float send = up ? v[j] : v[j + sft];
      const float keep = up ? v[j + sft] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
    }
  }
  return v[0];
}

constexpr int kExpWarps = 4;   // warps per CTA of the expansion kernels
constexpr int kMomLanes = 4;   // radiation: lanes per leaf
constexpr int kMomLeavesPerWarp = 32 / kMomLanes;

// w^e (e >= 0) by binary powering
__device__ __forceinline__ float2 cpowf(float2 w, int e) {
  float2 r = make_float2(1.f, 0.f);
  while (e) {
    if (e & 1) r = cmulf(r, w);
    w = cmulf(w, w);
    e >>= 1;
  }
  return r;
}

// w^E for a compile-time E (unrolled square-and-multiply)
template <int E>
__device__ __forceinline__ float2 cpow_const(float2 w) {
  if constexpr (E == 0) {
    return make_float2(1.f, 0.f);
  } else if constexpr (E == 1) {
    return w;
  } else {
    const float2 h = cpow_const<E / 2>(w);
    const float2 h2 = cmulf(h, h);
    if constexpr (E % 2) return cmulf(h2, w);
    else return h2;
  }
}


// Radiation through outgoing moments.  Lane group of kMomLanes lanes per
// leaf, kMomLeavesPerWarp leaves per warp.  The batch's points (contiguous)
// are staged in shared memory by cp.async; the next batch's copy is issued
// as soon as the moments are formed, so it overlaps the A-phase.  Each lane
// accumulates the moments of every kMomLanes-th point of its leaf in
// registers (passes of MP moments, 2 R MP = 80 accumulators), the group
// combines them with a transpose reduction (fixed pairing), then the warp
// applies A (read through L1, shared by every leaf) to its leaves' moments.
// smem per warp: points [bufpts] float2, q [bufpts][R], mu
// [leaves][nm][R] float2 (16-byte rows).
// Register budget for 4 CTAs / SM (<= 128 registers, no spills): at the
// natural 169 registers only 2 CTAs fit (measured 531 vs 537 us at C4).
template <int R>
__global__ void __launch_bounds__(32 * kExpWarps, 4) radiation_mom_kernel(
    const float2* __restrict__ prel, const int64_t* __restrict__ leaf_start,
    const int64_t* __restrict__ leaf_stop, const float* __restrict__ leaf_r,
    const float2* __restrict__ A, const float* __restrict__ qt, float* __restrict__ s,
    int64_t leaf0, int64_t nleaf, int Q, int nm, int bufpts) {
  KtScope kt_(60);
  constexpr int MP = 40 / R;  // moments per pass
  constexpr int NV = 2 * R * MP;       // 80 accumulators
  constexpr int NV2 = NV / 2, NV4 = NV / 4;
  constexpr int LW = kMomLeavesPerWarp;
  extern __shared__ float4 sm4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mu_stride = (nm * R + 1) & ~1;  // float2 per leaf, even => 16-byte rows
  const size_t per_warp = size_t(bufpts) * (2 + R) + size_t(LW) * mu_stride * 2;  // floats
  float* wbase = reinterpret_cast<float*>(sm4) + warp * per_warp;
  float2* Pb = reinterpret_cast<float2*>(wbase);
  float* Qb = wbase + 2 * bufpts;
  float2* mu = reinterpret_cast<float2*>(wbase + size_t(bufpts) * (2 + R));
  const int slot = lane / kMomLanes, g = lane % kMomLanes;
  const int64_t stride = int64_t(gridDim.x) * kExpWarps * LW;
  // stage the points of batch lw (if they fit); returns whether staged
  auto stage = [&](int64_t lw) -> bool {
    if (lw >= nleaf) return false;
    const int64_t le = lw + LW < nleaf ? lw + LW : nleaf;
    const int64_t b0 = leaf_start[leaf0 + lw], b1 = leaf_stop[leaf0 + le - 1];
    const int np = int(b1 - b0);
    if (np > bufpts) return false;
    for (int t = lane; t < np; t += 32) {
      cp_async<8>(Pb + t, prel + b0 + t);
      cp_async_n<R * 4>(Qb + t * R, qt + (b0 + t) * R);
    }
    cp_async_commit();
    return true;
  };
  int64_t lw = (int64_t(blockIdx.x) * kExpWarps + warp) * LW;
  bool staged = stage(lw);
  for (; lw < nleaf; lw += stride) {
    const int64_t li = lw + slot;
    const bool live = li < nleaf;
    const int64_t leaf = leaf0 + (live ? li : 0);
    const int64_t b = leaf_start[leaf];
    const int n = live ? int(leaf_stop[leaf] - b) : 0;
    const float inv = 1.f / leaf_r[leaf];
    const int64_t b0 = leaf_start[leaf0 + lw];
    if (staged) cp_async_wait_all();
    __syncwarp();
    float* muf = reinterpret_cast<float*>(mu + slot * mu_stride);
    for (int m0 = 0; m0 < nm; m0 += MP) {
      float v[NV];
#pragma unroll
      for (int t = 0; t < NV; ++t) v[t] = 0.f;
      for (int j = g; j < n; j += kMomLanes) {
        float2 p;
        float qv[R];
        if (staged) {
          const int t = int(b + j - b0);
          p = Pb[t];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) qv[rr] = Qb[t * R + rr];
        } else {
          p = prel[b + j];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) qv[rr] = qt[(b + j) * R + rr];
        }
        const float2 w = make_float2(p.x * inv, p.y * inv);
        // two interleaved power chains (even / odd terms, each stepping by w^2)
        // halve the dependent complex-multiply latency per point
        const float2 w2 = cmulf(w, w);
        const float2 W1 = w2, W2 = make_float2(-w2.y, w2.x);
        float2 zc[2];
        zc[0] = make_float2(1.f, 0.f);
        if (m0) {
          const float2 wp = cpow_const<MP>(w);
          zc[0] = wp;
          for (int e = MP; e < m0; e += MP) zc[0] = cmulf(zc[0], wp);
        }
        zc[1] = cmulf(zc[0], w);
#pragma unroll
        for (int mm = 0; mm < MP; ++mm) {
          const float2 z = zc[mm & 1];
          // v layout [moment][re, im][rhs column] (column pairs share an FFMA2)
          if constexpr (R % 2 == 0) {
#pragma unroll
            for (int rr = 0; rr < R; rr += 2) {
              ffma2(v[(mm * 2) * R + rr], v[(mm * 2) * R + rr + 1], z.x, qv[rr], qv[rr + 1]);
              ffma2(v[(mm * 2 + 1) * R + rr], v[(mm * 2 + 1) * R + rr + 1], z.y, qv[rr], qv[rr + 1]);
            }
          } else {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              v[(mm * 2) * R + rr] = fmaf(z.x, qv[rr], v[(mm * 2) * R + rr]);
              v[(mm * 2 + 1) * R + rr] = fmaf(z.y, qv[rr], v[(mm * 2 + 1) * R + rr]);
            }
          }
          zc[mm & 1] = cmul_pk(z, W1, W2);
        }
      }
      // transpose reduction over the 4 lanes of the group: lane g ends with
      // values [vb, vb + NV4)
      {
        const bool up = g & 2;
#pragma unroll
        for (int t = 0; t < NV2; ++t) {
          const float send = up ? v[t] : v[t + NV2];
          const float keep = up ? v[t + NV2] : v[t];
          v[t] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
      }
      {
        const bool up = g & 1;
#pragma unroll
        for (int t = 0; t < NV4; ++t) {
          const float send = up ? v[t] : v[t + NV4];
          const float keep = up ? v[t + NV4] : v[t];
          v[t] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
      }
      const int vb = ((g & 2) ? NV2 : 0) + ((g & 1) ? NV4 : 0);
      const int lim = (nm - m0) * R * 2;  // values of moments < nm
#pragma unroll
      for (int t = 0; t < NV4; ++t)
        if (vb + t < lim) muf[m0 * R * 2 + vb + t] = v[t];
    }
    __syncwarp();  // moments visible; the point buffer is free
    staged = stage(lw + stride);
    // s_k = -log(r) F_k mu_0 + sum_m Re(A_km mu_m): lane owns k = kb + lane
    // and kb + 32 + lane for all the warp's leaves
    for (int kb = 0; kb < Q; kb += 64) {
      const int k0 = kb + lane, k1 = kb + 32 + lane;
      const bool h0 = k0 < Q, h1 = k1 < Q;
      float acc[2][LW][R];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int l = 0; l < LW; ++l)
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc[h][l][rr] = 0.f;
      // A rows prefetched PF steps ahead (the A-apply was stalled on these
      // L1/L2 loads: ncu long-scoreboard at the first use)
      constexpr int PF = 4;
      float2 ap0[PF], ap1[PF];
#pragma unroll
      for (int i = 0; i < PF; ++i) {
        const int mm = 1 + i;
        ap0[i] = (h0 && mm < nm) ? __ldg(A + mm * Q + k0) : make_float2(0.f, 0.f);
        ap1[i] = (h1 && mm < nm) ? __ldg(A + mm * Q + k1) : make_float2(0.f, 0.f);
      }
      for (int mb = 1; mb < nm; mb += PF) {
#pragma unroll
        for (int i = 0; i < PF; ++i) {
        const int m = mb + i;
        if (m >= nm) break;
        const float2 a0 = ap0[i], a1 = ap1[i];
        {
          const int mn = m + PF;
          ap0[i] = (h0 && mn < nm) ? __ldg(A + mn * Q + k0) : make_float2(0.f, 0.f);
          ap1[i] = (h1 && mn < nm) ? __ldg(A + mn * Q + k1) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int l = 0; l < LW; ++l) {
          // mu_m: re[R] then im[R]
          const float* um = reinterpret_cast<const float*>(mu + l * mu_stride) + (m * 2) * R;
          float ur[R], ui[R];
          if constexpr (R == 2) {
            const float4 t = *reinterpret_cast<const float4*>(um);
            ur[0] = t.x; ur[1] = t.y; ui[0] = t.z; ui[1] = t.w;
          } else {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              ur[rr] = um[rr];
              ui[rr] = um[R + rr];
            }
          }
          if constexpr (R % 2 == 0) {
#pragma unroll
            for (int rr = 0; rr < R; rr += 2) {
              ffma2(acc[0][l][rr], acc[0][l][rr + 1], -a0.y, ui[rr], ui[rr + 1]);
              ffma2(acc[0][l][rr], acc[0][l][rr + 1], a0.x, ur[rr], ur[rr + 1]);
              ffma2(acc[1][l][rr], acc[1][l][rr + 1], -a1.y, ui[rr], ui[rr + 1]);
              ffma2(acc[1][l][rr], acc[1][l][rr + 1], a1.x, ur[rr], ur[rr + 1]);
            }
          } else {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              acc[0][l][rr] = fmaf(a0.x, ur[rr], fmaf(-a0.y, ui[rr], acc[0][l][rr]));
              acc[1][l][rr] = fmaf(a1.x, ur[rr], fmaf(-a1.y, ui[rr], acc[1][l][rr]));
            }
          }
        }
        }
      }
      const float f0 = h0 ? __ldg(A + k0).x : 0.f, f1 = h1 ? __ldg(A + k1).x : 0.f;
#pragma unroll
      for (int l = 0; l < LW; ++l) {
        const int64_t li2 = lw + l;
        if (li2 >= nleaf) break;
        const int64_t lf = leaf0 + li2;
        const float nl = -logf(leaf_r[lf]);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const float u0 = reinterpret_cast<const float*>(mu + l * mu_stride)[rr];
          if (h0) s[(lf * Q + k0) * R + rr] = fmaf(nl * f0, u0, acc[0][l][rr]);
          if (h1) s[(lf * Q + k1) * R + rr] = fmaf(nl * f1, u0, acc[1][l][rr]);
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait_all();
}

// ----------------------------------------------------------------------------
// Radiation on FP32 pipes + tensor cores (float32 plans from geometry, Q = 64,
// R <= 2, nm <= 38).  The moments mu_m = sum_j w_j^m q_j (m < nm) of a leaf
// come from 8 lanes: lanes 0-3 take the even moments, lanes 4-7 the odd ones
// (chains start at 1 / w and step by w^2, two interleaved chains stepping by
// w^4 for ILP), each lane every 4th point of the leaf, then a fixed
// transpose reduction over the 4 lanes of a half (deterministic).  The moment map s = A^ mu^ (operators.py:107-112
// through the circle expansion, see the section comment above) runs on the
// tensor cores: rows = (leaf, column) of a 32-leaf tile, K = 80 real moment
// rows (row 0 = -log(r) mu_0, rows 2m-1 / 2m = Re / Im mu_m), N = 64 outputs,
// tf32x3 with A^ pre-split on the host.  Persistent CTAs of 8 warps (4 leaves
// per warp); warps 0-3 own the 128 TMEM lanes and do the tensor-core part
// while warps 4-7 already form the next tile's moments.
// ----------------------------------------------------------------------------
constexpr int kRadTcWarps = 8;
constexpr int kRadTcLeaves = kRadTcWarps * 4;  // leaves per tile
constexpr int kRadTcK = 80;                    // moment rows (K) of the map
constexpr int kRadTcMH = 19;                   // moments per lane half (nm <= 38: C4 uses 38)
constexpr uint32_t kRadTcSBO = kRadTcK * 8 * 4;  // bytes between 8-row groups of A^
constexpr int kRadTcKP = kRadTcK + 4;          // mu^ row stride in smem (conflict-free 16-byte reads)

__device__ __forceinline__ uint64_t umma_desc_kmajor_sbo(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((kTcLBO >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}

template <int R>
constexpr size_t radiation_tc_smem_bytes() {
  // A^ hi | lo, mu^ tile, output stage, barriers / TMEM slot
  return size_t(2) * 64 * kRadTcK * 4 + size_t(kRadTcLeaves) * kRadTcKP * R * 4 +
         size_t(kRadTcLeaves) * (64 * R + 4) * 4 + 128 + 8 * kRadTcLeaves;
}

// Registers: beside the near field's two CTAs only ONE radiation CTA fits an
// SM (8 warps: 2 per sub-partition, 2 x 160 x 32 + the near field's 6144 =
// 16384), so the former 128-register squeeze for two CTAs per SM bought
// nothing inside the product (A/B 475.3 -> 470.4 us at the natural 148-160).
template <int R>
__global__ void __maxnreg__(kTcFarMaxReg) radiation_tc_kernel(
    const float2* __restrict__ prel, const int64_t* __restrict__ leaf_start,
    const int64_t* __restrict__ leaf_stop, const float* __restrict__ leaf_r,
    const float* __restrict__ ATC, const float* __restrict__ qt, float* __restrict__ s,
    const int32_t* __restrict__ leaf_order, int64_t nleaf, int nm) {
  static_assert(R == 1 || R == 2, "radiation_tc_kernel: R <= 2");
  KtScope kt_(62);
  constexpr int QR = 64 * R, OS = QR + 4;
  constexpr int NV = 2 * R * kRadTcMH;  // accumulators per lane
  constexpr int NV2 = NV / 2, NV4 = NV / 4;
  extern __shared__ __align__(128) unsigned char smem[];
  float* Ah = reinterpret_cast<float*>(smem);                 // A^ hi (canonical, 64 x 80)
  float* smu = Ah + 2 * 64 * kRadTcK;                         // [leaf][R][KP] (mu^ rows)
  float* stage = smu + kRadTcLeaves * kRadTcKP * R;           // [leaf][OS]
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + kRadTcLeaves * OS);  // [0] A^, [1] MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  int32_t* tleaf2 = reinterpret_cast<int32_t*>(tslot + 2);   // [2][kRadTcLeaves] leaf of each tile row
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar[0], 2 * 64 * kRadTcK * 4);
    bulk_g2s(Ah, ATC, 2 * 64 * kRadTcK * 4, &bar[0]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int g8 = lane & 7, half = g8 >> 2, g = g8 & 3;
  const int cnt = half ? nm >> 1 : (nm + 1) >> 1;  // odd / even moments below nm
  const int64_t ntiles = (nleaf + kRadTcLeaves - 1) / kRadTcLeaves;
  uint32_t mma_phase = 0;
  bool first = true;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    // double-buffered: warps 4-7 fill the next tile's entries while warps
    // 0-3 still store this one's rows
    int32_t* tleaf = tleaf2 + (it & 1) * kRadTcLeaves;
    // tiles hold leaves of similar size (leaf_order: descending point
    // count), so a tile is not held up by one large leaf
    const int le = warp * 4 + (lane >> 3);  // leaf of the tile
    const int64_t li = tile * kRadTcLeaves + le;
    const bool live = li < nleaf;
    const int64_t leaf = live ? int64_t(leaf_order[li]) : int64_t(leaf_order[0]);
    if ((lane & 7) == 0) tleaf[le] = int32_t(leaf);
    const int64_t b = leaf_start[leaf];
    const int n = live ? int(leaf_stop[leaf] - b) : 0;
    const float rc = leaf_r[leaf];
    const float inv = 1.f / rc;
    // ---- moments of this lane's half over every 4th point (each point's
    // data loaded two steps ahead)
    float v[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) v[t] = 0.f;
    float2 p0 = make_float2(0.f, 0.f), p1 = make_float2(0.f, 0.f);
    float q0[R], q1[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) q0[rr] = q1[rr] = 0.f;
    auto fetch = [&](int j, float2& pp, float (&qq)[R]) {
      if (j < n) {
        pp = prel[b + j];
        if constexpr (R == 2) {
          const float2 t = *reinterpret_cast<const float2*>(qt + (b + j) * 2);
          qq[0] = t.x;
          qq[1] = t.y;
        } else {
          qq[0] = qt[b + j];
        }
      }
    };
    auto point = [&](const float2 p, const float (&qv)[R]) {
        const float2 w = make_float2(p.x * inv, p.y * inv);
        const float2 w2 = cmulf(w, w);
        const float2 w4 = cmulf(w2, w2);
        const float2 W1 = w4, W2 = make_float2(-w4.y, w4.x);
        float2 zc[2];
        zc[0] = half ? w : make_float2(1.f, 0.f);   // moment 2 mm + half
        zc[1] = cmulf(zc[0], w2);
#pragma unroll
        for (int mm = 0; mm < kRadTcMH; ++mm) {
          const float2 z = zc[mm & 1];
          // v layout [moment][re, im][rhs column] (column pairs share an FFMA2)
          if constexpr (R == 2) {
            ffma2(v[(mm * 2) * R], v[(mm * 2) * R + 1], z.x, qv[0], qv[1]);
            ffma2(v[(mm * 2 + 1) * R], v[(mm * 2 + 1) * R + 1], z.y, qv[0], qv[1]);
          } else {
            v[mm * 2] = fmaf(z.x, qv[0], v[mm * 2]);
            v[mm * 2 + 1] = fmaf(z.y, qv[0], v[mm * 2 + 1]);
          }
          zc[mm & 1] = cmul_pk(z, W1, W2);
        }
    };
    // two points at a time: four independent power chains per lane (with one
    // CTA per SM beside the near field, two chains left the FP32 pipes idle)
    auto point2 = [&](const float2 pa, const float (&qa)[R], const float2 pb, const float (&qb)[R]) {
      const float2 wa = make_float2(pa.x * inv, pa.y * inv), wb = make_float2(pb.x * inv, pb.y * inv);
      const float2 wa2 = cmulf(wa, wa), wb2 = cmulf(wb, wb);
      const float2 wa4 = cmulf(wa2, wa2), wb4 = cmulf(wb2, wb2);
      const float2 A1 = wa4, A2 = make_float2(-wa4.y, wa4.x);
      const float2 B1 = wb4, B2 = make_float2(-wb4.y, wb4.x);
      float2 za[2], zb[2];
      za[0] = half ? wa : make_float2(1.f, 0.f);
      zb[0] = half ? wb : make_float2(1.f, 0.f);
      za[1] = cmulf(za[0], wa2);
      zb[1] = cmulf(zb[0], wb2);
#pragma unroll
      for (int mm = 0; mm < kRadTcMH; ++mm) {
        const float2 ya = za[mm & 1], yb = zb[mm & 1];
        if constexpr (R == 2) {
          ffma2(v[(mm * 2) * R], v[(mm * 2) * R + 1], ya.x, qa[0], qa[1]);
          ffma2(v[(mm * 2 + 1) * R], v[(mm * 2 + 1) * R + 1], ya.y, qa[0], qa[1]);
          ffma2(v[(mm * 2) * R], v[(mm * 2) * R + 1], yb.x, qb[0], qb[1]);
          ffma2(v[(mm * 2 + 1) * R], v[(mm * 2 + 1) * R + 1], yb.y, qb[0], qb[1]);
        } else {
          v[mm * 2] = fmaf(ya.x, qa[0], v[mm * 2]);
          v[mm * 2 + 1] = fmaf(ya.y, qa[0], v[mm * 2 + 1]);
          v[mm * 2] = fmaf(yb.x, qb[0], v[mm * 2]);
          v[mm * 2 + 1] = fmaf(yb.y, qb[0], v[mm * 2 + 1]);
        }
        za[mm & 1] = cmul_pk(ya, A1, A2);
        zb[mm & 1] = cmul_pk(yb, B1, B2);
      }
    };
    fetch(g, p0, q0);
    fetch(g + 4, p1, q1);
    for (int j = g; j < n; j += 8) {
      const float2 pa = p0, pb = p1;
      float qa[R], qb[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        qa[rr] = q0[rr];
        qb[rr] = q1[rr];
      }
      const bool two = j + 4 < n;
      fetch(j + 8, p0, q0);
      fetch(j + 12, p1, q1);
      if (two)
        point2(pa, qa, pb, qb);
      else
        point(pa, qa);
    }
    // ---- transpose reduction over the 4 lanes of the half: lane g keeps
    // values [vb, vb + NV4)
    {
      const bool up = g & 2;
#pragma unroll
      for (int t = 0; t < NV2; ++t) {
        const float send = up ? v[t] : v[t + NV2];
        const float keep = up ? v[t + NV2] : v[t];
        v[t] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
    }
    {
      const bool up = g & 1;
#pragma unroll
      for (int t = 0; t < NV4; ++t) {
        const float send = up ? v[t] : v[t + NV4];
        const float keep = up ? v[t + NV4] : v[t];
        v[t] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
    }
    __syncthreads();  // the previous tile's mu^ has been moved into TMEM
    {
      // value index x = (mm * 2 + c) * R + rr -> mu^ row of moment m = 2 mm + half
      const int vb = ((g & 2) ? NV2 : 0) + ((g & 1) ? NV4 : 0);
      float* mrow = smu + le * R * kRadTcKP;  // column rr's rows at rr * KP
      const float nl = -logf(rc);
#pragma unroll
      for (int t = 0; t < NV4; ++t) {
        const int x = vb + t;
        const int mm = x / (2 * R), c = (x / R) & 1, rr = x % R;
        const int m = 2 * mm + half;
        if (mm >= cnt) continue;
        if (m == 0) {
          if (c == 0) mrow[rr * kRadTcKP] = nl * v[t];  // row 0: -log(r) mu_0 (mu_0 is real)
        } else {
          mrow[rr * kRadTcKP + 2 * m - 1 + c] = v[t];
        }
      }
      // zero rows past 2 nm - 1 (written once per tile by the second half's lane 0)
      if (half && g == 0)
        for (int row = 2 * nm - 1; row < kRadTcK; ++row)
#pragma unroll
          for (int rr = 0; rr < R; ++rr) mrow[rr * kRadTcKP + row] = 0.f;
    }
    __syncthreads();  // mu^ tile complete
    {
      // ---- rows -> TMEM: thread row m = tid % 128 (leaf m / R, column m % R;
      // warp w reaches TMEM lanes 32 (w % 4) ..): warps 0-3 store the tf32 hi
      // part, warps 4-7 the lo part; rows past the 32 leaves are zero
      const int m = tid & 127;
      const int e = m / R, rr = m - (m / R) * R;
      const bool row_live = e < kRadTcLeaves && tile * kRadTcLeaves + e < nleaf;
      const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
      const uint32_t t_dst = tmem + lane_base + 64 + (warp >= 4 ? kRadTcK : 0);
      const float* mr = smu + ((e < kRadTcLeaves ? e : 0) * R + rr) * kRadTcKP;
#pragma unroll 4
      for (int kb = 0; kb < kRadTcK / 4; ++kb) {
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row_live) x = *reinterpret_cast<const float4*>(mr + 4 * kb);
        float4 h;
        h.x = tf32_rna(x.x);
        h.y = tf32_rna(x.y);
        h.z = tf32_rna(x.z);
        h.w = tf32_rna(x.w);
        if (warp >= 4) {
          h.x = tf32_rna(x.x - h.x);
          h.y = tf32_rna(x.y - h.y);
          h.z = tf32_rna(x.z - h.z);
          h.w = tf32_rna(x.w - h.w);
        }
        tmem_st4(t_dst + 4 * kb, h);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();  // TMEM rows written; smu free for the next tile
    if (warp < 4) {
      if (tid == 0) {
        if (first) mbar_wait(&bar[0], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bh = smem_u32(Ah), bl = smem_u32(Ah + 64 * kRadTcK);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          const uint32_t a0 = tmem + (cc == 2 ? 64u + kRadTcK : 64u), b0 = cc == 1 ? bl : bh;
#pragma unroll
          for (int ks = 0; ks < kRadTcK / 8; ++ks)
            umma_tf32_ts(tmem, a0 + ks * 8, umma_desc_kmajor_sbo(b0 + ks * 2 * kTcLBO, kRadTcSBO),
                         (cc | ks) != 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar[1]))
                     : "memory");
      }
      first = false;
      mbar_wait(&bar[1], mma_phase);
      mma_phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[64];
      tmem_ld64(tmem + (uint32_t(warp * 32) << 16), r);
      const int e = tid / R, rr = tid - (tid / R) * R;
      if (e < kRadTcLeaves)
#pragma unroll
        for (int k = 0; k < 64; ++k) stage[e * OS + k * R + rr] = __uint_as_float(r[k]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      named_bar_sync(2, 128);
      const int64_t l0t = tile * kRadTcLeaves;
      const int nt = int(nleaf - l0t < kRadTcLeaves ? nleaf - l0t : int64_t(kRadTcLeaves));
      constexpr int NVQ = QR / 4;
      for (int i = tid; i < nt * NVQ; i += 128) {
        const int ee = i / NVQ, vq = i - (i / NVQ) * NVQ;
        *reinterpret_cast<float4*>(s + int64_t(tleaf[ee]) * QR + 4 * vq) =
            *reinterpret_cast<const float4*>(stage + ee * OS + 4 * vq);
      }
      named_bar_sync(2, 128);  // stage reusable
    } else {
      first = false;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// Reception through the incoming expansion.  One warp per leaf, one lane per
// point; the point data and the leaf's amplitudes are loaded before the
// coefficient phase so their latency overlaps it.  E [Q][nt + 1] float2
// (column 0 = 1, column m = (1/m) e^{-i m theta_k}) is read through L1.
// smem per warp: beta [nt + 1][R] float2 (16-byte aligned), o [Q][R].
// BETA_IN: `o` holds beta^[leaf][64][R] (row 0 = sum_k o_k, rows 2m-1 / 2m =
// Re / Im beta_m) from the tensor-core GEMM beta^ = E^ o; the coefficient
// phase is skipped.
// Register budget for 6 CTAs / SM with beta^ in (measured 37 vs 39 us at C4).
template <int R, bool BETA_IN>
__global__ void __launch_bounds__(32 * kExpWarps, BETA_IN ? 6 : 1) reception_exp_kernel(
    const float2* __restrict__ prel, const int64_t* __restrict__ leaf_start,
    const int64_t* __restrict__ leaf_stop, const float* __restrict__ leaf_r,
    const float2* __restrict__ E, const float* __restrict__ o, const float* __restrict__ phin,
    const int64_t* __restrict__ perm, float* __restrict__ phi, int64_t leaf0, int64_t nleaf, int Q,
    int nt, int ldp) {
  KtScope kt_(70 + int(BETA_IN));
  extern __shared__ float4 sm4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = ((nt + 1) * R + 1) & ~1;            // beta float2, even
  const int per_warp = nb + ((Q * R + 3) & ~3) / 2;  // + o floats, 16-byte multiple
  float2* beta = reinterpret_cast<float2*>(sm4) + warp * per_warp;
  float* os = reinterpret_cast<float*>(beta + nb);
  const int ne = nt + 1;
  constexpr int kSlots = 4;
  const int nq = BETA_IN ? 64 * R : Q * R;
  constexpr int NOV = BETA_IN ? 2 * R : 4;  // prefetched words per lane
  const int64_t stride = int64_t(gridDim.x) * kExpWarps;
  // the next leaf's extent, radius and amplitudes (or coefficients) are
  // loaded one leaf ahead, so a leaf starts with one memory round trip (its
  // points) instead of a chain of dependent loads
  int64_t nx_b = 0;
  int nx_n = 0;
  float nx_r = 1.f;
  float nx_ov[NOV];
  auto meta = [&](int64_t l) {
    if (l < nleaf) {
      const int64_t lf = leaf0 + l;
      const int64_t b0 = leaf_start[lf], b1 = leaf_stop[lf];
      nx_r = leaf_r[lf];
#pragma unroll
      for (int t = 0; t < NOV; ++t) nx_ov[t] = lane + 32 * t < nq ? o[lf * nq + lane + 32 * t] : 0.f;
      nx_b = b0;
      nx_n = int(b1 - b0);
    }
  };
  meta(int64_t(blockIdx.x) * kExpWarps + warp);
  for (int64_t li = int64_t(blockIdx.x) * kExpWarps + warp; li < nleaf; li += stride) {
    const int64_t leaf = leaf0 + li;
    const int64_t b = nx_b;
    const int n = nx_n;
    const float r = nx_r;
    float ov[NOV];
#pragma unroll
    for (int t = 0; t < NOV; ++t) ov[t] = nx_ov[t];
    meta(li + stride);
    // the first kSlots * 32 points
    float2 pp[kSlots];
    int64_t dd[kSlots];
    float bb[kSlots][R];
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
      const int j = lane + 32 * i;
      if (j < n) {
        pp[i] = prel[b + j];
        dd[i] = perm ? perm[b + j] : b + j;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) bb[i][rr] = phin ? phin[(b + j) * R + rr] : 0.f;
      }
    }
    const float nlr = -logf(r);
    if constexpr (BETA_IN) {
      // beta^ row 0 -> beta_0 = -log(r) sum o; rows (2m-1, 2m) -> beta_m
#pragma unroll
      for (int t = 0; t < NOV; ++t) {
        const int idx = lane + 32 * t;
        if (idx < nq) {
          const int row = idx / R, rr = idx - (idx / R) * R;
          const int m = (row + 1) >> 1;
          // beta layout (floats): [m][re | -im][rr] (column pairs share an FFMA2)
          float* bf = reinterpret_cast<float*>(beta);
          if (row == 0) {
            bf[rr] = nlr * ov[t];
            bf[R + rr] = 0.f;
          } else if (m <= nt) {
            bf[m * 2 * R + ((row & 1) ? 0 : R) + rr] = (row & 1) ? ov[t] : -ov[t];
          }
        }
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int t = 0; t < NOV; ++t)
        if (lane + 32 * t < nq) os[lane + 32 * t] = ov[t];
      for (int t = lane + 32 * NOV; t < nq; t += 32) os[t] = o[leaf * nq + t];
      __syncwarp();
      for (int m = lane; m < ne; m += 32) {
        float2 acc[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int k = 0; k < Q; ++k) {
          const float2 e = __ldg(E + k * ne + m);
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const float ok = os[k * R + rr];
            acc[rr].x = fmaf(e.x, ok, acc[rr].x);
            acc[rr].y = fmaf(e.y, ok, acc[rr].y);
          }
        }
        float* bf = reinterpret_cast<float*>(beta) + m * 2 * R;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          bf[rr] = m ? acc[rr].x : nlr * acc[rr].x;
          bf[R + rr] = m ? -acc[rr].y : 0.f;
        }
      }
      __syncwarp();
    }
    const float inv = 1.f / r;
    const float* bf = reinterpret_cast<const float*>(beta);
    auto coef = [&](int m, float (&br)[R], float (&nbi)[R]) {  // re and -im of beta_m per column
      if constexpr (R == 2) {
        const float4 t = *reinterpret_cast<const float4*>(bf + m * 4);
        br[0] = t.x; br[1] = t.y; nbi[0] = t.z; nbi[1] = t.w;
      } else {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          br[rr] = bf[m * 2 * R + rr];
          nbi[rr] = bf[m * 2 * R + R + rr];
        }
      }
    };
    // acc += Re(beta_m z) = re z.x - im z.y (the -im term first)
    auto term = [&](float (&acc)[R], float2 z, const float (&br)[R], const float (&nbi)[R]) {
      if constexpr (R % 2 == 0) {
#pragma unroll
        for (int rr = 0; rr < R; rr += 2) {
          ffma2(acc[rr], acc[rr + 1], z.y, nbi[rr], nbi[rr + 1]);
          ffma2(acc[rr], acc[rr + 1], z.x, br[rr], br[rr + 1]);
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = fmaf(br[rr], z.x, fmaf(nbi[rr], z.y, acc[rr]));
      }
    };
    // two points per pass: their power and sum chains interleave (the series
    // is a dependent chain per point); per-point arithmetic as one point alone
    auto eval2 = [&](float2 pa, int64_t da, const float* ba, float2 pb, int64_t db, const float* bb2,
                     bool two) {
      const float2 wa = make_float2(pa.x * inv, pa.y * inv), wb = make_float2(pb.x * inv, pb.y * inv);
      const float2 Wa2 = make_float2(-wa.y, wa.x), Wb2 = make_float2(-wb.y, wb.x);
      float2 za = wa, zb = wb;
      float acca[R], accb[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acca[rr] = accb[rr] = bf[rr];
#pragma unroll 2
      for (int m = 1; m <= nt; ++m) {
        float br[R], nbi[R];
        coef(m, br, nbi);
        term(acca, za, br, nbi);
        term(accb, zb, br, nbi);
        za = cmul_pk(za, wa, Wa2);
        zb = cmul_pk(zb, wb, Wb2);
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) phi[da * ldp + rr] = ba[rr] + acca[rr];
      if (two)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) phi[db * ldp + rr] = bb2[rr] + accb[rr];
    };
    // one point per lane: the last pass of a leaf whose remainder fits 32
    // lanes (3 of 4 leaves at C4: 65-96 points) costs half the two-point pass
    auto eval1 = [&](float2 pa, int64_t da, const float* ba) {
      const float2 wa = make_float2(pa.x * inv, pa.y * inv);
      const float2 Wa2 = make_float2(-wa.y, wa.x);
      float2 za = wa;
      float acca[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acca[rr] = bf[rr];
#pragma unroll 2
      for (int m = 1; m <= nt; ++m) {
        float br[R], nbi[R];
        coef(m, br, nbi);
        term(acca, za, br, nbi);
        za = cmul_pk(za, wa, Wa2);
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) phi[da * ldp + rr] = ba[rr] + acca[rr];
    };
#pragma unroll
    for (int i = 0; i < kSlots; i += 2) {
      if (32 * (i + 1) >= n) {  // (warp-uniform) no lane has a second point in this pass
        if (lane + 32 * i < n) eval1(pp[i], dd[i], bb[i]);
      } else if (lane + 32 * i < n) {
        eval2(pp[i], dd[i], bb[i], pp[i + 1], dd[i + 1], bb[i + 1], lane + 32 * (i + 1) < n);
      }
    }
    for (int j = lane + 32 * kSlots; j < n; j += 32) {
      float base[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) base[rr] = phin ? phin[(b + j) * R + rr] : 0.f;
      const float2 p = prel[b + j];
      eval2(p, perm ? perm[b + j] : b + j, base, p, 0, base, false);
    }
    __syncwarp();
  }
}

// float64 plans: the same incoming expansion in float64 (the reference's
// precision).  Per leaf one warp forms beta_m = sum_k (1/m) e^{-i m theta_k}
// o_k (beta_0 = -log(r) sum_k o_k) in shared memory, then every lane
// evaluates phi_j = phi_near_j + Re sum_m beta_m w_j^m for its points; the
// plan sets the number of terms for a float64 truncation (<= 1e-15 relative
// at the largest |w|).  Replaces streaming the stored float64 U (1 GB at C4)
// by ~8 FP64 FMAs per point, term and column.
template <int R>
__global__ void __launch_bounds__(32 * kExpWarps) reception_exp64_kernel(
    const double2* __restrict__ prel, const int64_t* __restrict__ leaf_start,
    const int64_t* __restrict__ leaf_stop, const double* __restrict__ leaf_r,
    const double2* __restrict__ E, const double* __restrict__ o, const double* __restrict__ phin,
    const int64_t* __restrict__ perm, double* __restrict__ phi, int64_t leaf0, int64_t nleaf, int Q, int nt,
    int ldp) {
  KtScope kt_(72);
  extern __shared__ double2 smd[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ne = nt + 1;
  double2* beta = smd + size_t(warp) * (size_t(ne) * R + (size_t(Q) * R + 1) / 2);  // [m][rr] (re, -im)
  double* os = reinterpret_cast<double*>(beta + size_t(ne) * R);
  const int64_t stride = int64_t(gridDim.x) * kExpWarps;
  for (int64_t li = int64_t(blockIdx.x) * kExpWarps + warp; li < nleaf; li += stride) {
    const int64_t leaf = leaf0 + li;
    const int64_t b = leaf_start[leaf];
    const int n = int(leaf_stop[leaf] - b);
    const double r = leaf_r[leaf];
    for (int t = lane; t < Q * R; t += 32) os[t] = o[leaf * int64_t(Q) * R + t];
    __syncwarp();
    const double nlr = -log(r);
    for (int m = lane; m < ne; m += 32) {
      double ar[R], ai[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) ar[rr] = ai[rr] = 0.0;
      for (int k = 0; k < Q; ++k) {
        const double2 e = __ldg(E + k * ne + m);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const double ok = os[k * R + rr];
          ar[rr] = fma(e.x, ok, ar[rr]);
          ai[rr] = fma(e.y, ok, ai[rr]);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr)
        beta[m * R + rr] = m ? make_double2(ar[rr], -ai[rr]) : make_double2(nlr * ar[rr], 0.0);
    }
    __syncwarp();
    const double inv = 1.0 / r;
    for (int j = lane; j < n; j += 32) {
      const double2 p = prel[b + j];
      const double2 w = make_double2(p.x * inv, p.y * inv);
      double2 z = w;
      double acc[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[rr] = beta[rr].x;
      for (int m = 1; m <= nt; ++m) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const double2 bm = beta[m * R + rr];  // (re, -im): Re(beta z) = re z.x - im z.y
          acc[rr] = fma(bm.x, z.x, fma(bm.y, z.y, acc[rr]));
        }
        z = make_double2(z.x * w.x - z.y * w.y, z.x * w.y + z.y * w.x);
      }
      const int64_t dst = perm ? perm[b + j] : b + j;
#pragma unroll
      for (int rr = 0; rr < R; ++rr) phi[dst * ldp + rr] = (phin ? phin[(b + j) * R + rr] : 0.0) + acc[rr];
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// Near field for many right-hand sides on the tensor cores (float32 plans;
// C5: 64 plane waves = 128 real columns).  phi[perm p] += sum_j K_pj q_j for
// up to 128 real columns at once.  An item = <= 128 target rows of a leaf
// (padded to N = 16 k) against the leaf's near slab (W source points).  The
// MMA computes D (128 x N) = X^T (128 x W) K^T (W x N): M = the right-hand-side
// columns, so one tile covers 128 columns and the operator is streamed ONCE
// for all of them (the 4-column blocks streamed it 32 times).  K arrives by
// bulk copy in chunks of 32 source points, tf32 hi | lo pre-split in the
// canonical K-major layout (N rows x 32 k); X^T rows (thread r = column r)
// are read straight from the caller's q in ORIGINAL order (the permutation is
// folded into the item's source table: coalesced 512-byte rows), split and
// stored to TMEM; the chunk pipeline keeps the next chunk's X in registers
// and its K in flight while the tensor core works.  The epilogue adds the
// 128 x N tile into phi (each target row a coalesced 512-byte row).
// ----------------------------------------------------------------------------
struct NearTcItem {
  int64_t b_off;      // float offset of the item's canonical blob (kchunks x [hi | lo] x npad x 32)
  int64_t a_off;      // column-major near blob offset of the block item (packing input)
  int32_t m, npad;    // target rows, rows padded to a multiple of 16 (<= 256)
  int32_t w, kchunks; // slab width (source points), 32-point chunks
  int32_t y_row0;     // first target row (tree order)
  int32_t src_off;    // first entry of the item's source table (original indices)
  int32_t ld, r0;     // packing: leading dimension and first row within the block item
};
constexpr int kNearTcK = 32;
constexpr int kNearTcMaxN = 128;  // target rows per item: 256 TMEM columns, two CTAs per SM
constexpr uint32_t kNearTcSBO = kNearTcK * 8 * 4;  // bytes between 8-row groups of a chunk

// column-major near blob -> per-item canonical tf32 hi | lo chunks
__global__ void near_tc_pack_kernel(const NearTcItem* __restrict__ items, const float* __restrict__ blob,
                                    float* __restrict__ out) {
  const NearTcItem it = items[blockIdx.x];
  const int64_t per_chunk = int64_t(it.npad) * kNearTcK;
  for (int64_t e = threadIdx.x; e < int64_t(it.kchunks) * per_chunk; e += blockDim.x) {
    const int c = int(e / per_chunk);
    const int rem = int(e - int64_t(c) * per_chunk);
    const int n = rem / kNearTcK, kk = rem - (rem / kNearTcK) * kNearTcK;
    const int k = c * kNearTcK + kk;
    const float x = (n < it.m && k < it.w) ? blob[it.a_off + int64_t(k) * it.ld + it.r0 + n] : 0.f;
    const float hi = tf32_rna(x), lo = tf32_rna(x - hi);
    const int64_t base = it.b_off + int64_t(c) * 2 * per_chunk;
    const int off = (n >> 3) * (kNearTcK * 8) + (kk >> 2) * 32 + (n & 7) * 4 + (kk & 3);
    out[base + off] = hi;
    out[base + per_chunk + off] = lo;
  }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void umma_tf32_ts_n(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(accumulate), "r"(idesc), "r"(0u));
}

constexpr size_t near_tc_smem_bytes() {
  return size_t(2) * 2 * kNearTcMaxN * kNearTcK * 4 + 64;
}

__global__ void __launch_bounds__(128, 2) near_tc_kernel(const NearTcItem* __restrict__ items, int n_items,
                                                         const int32_t* __restrict__ src,
                                                         const float* __restrict__ blob,
                                                         const float* __restrict__ q, int ldq, int c0,
                                                         int ncols, const int64_t* __restrict__ perm,
                                                         float* __restrict__ phi, int accumulate) {
  KtScope kt_(90);
  extern __shared__ __align__(128) unsigned char smem[];
  float* Bs = reinterpret_cast<float*>(smem);  // 2 buffers x [hi | lo] x npad x 32
  constexpr int kBufFloats = 2 * kNearTcMaxN * kNearTcK;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + size_t(2) * kBufFloats * 4);  // [0,1] B, [2,3] MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  const bool col_live = tid < ncols;
  const float* qc = q + c0 + tid;
  // per-slot state as bits (slot s = bit s): barrier phases, MMA outstanding
  uint32_t bphase = 0u, mphase = 0u, pending = 0u;
  auto wait_mma = [&](int slot) {
    if (pending & (1u << slot)) {
      mbar_wait(&bar[2 + slot], (mphase >> slot) & 1u);
      mphase ^= 1u << slot;
      pending &= ~(1u << slot);
    }
  };
  auto issue_b = [&](const NearTcItem& it, int c, int slot) {
    const uint32_t bytes = uint32_t(it.npad) * kNearTcK * 4 * 2;
    mbar_arrive_expect_tx(&bar[slot], bytes);
    bulk_g2s(Bs + slot * kBufFloats, blob + it.b_off + int64_t(c) * 2 * it.npad * kNearTcK, bytes, &bar[slot]);
  };
  // X^T values of chunk c of item it for this thread's column: 32 source rows
  auto load_x = [&](const NearTcItem& it, int c, float (&x)[kNearTcK]) {
#pragma unroll
    for (int kk = 0; kk < kNearTcK; ++kk) {
      const int k = c * kNearTcK + kk;
      x[kk] = (col_live && k < it.w) ? __ldg(qc + int64_t(src[it.src_off + k]) * ldq) : 0.f;
    }
  };
  int gc = 0;  // chunks issued by this CTA (slot = gc & 1)
  int item = blockIdx.x;
  NearTcItem it{};
  float xn[kNearTcK];
  if (item < n_items) {
    it = items[item];
    if (tid == 0) issue_b(it, 0, 0);
    load_x(it, 0, xn);
  }
  while (item < n_items) {
    const int next_item = item + int(gridDim.x);
    NearTcItem nx{};
    if (next_item < n_items) nx = items[next_item];
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(it.npad) >> 3) << 17) |
                           ((128u >> 4) << 24);
    for (int c = 0; c < it.kchunks; ++c, ++gc) {
      const int slot = gc & 1;
      float x[kNearTcK];
#pragma unroll
      for (int kk = 0; kk < kNearTcK; ++kk) x[kk] = xn[kk];
      // the next chunk (this item's or the next item's first) in flight
      const bool last = c + 1 == it.kchunks;
      if (!last)
        load_x(it, c + 1, xn);
      else if (next_item < n_items)
        load_x(nx, 0, xn);
      wait_mma(slot);  // chunk gc - 2 released this A slot
      const uint32_t t_hi = tmem + lane_base + kNearTcMaxN + 64 * slot, t_lo = t_hi + 32;
#pragma unroll
      for (int kb = 0; kb < kNearTcK / 4; ++kb)
        tc_put4(t_hi, t_lo, kb, make_float4(x[4 * kb], x[4 * kb + 1], x[4 * kb + 2], x[4 * kb + 3]));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        mbar_wait(&bar[slot], (bphase >> slot) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bh = smem_u32(Bs + slot * kBufFloats);
        const uint32_t bl = bh + uint32_t(it.npad) * kNearTcK * 4;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          const uint32_t a0 = tmem + kNearTcMaxN + 64 * slot + (cc == 2 ? 32u : 0u), b0 = cc == 1 ? bl : bh;
#pragma unroll
          for (int ks = 0; ks < kNearTcK / 8; ++ks)
            umma_tf32_ts_n(tmem, a0 + ks * 8, umma_desc_kmajor_sbo(b0 + ks * 2 * kTcLBO, kNearTcSBO), idesc,
                           (c | cc | ks) != 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar[2 + slot]))
                     : "memory");
      }
      bphase ^= 1u << slot;
      pending |= 1u << slot;
      // the next chunk's K into the other buffer once its previous MMA is done
      if (!last || next_item < n_items) {
        const int ns = (gc + 1) & 1;
        wait_mma(ns);
        if (tid == 0) issue_b(last ? nx : it, last ? 0 : c + 1, ns);
      }
    }
    // ---- epilogue: the item's 128 x npad tile into phi (rows = targets)
    wait_mma((gc - 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int n0 = 0; n0 < it.m; n0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + uint32_t(n0), r);
      const int nn = it.m - n0 < 32 ? it.m - n0 : 32;
      int64_t dst[32];
      float cur[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) dst[j] = j < nn ? perm[it.y_row0 + n0 + j] : 0;
      if (col_live) {
#pragma unroll
        for (int j = 0; j < 32; ++j) cur[j] = (accumulate && j < nn) ? phi[dst[j] * ldq + c0 + tid] : 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nn) phi[dst[j] * ldq + c0 + tid] = cur[j] + __uint_as_float(r[j]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // accumulator read before the next item overwrites it
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    item = next_item;
    it = nx;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// ----------------------------------------------------------------------------
// Many right-hand sides (C5): the far field as batched GEMMs over up to 128
// columns.  With one or two columns every far-field step is a latency-bound
// GEMV; with 128 it is a dense GEMM per group (M = Q or leaf rows, N = 128,
// K = Q or leaf points), so the whole chain -- radiation V q, the upward
// C s, translation D s plus downward B o, reception U o -- runs through ONE
// register-tiled kernel fed by host-built work lists:
//
//   item  = one output tile (<= 64 rows x 128 columns: a group's s or o, or
//           a leaf panel of phi), written by exactly one CTA;
//   terms = the (matrix, input rows) products summed into it, in the
//           reference's order (children in id order; interaction entries in
//           list order, then B o_parent -- fastmvp.py:160-169).
//
// Matrices are column-major with a leading dimension (the plan's transposed
// C / B / D tables, the stored V / U blobs), inputs are rows of kWCols
// values (tree-order charges, s, o).  Each CTA stages K chunks of A and X in
// shared memory (double-buffered through registers) and every thread owns a
// 4 x 8 tile (FFMA2 on column pairs for float32).  One launch per stage and
// level, every launch independent of the column count up to 128.
// ----------------------------------------------------------------------------
constexpr int kWCols = 128;
constexpr int kWRows = 64;
constexpr int kWThreads = 256;

struct WTerm {
  int64_t a_off;  // A(0, 0) of the tile: element offset in matrix base `abase`
  int64_t x_row;  // first input row (K rows of kWCols values)
  int32_t lda;    // column stride of A (multiple of 4)
  int32_t k;      // inner dimension
  int32_t abase;  // 0 C table, 1 B table, 2 D table, 3 V blob, 4 U blob
  int32_t xsel;   // 0 charges (tree order), 1 s, 2 o
};
struct WItem {
  int64_t y_row;  // first output row (workspace row, or tree row when scattering)
  int32_t m;      // rows of the tile (<= kWRows)
  int32_t t0, t1; // terms
  int32_t pad;
};
static_assert(sizeof(WTerm) == 32 && sizeof(WItem) == 24, "work-list records");

template <typename T>
struct WArgs {
  const WItem* items;
  const WTerm* terms;
  const T* abase[5];
  const T* xs[3];       // xsel 1 s, 2 o (rows of kWCols); xsel 0 reads the caller's q
  T* y;                 // store: workspace rows of kWCols; scatter: phi rows of ldy
  const int64_t* perm;  // tree row -> original row (charges in, phi out)
  const T* q;           // xsel 0: the caller's charges, (N, ldy) in original order
  int64_t ldy;
  int col0, ncols;      // the caller's columns [col0, col0 + ncols)
  int vec4;             // ldy and col0 multiples of 16 bytes: vector loads of q rows
};
enum { kWStore = 0, kWScatter = 1, kWScatterAdd = 2 };

// Tile geometry: NC output columns per CTA (blockIdx.y picks the column
// block), KG groups of 256 / KG threads that split an item's terms between
// them (term-strided; each group has its own barrier and double buffer) and
// add their partial tiles in a fixed order at the end.  Wide levels use
// <128, 1>; the coarse levels -- few groups, many terms each -- <32, 4>,
// which gives 16x the CTAs and a quarter of the serial chunk chain.
template <typename T, int NC, int KG, int TR>
struct WTile {
  static constexpr int KC = sizeof(T) == 4 ? 16 : 8;  // K chunk
  static constexpr int CG = NC / 8;                   // column groups (8 columns per thread)
  static constexpr int GT = (kWRows / TR) * CG;       // threads per group (TR rows x 8 columns each)
  static constexpr int kThreads = GT * KG;
  static constexpr int AV = KC * kWRows / GT;         // A values per thread per chunk
  static constexpr int XV = KC * NC / GT;             // X values per thread per chunk
  static constexpr int kBuf = 2 * KC * (kWRows + NC); // one group's double buffer (elements)
  static constexpr size_t kSmem =
      sizeof(T) * (size_t(KG) * kBuf > (KG > 1 ? size_t(KG) * kWRows * NC : 0)
                       ? size_t(KG) * kBuf
                       : size_t(KG) * kWRows * NC);
  static_assert(kThreads <= 256 && kWRows % TR == 0, "TR x 8 thread tiles cover 64 rows x NC columns");
  static_assert(AV % (16 / sizeof(T)) == 0 && XV >= 4 && XV % 4 == 0 && TR % (16 / sizeof(T)) == 0,
                "loader geometry (16-byte vectors)");
};

template <typename T, int MODE, int NC, int KG, int TR>
__global__ void __launch_bounds__(WTile<T, NC, KG, TR>::kThreads) wgemm_kernel(const __grid_constant__ WArgs<T> a) {
  using W = WTile<T, NC, KG, TR>;
  constexpr int KC = W::KC, AV = W::AV, XV = W::XV, GT = W::GT, CG = W::CG;
  extern __shared__ __align__(16) unsigned char wsm[];
  const int tid = threadIdx.x, grp = tid / GT, lt = tid % GT;
  const int tx = lt % CG, ty = lt / CG;
  T* const gbuf = reinterpret_cast<T*>(wsm) + size_t(grp) * W::kBuf;
  auto As = [&](int buf, int k) { return gbuf + (buf * KC + k) * kWRows; };
  auto Xs = [&](int buf, int k) { return gbuf + 2 * KC * kWRows + (buf * KC + k) * NC; };
  auto gsync = [&]() {
    if constexpr (KG == 1)
      __syncthreads();
    else
      named_bar_sync(1 + grp, GT);
  };
  const WItem it = a.items[blockIdx.x];
  const int cb = blockIdx.y * NC;  // first column of this CTA
  const int a_k = lt / (kWRows / AV), a_r = (lt % (kWRows / AV)) * AV;
  const int x_k = lt / (NC / XV), x_c = (lt % (NC / XV)) * XV;
  T ra[AV], rx[XV];
  auto load = [&](int tt, int kk0) {
    const WTerm w = a.terms[tt];
    const int k = kk0 + a_k;
    const T* A = a.abase[w.abase] + w.a_off + int64_t(k) * w.lda + a_r;
#pragma unroll
    for (int v = 0; v < AV; ++v) ra[v] = (k < w.k && a_r + v < it.m) ? A[v] : T(0);
    const int kx = kk0 + x_k;
    const int col = cb + x_c;  // column within the pass
    if (kx < w.k && w.xsel == 0) {
      // charges straight from the caller's q through perm (no gather pass)
      const T* X = a.q + a.perm[w.x_row + kx] * a.ldy + a.col0 + col;
      if (a.vec4 && col + XV <= a.ncols) {
#pragma unroll
        for (int v = 0; v < XV; v += 16 / int(sizeof(T))) {
          if constexpr (sizeof(T) == 4) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(X + v));
            rx[v] = f.x; rx[v + 1] = f.y; rx[v + 2] = f.z; rx[v + 3] = f.w;
          } else {
            const double2 f = __ldg(reinterpret_cast<const double2*>(X + v));
            rx[v] = f.x; rx[v + 1] = f.y;
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < XV; ++v) rx[v] = col + v < a.ncols ? __ldg(X + v) : T(0);
      }
    } else if (kx < w.k) {
      const T* X = a.xs[w.xsel] + (w.x_row + kx) * kWCols + col;
#pragma unroll
      for (int v = 0; v < XV; v += 16 / int(sizeof(T))) {
        if constexpr (sizeof(T) == 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(X + v));
          rx[v] = f.x; rx[v + 1] = f.y; rx[v + 2] = f.z; rx[v + 3] = f.w;
        } else {
          const double2 f = __ldg(reinterpret_cast<const double2*>(X + v));
          rx[v] = f.x; rx[v + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < XV; ++v) rx[v] = T(0);
    }
  };
  // 16-byte shared accesses throughout (every offset is a multiple of 16 bytes)
  using V4 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int VW = 16 / int(sizeof(T));  // elements per 16-byte vector
  auto st16 = [&](T* p, const T* v) {
    if constexpr (sizeof(T) == 4)
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else
      *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  };
  auto ld16 = [&](const T* p, T* v) {
    const V4 x = *reinterpret_cast<const V4*>(p);
    if constexpr (sizeof(T) == 4) {
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      v[0] = x.x; v[1] = x.y;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int v = 0; v < AV; v += VW) st16(As(buf, a_k) + a_r + v, ra + v);
#pragma unroll
    for (int v = 0; v < XV; v += VW) st16(Xs(buf, x_k) + x_c + v, rx + v);
  };
  T acc[TR][8];
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);
  // this group's terms: t0 + grp, t0 + grp + KG, ...
  int t = it.t0 + grp, k0 = 0, buf = 0;
  bool have = t < it.t1;
  if (have) load(t, 0);
  while (have) {
    store(buf);
    gsync();
    const int kt = a.terms[t].k;
    k0 += KC;
    if (k0 >= kt) {
      k0 = 0;
      t += KG;
    }
    have = t < it.t1;
    if (have) load(t, k0);
    // row groups entirely past the tile's rows (Q = 48 in a 64-row tile,
    // the short last panel of a leaf) skip the math -- whole warps for 8-row
    // thread tiles
#pragma unroll
    for (int kk = 0; kk < KC && ty * TR < it.m; ++kk) {
      const T* Ap = As(buf, kk) + ty * TR;
      const T* Xp = Xs(buf, kk) + tx * 4;
      T av[TR], x0[4], x1[4];
#pragma unroll
      for (int i = 0; i < TR; i += VW) ld16(Ap + i, av + i);
#pragma unroll
      for (int j = 0; j < 4; j += VW) {
        ld16(Xp + j, x0 + j);
        ld16(Xp + NC / 2 + j, x1 + j);
      }
#pragma unroll
      for (int i = 0; i < TR; ++i) {
        if constexpr (sizeof(T) == 4) {
          ffma2(acc[i][0], acc[i][1], av[i], x0[0], x0[1]);
          ffma2(acc[i][2], acc[i][3], av[i], x0[2], x0[3]);
          ffma2(acc[i][4], acc[i][5], av[i], x1[0], x1[1]);
          ffma2(acc[i][6], acc[i][7], av[i], x1[2], x1[3]);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][j] = fma(av[i], x0[j], acc[i][j]);
            acc[i][4 + j] = fma(av[i], x1[j], acc[i][4 + j]);
          }
        }
      }
    }
    buf ^= 1;
    // the other buffer is rewritten only after every thread of the group
    // passed this iteration's barrier (two-deep ring, one barrier per chunk)
  }
  // columns of this thread: cb + tx*4 + j and cb + NC/2 + tx*4 + j
  if constexpr (KG > 1) {
    // add the groups' partial tiles in group order (deterministic)
    __syncthreads();
    T* red = reinterpret_cast<T*>(wsm);
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        red[(size_t(grp) * kWRows + ty * TR + i) * NC + tx * 4 + j] = acc[i][j];
        red[(size_t(grp) * kWRows + ty * TR + i) * NC + NC / 2 + tx * 4 + j] = acc[i][4 + j];
      }
    __syncthreads();
    for (int e = tid; e < kWRows * NC; e += W::kThreads) {
      const int r = e / NC, c = e - (e / NC) * NC;
      if (r >= it.m) continue;
      T v = red[e];
#pragma unroll
      for (int g = 1; g < KG; ++g) v += red[size_t(g) * kWRows * NC + e];
      if constexpr (MODE == kWStore) {
        a.y[(it.y_row + r) * kWCols + cb + c] = v;
      } else {
        if (cb + c < a.ncols) {
          T* y = a.y + a.perm[it.y_row + r] * a.ldy + a.col0 + cb + c;
          *y = (MODE == kWScatterAdd ? *y : T(0)) + v;
        }
      }
    }
  } else {
  // epilogue: this CTA is the tile's only writer; 16-byte stores
  // (4 consecutive columns per thread and half)
  auto put4 = [&](T* y, const T* v, int ncol_left) {
    if constexpr (sizeof(T) == 4) {
      if (ncol_left >= 4 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
        float4 o = make_float4(v[0], v[1], v[2], v[3]);
        if (MODE == kWScatterAdd) {
          const float4 c = *reinterpret_cast<const float4*>(y);
          o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
        }
        *reinterpret_cast<float4*>(y) = o;
        return;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ncol_left) y[j] = (MODE == kWScatterAdd ? y[j] : T(0)) + v[j];
  };
#pragma unroll
  for (int i = 0; i < TR; ++i) {
    const int r = ty * TR + i;
    if (r >= it.m) continue;
    if constexpr (MODE == kWStore) {
      T* y = a.y + (it.y_row + r) * kWCols + cb;
      put4(y + tx * 4, &acc[i][0], 4);
      put4(y + NC / 2 + tx * 4, &acc[i][4], 4);
    } else {
      T* y = a.y + a.perm[it.y_row + r] * a.ldy + a.col0 + cb;
      put4(y + tx * 4, &acc[i][0], a.ncols - (cb + tx * 4));
      put4(y + NC / 2 + tx * 4, &acc[i][4], a.ncols - (cb + NC / 2 + tx * 4));
    }
  }
  }
}

// ----------------------------------------------------------------------------
// Multi-GPU halo exchange (paper_1801_03589_b200/dist.py):
// pack this rank's partial source amplitudes that other ranks need into the
// all_gather send buffer, and complete the needed groups' amplitudes as the
// rank-ordered sum of their contributors' partials (contrib rows < n_recv
// index the gathered buffer, rows >= n_recv this rank's own s[row - n_recv]).
// ----------------------------------------------------------------------------
template <typename T>
__global__ void xpack_kernel(const T* __restrict__ s, const int64_t* __restrict__ ids, int64_t n_ids,
                             int64_t rows, int qr, T* __restrict__ send) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < rows * qr;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / qr, w = t - r * qr;
    send[t] = r < n_ids ? s[ids[r] * qr + w] : T(0);
  }
}

template <typename T>
__global__ void xcombine_kernel(T* s, const T* __restrict__ recv, const int64_t* __restrict__ imp,
                                const int64_t* __restrict__ contrib, int64_t n_imp, int max_c,
                                int64_t n_recv, int qr) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n_imp * qr;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / qr, w = t - i * qr;
    T acc = T(0);
    for (int k = 0; k < max_c; ++k) {  // fixed rank order: deterministic
      const int64_t c = contrib[i * max_c + k];
      if (c < 0) continue;
      acc += c < n_recv ? recv[c * qr + w] : s[(c - n_recv) * qr + w];
    }
    s[imp[i] * qr + w] = acc;  // the only local row read is imp[i]'s own
  }
}


}  // namespace nesa
