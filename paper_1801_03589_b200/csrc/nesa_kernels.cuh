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

struct BlockItem {
  int64_t a_off;     // element offset of the column-major block in blob
  int32_t m, n;      // rows, columns
  int32_t y_row0;    // first output row
  int32_t seg_begin; // segments [seg_begin, seg_begin + seg_count)
  int32_t seg_count;
  int32_t pad;
};
struct BlockSeg {
  int32_t x_row0;  // first x row of the segment
  int32_t col0;    // first column (within the item) of the segment
};
struct BlockChunk {
  int32_t item;
  int32_t col0;
  int32_t ncols;
  int32_t pad;
};

constexpr int kStages = 4;
constexpr int kABytes = 24 * 1024;         // payload per stage
constexpr int kAStride = kABytes + 128;    // + alignment slack, keeps 128 B alignment
constexpr int kMaxC = 256;                 // columns per chunk
constexpr int kNCW = 8;                    // consumer warps
constexpr int kNCT = kNCW * 32;            // consumer threads
constexpr int kBGThreads = kNCT + 32;      // + producer warp
constexpr int kMaxRows = 2 * kNCT;         // rows per item (taller blocks are paneled)

enum { kModeStore = 0, kModeScatter = 1 };

template <typename T>
struct BlockGemvArgs {
  const T* blob;
  const BlockItem* items;
  const BlockSeg* segs;
  const BlockChunk* chunks;
  const int32_t* cta_chunk_ptr;  // [grid + 1]
  const T* x;                    // x rows (R values each)
  T* y;                          // store: y rows; scatter: output in original order
  const T* base;                 // scatter: added per tree row (may be null)
  const int64_t* perm;           // scatter: tree row -> original row
  int64_t perm_offset;           // scatter: tree row of perm[0] (sub-plans)
};

template <typename T, int R>
constexpr size_t blockgemv_smem_bytes() {
  return size_t(kStages) * kAStride + size_t(kStages) * kMaxC * R * sizeof(T) +
         size_t(kNCT) * R * sizeof(T) + 2 * kStages * sizeof(uint64_t) + 16;
}

template <typename T, int R, int MODE>
__device__ __forceinline__ void bg_write(const BlockGemvArgs<T>& a, int row, const T* v) {
  if constexpr (MODE == kModeStore) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) a.y[int64_t(row) * R + rr] = v[rr];
  } else {
    const int64_t dst = a.perm[row - a.perm_offset];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      T b = a.base ? a.base[int64_t(row) * R + rr] : T(0);
      a.y[dst * R + rr] = b + v[rr];
    }
  }
}

template <typename T, int R, int MODE>
__global__ void __launch_bounds__(kBGThreads, 1) blockgemv_kernel(const BlockGemvArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sA = smem;
  T* sX = reinterpret_cast<T*>(smem + size_t(kStages) * kAStride);
  T* sRed = sX + kStages * kMaxC * R;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(sRed + kNCT * R) + 15) & ~uintptr_t(15));
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
    for (int i = c0; i < c1; ++i) {
      const int k = i - c0, st = k % kStages;
      const uint32_t round = uint32_t(k / kStages);
      mbar_wait(&empty[st], (round & 1u) ^ 1u);
      const BlockChunk ch = a.chunks[i];
      const BlockItem it = a.items[ch.item];
      const uintptr_t src =
          reinterpret_cast<uintptr_t>(a.blob + it.a_off + int64_t(ch.col0) * it.m);
      const uint32_t bytes = uint32_t(ch.ncols) * uint32_t(it.m) * uint32_t(sizeof(T));
      const uintptr_t s0 = src & ~uintptr_t(15);
      const uintptr_t s1 = (src + bytes + 15) & ~uintptr_t(15);
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[st], uint32_t(s1 - s0));
        bulk_g2s(sA + size_t(st) * kAStride, reinterpret_cast<const void*>(s0),
                 uint32_t(s1 - s0), &full[st]);
      }
      T* xs = sX + st * kMaxC * R;
      const int cend = ch.col0 + ch.ncols;
      for (int sg = it.seg_begin; sg < it.seg_begin + it.seg_count; ++sg) {
        const BlockSeg S = a.segs[sg];
        const int scol1 = (sg + 1 < it.seg_begin + it.seg_count) ? a.segs[sg + 1].col0 : it.n;
        const int lo = max(S.col0, ch.col0), hi = min(scol1, cend);
        for (int c = lo + lane; c < hi; c += 32)
          cp_async_n<R * sizeof(T)>(xs + (c - ch.col0) * R,
                                  a.x + int64_t(S.x_row0 + (c - S.col0)) * R);
      }
      cp_async_mbar_arrive_noinc(&full[st]);
    }
  } else {
    // ------------------------------ consumers -----------------------------
    const int tid = threadIdx.x;
    T acc0[R], acc1[R], accB[R];
    for (int i = c0; i < c1; ++i) {
      const int k = i - c0, st = k % kStages;
      const uint32_t round = uint32_t(k / kStages);
      const BlockChunk ch = a.chunks[i];
      const BlockItem it = a.items[ch.item];
      const int m = it.m, nc = ch.ncols;
      const uintptr_t src =
          reinterpret_cast<uintptr_t>(a.blob + it.a_off + int64_t(ch.col0) * m);
      const T* A = reinterpret_cast<const T*>(sA + size_t(st) * kAStride + (src & 15));
      const T* X = sX + st * kMaxC * R;
      if (ch.col0 == 0) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc0[rr] = acc1[rr] = T(0);
      }
      mbar_wait(&full[st], round & 1u);
      if (m <= kNCT) {
        const int CL = kNCT / m;
        const int r = tid % m, cl = tid / m;
        if (cl < CL) {
#pragma unroll
          for (int rr = 0; rr < R; ++rr) accB[rr] = T(0);
          int c = cl;
          for (; c + CL < nc; c += 2 * CL) {
            const T a0 = A[c * m + r], a1 = A[(c + CL) * m + r];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              acc0[rr] = fma(a0, X[c * R + rr], acc0[rr]);
              accB[rr] = fma(a1, X[(c + CL) * R + rr], accB[rr]);
            }
          }
          if (c < nc) {
            const T a0 = A[c * m + r];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) acc0[rr] = fma(a0, X[c * R + rr], acc0[rr]);
          }
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc0[rr] += accB[rr];
        }
      } else {
        const int r1 = tid + kNCT;
        for (int c = 0; c < nc; ++c) {
          const T a0 = A[c * m + tid];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc0[rr] = fma(a0, X[c * R + rr], acc0[rr]);
          if (r1 < m) {
            const T a1 = A[c * m + r1];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) acc1[rr] = fma(a1, X[c * R + rr], acc1[rr]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);

      if (ch.col0 + nc == it.n) {  // last chunk of the item: reduce + write
        if (m <= kNCT / 2) {
          const int CL = kNCT / m;
          const int r = tid % m, cl = tid / m;
          if (cl < CL) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) sRed[(cl * m + r) * R + rr] = acc0[rr];
          }
          named_bar_sync(1, kNCT);
          if (tid < m) {
            T v[R];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) v[rr] = sRed[tid * R + rr];
            for (int l = 1; l < CL; ++l) {
#pragma unroll
              for (int rr = 0; rr < R; ++rr) v[rr] += sRed[(l * m + tid) * R + rr];
            }
            bg_write<T, R, MODE>(a, it.y_row0 + tid, v);
          }
          named_bar_sync(1, kNCT);
        } else {
          if (tid < m) bg_write<T, R, MODE>(a, it.y_row0 + tid, acc0);
          if (tid + kNCT < m) bg_write<T, R, MODE>(a, it.y_row0 + tid + kNCT, acc1);
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------
// gather qt[i] = q[perm[i]]; scatter phi[perm[i]] = phin[i]
// ----------------------------------------------------------------------------
template <typename T, int R>
__global__ void gather_kernel(const T* __restrict__ q, const int64_t* __restrict__ perm,
                              T* __restrict__ qt, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = perm[i];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) qt[i * R + rr] = q[j * R + rr];
  }
}

template <typename T, int R>
__global__ void scatter_kernel(const T* __restrict__ phin, const int64_t* __restrict__ perm,
                               T* __restrict__ phi, int64_t row0, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = perm[i];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) phi[j * R + rr] = phin[(row0 + i) * R + rr];
  }
}

// ----------------------------------------------------------------------------
// Level transfers.  CT/BT hold the four quadrant matrices of one level,
// transposed (MT[q][j][k] = M[q][k][j]) so thread k reads consecutive words.
// ----------------------------------------------------------------------------
constexpr int kLvlThreads = 256;

// s[p] = sum over local children c of C[quad c] s[c]   (parents pf .. pf+pc-1)
template <typename T, int R>
__global__ void __launch_bounds__(kLvlThreads) upward_kernel(
    const T* __restrict__ CT, const int32_t* __restrict__ quad,
    const int64_t* __restrict__ child_first, const int32_t* __restrict__ n_child,
    int64_t pf, int64_t pc, int64_t cf, int64_t cl, T* s, int Q) {
  const int NG = kLvlThreads / Q;
  const int g = threadIdx.x / Q, k = threadIdx.x % Q;
  if (g >= NG) return;
  const int64_t QQ = int64_t(Q) * Q;
  for (int64_t pi = int64_t(blockIdx.x) * NG + g; pi < pc; pi += int64_t(gridDim.x) * NG) {
    const int64_t p = pf + pi;
    const int64_t c_lo = max(child_first[p], cf);
    const int64_t c_hi = min(child_first[p] + n_child[p], cl);
    T acc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) acc[rr] = T(0);
    for (int64_t c = c_lo; c < c_hi; ++c) {
      const T* M = CT + quad[c] * QQ;
      const T* sv = s + c * Q * R;
      T part[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) part[rr] = T(0);
      for (int j = 0; j < Q; ++j) {
        const T mv = __ldg(M + j * Q + k);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) part[rr] = fma(mv, __ldg(sv + j * R + rr), part[rr]);
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[rr] += part[rr];
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) s[(p * Q + k) * R + rr] = acc[rr];
  }
}

// o[c] += B[quad c] o[parent c]   (children cf .. cf+cc-1)
template <typename T, int R>
__global__ void __launch_bounds__(kLvlThreads) downward_kernel(
    const T* __restrict__ BT, const int32_t* __restrict__ quad,
    const int64_t* __restrict__ parent, int64_t cf, int64_t cc, T* o, int Q) {
  const int NG = kLvlThreads / Q;
  const int g = threadIdx.x / Q, k = threadIdx.x % Q;
  if (g >= NG) return;
  const int64_t QQ = int64_t(Q) * Q;
  for (int64_t ci = int64_t(blockIdx.x) * NG + g; ci < cc; ci += int64_t(gridDim.x) * NG) {
    const int64_t c = cf + ci;
    const T* M = BT + quad[c] * QQ;
    const T* ov = o + parent[c] * Q * R;
    T acc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) acc[rr] = T(0);
    for (int j = 0; j < Q; ++j) {
      const T mv = __ldg(M + j * Q + k);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[rr] = fma(mv, ov[j * R + rr], acc[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) o[(c * Q + k) * R + rr] += acc[rr];
  }
}

// ----------------------------------------------------------------------------
// Translation: one CTA per tile of <= kTransTile consecutive same-level
// targets.  The tile's (target, source) pairs are grouped in runs that share
// one D matrix (same level and offset; operators.py:225-239 caches D by
// exactly that key).  Each D is bulk-copied once per tile into a double-
// buffered smem slot and applied to every pair of its run; a run touches
// each target at most once, so the pairs of a run accumulate into the tile's
// smem o buffer without races.
// ----------------------------------------------------------------------------
constexpr int kTransTile = 32;
constexpr int kTransThreads = 256;

struct TransTile {
  int32_t first_target;
  int32_t n_targets;
  int32_t run_begin;
  int32_t run_end;
};
struct TransRun {
  int32_t dtab;
  int32_t pair_begin;
  int32_t pair_end;
  int32_t pad;
};
struct TransPair {
  int32_t tgt;  // local target index in the tile
  int32_t src;  // source group id
};

template <typename T>
struct TransArgs {
  const TransTile* tiles;
  const TransRun* runs;
  const TransPair* pairs;
  const T* DT;        // transposed D table, stride dstride elements
  int64_t dstride;
  const T* s;
  T* o;
  int Q;
};

template <typename T, int R>
size_t trans_smem_bytes(int Q, int64_t dstride) {
  size_t oacc = (size_t(kTransTile) * Q * R * sizeof(T) + 127) & ~size_t(127);
  return oacc + 2 * size_t(dstride) * sizeof(T) + 2 * sizeof(uint64_t) + 16;
}

template <typename T, int R>
__global__ void __launch_bounds__(kTransThreads) translate_kernel(const TransArgs<T> a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int Q = a.Q;
  const TransTile tile = a.tiles[blockIdx.x];
  T* oacc = reinterpret_cast<T*>(smem);
  const size_t oacc_bytes = (size_t(kTransTile) * Q * R * sizeof(T) + 127) & ~size_t(127);
  T* Ds0 = reinterpret_cast<T*>(smem + oacc_bytes);
  T* Ds1 = Ds0 + a.dstride;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Ds1 + a.dstride);
  const uint32_t dbytes = uint32_t(a.dstride * sizeof(T));

  const int n_out = tile.n_targets * Q * R;
  for (int i = threadIdx.x; i < n_out; i += kTransThreads) oacc[i] = T(0);
  const int nruns = tile.run_end - tile.run_begin;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    if (nruns > 0) {
      mbar_arrive_expect_tx(&bar[0], dbytes);
      bulk_g2s(Ds0, a.DT + int64_t(a.runs[tile.run_begin].dtab) * a.dstride, dbytes, &bar[0]);
    }
  }
  __syncthreads();
  const int NG = kTransThreads / Q;
  const int g = threadIdx.x / Q, k = threadIdx.x % Q;
  for (int r = 0; r < nruns; ++r) {
    const int buf = r & 1;
    if (threadIdx.x == 0 && r + 1 < nruns) {
      mbar_arrive_expect_tx(&bar[buf ^ 1], dbytes);
      bulk_g2s(buf ? Ds0 : Ds1,
               a.DT + int64_t(a.runs[tile.run_begin + r + 1].dtab) * a.dstride, dbytes,
               &bar[buf ^ 1]);
    }
    mbar_wait(&bar[buf], uint32_t(r >> 1) & 1u);
    const TransRun run = a.runs[tile.run_begin + r];
    const T* Dm = buf ? Ds1 : Ds0;
    if (g < NG) {
      for (int p = run.pair_begin + g; p < run.pair_end; p += NG) {
        const TransPair pr = a.pairs[p];
        const T* sv = a.s + int64_t(pr.src) * Q * R;
        T acc[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = T(0);
#pragma unroll 4
        for (int j = 0; j < Q; ++j) {
          const T d = Dm[j * Q + k];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc[rr] = fma(d, __ldg(sv + j * R + rr), acc[rr]);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) oacc[(pr.tgt * Q + k) * R + rr] += acc[rr];
      }
    }
    __syncthreads();
  }
  T* dst = a.o + int64_t(tile.first_target) * Q * R;
  for (int i = threadIdx.x; i < n_out; i += kTransThreads) dst[i] = oacc[i];
}

}  // namespace nesa
