// nesa_plan.cu -- plan construction, device operator assembly, CUDA-graph
// launch and the C ABI declared in include/nesa_b200.h.
//
// The plan is the GPU form of the reference's Tree + OperatorSet +
// StageVectors (quadtree.py:71-93, operators.py:158-253, fastmvp.py:24-59):
// every per-task gemv of fastmvp.mvp becomes a row of a batched launch, the
// handle generations of runtime.py:137-161 become the edges of a CUDA graph
// (gather -> {near | radiation -> upward levels -> translation -> downward
// levels} -> reception), and the near-field branch runs concurrently with the
// far-field chain (the paper's near/far task mixing).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <utility>
#include <map>
#include <string>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "../../include/nesa_b200.h"
#include "nesa_kernels.cuh"
constexpr int64_t kLevelTcMin = 2048;  // groups of a level for the tensor-core level kernels

using namespace nesa;

namespace {

thread_local std::string g_last_error;

struct NesaError : std::runtime_error {
  int code;
  NesaError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(expr)                                                                \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      throw NesaError(_e == cudaErrorMemoryAllocation ? NESA_ERR_OOM : NESA_ERR_CUDA, \
                      std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

void require(bool ok, const std::string& msg) {
  if (!ok) throw NesaError(NESA_ERR_INVALID, msg);
}

// NCCL, resolved at run time (dlopen "libnccl.so.2": the copy the process
// already has -- e.g. torch's -- or the system one), so the library has no
// link-time dependency and single-GPU use never touches it.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw NesaError(NESA_ERR_UNSUPPORTED, std::string("libnccl.so.2 not found: ") + dlerror());
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) throw NesaError(NESA_ERR_UNSUPPORTED, std::string("NCCL symbol missing: ") + name);
      return f;
    };
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
    api.h = h;
  }
  return api;
}

#define NCCL_OK(expr)                                                                           \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess)                                                                      \
      throw NesaError(NESA_ERR_CUDA, std::string(#expr) + ": " + nccl().errorString(_r));       \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool own = true;  // false: a view into another buffer
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), own(o.own) {
    o.p = nullptr;
    o.n = 0;
  }
  ~DevBuf() {
    if (p && own) cudaFree(p);
  }
  void view(T* ptr, size_t count) {
    if (p && own) cudaFree(p);
    p = ptr;
    n = count;
    own = false;
  }
  void alloc(size_t count, size_t pad_bytes = 0) {
    if (p && own) cudaFree(p);
    own = true;
    p = nullptr;
    n = count;
    size_t bytes = count * sizeof(T) + pad_bytes;
    if (bytes == 0) bytes = 16;
    CUDA_OK(cudaMalloc(&p, bytes));
    CUDA_OK(cudaMemset(p, 0, bytes));
  }
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty()) CUDA_OK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
};

// Host description of one batched block-GEMV launch.
struct HostBlockSet {
  std::vector<BlockItem> items;
  std::vector<BlockSeg> segs;
  std::vector<ChunkRec> recs;
  std::vector<int32_t> cta_ptr;
  int64_t blob_elems = 0;
  int64_t entries = 0;
};

struct DevBlockSet {
  DevBuf<unsigned char> blob;  // T elements
  DevBuf<BlockItem> items;
  DevBuf<BlockSeg> segs;
  DevBuf<ChunkRec> recs;
  DevBuf<int32_t> cta_ptr;
  int grid = 0;
  int64_t n_items = 0;
  int64_t entries = 0;
};

// Split items into bulk-copy chunks and give each CTA a contiguous,
// byte-balanced range of whole items (a target row is never split across
// CTAs, so it has exactly one writer).
void chunk_and_balance(HostBlockSet& hs, size_t elem_bytes, int max_grid, int ab = kABytes,
                       int nct = kNCT) {
  hs.recs.clear();
  std::vector<int64_t> item_first_chunk(hs.items.size() + 1);
  std::vector<double> item_bytes(hs.items.size());
  for (size_t i = 0; i < hs.items.size(); ++i) {
    const BlockItem& it = hs.items[i];
    item_first_chunk[i] = int64_t(hs.recs.size());
    int per = int(std::min<int64_t>(ab / 64, ab / (int64_t(it.ld) * int64_t(elem_bytes))));
    per = std::max(per, 1);
    const int RQ = it.ld / 4;
    const int seg_end = it.seg_begin + it.seg_count;
    int c = 0;
    while (c < it.n) {
      ChunkRec r{};
      r.src_off = it.a_off + int64_t(c) * it.ld;
      r.m = it.m;
      r.ld = it.ld;
      r.y_row0 = it.y_row0;
      r.magic = RQ == 1 ? 0u : uint32_t(((uint64_t(1) << 32) + RQ - 1) / RQ);
      r.CL = nct / RQ;
      int ce = std::min(it.n, c + per);
      // segments overlapping [c, ce); cut the chunk if more than kRecSegs
      int ns = 0;
      for (int sg = it.seg_begin; sg < seg_end; ++sg) {
        const int s0 = hs.segs[sg].col0;
        const int s1 = sg + 1 < seg_end ? hs.segs[sg + 1].col0 : it.n;
        const int lo = std::max(s0, c), hi = std::min(s1, ce);
        if (lo >= hi) continue;
        if (ns == kRecSegs) {
          ce = lo;
          break;
        }
        r.seg[2 * ns] = hs.segs[sg].x_row0 + (lo - s0);
        r.seg[2 * ns + 1] = lo - c;
        ++ns;
      }
      r.nseg = ns;
      r.ncols = ce - c;
      r.flags = (c == 0 ? 1 : 0) | (ce == it.n ? 2 : 0);
      hs.recs.push_back(r);
      c = ce;
    }
    item_bytes[i] = double(it.ld) * it.n * elem_bytes + 256.0;  // + per-item overhead
  }
  item_first_chunk[hs.items.size()] = int64_t(hs.recs.size());
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(max_grid, int64_t(hs.items.size()))));
  double total = 0;
  for (double b : item_bytes) total += b;
  hs.cta_ptr.assign(grid + 1, 0);
  size_t it = 0;
  double acc = 0;
  for (int c = 0; c < grid; ++c) {
    hs.cta_ptr[c] = int32_t(item_first_chunk[it]);
    const double target = total * double(c + 1) / grid;
    while (it < hs.items.size() && c < grid - 1) {
      const double nb = acc + item_bytes[it];
      // stop before an item that overshoots the target by more than it undershoots
      if (nb > target && (nb - target) > (target - acc) && int64_t(hs.cta_ptr[c]) != item_first_chunk[it])
        break;
      acc = nb;
      ++it;
      if (acc >= target) break;
    }
  }
  hs.cta_ptr[grid] = int32_t(hs.recs.size());
}

template <typename T>
void upload_blockset(DevBlockSet& d, const HostBlockSet& h) {
  d.blob.alloc(size_t(h.blob_elems) * sizeof(T), 256);
  d.items.upload(h.items);
  d.segs.upload(h.segs);
  d.recs.upload(h.recs);
  d.cta_ptr.upload(h.cta_ptr);
  d.grid = int(h.cta_ptr.size()) - 1;
  d.n_items = int64_t(h.items.size());
  d.entries = h.entries;
}

// ---------------------------------------------------------------------------
// Device assembly of near / V / U blocks (operators.py:107-155 on the GPU).
// Entries are evaluated in float64 exactly as linalg.kernel_matrix does:
// d2 = (t - s)_x^2 + (t - s)_y^2 without contraction, -0.5 * log(d2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double kernel_entry(double tx, double ty, double sx, double sy) {
  const double dx = __dsub_rn(tx, sx), dy = __dsub_rn(ty, sy);
  const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  return -0.5 * log(d2);
}

template <typename T>
__global__ void assemble_near_kernel(const BlockItem* items, const BlockSeg* segs,
                                     const double* pts, T* blob) {
  const BlockItem it = items[blockIdx.x];
  for (int sg = it.seg_begin; sg < it.seg_begin + it.seg_count; ++sg) {
    const BlockSeg S = segs[sg];
    const int scol1 = (sg + 1 < it.seg_begin + it.seg_count) ? segs[sg + 1].col0 : it.n;
    const int64_t cnt = int64_t(scol1 - S.col0) * it.m;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int c = S.col0 + int(e / it.m), r = int(e % it.m);
      const int64_t i = it.y_row0 + r, j = S.x_row0 + (c - S.col0);
      const double v = (i == j) ? 0.0
                                : kernel_entry(pts[2 * i], pts[2 * i + 1], pts[2 * j], pts[2 * j + 1]);
      blob[it.a_off + int64_t(c) * it.ld + r] = T(v);
    }
  }
}

// Track B near blocks, row-split complex (NESA_PLAN_HELMHOLTZ_NEAR): item
// rows 2r / 2r+1 = Re / Im of G(x_i, x_j) = exp(-j k r) / (4 pi r) for the
// complex target row r (point i = y_row0 + r) and source column c (point j
// from the item's segments); zero for i == j (helmholtz.helmholtz_matrix).
template <typename T>
__global__ void assemble_near_helm_kernel(const BlockItem* items, const BlockSeg* segs,
                                          const double* pts3, double k, T* blob) {
  const BlockItem it = items[blockIdx.x];
  const int mc = it.m / 2;  // complex rows
  const double inv4pi = 1.0 / (4.0 * 3.14159265358979323846);
  for (int sg = it.seg_begin; sg < it.seg_begin + it.seg_count; ++sg) {
    const BlockSeg S = segs[sg];
    const int scol1 = (sg + 1 < it.seg_begin + it.seg_count) ? segs[sg + 1].col0 : it.n;
    const int64_t cnt = int64_t(scol1 - S.col0) * mc;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int c = S.col0 + int(e / mc), r = int(e % mc);
      const int64_t i = it.y_row0 + r, j = S.x_row0 + (c - S.col0);
      double re = 0.0, im = 0.0;
      if (i != j) {
        const double dx = __dsub_rn(pts3[3 * i], pts3[3 * j]);
        const double dy = __dsub_rn(pts3[3 * i + 1], pts3[3 * j + 1]);
        const double dz = __dsub_rn(pts3[3 * i + 2], pts3[3 * j + 2]);
        const double d = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        double sn, cs;
        sincos(k * d, &sn, &cs);
        const double a = inv4pi / d;
        re = cs * a;
        im = -sn * a;
      }
      blob[it.a_off + int64_t(c) * it.ld + 2 * r] = T(re);
      blob[it.a_off + int64_t(c) * it.ld + 2 * r + 1] = T(im);
    }
  }
}

// V_b = fit @ K(out_check_b, pts_b): item m = Q rows, n = n_b columns.
template <typename T>
__global__ void assemble_V_kernel(const BlockItem* items, const int64_t* item_leaf,
                                  const double* pts, const double* center, const double* r_check,
                                  const double* fit, const double* ccos, const double* csin,
                                  int Q, int n_check, T* blob) {
  extern __shared__ double kc[];  // n_check
  const BlockItem it = items[blockIdx.x];
  const int64_t leaf = item_leaf[blockIdx.x];
  const double cx = center[2 * leaf], cy = center[2 * leaf + 1], rc = r_check[leaf];
  for (int c = 0; c < it.n; ++c) {
    // column c is point (segment x_row0 + c); V items carry one segment.
    const int64_t j = int64_t(it.x0) + c;
    const double px = pts[2 * j], py = pts[2 * j + 1];
    __syncthreads();
    for (int i = threadIdx.x; i < n_check; i += blockDim.x) {
      const double chx = __dadd_rn(cx, __dmul_rn(rc, ccos[i]));
      const double chy = __dadd_rn(cy, __dmul_rn(rc, csin[i]));
      kc[i] = kernel_entry(chx, chy, px, py);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < Q; k += blockDim.x) {
      double acc = 0.0;
      for (int i = 0; i < n_check; ++i) acc = fma(fit[int64_t(k) * n_check + i], kc[i], acc);
      blob[it.a_off + int64_t(c) * it.ld + k] = T(acc);
    }
  }
}

// U_a = K(pts_a, in_aux_a): item m = rows of the panel, n = Q columns.
template <typename T>
__global__ void assemble_U_kernel(const BlockItem* items, const int64_t* item_leaf,
                                  const double* pts, const double* center, const double* r_aux,
                                  const double* acos_, const double* asin_, T* blob) {
  const BlockItem it = items[blockIdx.x];
  const int64_t leaf = item_leaf[blockIdx.x];
  const double cx = center[2 * leaf], cy = center[2 * leaf + 1], ra = r_aux[leaf];
  const int64_t cnt = int64_t(it.m) * it.n;
  for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
    const int k = int(e / it.m), r = int(e % it.m);
    const int64_t i = it.y_row0 + r;
    const double ax = __dadd_rn(cx, __dmul_rn(ra, acos_[k]));
    const double ay = __dadd_rn(cy, __dmul_rn(ra, asin_[k]));
    blob[it.a_off + int64_t(k) * it.ld + r] = T(kernel_entry(pts[2 * i], pts[2 * i + 1], ax, ay));
  }
}

template <typename T>
__global__ void convert_kernel(const double* src, T* dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = T(src[i]);
}

}  // namespace

// ---------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------
constexpr int kTraceSlots = 64;

struct nesa_plan {
  int device = 0;
  int dtype = NESA_F64;
  size_t esz = 8;
  int Q = 0, n_check = 0, l0 = 0, L = 0;
  int64_t N = 0, NL = 0, G = 0;
  int64_t leaf_begin = 0, leaf_end = 0;  // local target leaves
  bool far_only = false;                 // NESA_PLAN_FAR_ONLY: no near operator at all
  bool cnear = false;                    // NESA_PLAN_COMPLEX_NEAR: row-split complex near blob
  int nkind = 4;                         // child kinds per level (NESA_PLAN_OCTREE: 8)
  int64_t pt_begin = 0, pt_end = 0;      // local tree-order point range
  int n_sm = 148;

  std::vector<int64_t> lvl_first, lvl_count;  // global, index level - l0
  std::vector<int64_t> loc_first, loc_count;  // local (ancestors of local leaves)

  DevBuf<int64_t> perm;        // [N]
  DevBuf<int32_t> iperm;       // [N] original index -> tree index
  DevBuf<int32_t> quad;        // [G]
  DevBuf<int64_t> parent;      // [G]
  DevBuf<int64_t> child_first; // [G]
  DevBuf<int32_t> n_child;     // [G]
  DevBuf<unsigned char> CT, BT, DT;  // T tables (transposed)
  int64_t n_dtab = 0, d_refs = 0;

  DevBlockSet nearset, Vset, Uset;
  // many right-hand sides (float32 with tensor cores): the near field as one
  // tcgen05 GEMM over up to 128 columns (near_tc_kernel); its canonical tf32
  // blob is packed from the near blob on first use
  bool near_tc = false;                     // float32 and NESA_TC != 0 (any Q)
  DevBuf<NearTcItem> ntc_items;
  DevBuf<int32_t> ntc_src;                  // slab columns -> original point index
  DevBuf<float> ntc_blob;
  int64_t ntc_floats = 0;
  int ntc_n = 0;

  // translation: entries grouped by unique D (see tgemm_kernel)
  DevBuf<TUnit> tunits;
  DevBuf<TEnt> tents;
  int n_tunits = 0;
  DevBuf<int64_t> int_ptr;  // [G+1] interaction CSR (Y rows of each target)
  int64_t nnz = 0;
  size_t mbytes = 0;                       // padded matrix stride (bytes)
  DevBuf<int32_t> red_ids;                  // local groups (translation-sum targets)
  int64_t n_red = 0;
  std::vector<DevBuf<int32_t>> down_order;  // per level (index lv-l0): children by quadrant
  std::vector<DevBuf<int32_t>> down_par;    // parents of down_order
  std::vector<DevBuf<int2>> down_child;     // local child range of down_order entries
  // tensor-core level transfers (float32, Q = 64; level_tc_kernel)
  bool level_tc = false;
  DevBuf<float> CTC, BTC;                   // [(L-l0) * 4][hi | lo][4096] canonical tf32 C / B
  std::vector<DevBuf<int4>> lvl_tiles;      // [(lv - l0) * 3 + r]: quadrant-pure tiles, R = 1 << r
  // fused coarse levels l0+1 .. fused_lf (one kernel per pass; see
  // nesa_kernels.cuh "Fused coarse levels"); fused_lf == l0: off
  bool fused = true;
  int fused_lf = 0;
  DevBuf<int2> uchild;                      // [G] local children (first, count)
  DevBuf<int32_t> fused_anc;                // [count(lf)][lf - l0 - 1] ancestors
  DevBuf<int> fused_cnt, fused_state;       // [G] arrival counters / done flags
  DevBuf<int4> fused_chain_up, fused_chain_down;  // packed per-CTA chain records (see build)
  DevBuf<int32_t> fused_own;                // [count(lf)] ancestors owned by each level-lf group's CTA
  DevBuf<int> fused_ticket;                 // [2] fused_down start-order counter
  int64_t wide_level = 1024;                // per-level (warp-tiled / tensor-core) kernels from this size
                                            // (NESA_WIDE_LEVEL: tests force them on small trees)
  bool u_mf = false;                        // matrix-free reception (float32 plans)
  DevBuf<float2> mf_prel;                   // [N] point - leaf center (float32)
  DevBuf<int64_t> gstart, gstop;            // [NL] leaf point ranges
  DevBuf<float> mf_leaf_r;                  // [NL] rho_in_aux * half side (float32)
  // radiation through outgoing moments (float32 plans from geometry)
  bool v_mom = false;
  int v_nm = 0;                             // moments m = 0 .. v_nm - 1
  int u_nt = 0;                             // reception terms m = 1 .. u_nt
  DevBuf<float2> mom_A;                     // [v_nm][Q]: row 0 = (F_k, 0), row m = A_km
  bool rad_tc = false;                      // moment map on the tensor cores (radiation_tc_kernel)
  DevBuf<float> ATC;                        // [hi | lo][64 x 80] canonical tf32 A^ (K = 80)
  DevBuf<int32_t> rad_order;                // local leaves by descending point count
  DevBuf<float2> exp_E;                     // [Q][u_nt + 1]: 1, (1/m) e^{-i m theta_k}
  DevBuf<double2> mf_prel64, exp_E64;       // float64 plans: the same inputs in float64
  DevBuf<double> mf_leaf_r64;
  // many right-hand sides: the far field as batched GEMMs over up to 128
  // columns (wgemm_kernel; plans with stored V and U)
  struct WStage {
    int64_t begin, end;  // item range
    int ysel;            // 0 s, 1 o, 2 phi (scatter)
  };
  bool wide_far = false;
  DevBuf<WItem> w_items;
  DevBuf<WTerm> w_terms;
  std::vector<WStage> w_stages;
  DevBuf<unsigned char> w_s, w_o;  // G x Q x 128 (allocated on first use)
  cudaEvent_t w_ev_fork = nullptr, w_ev_near = nullptr;
  DevBuf<float> mf_leaf_rc;                 // [NL] rho_out_check * half side (float32)
  bool tc = true;                           // translation on the tensor cores (float32, Q = 64;
                                            // NESA_TC=0 selects the FFMA kernel, as float64 plans)
  DevBuf<float> DTC;                        // [n_dtab + 1][hi | lo][64 x 64] canonical tf32 D (+ zero)
  DevBuf<TUnit> mom_units;                  // reception coefficient GEMM: 32 leaves per unit
  DevBuf<TEnt> mom_ents;
  int n_mom_units = 0;
  bool beta_tc = false;                     // reception coefficients by tgemm_tc2 (E^ o)
  bool beta_fused = false;                  // leaf down + beta in one kernel (reception separate)
  DevBuf<float> ET;                         // [64][64] E^ transposed for the warp-tiled GEMM
  DevBuf<float> ETC;                        // [hi | lo][64 x 64] canonical tf32 E^
  DevBuf<unsigned char> beta;               // [NL][64][R] reception coefficients

  // multi-GPU plan (nesa_plan_create_dist): the halo exchange of partial
  // source amplitudes inside the product graph (pack -> ncclAllGather ->
  // combine), so a distributed product is one graph launch per rank
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t x_n_export = 0, x_max_export = 1, x_n_import = 0;
  int x_max_contrib = 1;
  DevBuf<int64_t> x_export, x_import, x_contrib;
  DevBuf<unsigned char> x_send, x_recv;      // [max_export][Q R] / [nranks * max_export][Q R]

  // workspace for R real columns
  int ws_R = 0;
  uint64_t ws_gen = 0;                      // bumped when the workspace is reallocated
  DevBuf<unsigned char> qt, phin, s, o, Y, Tup;
  DevBuf<unsigned char> farws;              // s | Tup | o, contiguous

  cudaStream_t s0 = nullptr, s1 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_tx = nullptr;
  cudaStream_t s2 = nullptr, s3 = nullptr;   // fine-level translation branch, leaf-level translation sums
  int split_lv = 0;                          // levels >= split_lv: translated on s2
  int n_tunits_fine = 0;                     // units [0, n_tunits_fine) are fine levels
  // per level (index lv - l0): translation units and translation-sum groups,
  // so each fine level is translated as soon as its own s is final
  std::vector<int> tunit_lv_begin, tunit_lv_end;
  std::vector<int64_t> red_lv_begin, red_lv_end;
  std::vector<cudaEvent_t> ev_s_lv, ev_t_lv;
  int64_t n_red_fine = 0;                    // red_ids [0, n_red_fine) are fine levels

  // One captured graph per (R, flags, stage, ldv).  The caller's q / phi
  // pointers appear only in the gather and the reception / scatter nodes;
  // a launch with other buffers patches those nodes in the instantiated
  // graph (cudaGraphExecKernelNodeSetParams) instead of capturing again.
  struct GraphKey {
    int R;
    uint32_t flags;
    int stage;
    int ldv;
    bool operator<(const GraphKey& o) const {
      return std::tie(R, flags, stage, ldv) < std::tie(o.R, o.flags, o.stage, o.ldv);
    }
  };
  struct IoPatch {
    cudaGraphNode_t node = nullptr;  // node of the captured graph (addresses the exec's copy)
    std::function<cudaError_t(cudaGraphExec_t, cudaGraphNode_t, const void*, void*)> apply;
  };
  struct GraphEntry {
    cudaGraph_t graph = nullptr;  // kept alive: its nodes address the exec's nodes
    cudaGraphExec_t exec = nullptr;
    std::vector<std::pair<cudaGraphNode_t, int>> ev_nodes;  // node, slot (stage*2+end)
    std::vector<IoPatch> io;       // nodes that read q / write phi
    const void* q = nullptr;       // buffers the exec currently addresses
    void* phi = nullptr;
    uint64_t gen = 0;              // workspace generation it was captured against
  };
  std::map<GraphKey, GraphEntry> graphs;
  std::vector<IoPatch>* capturing_io = nullptr;  // set while a graph is being captured
  int64_t graph_captures = 0;                    // diagnostics (NESA_STAT_GRAPH_CAPTURES)
  int kernels_per_matvec = 0;

  // profiling: per matvec a set of 2*NESA_N_STAGES events
  std::vector<std::vector<cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  cudaEvent_t cap_events[2 * NESA_N_STAGES + kTraceSlots] = {};
  bool trace = false;                       // NESA_TRACE: an event after every kernel
  std::vector<std::string> trace_names;

  void drop_graphs() {
    for (auto& kv : graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
    }
    graphs.clear();
  }

  ~nesa_plan() {
    cudaSetDevice(device);
    drop_graphs();
    for (auto& v : prof_events)
      for (auto e : v) cudaEventDestroy(e);
    for (auto e : cap_events)
      if (e) cudaEventDestroy(e);
    if (w_ev_fork) cudaEventDestroy(w_ev_fork);
    for (auto e : ev_s_lv) cudaEventDestroy(e);
    for (auto e : ev_t_lv) cudaEventDestroy(e);
    if (w_ev_near) cudaEventDestroy(w_ev_near);
    if (s2) cudaStreamDestroy(s2);
    if (s3) cudaStreamDestroy(s3);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_tx) cudaEventDestroy(ev_tx);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s0) cudaStreamDestroy(s0);
    if (s1) cudaStreamDestroy(s1);
  }
};

namespace {

// round to tf32 (nearest, ties away: cvt.rna.tf32.f32 on the device)
float tf32_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

// n_mats row-major 64 x 64 float64 matrices (y = M x) -> the canonical no-swizzle
// K-major tf32 layout of a tcgen05 B operand, hi then lo per matrix (see
// tgemm_tc2_kernel), plus `extra` zero matrices
std::vector<float> canon_tf32(const double* M, int64_t n_mats, int64_t extra = 0) {
  std::vector<float> h(size_t(n_mats + extra) * 8192, 0.f);
  for (int64_t t = 0; t < n_mats; ++t)
    for (int nn = 0; nn < 64; ++nn)
      for (int k = 0; k < 64; ++k) {
        const float x = float(M[(t * 64 + nn) * 64 + k]);
        const float hi = tf32_host(x), lo = tf32_host(x - hi);
        const size_t off = size_t(nn / 8) * 512 + size_t(k / 4) * 32 + size_t(nn % 8) * 4 + (k % 4);
        h[size_t(t) * 8192 + off] = hi;
        h[size_t(t) * 8192 + 4096 + off] = lo;
      }
  return h;
}

// Q x Q float64 row-major matrices -> padded transposed device layout
// MT[j * Qp + k] = M[k][j], matrix stride mat_bytes(Q) (see nesa_kernels.cuh).
template <typename T>
void upload_table_T(DevBuf<unsigned char>& dst, const double* src, int64_t n_mats, int Q) {
  const int Qp = (Q + 3) / 4 * 4;
  const size_t stride = mat_bytes(Q, sizeof(T)) / sizeof(T);
  std::vector<T> h(size_t(std::max<int64_t>(n_mats, 1)) * stride, T(0));
  for (int64_t m = 0; m < n_mats; ++m)
    for (int k = 0; k < Q; ++k)
      for (int j = 0; j < Q; ++j) h[m * stride + size_t(j) * Qp + k] = T(src[(m * Q + k) * Q + j]);
  dst.alloc(h.size() * sizeof(T));
  CUDA_OK(cudaMemcpy(dst.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// Host blob (reference layout, float64) -> device layout (type T, paneled).
template <typename T>
void upload_host_blob(DevBlockSet& d, const HostBlockSet& h, const double* src,
                      const std::vector<int64_t>& item_src_off,
                      const std::vector<int32_t>& item_src_rows,
                      const std::vector<int32_t>& item_row0) {
  std::vector<T> stage(size_t(h.blob_elems));
  for (size_t i = 0; i < h.items.size(); ++i) {
    const BlockItem& it = h.items[i];
    const int64_t so = item_src_off[i];
    const int32_t ld = item_src_rows[i], r0 = item_row0[i];
    for (int c = 0; c < it.n; ++c)
      for (int r = 0; r < it.m; ++r)
        stage[it.a_off + int64_t(c) * it.ld + r] = T(src[so + int64_t(c) * ld + r0 + r]);
  }
  if (!stage.empty())
    CUDA_OK(cudaMemcpy(d.blob.p, stage.data(), stage.size() * sizeof(T), cudaMemcpyHostToDevice));
}

template <typename T>
void build_plan_T(nesa_plan* P, const nesa_plan_desc* d) {
  const int Q = P->Q;
  const int64_t NL = P->NL, G = P->G;
  const size_t es = sizeof(T);
  const int64_t lb = P->leaf_begin, le = P->leaf_end;

  // ---- tree arrays
  {
    std::vector<int64_t> perm(d->perm, d->perm + P->N);  // full: near halo columns
    for (auto v : perm) require(v >= 0 && v < P->N, "perm out of range");
    P->perm.upload(perm);
    {
      std::vector<int32_t> iperm(P->N, -1);
      for (int64_t i = 0; i < P->N; ++i) {
        require(iperm[perm[i]] < 0, "perm is not a permutation");
        iperm[perm[i]] = int32_t(i);
      }
      P->iperm.upload(iperm);
    }
    std::vector<int32_t> quad(d->quad, d->quad + G);
    P->quad.upload(quad);
    std::vector<int64_t> parent(d->parent, d->parent + G);
    P->parent.upload(parent);
    std::vector<int64_t> cf(G, -1);
    std::vector<int32_t> nc(G, 0);
    for (int64_t g = G - 1; g >= 0; --g) {
      const int64_t p = parent[g];
      if (p >= 0) {
        require(p < G && p > g, "parent ids must follow child ids");
        cf[p] = g;  // smallest child id wins (iterating downward)
        nc[p] += 1;
      }
    }
    P->child_first.upload(cf);
    P->n_child.upload(nc);
  }

  // ---- local (ancestor) level ranges
  const int nlev = P->L - P->l0 + 1;
  P->loc_first.assign(nlev, 0);
  P->loc_count.assign(nlev, 0);
  {
    int64_t lo = lb, hi = le - 1;  // ids at level L
    for (int lv = P->L; lv >= P->l0; --lv) {
      const int li = lv - P->l0;
      if (le > lb) {
        P->loc_first[li] = lo;
        P->loc_count[li] = hi - lo + 1;
        if (lv > P->l0) {
          lo = d->parent[lo];
          hi = d->parent[hi];
        }
      }
    }
  }

  // the many-RHS near field on the tensor cores works for any Q (real operators)
  P->near_tc = std::is_same<T, float>::value && P->tc && !P->cnear;
  // ---- tables
  const int64_t nlt = P->L - P->l0;
  P->mbytes = mat_bytes(Q, sizeof(T));
  if (nlt > 0) {
    upload_table_T<T>(P->CT, d->C, nlt * P->nkind, Q);
    upload_table_T<T>(P->BT, d->B, nlt * P->nkind, Q);
  }
  P->n_dtab = d->n_dtab;
  upload_table_T<T>(P->DT, d->D, d->n_dtab, Q);
  // tensor-core translation (float32, Q = 64): D split into tf32 hi / lo in
  // the canonical K-major core-matrix layout (see tgemm_tc_kernel)
  if (std::is_same<T, float>::value && Q == 64 && P->tc && d->n_dtab > 0) {
    // + one zero matrix at index n_dtab
    P->DTC.upload(canon_tf32(d->D, d->n_dtab, 1));
  } else {
    P->tc = false;
  }
  require(fused_smem_bytes<T>(Q, 4, 2, 64) <= 200 * 1024 && tgemm_smem_bytes<T, 4>(Q) <= 200 * 1024,
          "Q too large for the far-field kernels");
  // per-level gather tables (see nesa_kernels.cuh "Level transfers")
  P->down_order.resize(nlev);
  P->lvl_tiles.resize(size_t(nlev) * 3);
  P->down_par.resize(nlev);
  P->down_child.resize(nlev);
  for (int lv = P->l0 + 1; lv <= P->L; ++lv) {
    const int li = lv - P->l0;
    const int64_t cf = P->loc_first[li], cn = P->loc_count[li];
    const int64_t pf = P->loc_first[li - 1], pn = P->loc_count[li - 1];
    for (int64_t c = cf; c < cf + cn; ++c) {
      const int64_t pl = d->parent[c] - pf;
      require(pl >= 0 && pl < pn, "local child with a non-local parent");
    }
    std::vector<int32_t> ord(static_cast<size_t>(cn)), par(static_cast<size_t>(cn));
    for (int64_t i = 0; i < cn; ++i) ord[i] = int32_t(cf + i);
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int32_t x, int32_t y) { return d->quad[x] < d->quad[y]; });
    for (int64_t i = 0; i < cn; ++i) par[i] = int32_t(d->parent[ord[i]]);
    // quadrant-pure tiles of <= 128 / R groups (level_tc_kernel)
    for (int r = 0; r < 3; ++r) {
      const int ept = 128 >> r;
      std::vector<int4> tl;
      for (int64_t i = 0; i < cn;) {
        const int qd = d->quad[ord[i]];
        int64_t j = i;
        while (j < cn && j - i < ept && d->quad[ord[j]] == qd) ++j;
        tl.push_back(int4{int(i), int(j - i), qd, 0});
        i = j;
      }
      P->lvl_tiles[size_t(li) * 3 + r].upload(tl);
    }
    P->down_order[li].upload(ord);
    P->down_par[li].upload(par);
    // children of each ordered group, clipped to the local range of level lv+1
    std::vector<int2> och(static_cast<size_t>(cn), int2{0, 0});
    if (lv < P->L) {
      std::vector<int64_t> first(static_cast<size_t>(cn), -1), cnt(static_cast<size_t>(cn), 0);
      const int64_t lo = P->loc_first[li + 1], hi = lo + P->loc_count[li + 1];
      std::vector<int64_t> pos(static_cast<size_t>(P->G), -1);
      for (int64_t i = 0; i < cn; ++i) pos[ord[i]] = i;
      for (int64_t k = lo; k < hi; ++k) {
        const int64_t i = pos[d->parent[k]];
        require(i >= 0, "child of a non-local parent");
        if (first[i] < 0) first[i] = k;
        require(k == first[i] + cnt[i], "children must be consecutive ids");
        cnt[i]++;
      }
      for (int64_t i = 0; i < cn; ++i) {
        require(cnt[i] <= P->nkind, "more children than child kinds");
        och[i] = int2{int(std::max<int64_t>(first[i], 0)), int(cnt[i])};
      }
    }
    P->down_child[li].upload(och);
  }
  // fused coarse levels: l0+1 .. fused_lf are the levels the wide kernels do
  // not take (contiguous from the top)
  P->fused_lf = P->l0;
  if (P->fused) {
    for (int lv = P->l0 + 1; lv <= P->L; ++lv) {
      // warp-tiled level kernels: Q = 64, and Q = 128 when their shared
      // memory fits (float32: Track B's embedded complex Q = 64)
      const bool wide_q = Q == 64 || (Q == 128 && LVW<T, 4, 128, kLvlDown>::SMEM <= 220 * 1024);
      const bool wide = wide_q && P->loc_count[lv - P->l0] >= P->wide_level;
      // level l0 + 1 always stays fused: the fused up kernel also forms the
      // top level's sums (no per-level kernel does)
      if ((wide && lv > P->l0 + 1) || P->loc_count[lv - P->l0] == 0) break;
      P->fused_lf = lv;
    }
  }
  P->level_tc = std::is_same<T, float>::value && Q == 64 && P->tc && nlt > 0 && P->fused_lf < P->L;
  if (P->level_tc) {
    P->CTC.upload(canon_tf32(d->C, nlt * 4));
    P->BTC.upload(canon_tf32(d->B, nlt * 4));
  }
  if (P->fused_lf > P->l0) {
    std::vector<int2> uc(static_cast<size_t>(G), int2{0, 0});
    for (int lv = P->l0; lv < P->L; ++lv) {
      const int li = lv - P->l0;
      const int64_t lo = P->loc_first[li + 1], hi = lo + P->loc_count[li + 1];
      for (int64_t k = lo; k < hi; ++k) {
        const int64_t p = d->parent[k];
        if (uc[p].y == 0) uc[p].x = int(k);
        require(k == uc[p].x + uc[p].y, "children must be consecutive ids");
        uc[p].y += 1;
      }
    }
    P->uchild.upload(uc);
    const int li = P->fused_lf - P->l0;
    const int D = P->fused_lf - P->l0 - 1;
    std::vector<int32_t> anc(static_cast<size_t>(std::max<int64_t>(1, P->loc_count[li] * D)), 0);
    for (int64_t i = 0; i < P->loc_count[li]; ++i) {
      int64_t x = P->loc_first[li] + i;
      for (int k = 0; k < D; ++k) {
        x = d->parent[x];
        anc[size_t(i * D + k)] = int32_t(x);
      }
    }
    P->fused_anc.upload(anc);
    // ownership: a coarse group is computed by its first level-lf
    // descendant's CTA, i.e. g owns its ancestors while it is a first child
    std::vector<int32_t> own(static_cast<size_t>(std::max<int64_t>(1, P->loc_count[li])), 0);
    for (int64_t i = 0; i < P->loc_count[li]; ++i) {
      int64_t x = P->loc_first[li] + i;
      int k = 0;
      while (k < D && uc[size_t(d->parent[x])].x == x) {
        x = d->parent[x];
        ++k;
      }
      own[size_t(i)] = k;
    }
    P->fused_own.upload(own);
    // packed chain records, one 16-byte load per step (the kernels fetch a
    // CTA's whole chain in one round trip instead of walking anc -> parent /
    // quad / uchild):
    //   up   [i][k], k = 0 .. D+1: (group at level lf-k, first child, children, quad)
    //   down [i][st], st = 0 .. own: (x = anc[own-1-st] or g, parent x, quad x, own)
    {
      const int64_t cnt = P->loc_count[li];
      std::vector<int4> cup(static_cast<size_t>(std::max<int64_t>(1, cnt * (D + 2))), int4{0, 0, 0, 0});
      std::vector<int4> cdn(static_cast<size_t>(std::max<int64_t>(1, cnt * (D + 1))), int4{0, 0, 0, 0});
      for (int64_t i = 0; i < cnt; ++i) {
        int64_t x = P->loc_first[li] + i;
        for (int k = 0; k <= D + 1; ++k) {
          cup[size_t(i * (D + 2) + k)] = int4{int(x), uc[size_t(x)].x, uc[size_t(x)].y, d->quad[x]};
          if (k <= D) x = d->parent[x];
        }
        const int ow = own[size_t(i)];
        for (int st = 0; st <= ow; ++st) {
          const int a = ow - 1 - st;
          const int64_t y = a >= 0 ? int64_t(anc[size_t(i * D + a)]) : P->loc_first[li] + i;
          cdn[size_t(i * (D + 1) + st)] = int4{int(y), int(d->parent[y]), d->quad[y], ow};
        }
      }
      P->fused_chain_up.upload(cup);
      P->fused_chain_down.upload(cdn);
    }
    P->fused_ticket.alloc(2);
    P->fused_cnt.alloc(size_t(G));    // zero-filled
    P->fused_state.alloc(size_t(G));
  }
  // wide levels (>= split_lv) get their translation on a side stream as soon
  // as their source amplitudes are final (see enqueue_T)
  P->split_lv = P->L + 1;
  for (int lv = P->L; lv >= P->l0 && P->loc_count[lv - P->l0] >= P->wide_level; --lv) P->split_lv = lv;
  // the split point must be a per-level kernel's output: levels inside the
  // fused coarse range are all produced by one kernel at its end
  if (P->fused_lf > P->l0 && P->split_lv <= P->fused_lf) P->split_lv = P->fused_lf + 1;
  {
    std::vector<int32_t> ids;  // fine levels first
    P->red_lv_begin.assign(size_t(nlev), 0);
    P->red_lv_end.assign(size_t(nlev), 0);
    for (int lv = P->L; lv >= P->l0; --lv) {
      const int li = lv - P->l0;
      P->red_lv_begin[size_t(li)] = int64_t(ids.size());
      for (int64_t g = P->loc_first[li]; g < P->loc_first[li] + P->loc_count[li]; ++g)
        ids.push_back(int32_t(g));
      P->red_lv_end[size_t(li)] = int64_t(ids.size());
      if (lv == P->split_lv) P->n_red_fine = int64_t(ids.size());
    }
    P->n_red = int64_t(ids.size());
    P->red_ids.upload(ids);
  }
  // ---- circle expansions (float32 plans from geometry): the number of
  // terms follows the largest |p - c| / r of the plan's points
  {
    const bool geom = d->points_tree && d->leaf_center && d->leaf_r_check && d->leaf_r_inaux &&
                      d->out_fit_leaf && d->check_cos && d->check_sin && d->aux_cos && d->aux_sin;
    const bool f32 = std::is_same<T, float>::value;
    P->v_mom = P->v_mom && f32 && !d->V_blob && geom;
    P->u_mf = P->u_mf && !d->U_blob && geom;
    if (P->v_mom || P->u_mf) {
      double rv = 0, ru = 0;
      for (int64_t a = lb; a < le; ++a) {
        const double cx = d->leaf_center[2 * a], cy = d->leaf_center[2 * a + 1];
        double dm = 0;
        for (int64_t i = d->group_start[a]; i < d->group_stop[a]; ++i)
          dm = std::max(dm, std::hypot(d->points_tree[2 * i] - cx, d->points_tree[2 * i + 1] - cy));
        rv = std::max(rv, dm / d->leaf_r_check[a]);
        ru = std::max(ru, dm / d->leaf_r_inaux[a]);
      }
      // smallest M with rho^(M+1) / (1 - rho) <= tol
      auto terms = [](double rho, double tol) {
        int M = 1;
        while (M < 96 && std::pow(rho, M + 1) / (1.0 - rho) > tol) ++M;
        return M;
      };
      if (rv >= 0.9) P->v_mom = false;  // stored V for (non-quadtree) geometry this far out
      if (ru >= 0.9) P->u_mf = false;
      P->v_nm = terms(rv, 1e-9) + 1;     // V: the fit amplifies truncation; keep a margin
      P->u_nt = terms(ru, f32 ? 1e-8 : 1e-15);  // float64: truncation below its rounding
      if (const char* e = std::getenv("NESA_V_MOMENTS")) P->v_nm = std::max(2, std::atoi(e));
      if (const char* e = std::getenv("NESA_U_TERMS")) P->u_nt = std::max(1, std::atoi(e));
    }
  }
  // ---- near / V / U block sets (local leaves)
  HostBlockSet hn, hv, hu;
  std::vector<int64_t> near_src_off, v_src_off, u_src_off;
  std::vector<int32_t> near_src_rows, near_row0, u_src_rows, u_row0, v_src_rows, v_row0;
  std::vector<int64_t> v_leaf, u_leaf;
  {
    // host-blob offsets of every leaf (reference layout, whole leaves)
    int64_t near_off = 0, v_off = 0, u_off = 0;
    for (int64_t a = 0; a < NL; ++a) {
      const int64_t na = d->group_stop[a] - d->group_start[a];
      require(na >= 1, "empty leaf");
      // complex near (NESA_PLAN_COMPLEX_NEAR): slab columns and x rows
      // count complex points (half the embedded ones); rows stay re / im
      const int64_t cdiv = P->cnear ? 2 : 1;
      int64_t W = 0;
      for (int64_t e = d->nbr_ptr[a]; e < d->nbr_ptr[a + 1]; ++e) {
        const int64_t b = d->nbr_idx[e];
        require(b >= 0 && b < NL, "neighbor id out of range");
        W += (d->group_stop[b] - d->group_start[b]) / cdiv;
      }
      require(W < (int64_t(1) << 31), "near slab too wide");
      if (a >= lb && a < le && !P->far_only) {
        // near item(s): panels of <= kMaxRows rows
        const int32_t seg_begin = int32_t(hn.segs.size());
        int32_t col = 0;
        for (int64_t e = d->nbr_ptr[a]; e < d->nbr_ptr[a + 1]; ++e) {
          const int64_t b = d->nbr_idx[e];
          const int64_t bs = d->group_start[b] / cdiv, bn = (d->group_stop[b] - d->group_start[b]) / cdiv;
          if (int32_t(hn.segs.size()) > seg_begin) {
            BlockSeg& last = hn.segs.back();
            if (int64_t(last.x_row0) + (col - last.col0) == bs) {
              col += int32_t(bn);
              continue;
            }
          }
          hn.segs.push_back(BlockSeg{int32_t(bs), col});
          col += int32_t(bn);
        }
        const int32_t seg_count = int32_t(hn.segs.size()) - seg_begin;
        for (int64_t r0 = 0; r0 < na; r0 += kMaxRows) {
          const int32_t m = int32_t(std::min<int64_t>(kMaxRows, na - r0));
          const int32_t ld = (m + 3) / 4 * 4;
          hn.items.push_back(BlockItem{hn.blob_elems, m, int32_t(W), ld,
                                       int32_t((d->group_start[a] + r0) / cdiv), seg_begin, seg_count, 0, 0});
          near_src_off.push_back(near_off);
          near_src_rows.push_back(int32_t(na));
          near_row0.push_back(int32_t(r0));
          hn.blob_elems += int64_t(ld) * W;
          hn.entries += int64_t(m) * W;
        }
      }
      if (a >= lb && a < le) {
        // V: Q x na, x = qt rows of the leaf, y = s rows of leaf a
        {
          // (complex operators, NESA_PLAN_COMPLEX_NEAR: V row-split like the
          // near blocks -- columns and x rows in complex points, output rows
          // combined pairwise into complex s rows)
          const int32_t sb = int32_t(hv.segs.size());
          hv.segs.push_back(BlockSeg{int32_t(d->group_start[a] / cdiv), 0});
          const int32_t ld = (Q + 3) / 4 * 4;
          const int64_t vn = na / cdiv;
          BlockItem it{hv.blob_elems, Q, int32_t(vn), ld, int32_t(a * Q / cdiv), sb, 1,
                       int32_t(d->group_start[a] / cdiv), 0};
          hv.items.push_back(it);
          v_src_off.push_back(v_off);
          v_src_rows.push_back(Q);
          v_row0.push_back(0);
          v_leaf.push_back(a);
          hv.blob_elems += int64_t(ld) * vn;
          hv.entries += int64_t(Q) * vn;
        }
        // U: na x Q, x = o rows of leaf a, y = phi rows (stored mode only)
        if (!P->u_mf) {
          // (complex operators: U row-split, columns / x rows / output rows
          // in complex units, kModeScatterCplx)
          const int32_t sb = int32_t(hu.segs.size());
          const int32_t uq = int32_t(Q / cdiv);
          hu.segs.push_back(BlockSeg{int32_t(a * uq), 0});
          for (int64_t r0 = 0; r0 < na; r0 += kMaxRows) {
            const int32_t m = int32_t(std::min<int64_t>(kMaxRows, na - r0));
            const int32_t ld = (m + 3) / 4 * 4;
            hu.items.push_back(BlockItem{hu.blob_elems, m, uq, ld,
                                         int32_t((d->group_start[a] + r0) / cdiv), sb, 1, 0, 0});
            u_src_off.push_back(u_off);
            u_src_rows.push_back(int32_t(na));
            u_row0.push_back(int32_t(r0));
            u_leaf.push_back(a);
            hu.blob_elems += int64_t(ld) * uq;
            hu.entries += int64_t(m) * uq;
          }
        }
      }
      near_off += na * W;
      v_off += int64_t(Q) * na / cdiv;
      u_off += na * Q / cdiv;
    }
    require(int64_t(NL) * Q < (int64_t(1) << 31), "too many groups for int32 rows");
  }
  // near field: two persistent CTAs per SM (4 consumer warps, 2 x 24 KB ring);
  // V / U: the generic 8-warp, 3 x 16 KB geometry
  chunk_and_balance(hn, es, kBGPerSM * P->n_sm, kNearABytes, kNearNCW * 32);
  chunk_and_balance(hv, es, kBGPerSM * P->n_sm);
  chunk_and_balance(hu, es, kBGPerSM * P->n_sm);
  upload_blockset<T>(P->nearset, hn);
  if (P->near_tc && !hn.items.empty()) {
    // tensor-core items: <= 128 target rows each, the slab's source points
    // as original indices (the caller's q is read without a gather)
    std::vector<NearTcItem> ti;
    std::vector<int32_t> src;
    int64_t off = 0;
    for (const BlockItem& bi : hn.items) {
      const int32_t src_off = int32_t(src.size());
      require(int64_t(src.size()) + bi.n < (int64_t(1) << 31), "near source table too large");
      for (int sg = bi.seg_begin; sg < bi.seg_begin + bi.seg_count; ++sg) {
        const BlockSeg S = hn.segs[size_t(sg)];
        const int c1 = sg + 1 < bi.seg_begin + bi.seg_count ? hn.segs[size_t(sg) + 1].col0 : bi.n;
        for (int c = S.col0; c < c1; ++c) src.push_back(int32_t(d->perm[S.x_row0 + (c - S.col0)]));
      }
      for (int r0 = 0; r0 < bi.m; r0 += kNearTcMaxN) {
        NearTcItem t{};
        t.b_off = off;
        t.a_off = bi.a_off;
        t.m = std::min(kNearTcMaxN, bi.m - r0);
        t.npad = (t.m + 15) / 16 * 16;
        t.w = bi.n;
        t.kchunks = (bi.n + kNearTcK - 1) / kNearTcK;
        t.y_row0 = bi.y_row0 + r0;
        t.src_off = src_off;
        t.ld = bi.ld;
        t.r0 = r0;
        off += int64_t(t.kchunks) * 2 * t.npad * kNearTcK;
        ti.push_back(t);
      }
    }
    P->ntc_items.upload(ti);
    P->ntc_src.upload(src);
    P->ntc_floats = off;
    P->ntc_n = int(ti.size());
  }
  if (!P->v_mom) upload_blockset<T>(P->Vset, hv);
  upload_blockset<T>(P->Uset, hu);
  // ---- many right-hand sides: work lists of the wide far field
  if (!P->v_mom && !P->u_mf && !P->cnear && lb == 0 && le == NL) {
    const int Qp = (Q + 3) / 4 * 4;
    const int64_t ms = int64_t(mat_bytes(Q, sizeof(T)) / sizeof(T));
    std::vector<WItem> wi;
    std::vector<WTerm> wt;
    // one item per <= kWRows output rows; add(r0) appends the tile's terms
    auto tiles = [&](int64_t y_row, int m_total, const std::function<void(int)>& add) {
      for (int r0 = 0; r0 < m_total; r0 += kWRows) {
        WItem I{};
        I.y_row = y_row + r0;
        I.m = std::min(kWRows, m_total - r0);
        I.t0 = int32_t(wt.size());
        add(r0);
        I.t1 = int32_t(wt.size());
        wi.push_back(I);
      }
    };
    auto stage = [&](int64_t b, int ysel) { P->w_stages.push_back({b, int64_t(wi.size()), ysel}); };
    std::vector<int64_t> cfirst(size_t(G), -1);
    std::vector<int32_t> ccount(size_t(G), 0);
    for (int64_t g = 0; g < G; ++g) {
      const int64_t p = d->parent[g];
      if (p < 0) continue;
      if (cfirst[size_t(p)] < 0) cfirst[size_t(p)] = g;
      ccount[size_t(p)]++;
    }
    // radiation: s_leaf = V_leaf q_leaf (fastmvp.py:158-159)
    int64_t b = int64_t(wi.size());
    for (const BlockItem& v : hv.items)
      tiles(v.y_row0, Q, [&](int r0) {
        wt.push_back(WTerm{v.a_off + r0, int64_t(v.x0), v.ld, v.n, 3, 0});
      });
    stage(b, 0);
    // source transfer, levels L-1 .. l0: s_p = sum_children C_{quad c} s_c (160-162)
    for (int lv = P->L - 1; lv >= P->l0; --lv) {
      b = int64_t(wi.size());
      const int64_t f = P->lvl_first[lv - P->l0], n = P->lvl_count[lv - P->l0];
      for (int64_t p = f; p < f + n; ++p)
        tiles(p * Q, Q, [&](int r0) {
          for (int k = 0; k < ccount[size_t(p)]; ++k) {
            const int64_t c = cfirst[size_t(p)] + k;
            wt.push_back(WTerm{(int64_t(lv - P->l0) * P->nkind + d->quad[c]) * ms + r0, c * Q, Qp, Q, 0, 1});
          }
        });
      stage(b, 0);
    }
    // translation + potential transfer, levels l0 .. L:
    // o_g = sum_e D_e s_src(e) (163-166) + B_{quad g} o_parent (167-169)
    for (int lv = P->l0; lv <= P->L; ++lv) {
      b = int64_t(wi.size());
      const int64_t f = P->lvl_first[lv - P->l0], n = P->lvl_count[lv - P->l0];
      for (int64_t g = f; g < f + n; ++g)
        tiles(g * Q, Q, [&](int r0) {
          for (int64_t e = d->int_ptr[g]; e < d->int_ptr[g + 1]; ++e)
            wt.push_back(WTerm{d->int_dtab[e] * ms + r0, d->int_idx[e] * Q, Qp, Q, 2, 1});
          if (lv > P->l0)
            wt.push_back(WTerm{(int64_t(lv - P->l0 - 1) * P->nkind + d->quad[g]) * ms + r0,
                               d->parent[g] * Q, Qp, Q, 1, 2});
        });
      stage(b, 1);
    }
    // reception: phi[perm] = U_leaf o_leaf (170-172), panels of the stored U
    b = int64_t(wi.size());
    for (size_t i = 0; i < hu.items.size(); ++i) {
      const BlockItem& u = hu.items[i];
      tiles(u.y_row0, u.m, [&](int r0) {
        wt.push_back(WTerm{u.a_off + r0, u_leaf[i] * Q, u.ld, Q, 4, 2});
      });
    }
    stage(b, 2);
    require(wt.size() < (size_t(1) << 31), "wide work list too large");
    P->w_items.upload(wi);
    P->w_terms.upload(wt);
    P->wide_far = true;
  }

  // ---- fill the blobs: from host operators or assembled on the device
  DevBuf<double> pts;
  const bool helm_near = !d->near_blob && (d->options & NESA_PLAN_HELMHOLTZ_NEAR);
  const bool need_geom = (!d->near_blob && !helm_near) || !d->V_blob || !d->U_blob;
  if (need_geom) {
    require(d->points_tree && d->leaf_center && d->leaf_r_check && d->leaf_r_inaux &&
                d->out_fit_leaf && d->check_cos && d->check_sin && d->aux_cos && d->aux_sin,
            "device assembly needs the geometry fields of nesa_plan_desc");
    pts.upload(std::vector<double>(d->points_tree, d->points_tree + 2 * P->N));
  }
  T* nblob = reinterpret_cast<T*>(P->nearset.blob.p);
  T* vblob = reinterpret_cast<T*>(P->Vset.blob.p);
  T* ublob = reinterpret_cast<T*>(P->Uset.blob.p);
  if (d->near_blob) {
    upload_host_blob<T>(P->nearset, hn, d->near_blob, near_src_off, near_src_rows, near_row0);
  } else if (helm_near) {
    if (!hn.items.empty()) {
      DevBuf<double> p3;
      p3.upload(std::vector<double>(d->points3, d->points3 + 3 * (P->N / 2)));
      assemble_near_helm_kernel<T><<<int(hn.items.size()), 256>>>(P->nearset.items.p, P->nearset.segs.p, p3.p,
                                                                  d->wavenumber, nblob);
      CUDA_OK(cudaGetLastError());
      CUDA_OK(cudaDeviceSynchronize());
    }
  } else if (!hn.items.empty()) {
    assemble_near_kernel<T><<<int(hn.items.size()), 256>>>(P->nearset.items.p, P->nearset.segs.p,
                                                            pts.p, nblob);
    CUDA_OK(cudaGetLastError());
  }
  DevBuf<double> center, rck, rax, fit, cc, cs, ac, as;
  DevBuf<int64_t> vleaf, uleaf;
  if (!d->V_blob || !d->U_blob) {
    center.upload(std::vector<double>(d->leaf_center, d->leaf_center + 2 * NL));
    rck.upload(std::vector<double>(d->leaf_r_check, d->leaf_r_check + NL));
    rax.upload(std::vector<double>(d->leaf_r_inaux, d->leaf_r_inaux + NL));
    fit.upload(std::vector<double>(d->out_fit_leaf, d->out_fit_leaf + int64_t(Q) * P->n_check));
    cc.upload(std::vector<double>(d->check_cos, d->check_cos + P->n_check));
    cs.upload(std::vector<double>(d->check_sin, d->check_sin + P->n_check));
    ac.upload(std::vector<double>(d->aux_cos, d->aux_cos + Q));
    as.upload(std::vector<double>(d->aux_sin, d->aux_sin + Q));
    vleaf.upload(v_leaf);
    uleaf.upload(u_leaf);
  }
  if (d->V_blob) {
    upload_host_blob<T>(P->Vset, hv, d->V_blob, v_src_off, v_src_rows, v_row0);
  } else if (!hv.items.empty() && !P->v_mom) {
    assemble_V_kernel<T><<<int(hv.items.size()), 128, P->n_check * sizeof(double)>>>(
        P->Vset.items.p, vleaf.p, pts.p, center.p, rck.p, fit.p, cc.p, cs.p, Q, P->n_check, vblob);
    CUDA_OK(cudaGetLastError());
  }
  if (P->u_mf || P->v_mom) {
    // expansion inputs: leaf-relative float32 coordinates, radii, and the
    // per-plan coefficient tables (formed in float64)
    std::vector<float2> prel(static_cast<size_t>(P->N));
    std::vector<float> lr(static_cast<size_t>(NL)), lrc(static_cast<size_t>(NL));
    for (int64_t a = 0; a < NL; ++a) {
      const double cx = d->leaf_center[2 * a], cy = d->leaf_center[2 * a + 1];
      lr[a] = float(d->leaf_r_inaux[a]);
      lrc[a] = float(d->leaf_r_check[a]);
      for (int64_t i = d->group_start[a]; i < d->group_stop[a]; ++i) {
        prel[i] = float2{float(d->points_tree[2 * i] - cx), float(d->points_tree[2 * i + 1] - cy)};
      }
    }
    P->mf_prel.upload(prel);
    if (!std::is_same<T, float>::value && P->u_mf) {
      std::vector<double2> p64(static_cast<size_t>(P->N));
      std::vector<double> r64(static_cast<size_t>(NL));
      for (int64_t a = 0; a < NL; ++a) {
        const double cx = d->leaf_center[2 * a], cy = d->leaf_center[2 * a + 1];
        r64[a] = d->leaf_r_inaux[a];
        for (int64_t i = d->group_start[a]; i < d->group_stop[a]; ++i)
          p64[i] = double2{d->points_tree[2 * i] - cx, d->points_tree[2 * i + 1] - cy};
      }
      P->mf_prel64.upload(p64);
      P->mf_leaf_r64.upload(r64);
    }
    P->gstart.upload(std::vector<int64_t>(d->group_start, d->group_start + NL));
    P->gstop.upload(std::vector<int64_t>(d->group_stop, d->group_stop + NL));
    P->mf_leaf_r.upload(lr);
    P->mf_leaf_rc.upload(lrc);
    const int nc = P->n_check;
    if (P->v_mom) {
      std::vector<float2> A(size_t(P->v_nm) * Q);
      std::vector<double> Ad(size_t(P->v_nm) * Q * 2);  // float64 (re, im) for the stacked map
      std::vector<double> ang(nc);
      for (int l = 0; l < nc; ++l) ang[l] = std::atan2(d->check_sin[l], d->check_cos[l]);
      for (int k = 0; k < Q; ++k) {
        const double* f = d->out_fit_leaf + int64_t(k) * nc;
        double F = 0;
        for (int l = 0; l < nc; ++l) F += f[l];
        A[k] = float2{float(F), 0.f};
        Ad[2 * size_t(k)] = F;
        Ad[2 * size_t(k) + 1] = 0;
        for (int m = 1; m < P->v_nm; ++m) {
          double re = 0, im = 0;
          for (int l = 0; l < nc; ++l) {
            re += f[l] * std::cos(m * ang[l]);
            im -= f[l] * std::sin(m * ang[l]);
          }
          A[size_t(m) * Q + k] = float2{float(re / m), float(im / m)};
          Ad[2 * (size_t(m) * Q + k)] = re / m;
          Ad[2 * (size_t(m) * Q + k) + 1] = im / m;
        }
      }
      P->mom_A.upload(A);
      // Q = 64: s = A^ mu^ on the tensor cores (K = 2 nm - 1 <= 80 real rows:
      // 0 -> F_k, 2m-1 -> Re A_km, 2m -> -Im A_km)
      if (Q == 64 && P->tc && P->v_nm <= 2 * kRadTcMH) {
        std::vector<float> h(size_t(2) * 64 * kRadTcK, 0.f);
        for (int k = 0; k < 64; ++k)
          for (int j = 0; j < kRadTcK; ++j) {
            float x = 0.f;
            const int m = (j + 1) / 2;
            if (j == 0)
              x = A[k].x;
            else if (m < P->v_nm)
              x = (j & 1) ? A[size_t(m) * Q + k].x : -A[size_t(m) * Q + k].y;
            const float hi = tf32_host(x), lo = tf32_host(x - hi);
            const size_t off = size_t(k / 8) * (kRadTcK * 8) + size_t(j / 4) * 32 + size_t(k % 8) * 4 + (j % 4);
            h[off] = hi;
            h[size_t(64) * kRadTcK + off] = lo;
          }
        P->ATC.upload(h);
        std::vector<int32_t> ord;
        for (int64_t a = lb; a < le; ++a) ord.push_back(int32_t(a));
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
          return d->group_stop[x] - d->group_start[x] > d->group_stop[y] - d->group_start[y];
        });
        P->rad_order.upload(ord);
        P->rad_tc = true;
      }
    }
    if (P->u_mf) {
      const int ne = P->u_nt + 1;
      std::vector<float2> E(size_t(Q) * ne);
      for (int k = 0; k < Q; ++k) {
        const double th = std::atan2(d->aux_sin[k], d->aux_cos[k]);
        E[size_t(k) * ne] = float2{1.f, 0.f};
        for (int m = 1; m <= P->u_nt; ++m)
          E[size_t(k) * ne + m] = float2{float(std::cos(m * th) / m), float(-std::sin(m * th) / m)};
      }
      P->exp_E.upload(E);
      if (!std::is_same<T, float>::value) {
        std::vector<double2> E64(size_t(Q) * ne);
        for (int k = 0; k < Q; ++k) {
          const double th = std::atan2(d->aux_sin[k], d->aux_cos[k]);
          E64[size_t(k) * ne] = double2{1.0, 0.0};
          for (int m = 1; m <= P->u_nt; ++m)
            E64[size_t(k) * ne + m] = double2{std::cos(m * th) / m, -std::sin(m * th) / m};
        }
        P->exp_E64.upload(E64);
      }
      // Q = 64 with tensor cores: beta^ = E^ o for all leaves as one GEMM;
      // E^ rows 0 -> 1 (sum of o), 2m-1 / 2m -> Re / Im of (1/m) e^{-i m theta_k}
      if (Q == 64 && P->tc && 2 * P->u_nt + 1 <= 64) {
        std::vector<double> Em(64 * 64, 0.0);  // E^[row][k]
        for (int row = 0; row < 64; ++row)
          for (int k = 0; k < 64; ++k) {
            float x = 0.f;
            if (row == 0)
              x = 1.f;
            else if (row <= 2 * P->u_nt)
              x = (row & 1) ? E[size_t(k) * ne + (row + 1) / 2].x : E[size_t(k) * ne + row / 2].y;
            Em[size_t(row) * 64 + k] = x;
          }
        P->ETC.upload(canon_tf32(Em.data(), 1));
        P->beta_tc = true;
      }
      // leaf level handled by the wide kernels: its downward transfer and
      // beta^ = E^ o in one kernel (no o round trip before the reception)
      const bool leaf_wide = P->L > P->l0 && P->loc_count[P->L - P->l0] >= P->wide_level;
      if (Q == 64 && leaf_wide && P->beta_tc) {
        std::vector<float> et(64 * 64, 0.f);
        for (int row = 0; row < 64; ++row)
          for (int k = 0; k < 64; ++k) {
            float x = 0.f;
            if (row == 0)
              x = 1.f;
            else if (row <= 2 * P->u_nt)
              x = (row & 1) ? E[size_t(k) * ne + (row + 1) / 2].x : E[size_t(k) * ne + row / 2].y;
            et[size_t(k) * 64 + row] = x;
          }
        P->ET.upload(et);
        P->beta_fused = true;
      }
    }
    if (P->beta_tc) {
      // one entry per local leaf (src = dst = leaf), 32 leaves per unit
      std::vector<TUnit> units;
      std::vector<TEnt> ents;
      for (int64_t a = lb; a < le; ++a) ents.push_back(TEnt{int32_t(a), int32_t(a)});
      const int per = 32;  // one pass of 32 leaves per CTA: the GEMM is latency-bound
      for (size_t i = 0; i < ents.size(); i += per)
        units.push_back(TUnit{0, int32_t(i), int32_t(std::min(ents.size(), i + per)), 0});
      P->mom_units.upload(units);
      P->mom_ents.upload(ents);
      P->n_mom_units = int(units.size());
    }
  }
  if (P->u_mf) {
  } else if (d->U_blob) {
    upload_host_blob<T>(P->Uset, hu, d->U_blob, u_src_off, u_src_rows, u_row0);
  } else if (!hu.items.empty()) {
    assemble_U_kernel<T><<<int(hu.items.size()), 256>>>(P->Uset.items.p, uleaf.p, pts.p, center.p,
                                                         rax.p, ac.p, as.p, ublob);
    CUDA_OK(cudaGetLastError());
  }
  CUDA_OK(cudaDeviceSynchronize());

  // ---- translation entries of the local targets, grouped by unique D
  {
    P->nnz = d->int_ptr[G];
    P->int_ptr.upload(std::vector<int64_t>(d->int_ptr, d->int_ptr + G + 1));
    require(P->nnz < (int64_t(1) << 31), "too many interaction entries");
    // entries per unit: the FFMA kernel runs kTUnitPasses passes (sized for
    // R = 4); the tensor-core kernel loops over M = 128 tiles and amortises
    // its D load and TMEM allocation over longer units
    int per = kTUnitPasses * (tg_geom(Q).NC / 4);
    if (P->tc) per = 128;
    std::vector<TEnt> ents;
    std::vector<TUnit> units;
    std::vector<std::vector<TEnt>> by_d(size_t(std::max<int64_t>(d->n_dtab, 1)));
    // levels fine -> coarse; within a level grouped by unique D
    P->tunit_lv_begin.assign(size_t(P->L - P->l0 + 1), 0);
    P->tunit_lv_end.assign(size_t(P->L - P->l0 + 1), 0);
    for (int lv = P->L; lv >= P->l0; --lv) {
      const int li = lv - P->l0;
      P->tunit_lv_begin[size_t(li)] = int(units.size());
      std::vector<int64_t> used;
      for (int64_t g = P->loc_first[li]; g < P->loc_first[li] + P->loc_count[li]; ++g)
        for (int64_t e = d->int_ptr[g]; e < d->int_ptr[g + 1]; ++e) {
          const int64_t dt = d->int_dtab[e];
          require(dt >= 0 && dt < d->n_dtab, "D index out of range");
          require(d->int_idx[e] >= 0 && d->int_idx[e] < G, "interaction id out of range");
          if (by_d[dt].empty()) used.push_back(dt);
          by_d[dt].push_back(TEnt{int32_t(d->int_idx[e]), int32_t(e)});
        }
      std::sort(used.begin(), used.end());
      for (int64_t dt : used) {
        auto& v = by_d[dt];
        for (size_t i = 0; i < v.size(); i += size_t(per)) {
          const size_t j = std::min(v.size(), i + size_t(per));
          units.push_back(TUnit{int32_t(dt), int32_t(ents.size()), int32_t(ents.size() + (j - i)), 0});
          ents.insert(ents.end(), v.begin() + i, v.begin() + j);
        }
        P->d_refs += int64_t(v.size());
        v.clear();
      }
      if (lv == P->split_lv) P->n_tunits_fine = int(units.size());
      P->tunit_lv_end[size_t(li)] = int(units.size());
    }
    P->tunits.upload(units);
    P->tents.upload(ents);
    P->n_tunits = int(units.size());
  }
}



template <typename T>
void ensure_workspace(nesa_plan* P, int R) {
  if (P->ws_R >= R) return;
  // every captured graph addresses the old buffers: drop them (an exec still
  // in flight is freed by the driver when it completes; cudaFree below
  // synchronises the device first)
  P->drop_graphs();
  const size_t es = sizeof(T);
  P->qt.alloc(size_t(P->N) * R * es);
  P->phin.alloc(size_t(P->N) * R * es);
  if (P->beta_tc) P->beta.alloc(size_t(P->NL) * 64 * R * es);
  {
    const size_t fb = (size_t(P->G) * P->Q * R * es + 255) & ~size_t(255);
    P->farws.alloc(3 * fb);
    P->s.view(P->farws.p, fb);
    P->Tup.view(P->farws.p + fb, fb);
    P->o.view(P->farws.p + 2 * fb, fb);
  }
  P->Y.alloc(size_t(std::max<int64_t>(P->nnz, 1)) * P->Q * R * es);
  if (P->comm) {
    const size_t row = size_t(P->Q) * R * es;
    P->x_send.alloc(size_t(P->x_max_export) * row);
    P->x_recv.alloc(size_t(P->nranks) * P->x_max_export * row);
  }
  P->ws_R = R;
  P->ws_gen++;
}

inline int grid_for(int64_t n, int threads, int cap) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap)));
}

template <typename T, int R, int MODE, int NST = kStages, int NCW = kNCW, int AB = kABytes>
BlockGemvArgs<T> blockgemv_args(const DevBlockSet& bs, const T* x, T* y, const T* base,
                                const int64_t* perm, int ldy) {
  return BlockGemvArgs<T>{reinterpret_cast<const T*>(bs.blob.p), bs.recs.p, bs.cta_ptr.p, x, y,
                          base, perm, ldy};
}

// near field (store mode): 4 consumer warps, two 24 KB stages
template <typename T, int R>
void launch_near(const DevBlockSet& bs, const T* x, T* y, cudaStream_t st) {
  if (bs.n_items == 0) return;
  blockgemv_kernel<T, R, kModeStore, kNearStages, kNearNCW, kNearABytes>
      <<<bs.grid, kNearNCW * 32 + 32, blockgemv_smem_bytes<T, R, kModeStore, kNearStages, kNearNCW, kNearABytes>(),
         st>>>(blockgemv_args<T, R, kModeStore>(bs, x, y, nullptr, nullptr, 0));
}

// complex near field (NESA_PLAN_COMPLEX_NEAR): the same engine on the
// row-split complex blob, x / y read as complex (R = 2) values
template <typename T>
void launch_near_cplx(const DevBlockSet& bs, const T* x, T* y, cudaStream_t st) {
  if (bs.n_items == 0) return;
  blockgemv_kernel<T, 2, kModeStoreCplx, kNearStages, kNearNCW, kNearABytes>
      <<<bs.grid, kNearNCW * 32 + 32,
         blockgemv_smem_bytes<T, 2, kModeStoreCplx, kNearStages, kNearNCW, kNearABytes>(), st>>>(
          blockgemv_args<T, 2, kModeStoreCplx>(bs, x, y, nullptr, nullptr, 0));
}

template <typename T, int R>
void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  auto attr = [](auto* fn, int smem) {
    CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  };
  attr(blockgemv_kernel<T, R, kModeStore, kNearStages, kNearNCW, kNearABytes>,
       int(blockgemv_smem_bytes<T, R, kModeStore, kNearStages, kNearNCW, kNearABytes>()));
  attr(blockgemv_kernel<T, R, kModeStore>, int(blockgemv_smem_bytes<T, R, kModeStore>()));
  if constexpr (R == 1) {
    attr(blockgemv_kernel<T, 2, kModeStoreCplx, kNearStages, kNearNCW, kNearABytes>,
         int(blockgemv_smem_bytes<T, 2, kModeStoreCplx, kNearStages, kNearNCW, kNearABytes>()));
    attr(blockgemv_kernel<T, 2, kModeStoreCplx>, int(blockgemv_smem_bytes<T, 2, kModeStoreCplx>()));
    attr(blockgemv_kernel<T, 2, kModeScatterCplx>, int(blockgemv_smem_bytes<T, 2, kModeScatterCplx>()));
  }
  attr(blockgemv_kernel<T, R, kModeScatter>, int(blockgemv_smem_bytes<T, R, kModeScatter>()));
  const int lim = 220 * 1024;
  attr(tgemm_kernel<T, R>, lim);
  attr(tgemm_wt_kernel<T, R, 64>, lim);
  attr(tgemm_wt_kernel<T, R, 32>, lim);
  if constexpr (TGW<T, R, 128>::SMEM <= 220 * 1024) attr(tgemm_wt_kernel<T, R, 128>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlUpLeaf>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlUpSum>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlDown>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlDownBeta>, lim);
  if constexpr (LVW<T, R, 128, kLvlDown>::SMEM <= 220 * 1024) {
    attr(level_wt_kernel<T, R, 128, kLvlUpLeaf>, lim);
    attr(level_wt_kernel<T, R, 128, kLvlUpSum>, lim);
    attr(level_wt_kernel<T, R, 128, kLvlDown>, lim);
  }
  attr(fused_up_kernel<T, R>, lim);
  attr(fused_down_kernel<T, R>, lim);
  if constexpr (std::is_same<T, float>::value) {
    attr(radiation_mom_kernel<R>, lim);
    if constexpr (R == 2) attr(radiation_tc_kernel<R>, int(radiation_tc_smem_bytes<R>()));
    attr(tgemm_tc2_kernel<R>, int(tc2_smem_bytes<R>()));
    attr(tgemm_tc3_kernel<R>, int(tc2_smem_bytes<R>()));
    attr(level_tc_kernel<R, kLvlUpLeaf>, int(level_tc_smem_bytes<R>(kLvlUpLeaf)));
    attr(level_tc_kernel<R, kLvlUpSum>, int(level_tc_smem_bytes<R>(kLvlUpSum)));
    attr(level_tc_kernel<R, kLvlDown>, int(level_tc_smem_bytes<R>(kLvlDown)));
    attr(level_tc_kernel<R, kLvlDownBeta>, int(level_tc_smem_bytes<R>(kLvlDownBeta)));
    attr(reception_exp_kernel<R, false>, lim);
    attr(reception_exp_kernel<R, true>, lim);
  }
  done = true;
}

// Record a profiling event; during capture this becomes an event-record node
// on the stream the neighbouring kernels run on.
void prof_mark(nesa_plan* P, bool profile, int slot, cudaStream_t st) {
  if (!profile) return;
  CUDA_OK(cudaEventRecordWithFlags(P->cap_events[slot], st, cudaEventRecordExternal));
}

// Launch with programmatic dependent launch (PDL): the kernel may start its
// prologue while the previous kernel of the stream drains; it calls
// pdl_wait() before touching that kernel's outputs.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <typename Tuple, size_t... I>
void tuple_ptrs(Tuple& t, void** out, std::index_sequence<I...>) {
  ((out[I] = static_cast<void*>(&std::get<I>(t))), ...);
}

// Launch a kernel that reads the caller's q or writes the caller's phi.
// `make(q, phi)` builds its arguments; during a capture the node is
// recorded with a closure that re-points it at other buffers in the
// instantiated graph (run_block), so the graph cache is keyed without the
// caller's pointers.
template <typename F, typename... KArgs>
void io_launch(nesa_plan* P, void (*kern)(KArgs...), int grid, int block, size_t smem,
               cudaStream_t st, F make, const void* q, void* phi) {
  std::tuple<KArgs...> args = make(q, phi);
  std::apply([&](auto&... a) { kern<<<grid, block, smem, st>>>(a...); }, args);
  CUDA_OK(cudaGetLastError());
  if (!P->capturing_io) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CUDA_OK(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
  require(cs == cudaStreamCaptureStatusActive && nd == 1, "io kernel node not found in the capture");
  nesa_plan::IoPatch io;
  io.node = deps[0];
  io.apply = [kern, grid, block, smem, make](cudaGraphExec_t ex, cudaGraphNode_t node, const void* q2,
                                             void* phi2) {
    std::tuple<KArgs...> a2 = make(q2, phi2);
    void* ptrs[sizeof...(KArgs) > 0 ? sizeof...(KArgs) : 1];
    tuple_ptrs(a2, ptrs, std::index_sequence_for<KArgs...>{});
    cudaKernelNodeParams p = {};
    p.func = reinterpret_cast<void*>(kern);
    p.gridDim = dim3(unsigned(grid));
    p.blockDim = dim3(unsigned(block));
    p.sharedMemBytes = unsigned(smem);
    p.kernelParams = ptrs;
    return cudaGraphExecKernelNodeSetParams(ex, node, &p);
  };
  P->capturing_io->push_back(std::move(io));
}

constexpr int kExpCtasPerSM = 12;  // reception: two waves (A/B: 1.7 us faster than one)
constexpr int kMomCtasPerSM = 4;
constexpr int kMomBufPoints = 800;  // points staged per warp by the moment kernel

// s = V qt: outgoing moments (float32 plans from geometry) or stored V
template <typename T, int R>
int launch_radiation(nesa_plan* P, const T* qt, T* s, cudaStream_t st) {
  if constexpr (std::is_same<T, float>::value) {
    // the tensor-core moment map pairs the two real columns of one complex
    // right-hand side; one or four real columns take the FFMA2 moment kernel
    if (P->v_mom && P->rad_tc && R == 2) {
      if constexpr (R == 2) {
        const int64_t nleaf = P->leaf_end - P->leaf_begin;
        const int64_t ntiles = (nleaf + kRadTcLeaves - 1) / kRadTcLeaves;
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ntiles, 2 * P->n_sm)));
        radiation_tc_kernel<R><<<grid, 32 * kRadTcWarps, radiation_tc_smem_bytes<R>(), st>>>(
            P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_rc.p, P->ATC.p, qt, s, P->rad_order.p, nleaf,
            P->v_nm);
        return 1;
      }
    }
    if (P->v_mom) {
      const int64_t nleaf = P->leaf_end - P->leaf_begin;
      const int64_t per_cta = int64_t(kExpWarps) * kMomLeavesPerWarp;
      const int grid = int(std::max<int64_t>(
          1, std::min<int64_t>((nleaf + per_cta - 1) / per_cta, int64_t(kMomCtasPerSM) * P->n_sm)));
      const size_t sm = size_t(kExpWarps) *
                        (size_t(kMomBufPoints) * (2 + R) +
                         size_t(kMomLeavesPerWarp) * ((P->v_nm * R + 1) & ~1) * 2) *
                        sizeof(float);
      radiation_mom_kernel<R><<<grid, 32 * kExpWarps, sm, st>>>(
          P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_rc.p, P->mom_A.p, qt, s, P->leaf_begin,
          nleaf, P->Q, P->v_nm, kMomBufPoints);
      return 1;
    }
  }
  if (P->Vset.n_items == 0) return 0;
  if (P->cnear) {
    // complex V row-split (Track B): one complex column
    if constexpr (R == 1)
      blockgemv_kernel<T, 2, kModeStoreCplx><<<P->Vset.grid, kBGThreads, blockgemv_smem_bytes<T, 2, kModeStoreCplx>(),
                                               st>>>(blockgemv_args<T, 2, kModeStoreCplx>(P->Vset, qt, s, nullptr,
                                                                                          nullptr, 0));
    return 1;
  }
  blockgemv_kernel<T, R, kModeStore><<<P->Vset.grid, kBGThreads, blockgemv_smem_bytes<T, R, kModeStore>(), st>>>(
      blockgemv_args<T, R, kModeStore>(P->Vset, qt, s, nullptr, nullptr, 0));
  return 1;
}

// Enqueue one product, or one of its two stages (multi-GPU), on P->s0/P->s1.
//   stage 0: gather, radiation, fork{near | up, translate, down}, join, reception
//   stage 1: gather, fork{near | radiation, up}, join  (before the s halo exchange)
//   stage 2: translate, down, reception
template <typename T, int R>
int enqueue_T(nesa_plan* P, const T* q, T* phi, int ldv, uint32_t flags, int stage) {
  const bool near = flags & NESA_NEAR, far = flags & NESA_FAR, profn = flags & NESA_PROFILE;
  const bool prof = profn && !(flags & NESA_PROFILE_NEAR);  // stage marks on the far path
  cudaStream_t s0 = P->s0, s1 = P->s1;
  T* qt = reinterpret_cast<T*>(P->qt.p);
  T* phin = reinterpret_cast<T*>(P->phin.p);
  T* s = reinterpret_cast<T*>(P->s.p);
  T* o = reinterpret_cast<T*>(P->o.p);
  T* Tup = reinterpret_cast<T*>(P->Tup.p);
  T* Y = reinterpret_cast<T*>(P->Y.p);
  const T* CT = reinterpret_cast<const T*>(P->CT.p);
  const T* BT = reinterpret_cast<const T*>(P->BT.p);
  const int Q = P->Q;
  const int cap = P->n_sm * 8;
  const int64_t nloc = P->pt_end - P->pt_begin;
  const size_t mstride = P->mbytes / sizeof(T);
  int nk = 0;
  if (prof) P->trace_names.clear();
  // NESA_TRACE diagnostics: an event-record node after each kernel
  auto tr = [&](const char* name, cudaStream_t st) {
    if (!prof || !P->trace || P->trace_names.size() >= size_t(kTraceSlots)) return;
    prof_mark(P, true, 2 * NESA_N_STAGES + int(P->trace_names.size()), st);
    P->trace_names.emplace_back(name);
  };

  auto level_args = [&](int li, const T* M) {
    LevelArgs<T, R> la{};
    la.MT4 = M;
    la.quad = P->quad.p;
    la.order = P->down_order[li].p;
    la.opar = P->down_par[li].p;
    la.ochild = P->down_child[li].p;
    la.Tin = Tup;
    la.s = s;
    la.Tout = Tup;
    la.o = o;
    la.count = P->loc_count[li];
    la.Q = Q;
    return la;
  };
  const bool fused = P->fused_lf > P->l0;
  // every level is either one of the wide (warp-tiled, Q = 64) levels at the
  // fine end or inside the fused coarse range (see build_plan_T)
  auto wide = [&](int lv) { return lv > P->fused_lf; };
  constexpr int RI = R == 1 ? 0 : (R == 2 ? 1 : 2);
  // float32 Q = 64: the level GEMMs on the tensor cores (level_tc_kernel)
  auto level_tc = [&](int lv, int mode) -> bool {
    if constexpr (std::is_same<T, float>::value) {
      if (!P->level_tc) return false;
      const int ci = lv - P->l0;
      // tensor cores only from kLevelTcMin groups: every tf32x3 level adds a
      // systematic ~1.5e-6 to the complex64 error at C4 (the tensor core's
      // accumulator truncates; the errors of successive levels add linearly:
      // 0 / 1 / 2 / 3 / 4 / 5 levels -> 1.6 / 3.3 / 5.0 / 6.5 / 8.0 / 9.6e-6
      // against the exact sum), so the smallest per-level kernel stays on the
      // FFMA path and the product keeps its margin below 1e-5
      if (P->loc_count[ci] < kLevelTcMin) return false;
      const DevBuf<int4>& tiles = P->lvl_tiles[size_t(ci) * 3 + RI];
      LevelTcArgs ta{};
      const bool down = mode == kLvlDown || mode == kLvlDownBeta;
      ta.MTC = (down ? P->BTC.p : P->CTC.p) + size_t(ci - 1) * 4 * 8192;
      ta.ETC = P->ETC.p;
      ta.tiles = tiles.p;
      ta.order = P->down_order[ci].p;
      ta.opar = P->down_par[ci].p;
      ta.ochild = P->down_child[ci].p;
      ta.Tin = Tup;
      ta.s = s;
      ta.Tout = Tup;
      ta.o = o;
      ta.beta = reinterpret_cast<float*>(P->beta.p);
      const int grid = int(tiles.n);
      switch (mode) {
        case kLvlUpLeaf:
          launch_pdl(level_tc_kernel<R, kLvlUpLeaf>, grid, 128, level_tc_smem_bytes<R>(kLvlUpLeaf), s0, ta);
          break;
        case kLvlUpSum:
          launch_pdl(level_tc_kernel<R, kLvlUpSum>, grid, 128, level_tc_smem_bytes<R>(kLvlUpSum), s0, ta);
          break;
        case kLvlDown:
          launch_pdl(level_tc_kernel<R, kLvlDown>, grid, 128, level_tc_smem_bytes<R>(kLvlDown), s0, ta);
          break;
        default:
          launch_pdl(level_tc_kernel<R, kLvlDownBeta>, grid, 128, level_tc_smem_bytes<R>(kLvlDownBeta), s0,
                     ta);
      }
      return true;
    }
    return false;
  };
  auto up_level = [&](int lv) {
    // children-major: T[c] = C s[c]; s[parent] = sum of its children's T
    const int ci = lv - P->l0;
    if (P->loc_count[ci] == 0) return;
    if (level_tc(lv, lv == P->L ? kLvlUpLeaf : kLvlUpSum)) {
      nk++;
      tr("up_tc", s0);
      return;
    }
    const LevelArgs<T, R> la = level_args(ci, CT + size_t(ci - 1) * P->nkind * mstride);
    if (Q == 128) {
      // (Track B's complex Q = 64 in the real embedding)
      if constexpr (LVW<T, R, 128, kLvlDown>::SMEM <= 220 * 1024) {
        const int gw = int((la.count + TGW<T, R, 128>::PER - 1) / TGW<T, R, 128>::PER);
        if (lv == P->L)
          launch_pdl(level_wt_kernel<T, R, 128, kLvlUpLeaf>, gw, 128, LVW<T, R, 128, kLvlUpLeaf>::SMEM, s0, la,
                     RecvArgs{});
        else
          launch_pdl(level_wt_kernel<T, R, 128, kLvlUpSum>, gw, 128, LVW<T, R, 128, kLvlUpSum>::SMEM, s0, la,
                     RecvArgs{});
      }
      nk++;
      tr("up_wt", s0);
      return;
    }
    const int gw = int((la.count + TGW<T, R, 64>::PER - 1) / TGW<T, R, 64>::PER);
    if (lv == P->L)
      launch_pdl(level_wt_kernel<T, R, 64, kLvlUpLeaf>, gw, 128, LVW<T, R, 64, kLvlUpLeaf>::SMEM, s0, la, RecvArgs{});
    else
      launch_pdl(level_wt_kernel<T, R, 64, kLvlUpSum>, gw, 128, LVW<T, R, 64, kLvlUpSum>::SMEM, s0, la, RecvArgs{});
    nk++;
    tr("up_wt", s0);
  };
  auto translate = [&](int u0, int u1, cudaStream_t st, bool pdl = true) {
    if (u1 <= u0) return;
    const T* DTp = reinterpret_cast<const T*>(P->DT.p);
    const TUnit* up = P->tunits.p + u0;
    const bool pdl_ok = pdl && st == s0;
    auto go = [&](auto kern, int grid, size_t smem, auto... args) {
      if (pdl_ok)
        launch_pdl(kern, grid, 128, smem, st, args...);
      else
        kern<<<grid, 128, smem, st>>>(args...);
    };
    if constexpr (std::is_same<T, float>::value) {
      if (P->tc) {
        go(tgemm_tc3_kernel<R>, std::min(u1 - u0, kTc3CtasPerSM * P->n_sm), tc2_smem_bytes<R>(), up,
           u1 - u0, (const TEnt*)P->tents.p, (const float*)P->DTC.p, (const float*)s, Y,
           u0 < P->n_tunits_fine ? 44 : 45);  // (ktrace: fine / coarse units)
        nk++;
        tr("translate", st);
        return;
      }
    }
    if (Q == 64)
      go(tgemm_wt_kernel<T, R, 64>, u1 - u0, TGW<T, R, 64>::SMEM, up, (const TEnt*)P->tents.p, DTp,
         (const T*)s, Y);
    else if (Q == 32)
      go(tgemm_wt_kernel<T, R, 32>, u1 - u0, TGW<T, R, 32>::SMEM, up, (const TEnt*)P->tents.p, DTp,
         (const T*)s, Y);
    else if (Q == 128 && TGW<T, R, 128>::SMEM <= 220 * 1024)
      // (Track B's complex Q = 64 in the real embedding, or a real Q = 128)
      go(tgemm_wt_kernel<T, R, 128>, u1 - u0, TGW<T, R, 128>::SMEM, up, (const TEnt*)P->tents.p, DTp,
         (const T*)s, Y);
    else
      tgemm_kernel<T, R><<<u1 - u0, kTGThreads, tgemm_smem_bytes<T, R>(Q), st>>>(up, P->tents.p, DTp, s,
                                                                                Y, Q);
    nk++;
    tr("translate", st);
  };
  auto reduce = [&](int64_t i0, int64_t i1, cudaStream_t st, int per_sm = 8) {
    // o[g] = translation sum of the listed local groups
    if (i1 <= i0) return;
    const int grid = grid_for((i1 - i0) * 32, 256, P->n_sm * per_sm);
    const int32_t* ids = P->red_ids.p + i0;
    const int64_t* ip = P->int_ptr.p;
    if (st == s0)
      launch_pdl(reduce_kernel<T, R>, grid, 256, 0, st, ids, i1 - i0, ip, (const T*)Y, o, Q);
    else
      reduce_kernel<T, R><<<grid, 256, 0, st>>>(ids, i1 - i0, ip, (const T*)Y, o, Q);
    nk++;
    tr("reduce", st);
  };
  const bool far_recv = far && (stage == 0 || stage == 2);
  auto down_level = [&](int lv) {
    const int ci = lv - P->l0;
    if (P->loc_count[ci] == 0) return;
    if (level_tc(lv, lv == P->L && P->beta_fused && far_recv ? kLvlDownBeta : kLvlDown)) {
      nk++;
      tr("down_tc", s0);
      return;
    }
    const LevelArgs<T, R> la = level_args(ci, BT + size_t(ci - 1) * P->nkind * mstride);
    if (Q == 128) {
      if constexpr (LVW<T, R, 128, kLvlDown>::SMEM <= 220 * 1024) {
        const int gw = int((la.count + TGW<T, R, 128>::PER - 1) / TGW<T, R, 128>::PER);
        launch_pdl(level_wt_kernel<T, R, 128, kLvlDown>, gw, 128, LVW<T, R, 128, kLvlDown>::SMEM, s0, la,
                   RecvArgs{});
      }
      nk++;
      tr("down_wt", s0);
      return;
    }
    const int gw = int((la.count + TGW<T, R, 64>::PER - 1) / TGW<T, R, 64>::PER);
    if (lv == P->L && P->beta_fused && far_recv) {
      // leaf level + reception coefficients beta^ = E^ o in one kernel
      if constexpr (std::is_same<T, float>::value) {
        RecvArgs rv{};
        rv.ET = P->ET.p;
        rv.beta = reinterpret_cast<float*>(P->beta.p);
        launch_pdl(level_wt_kernel<T, R, 64, kLvlDownBeta>, gw, 128, LVW<T, R, 64, kLvlDownBeta>::SMEM, s0,
                   la, rv);
      }
    } else {
      launch_pdl(level_wt_kernel<T, R, 64, kLvlDown>, gw, 128, LVW<T, R, 64, kLvlDown>::SMEM, s0, la,
                 RecvArgs{});
    }
    nk++;
    tr("down_wt", s0);
  };
  auto fused_args = [&](const T* MT) {
    FusedArgs<T> fa{};
    fa.MT = MT;
    fa.mstride = mstride;
    fa.quad = P->quad.p;
    fa.nkind = P->nkind;
    fa.parent = P->parent.p;
    fa.uchild = P->uchild.p;
    fa.anc = P->fused_anc.p;
    fa.cnt = P->fused_cnt.p;
    fa.state = P->fused_state.p;
    fa.own = P->fused_own.p;
    fa.chain_up = P->fused_chain_up.p;
    fa.chain_down = P->fused_chain_down.p;
    fa.ticket = P->fused_ticket.p;
    fa.Tup = Tup;
    fa.s = s;
    fa.o = o;
    const int li = P->fused_lf - P->l0;
    fa.first = P->loc_first[li];
    fa.count = P->loc_count[li];
    fa.lf = P->fused_lf;
    fa.l0 = P->l0;
    fa.L = P->L;
    fa.Q = Q;
    fa.D = P->fused_lf - P->l0 - 1;
    return fa;
  };
  const int nchain = P->fused_lf - P->l0 + 1;
  const size_t fsm_up = fused_smem_bytes<T>(Q, R, 1, nchain), fsm = fused_smem_bytes<T>(Q, R, 2, nchain);
  // upward transfers of the fused coarse levels + the top-level sum
  auto fused_up = [&]() {
    const FusedArgs<T> fa = fused_args(CT);
    launch_pdl(fused_up_kernel<T, R>, int(fa.count), kFusedThreads, fsm_up, s0, fa);
    nk++;
    tr("up_fused", s0);
  };
  auto fused_down = [&]() {
    const FusedArgs<T> fa = fused_args(BT);
    launch_pdl(fused_down_kernel<T, R>, int(fa.count), kFusedThreads, fsm, s0, fa);
    nk++;
    tr("down_fused", s0);
  };
  // Far field.  The wide (fine) levels' translation + reduce run on s2 as
  // soon as their s is final, concurrently with the coarse end of the
  // upward chain, the coarse translations and the coarse downward levels.
  // split: fine translation on the side stream (stage 0); stage 1 / 2 split
  // the product at the halo exchange instead
  // fine levels: level lv's s is final after the radiation (lv = L) or
  // after up_level(lv); its translation + translation sums go to s2 right
  // then, one level at a time, and down_level(lv) waits for its own level
  auto up_pass = [&](bool split) {
    const bool fine = split && P->split_lv <= P->L;
    for (int lv = P->L; lv > P->l0; --lv) {
      if (!wide(lv)) break;
      if (fine && lv == P->L) CUDA_OK(cudaEventRecord(P->ev_s_lv[size_t(lv - P->l0)], s0));
      up_level(lv);
      if (fine && lv < P->L && lv >= P->split_lv)
        CUDA_OK(cudaEventRecord(P->ev_s_lv[size_t(lv - P->l0)], s0));
    }
    if (fused) fused_up();
    return fine;
  };
  auto down_pass = [&](bool fine) {
    if (fine) {
      // Side stream s2: the leaf level's translation (its s is final right
      // after the radiation), then the other wide levels' in one launch once
      // the coarsest of them is final -- back to back, so the second
      // persistent launch takes the SM slots the first one's CTAs leave
      // (beside the near field's two CTAs an SM holds ONE more 50 KB
      // tensor-core CTA plus a level kernel or three fused-chain CTAs; two
      // resident translations starve the upward chain).  The leaf level's
      // translation sums run on a third stream beside the second
      // translation; the other levels' sums follow it.  The coarse
      // translation on s0 gets no early programmatic start: its persistent
      // CTAs would hold their slots idle until the fused upward chain ends.
      // (ktrace before / after: profiles/r2_ktrace_sched.txt)
      {
        const size_t li = size_t(P->L - P->l0);
        const size_t lo = size_t(P->split_lv - P->l0);
        // FFMA translation (float64 / no tensor cores): its CTAs fill the
        // shared memory the upward level kernels need (ktrace at C4 float64:
        // the upward chain stalled 190 us behind the leaf translation), so
        // there the side stream waits for the wide levels' upward pass
        // (C4 complex128 1340 -> 1316 us)
        const bool tc_tr = std::is_same<T, float>::value && P->tc;
        CUDA_OK(cudaStreamWaitEvent(P->s2, P->ev_s_lv[tc_tr ? li : lo], 0));
        translate(P->tunit_lv_begin[li], P->tunit_lv_end[li], P->s2);
        if (P->split_lv < P->L) {
          CUDA_OK(cudaEventRecord(P->ev_tx, P->s2));
          CUDA_OK(cudaStreamWaitEvent(P->s3, P->ev_tx, 0));
          // (and not before the wide levels' upward pass is done: started
          // earlier, its 256-thread CTAs filled the register file and the
          // fused upward chain's CTAs waited ~10 us to become resident)
          CUDA_OK(cudaStreamWaitEvent(P->s3, P->ev_s_lv[lo], 0));
          // (half the usual grid: at 8 CTAs per SM this pass filled every
          // thread slot and kept the fused upward chain's CTAs out for 12 us;
          // its result is not needed before the leaf level's downward kernel)
          reduce(P->red_lv_begin[li], P->red_lv_end[li], P->s3, 4);
          CUDA_OK(cudaEventRecord(P->ev_t_lv[li], P->s3));
          CUDA_OK(cudaStreamWaitEvent(P->s2, P->ev_s_lv[lo], 0));
          translate(P->tunit_lv_begin[li - 1], P->tunit_lv_end[lo], P->s2);
          reduce(P->red_lv_begin[li - 1], P->red_lv_end[lo], P->s2);
          for (size_t l = lo; l < li; ++l) CUDA_OK(cudaEventRecord(P->ev_t_lv[l], P->s2));
        } else {
          reduce(P->red_lv_begin[li], P->red_lv_end[li], P->s2);
          CUDA_OK(cudaEventRecord(P->ev_t_lv[li], P->s2));
        }
      }
      translate(P->n_tunits_fine, P->n_tunits, s0, false);
      reduce(P->n_red_fine, P->n_red, s0);
    } else {
      translate(0, P->n_tunits, s0);
      reduce(0, P->n_red, s0);
    }
    if (fused) fused_down();
    for (int lv = P->l0 + 1; lv <= P->L; ++lv) {
      if (!wide(lv)) continue;
      if (fine && lv >= P->split_lv) CUDA_OK(cudaStreamWaitEvent(s0, P->ev_t_lv[size_t(lv - P->l0)], 0));
      down_level(lv);
    }
    // s2's work joins s0 (every fine level's event, also when a level had
    // no down kernel)
    if (fine)
      for (int lv = P->split_lv; lv <= P->L; ++lv)
        CUDA_OK(cudaStreamWaitEvent(s0, P->ev_t_lv[size_t(lv - P->l0)], 0));
  };
  auto gather = [&]() {
    const int32_t* ip = P->iperm.p;
    const int64_t n = P->N;
    io_launch(
        P, gather_inv_kernel<T, R>, grid_for((n + 3) / 4, 256, cap), 256, 0, s0,
        [=](const void* qq, void*) { return std::make_tuple(static_cast<const T*>(qq), ip, qt, n, ldv); },
        q, phi);
    nk++;
    tr("gather", s0);
  };
  auto finish = [&]() {
    prof_mark(P, prof, 2 * NESA_STAGE_RECEPTION, s0);
    const int64_t* pm = P->perm.p;
    const T* base = near ? phin : nullptr;
    if (far && P->u_mf) {
      if constexpr (std::is_same<T, float>::value) {
        const int64_t nleaf = P->leaf_end - P->leaf_begin;
        const int grid = int(std::max<int64_t>(
            1, std::min<int64_t>((nleaf + kExpWarps - 1) / kExpWarps, int64_t(kExpCtasPerSM) * P->n_sm)));
        const int nt = P->u_nt;
        const size_t nb = ((size_t(nt) + 1) * R + 1) & ~size_t(1);
        const size_t sm = size_t(kExpWarps) * (nb + ((size_t(Q) * R + 3) & ~size_t(3)) / 2) * sizeof(float2);
        const float2* prel = P->mf_prel.p;
        const int64_t *gs = P->gstart.p, *ge = P->gstop.p;
        const float* lr = P->mf_leaf_r.p;
        const float2* E = P->exp_E.p;
        const int64_t lb = P->leaf_begin;
        if (P->beta_tc) {
          // beta^ = E^ o for every leaf on the tensor cores (or already by the
          // fused leaf-level kernel), then the per-point series
          float* beta = reinterpret_cast<float*>(P->beta.p);
          if (!P->beta_fused) {
            tgemm_tc2_kernel<R><<<P->n_mom_units, 128, tc2_smem_bytes<R>(), s0>>>(
                P->mom_units.p, P->mom_ents.p, P->ETC.p, o, beta);
            nk++;
          }
          io_launch(
              P, reception_exp_kernel<R, true>, grid, 32 * kExpWarps, sm, s0,
              [=](const void*, void* pp) {
                return std::make_tuple(prel, gs, ge, lr, E, (const float*)beta, (const float*)base, pm,
                                       static_cast<float*>(pp), lb, nleaf, Q, nt, ldv);
              },
              q, phi);
        } else {
          io_launch(
              P, reception_exp_kernel<R, false>, grid, 32 * kExpWarps, sm, s0,
              [=](const void*, void* pp) {
                return std::make_tuple(prel, gs, ge, lr, E, (const float*)o, (const float*)base, pm,
                                       static_cast<float*>(pp), lb, nleaf, Q, nt, ldv);
              },
              q, phi);
        }
        nk++;
      } else {
        // float64: the expansion in float64 (reception_exp64_kernel)
        const int64_t nleaf = P->leaf_end - P->leaf_begin;
        const int grid = int(std::max<int64_t>(
            1, std::min<int64_t>((nleaf + kExpWarps - 1) / kExpWarps, int64_t(kExpCtasPerSM) * P->n_sm)));
        const int nt = P->u_nt;
        const size_t sm = size_t(kExpWarps) * (size_t(nt + 1) * R + (size_t(Q) * R + 1) / 2) * sizeof(double2);
        const double2* prel = P->mf_prel64.p;
        const int64_t *gs = P->gstart.p, *ge = P->gstop.p;
        const double* lr = P->mf_leaf_r64.p;
        const double2* E = P->exp_E64.p;
        const int64_t lb = P->leaf_begin;
        io_launch(
            P, reception_exp64_kernel<R>, grid, 32 * kExpWarps, sm, s0,
            [=](const void*, void* pp) {
              return std::make_tuple(prel, gs, ge, lr, E, (const double*)o, (const double*)base, pm,
                                     static_cast<double*>(pp), lb, nleaf, Q, nt, ldv);
            },
            q, phi);
        nk++;
      }
    } else if (far && P->cnear) {
      // complex U row-split (Track B): one complex column
      const DevBlockSet& U = P->Uset;
      if constexpr (R == 1) {
        if (U.n_items > 0) {
          io_launch(
              P, blockgemv_kernel<T, 2, kModeScatterCplx>, U.grid, kBGThreads,
              blockgemv_smem_bytes<T, 2, kModeScatterCplx>(), s0,
              [=, &U](const void*, void* pp) {
                return std::make_tuple(
                    blockgemv_args<T, 2, kModeScatterCplx>(U, o, static_cast<T*>(pp), base, pm, ldv));
              },
              q, phi);
          nk++;
        }
      }
    } else if (far) {
      const DevBlockSet& U = P->Uset;
      if (U.n_items > 0) {
        io_launch(
            P, blockgemv_kernel<T, R, kModeScatter>, U.grid, kBGThreads,
            blockgemv_smem_bytes<T, R, kModeScatter>(), s0,
            [=, &U](const void*, void* pp) {
              return std::make_tuple(blockgemv_args<T, R, kModeScatter>(U, o, static_cast<T*>(pp), base, pm, ldv));
            },
            q, phi);
        nk++;
      }
    } else {
      const int64_t pb = P->pt_begin;
      io_launch(
          P, scatter_kernel<T, R>, grid_for(nloc, 256, cap), 256, 0, s0,
          [=](const void*, void* pp) {
            return std::make_tuple(base, (const T*)nullptr, pm, static_cast<T*>(pp), pb, nloc, ldv);
          },
          q, phi);
      nk++;
    }
    tr("finish", s0);
    prof_mark(P, prof, 2 * NESA_STAGE_RECEPTION + 1, s0);
  };
  auto fork_near = [&]() {
    CUDA_OK(cudaEventRecord(P->ev_fork, s0));
    CUDA_OK(cudaStreamWaitEvent(s1, P->ev_fork, 0));
    if (!near) return;
    prof_mark(P, profn, 2 * NESA_STAGE_NEAR, s1);
    if (P->cnear) {
      // complex operator row-split: one complex column (R = 1 embedded)
      if constexpr (R == 1) launch_near_cplx<T>(P->nearset, qt, phin, s1);
    } else {
      launch_near<T, R>(P->nearset, qt, phin, s1);
    }
    nk++;
    prof_mark(P, profn, 2 * NESA_STAGE_NEAR + 1, s1);
    tr("near", s1);
  };
  auto join_near = [&]() {
    CUDA_OK(cudaEventRecord(P->ev_join, s1));
    CUDA_OK(cudaStreamWaitEvent(s0, P->ev_join, 0));
  };

  // halo exchange of a distributed plan (nesa_plan_create_dist): pack the
  // partials other ranks need, all_gather them over NCCL (captured into
  // this graph), complete the needed groups' s in rank order
  auto exchange = [&]() {
    const int qr = Q * R;
    T* send = reinterpret_cast<T*>(P->x_send.p);
    T* recv = reinterpret_cast<T*>(P->x_recv.p);
    const int64_t rows = P->x_max_export;
    xpack_kernel<T><<<grid_for(rows * qr, 256, 4096), 256, 0, s0>>>(s, P->x_export.p, P->x_n_export, rows, qr,
                                                                      send);
    NCCL_OK(nccl().allGather(send, recv, size_t(rows) * qr, sizeof(T) == 8 ? ncclFloat64 : ncclFloat32,
                             P->comm, s0));
    if (P->x_n_import > 0)
      xcombine_kernel<T><<<grid_for(P->x_n_import * qr, 256, 4096), 256, 0, s0>>>(
          s, recv, P->x_import.p, P->x_contrib.p, P->x_n_import, P->x_max_contrib, P->nranks * rows, qr);
    nk += 2;
    tr("exchange", s0);
  };

  if (stage == 0 && P->comm) {
    // distributed product, one graph per rank: gather -> fork {near (local
    // leaves) | radiation, upward pass -> halo exchange -> translation,
    // downward pass} -> join -> reception of the local points
    prof_mark(P, prof, 2 * NESA_STAGE_TOTAL, s0);
    gather();
    fork_near();
    if (far) {
      nk += launch_radiation<T, R>(P, qt, s, s0);
      up_pass(false);
      exchange();
      down_pass(false);
    }
    join_near();
    finish();
    prof_mark(P, prof, 2 * NESA_STAGE_TOTAL + 1, s0);
  } else if (stage == 0) {
    // gather -> fork {near | radiation, up, translate, down} -> join ->
    // reception
    prof_mark(P, prof, 2 * NESA_STAGE_TOTAL, s0);
    gather();
    // the radiation from outgoing moments is compute-bound: fork the near
    // field first (A/B: 5 us faster); stored V blocks stream from HBM like
    // the near operator, so they go first and the near field streams
    // beside the latency-bound chain that follows
    const bool v_first = far && !P->v_mom;
    if (!v_first) fork_near();
    if (far) {
      prof_mark(P, prof, 2 * NESA_STAGE_FAR, s0);
      nk += launch_radiation<T, R>(P, qt, s, s0);
      tr("radiation", s0);
    }
    if (v_first) fork_near();
    if (far) {
      const bool fine = up_pass(true);
      down_pass(fine);
      prof_mark(P, prof, 2 * NESA_STAGE_FAR + 1, s0);
    }
    join_near();
    finish();
    prof_mark(P, prof, 2 * NESA_STAGE_TOTAL + 1, s0);
  } else if (stage == 1) {
    // multi-GPU stage 1: the near field (local leaves) runs beside the
    // radiation and the upward pass, before the halo exchange; stage 2 is
    // the far field's second half and the reception
    gather();
    fork_near();
    if (far) {
      nk += launch_radiation<T, R>(P, qt, s, s0);
      up_pass(false);
    }
    join_near();
  } else {
    if (far) down_pass(false);
    finish();
  }
  return nk;
}

template <typename T>
int enqueue_dispatch(nesa_plan* P, const void* q, void* phi, int R, int ldv, uint32_t flags, int stage) {
  switch (R) {
    case 1:
      set_smem_attrs<T, 1>();
      return enqueue_T<T, 1>(P, static_cast<const T*>(q), static_cast<T*>(phi), ldv, flags, stage);
    case 2:
      set_smem_attrs<T, 2>();
      return enqueue_T<T, 2>(P, static_cast<const T*>(q), static_cast<T*>(phi), ldv, flags, stage);
    case 4:
      set_smem_attrs<T, 4>();
      return enqueue_T<T, 4>(P, static_cast<const T*>(q), static_cast<T*>(phi), ldv, flags, stage);
    default:
      throw NesaError(NESA_ERR_UNSUPPORTED, "nrhs * (1 + is_complex) must be 1, 2 or 4");
  }
}

int run_block(nesa_plan* P, const void* q, void* phi, int R, int ldv, uint32_t flags, void* stream,
              int stage);

bool near_wide_ok(const nesa_plan* P) { return P->dtype == NESA_F32 && P->near_tc && P->ntc_n > 0; }

// phi[:, col0 : col0 + ncols] += near(q) for real columns of (N, ld) blocks in
// original order, 128 columns per tensor-core pass (stream-ordered)
void run_near_wide(nesa_plan* P, const void* q, void* phi, int ld, int col0, int ncols, cudaStream_t st,
                   bool accumulate = true) {
  require(near_wide_ok(P), "the wide near field needs a float32 plan with tensor cores");
  require(ld >= 1 && col0 >= 0 && ncols >= 1 && col0 + ncols <= ld, "bad column range");
  CUDA_OK(cudaSetDevice(P->device));
  if (!P->ntc_blob.p) {
    P->ntc_blob.alloc(size_t(std::max<int64_t>(P->ntc_floats, 1)));
    near_tc_pack_kernel<<<P->ntc_n, 256>>>(P->ntc_items.p, reinterpret_cast<const float*>(P->nearset.blob.p),
                                           P->ntc_blob.p);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaFuncSetAttribute(near_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(near_tc_smem_bytes())));
  }
  const int grid = std::min(P->ntc_n, 2 * P->n_sm);
  for (int c = col0; c < col0 + ncols; c += 128) {
    const int nc = std::min(128, col0 + ncols - c);
    near_tc_kernel<<<grid, 128, near_tc_smem_bytes(), st>>>(
        P->ntc_items.p, P->ntc_n, P->ntc_src.p, P->ntc_blob.p, static_cast<const float*>(q), ld, c, nc,
        P->perm.p, static_cast<float*>(phi), accumulate ? 1 : 0);
    CUDA_OK(cudaGetLastError());
  }
}

// Far field of real columns [col0, col0 + ncols) (ncols <= kWCols) of
// (N, ld) row-major blocks in original order as batched GEMMs (wgemm_kernel):
// phi[:, cols] = far field (stored, not accumulated).  Stream-ordered.
template <typename T, int NC, int KG, int TR>
void launch_wgemm(const WArgs<T>& a, int mode, int64_t n, cudaStream_t st) {
  using W = WTile<T, NC, KG, TR>;
  static bool attr = false;
  if (!attr) {
    for (auto* f : {wgemm_kernel<T, kWStore, NC, KG, TR>, wgemm_kernel<T, kWScatter, NC, KG, TR>,
                    wgemm_kernel<T, kWScatterAdd, NC, KG, TR>})
      CUDA_OK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(W::kSmem)));
    attr = true;
  }
  const dim3 grid(unsigned(n), kWCols / NC);
  if (mode == kWStore)
    wgemm_kernel<T, kWStore, NC, KG, TR><<<grid, W::kThreads, W::kSmem, st>>>(a);
  else if (mode == kWScatter)
    wgemm_kernel<T, kWScatter, NC, KG, TR><<<grid, W::kThreads, W::kSmem, st>>>(a);
  else
    wgemm_kernel<T, kWScatterAdd, NC, KG, TR><<<grid, W::kThreads, W::kSmem, st>>>(a);
  CUDA_OK(cudaGetLastError());
}

template <typename T>
void run_far_wide_T(nesa_plan* P, const void* q, void* phi, int ld, int col0, int ncols, cudaStream_t st,
                    bool reception, bool rec_add) {
  const size_t es = sizeof(T);
  if (!P->w_s.p) {
    P->w_s.alloc(size_t(P->G) * P->Q * kWCols * es);
    P->w_o.alloc(size_t(P->G) * P->Q * kWCols * es);
  }
  T* s = reinterpret_cast<T*>(P->w_s.p);
  T* o = reinterpret_cast<T*>(P->w_o.p);
  WArgs<T> a{};
  a.terms = P->w_terms.p;
  a.abase[0] = reinterpret_cast<const T*>(P->CT.p);
  a.abase[1] = reinterpret_cast<const T*>(P->BT.p);
  a.abase[2] = reinterpret_cast<const T*>(P->DT.p);
  a.abase[3] = reinterpret_cast<const T*>(P->Vset.blob.p);
  a.abase[4] = reinterpret_cast<const T*>(P->Uset.blob.p);
  a.xs[0] = nullptr;
  a.xs[1] = s;
  a.xs[2] = o;
  a.perm = P->perm.p;
  a.q = static_cast<const T*>(q);
  a.ldy = ld;
  a.col0 = col0;
  a.ncols = ncols;
  a.vec4 = (size_t(ld) * es) % 16 == 0 && (size_t(col0) * es) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(q) % 16 == 0;
  for (const auto& S : P->w_stages) {
    if (S.end <= S.begin || (S.ysel == 2) != reception) continue;
    a.items = P->w_items.p + S.begin;
    a.y = S.ysel == 0 ? s : (S.ysel == 1 ? o : static_cast<T*>(phi));
    const int mode = S.ysel < 2 ? kWStore : (rec_add ? kWScatterAdd : kWScatter);
    const int64_t n = S.end - S.begin;
    // coarse levels (few items, many terms): 32-column blocks, terms split
    // over 4 thread groups; wide levels: one CTA per 64 x 128 tile
    if (n < 2 * P->n_sm)
      launch_wgemm<T, 32, 4, 4>(a, mode, n, st);
    else
      launch_wgemm<T, 128, 1, 8>(a, mode, n, st);
  }
}

// One product of nrhs right-hand sides: real columns are processed in blocks
// of <= 4 (one captured graph per block width; rows of q / phi keep their stride).
int run_matvec(nesa_plan* P, const void* q, void* phi, int32_t nrhs, int32_t is_complex,
               uint32_t flags, void* stream, int stage) {
  require(P != nullptr, "null plan");
  require(nrhs >= 1, "nrhs must be >= 1");
  require(q != nullptr && phi != nullptr, "null vector");
  require(stage == 0 || !(flags & NESA_PROFILE), "profiling needs a full product");
  const int Rt = nrhs * (is_complex ? 2 : 1);
  if (P->cnear) {
    // complex near field: one (embedded) column per block
    require(!is_complex, "an embedded complex plan takes real (embedded) vectors");
    for (int c = 0; c < Rt; ++c)
      run_block(P, static_cast<const char*>(q) + c * P->esz, static_cast<char*>(phi) + c * P->esz, 1, Rt,
                flags, stream, stage);
    return NESA_OK;
  }
  if (Rt == 1 || Rt == 2 || Rt == 4) return run_block(P, q, phi, Rt, Rt, flags, stream, stage);
  require(stage == 0, "the staged (multi-GPU) product takes at most 4 real columns");
  require(!(flags & NESA_PROFILE), "profiling takes at most 4 real columns");
  const size_t es = P->esz;
  if ((flags & NESA_FAR) && P->wide_far && P->comm == nullptr && (!(flags & NESA_NEAR) || near_wide_ok(P))) {
    // many right-hand sides: the near field's tensor-core GEMM (storing phi)
    // on a side stream, concurrently with the far field as batched GEMMs
    // over 128-column passes up to o; the reception then adds U o to phi
    CUDA_OK(cudaSetDevice(P->device));
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool near = (flags & NESA_NEAR) != 0;
    if (!P->w_ev_fork) {
      CUDA_OK(cudaEventCreateWithFlags(&P->w_ev_fork, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&P->w_ev_near, cudaEventDisableTiming));
    }
    if (near) {
      CUDA_OK(cudaEventRecord(P->w_ev_fork, st));
      CUDA_OK(cudaStreamWaitEvent(P->s1, P->w_ev_fork, 0));
      for (int c0 = 0; c0 < Rt; c0 += kWCols)
        run_near_wide(P, q, phi, Rt, c0, std::min(kWCols, Rt - c0), P->s1, /*accumulate=*/false);
      CUDA_OK(cudaEventRecord(P->w_ev_near, P->s1));
    }
    for (int c0 = 0; c0 < Rt; c0 += kWCols) {
      const int nc = std::min(kWCols, Rt - c0);
      for (int part = 0; part < 2; ++part) {
        if (part == 1 && c0 == 0 && near) CUDA_OK(cudaStreamWaitEvent(st, P->w_ev_near, 0));
        if (P->dtype == NESA_F64)
          run_far_wide_T<double>(P, q, phi, Rt, c0, nc, st, part == 1, near);
        else
          run_far_wide_T<float>(P, q, phi, Rt, c0, nc, st, part == 1, near);
      }
    }
    return NESA_OK;
  }
  // float32 with tensor cores: the far field in blocks of <= 4 columns, then
  // the near field ONCE for all columns (tcgen05 GEMM, operator read once)
  const bool wide = (flags & NESA_NEAR) && near_wide_ok(P) && P->comm == nullptr;
  const uint32_t bflags = wide ? (flags & ~NESA_NEAR) : flags;
  for (int c0 = 0; c0 < Rt;) {
    const int Rb = Rt - c0 >= 4 ? 4 : (Rt - c0 >= 2 ? 2 : 1);
    run_block(P, static_cast<const char*>(q) + c0 * es, static_cast<char*>(phi) + c0 * es, Rb, Rt,
              bflags, stream, stage);
    c0 += Rb;
  }
  if (wide) run_near_wide(P, q, phi, Rt, 0, Rt, static_cast<cudaStream_t>(stream));
  return NESA_OK;
}

int run_block(nesa_plan* P, const void* q, void* phi, int R, int ldv, uint32_t flags, void* stream,
              int stage) {
  CUDA_OK(cudaSetDevice(P->device));
  require(!(P->far_only && (flags & NESA_NEAR)), "this plan was created without the near field (NESA_PLAN_FAR_ONLY)");
  // the workspace for the widest block so far (growing it drops every graph)
  if (P->dtype == NESA_F64)
    ensure_workspace<double>(P, R);
  else
    ensure_workspace<float>(P, R);
  nesa_plan::GraphKey key{R, flags & (NESA_NEAR | NESA_FAR | NESA_PROFILE | NESA_PROFILE_NEAR), stage, ldv};
  auto itg = P->graphs.find(key);
  if (itg != P->graphs.end() && itg->second.gen != P->ws_gen) {  // (cannot happen: growth drops all)
    if (itg->second.exec) cudaGraphExecDestroy(itg->second.exec);
    if (itg->second.graph) cudaGraphDestroy(itg->second.graph);
    P->graphs.erase(itg);
    itg = P->graphs.end();
  }
  if (itg == P->graphs.end()) {
    nesa_plan::GraphEntry ent;
    cudaGraph_t g = nullptr;
    CUDA_OK(cudaStreamBeginCapture(P->s0, cudaStreamCaptureModeThreadLocal));
    int nk = 0;
    P->capturing_io = &ent.io;
    try {
      nk = P->dtype == NESA_F64 ? enqueue_dispatch<double>(P, q, phi, R, ldv, flags, stage)
                                : enqueue_dispatch<float>(P, q, phi, R, ldv, flags, stage);
    } catch (...) {
      P->capturing_io = nullptr;
      cudaStreamEndCapture(P->s0, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    P->capturing_io = nullptr;
    CUDA_OK(cudaStreamEndCapture(P->s0, &g));
    ent.graph = g;
    CUDA_OK(cudaGraphInstantiate(&ent.exec, g, 0));
    if (flags & NESA_PROFILE) {
      size_t n = 0;
      CUDA_OK(cudaGraphGetNodes(g, nullptr, &n));
      std::vector<cudaGraphNode_t> nodes(n);
      CUDA_OK(cudaGraphGetNodes(g, nodes.data(), &n));
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        CUDA_OK(cudaGraphNodeGetType(nd, &ty));
        if (ty != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev;
        CUDA_OK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
        for (int slot = 0; slot < 2 * NESA_N_STAGES + kTraceSlots; ++slot)
          if (P->cap_events[slot] == ev) ent.ev_nodes.emplace_back(nd, slot);
      }
    }
    ent.q = q;
    ent.phi = phi;
    ent.gen = P->ws_gen;
    P->graph_captures++;
    if (stage == 0 && (flags & NESA_NEAR) && (flags & NESA_FAR)) P->kernels_per_matvec = nk;  // full product
    itg = P->graphs.emplace(key, std::move(ent)).first;
  }
  nesa_plan::GraphEntry& ge = itg->second;
  if (ge.q != q || ge.phi != phi) {
    // same schedule, other caller buffers: re-point the io nodes
    for (auto& io : ge.io) CUDA_OK(io.apply(ge.exec, io.node, q, phi));
    ge.q = q;
    ge.phi = phi;
  }
  if (flags & NESA_PROFILE) {
    if (P->prof_used == P->prof_events.size()) {
      std::vector<cudaEvent_t> evs(2 * NESA_N_STAGES + kTraceSlots);
      for (auto& e : evs) CUDA_OK(cudaEventCreate(&e));
      P->prof_events.push_back(evs);
    }
    auto& evs = P->prof_events[P->prof_used++];
    for (auto& pr : ge.ev_nodes) CUDA_OK(cudaGraphExecEventRecordNodeSetEvent(ge.exec, pr.first, evs[pr.second]));
  }
  CUDA_OK(cudaGraphLaunch(ge.exec, static_cast<cudaStream_t>(stream)));
  return NESA_OK;
}

}  // namespace

#define NESA_API extern "C" __attribute__((visibility("default")))

#define NESA_GUARD(body)                              \
  try {                                               \
    body;                                             \
  } catch (const NesaError& e) {                      \
    g_last_error = e.what();                          \
    return e.code;                                    \
  } catch (const std::exception& e) {                 \
    g_last_error = e.what();                          \
    return NESA_ERR_INVALID;                          \
  }

nesa_plan* plan_create_impl(const nesa_plan_desc* d, int device, void* comm, int rank, int nranks,
                            const nesa_exchange_desc* xd);

NESA_API int nesa_plan_create(const nesa_plan_desc* d, int device, nesa_plan** out) {
  NESA_GUARD({
    require(out != nullptr, "null argument");
    *out = nullptr;
    *out = plan_create_impl(d, device, nullptr, 0, 1, nullptr);
    return NESA_OK;
  })
}

NESA_API int nesa_plan_create_dist(const nesa_plan_desc* d, int device, void* nccl_comm, int32_t rank,
                                   int32_t nranks, const nesa_exchange_desc* xd, nesa_plan** out) {
  NESA_GUARD({
    require(out != nullptr && nccl_comm != nullptr && xd != nullptr, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    *out = nullptr;
    *out = plan_create_impl(d, device, nccl_comm, rank, nranks, xd);
    return NESA_OK;
  })
}

NESA_API int nesa_nccl_unique_id(void* out, int32_t bytes) {
  NESA_GUARD({
    require(out != nullptr && bytes >= int32_t(sizeof(ncclUniqueId)), "need a 128-byte buffer");
    ncclUniqueId id;
    NCCL_OK(nccl().getUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return NESA_OK;
  })
}

NESA_API int nesa_nccl_comm_init(const void* unique_id, int32_t nranks, int32_t rank, int32_t device,
                                 void** comm_out) {
  NESA_GUARD({
    require(unique_id != nullptr && comm_out != nullptr, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    CUDA_OK(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t c = nullptr;
    NCCL_OK(nccl().commInitRank(&c, nranks, id, rank));
    *comm_out = c;
    return NESA_OK;
  })
}

NESA_API int nesa_nccl_comm_destroy(void* comm) {
  NESA_GUARD({
    if (comm) NCCL_OK(nccl().commDestroy(static_cast<ncclComm_t>(comm)));
    return NESA_OK;
  })
}

nesa_plan* plan_create_impl(const nesa_plan_desc* d, int device, void* comm, int rank, int nranks,
                            const nesa_exchange_desc* xd) {
  {
    require(d != nullptr, "null argument");
    require(d->abi_version == NESA_ABI_VERSION, "ABI version mismatch");
    require(d->op_dtype == NESA_F64 || d->op_dtype == NESA_F32, "op_dtype must be F64 or F32");
    require(d->Q >= 3 && d->Q <= 256, "Q must be in [3, 256]");
    require(d->N >= 1 && d->n_leaves >= 1 && d->n_groups >= d->n_leaves, "bad sizes");
    require(d->L >= d->l0 && d->l0 >= 0, "bad levels");
    require(d->N < (int64_t(1) << 31), "N must fit in int32");
    require(d->perm && d->group_start && d->group_stop && d->parent && d->quad && d->level_first &&
                d->level_count && d->nbr_ptr && d->nbr_idx && d->int_ptr && d->int_idx &&
                d->int_dtab && d->D,
            "missing tree / table arrays");
    require(d->L == d->l0 || (d->C && d->B), "missing C/B tables");
    std::unique_ptr<nesa_plan> P(new nesa_plan());
    P->device = device;
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaDeviceGetAttribute(&P->n_sm, cudaDevAttrMultiProcessorCount, device));
    P->dtype = d->op_dtype;
    P->esz = d->op_dtype == NESA_F64 ? 8 : 4;
    P->Q = d->Q;
    P->n_check = d->n_check;
    P->l0 = d->l0;
    P->L = d->L;
    P->N = d->N;
    P->NL = d->n_leaves;
    P->G = d->n_groups;
    if (const char* wl = std::getenv("NESA_WIDE_LEVEL")) P->wide_level = std::atoll(wl);
    if (const char* tc = std::getenv("NESA_TC")) P->tc = std::atoi(tc) != 0;
    P->u_mf = !d->U_blob;
    if (const char* us = std::getenv("NESA_U_STORED")) P->u_mf = P->u_mf && std::atoi(us) == 0;
    P->v_mom = d->op_dtype == NESA_F32 && !d->V_blob;
    if (const char* vs = std::getenv("NESA_V_STORED")) P->v_mom = P->v_mom && std::atoi(vs) == 0;
    if (d->options & NESA_PLAN_STORED_VU) {
      // many right-hand sides: stored V / U blocks (assembled on the device),
      // the far field then runs as batched GEMMs over all columns
      P->v_mom = false;
      P->u_mf = false;
    }
    if (const char* tr = std::getenv("NESA_TRACE")) P->trace = std::atoi(tr) != 0;
    P->leaf_begin = d->leaf_begin;
    P->leaf_end = d->leaf_end;
    P->far_only = (d->options & NESA_PLAN_FAR_ONLY) != 0;
    if (d->options & NESA_PLAN_OCTREE) {
      // Track B: octree (8 child kinds), operators from the host.  The
      // quadtree-specialised tensor-core kernels (levels, translation) and
      // the circle expansions do not apply; wide levels use the warp-tiled
      // FFMA kernels (per child kind, 8 matrices per level), the coarse
      // levels the fused kernels.
      P->nkind = 8;
      P->tc = false;
      require(d->V_blob && d->U_blob &&
                  (d->near_blob || P->far_only ||
                   ((d->options & NESA_PLAN_HELMHOLTZ_NEAR) && (d->options & NESA_PLAN_COMPLEX_NEAR) && d->points3)),
              "octree plans take their near (or NESA_PLAN_HELMHOLTZ_NEAR points) / V / U blocks from the host");
    }
    P->cnear = (d->options & NESA_PLAN_COMPLEX_NEAR) != 0;
    if (P->cnear) {
      require((d->near_blob || ((d->options & NESA_PLAN_HELMHOLTZ_NEAR) && d->points3)) && !P->far_only,
              "NESA_PLAN_COMPLEX_NEAR needs a near blob or NESA_PLAN_HELMHOLTZ_NEAR points");
      for (int64_t g = 0; g < d->n_leaves; ++g)
        require(d->group_start[g] % 2 == 0 && d->group_stop[g] % 2 == 0,
                "NESA_PLAN_COMPLEX_NEAR needs embedded (even) point ranges");
    }
    for (int64_t g = 0; g < d->n_groups; ++g)
      require(d->quad[g] >= 0 && d->quad[g] < P->nkind, "child kind out of range");
    if (P->leaf_end <= P->leaf_begin) {
      P->leaf_begin = 0;
      P->leaf_end = P->NL;
    }
    require(P->leaf_begin >= 0 && P->leaf_end <= P->NL, "leaf range out of bounds");
    P->pt_begin = d->group_start[P->leaf_begin];
    P->pt_end = d->group_stop[P->leaf_end - 1];
    const int nlev = P->L - P->l0 + 1;
    P->lvl_first.assign(d->level_first, d->level_first + nlev);
    P->lvl_count.assign(d->level_count, d->level_count + nlev);
    require(P->lvl_first[nlev - 1] == 0 && P->lvl_count[nlev - 1] == P->NL,
            "leaves must be ids 0..n_leaves-1");
    if (P->dtype == NESA_F64)
      build_plan_T<double>(P.get(), d);
    else
      build_plan_T<float>(P.get(), d);
    // graph replays do not apply stream priorities (equal-priority streams
    // measured fastest for this schedule)
    CUDA_OK(cudaStreamCreateWithFlags(&P->s0, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&P->s1, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&P->s2, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&P->s3, cudaStreamNonBlocking));
    for (int i = 0; i < P->L - P->l0 + 1; ++i) {
      cudaEvent_t a = nullptr, b = nullptr;
      CUDA_OK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      P->ev_s_lv.push_back(a);
      P->ev_t_lv.push_back(b);
    }
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_tx, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming));
    for (auto& e : P->cap_events) CUDA_OK(cudaEventCreate(&e));
    if (comm) {
      // the plan uses (does not own) the caller's communicator
      P->comm = static_cast<ncclComm_t>(comm);
      P->rank = rank;
      P->nranks = nranks;
      require(xd->n_export >= 0 && xd->max_export >= std::max<int64_t>(1, xd->n_export) &&
                  xd->n_import >= 0 && xd->max_contrib >= 1,
              "bad exchange descriptor");
      P->x_n_export = xd->n_export;
      P->x_max_export = xd->max_export;
      P->x_n_import = xd->n_import;
      P->x_max_contrib = xd->max_contrib;
      const int64_t n_recv = int64_t(nranks) * xd->max_export;
      std::vector<int64_t> ex(xd->export_ids, xd->export_ids + xd->n_export);
      std::vector<int64_t> im(xd->import_ids, xd->import_ids + xd->n_import);
      std::vector<int64_t> ct(xd->contrib, xd->contrib + xd->n_import * xd->max_contrib);
      for (auto v : ex) require(v >= 0 && v < P->G, "export id out of range");
      for (auto v : im) require(v >= 0 && v < P->G, "import id out of range");
      for (auto v : ct) require(v >= -1 && v < n_recv + P->G, "contribution row out of range");
      P->x_export.upload(ex);
      P->x_import.upload(im);
      P->x_contrib.upload(ct);
    }
    return P.release();
  }
}

NESA_API int nesa_matvec(nesa_plan* plan, const void* q_dev, void* phi_dev, int32_t nrhs,
                         int32_t is_complex, uint32_t flags, void* stream) {
  NESA_GUARD(return run_matvec(plan, q_dev, phi_dev, nrhs, is_complex, flags, stream, 0));
}

int run_cols(nesa_plan* P, const void* q, void* phi, int32_t ld, int32_t col0, int32_t ncols,
             uint32_t flags, void* stream) {
  require(P != nullptr, "null plan");
  require(q != nullptr && phi != nullptr, "null vector");
  require(ld >= 1 && col0 >= 0 && ncols >= 1 && col0 + ncols <= ld, "bad column range");
  require(!(flags & NESA_PROFILE), "profiling takes one block");
  const size_t es = P->esz;
  for (int c0 = col0; c0 < col0 + ncols;) {
    const int left = col0 + ncols - c0;
    const int Rb = left >= 4 ? 4 : (left >= 2 ? 2 : 1);
    run_block(P, static_cast<const char*>(q) + c0 * es, static_cast<char*>(phi) + c0 * es, Rb, ld,
              flags, stream, 0);
    c0 += Rb;
  }
  return NESA_OK;
}

NESA_API int nesa_matvec_near_wide(nesa_plan* plan, const void* q_dev, void* phi_dev, int32_t ld_real,
                                   int32_t col0, int32_t ncols_real, void* stream) {
  NESA_GUARD({
    require(plan != nullptr && q_dev != nullptr && phi_dev != nullptr, "null argument");
    run_near_wide(plan, q_dev, phi_dev, ld_real, col0, ncols_real, static_cast<cudaStream_t>(stream));
    return NESA_OK;
  })
}

NESA_API int nesa_matvec_cols(nesa_plan* plan, const void* q_dev, void* phi_dev, int32_t ld_real,
                              int32_t col0, int32_t ncols_real, uint32_t flags, void* stream) {
  NESA_GUARD(return run_cols(plan, q_dev, phi_dev, ld_real, col0, ncols_real, flags, stream));
}

NESA_API int nesa_matvec_stage(nesa_plan* plan, int32_t stage, const void* q_dev, void* phi_dev,
                               int32_t nrhs, int32_t is_complex, uint32_t flags, void* stream) {
  NESA_GUARD({
    require(stage == 1 || stage == 2, "stage must be 1 or 2");
    return run_matvec(plan, q_dev, phi_dev, nrhs, is_complex, flags, stream, stage);
  })
}

NESA_API void* nesa_plan_s_dev(nesa_plan* plan, int32_t nrhs_real) {
  try {
    if (!plan) return nullptr;
    CUDA_OK(cudaSetDevice(plan->device));
    if (plan->dtype == NESA_F64)
      ensure_workspace<double>(plan, nrhs_real);
    else
      ensure_workspace<float>(plan, nrhs_real);
    return plan->s.p;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return nullptr;
  }
}

NESA_API int nesa_plan_destroy(nesa_plan* plan) {
  NESA_GUARD({
    delete plan;
    return NESA_OK;
  })
}

// ---------------------------------------------------------------------------
// Exact O(N^2) potential sum on the GPU (dense.py:14-33): the approximation
// error oracle at sizes the CPU cannot reach.
// phi_i = sum_{j != i} -0.5 log(d2_ij) q_j with d2 = dx*dx + dy*dy formed
// without contraction as the reference's einsum does, float64 throughout.
// One thread per target; sources stream through shared memory in tiles.
// Coincident distinct points are counted (the reference raises ValueError).
// ---------------------------------------------------------------------------
namespace {
constexpr int kDenseTile = 256;

template <int R>
__global__ void __launch_bounds__(kDenseTile) dense_kernel(const double* __restrict__ pts,
                                                           const double* __restrict__ q,
                                                           double* __restrict__ phi, int64_t n,
                                                           unsigned long long* coincident) {
  __shared__ double sx[kDenseTile], sy[kDenseTile], sq[kDenseTile * R];
  const int64_t i = int64_t(blockIdx.x) * kDenseTile + threadIdx.x;
  const bool live = i < n;
  const double xi = live ? pts[2 * i] : 0.0, yi = live ? pts[2 * i + 1] : 0.0;
  double acc[R];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) acc[rr] = 0.0;
  unsigned long long bad = 0;
  for (int64_t j0 = 0; j0 < n; j0 += kDenseTile) {
    const int64_t j = j0 + threadIdx.x;
    __syncthreads();
    if (j < n) {
      sx[threadIdx.x] = pts[2 * j];
      sy[threadIdx.x] = pts[2 * j + 1];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) sq[threadIdx.x * R + rr] = q[j * R + rr];
    }
    __syncthreads();
    const int m = n - j0 < kDenseTile ? int(n - j0) : kDenseTile;
    if (!live) continue;
    for (int t = 0; t < m; ++t) {
      if (j0 + t == i) continue;
      const double dx = __dsub_rn(xi, sx[t]), dy = __dsub_rn(yi, sy[t]);
      const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      if (d2 == 0.0) {
        ++bad;
        continue;
      }
      const double k = -0.5 * log(d2);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[rr] = fma(k, sq[t * R + rr], acc[rr]);
    }
  }
  if (live) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) phi[i * R + rr] = acc[rr];
  }
  if (bad) atomicAdd(coincident, bad);
}
}  // namespace

int dense_run(const double* points_dev, const double* q_dev, double* phi_dev, int64_t n,
              int32_t ncols, void* stream) {
  require(n >= 2, "n must be >= 2");
  require(points_dev && q_dev && phi_dev, "null pointer");
  require(ncols >= 1 && ncols <= 4, "ncols must be 1..4 (real columns; complex = 2)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* cnt = nullptr;
  CUDA_OK(cudaMallocAsync(&cnt, sizeof(unsigned long long), st));
  CUDA_OK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
  const int grid = int((n + kDenseTile - 1) / kDenseTile);
  if (ncols == 1)
    dense_kernel<1><<<grid, kDenseTile, 0, st>>>(points_dev, q_dev, phi_dev, n, cnt);
  else if (ncols == 2)
    dense_kernel<2><<<grid, kDenseTile, 0, st>>>(points_dev, q_dev, phi_dev, n, cnt);
  else if (ncols == 3)
    dense_kernel<3><<<grid, kDenseTile, 0, st>>>(points_dev, q_dev, phi_dev, n, cnt);
  else
    dense_kernel<4><<<grid, kDenseTile, 0, st>>>(points_dev, q_dev, phi_dev, n, cnt);
  CUDA_OK(cudaGetLastError());
  unsigned long long h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  CUDA_OK(cudaFree(cnt));
  require(h == 0, "coincident points");
  return NESA_OK;
}

NESA_API int nesa_dense_matvec(const double* points_dev, const double* q_dev, double* phi_dev,
                               int64_t n, int32_t ncols, void* stream) {
  NESA_GUARD(return dense_run(points_dev, q_dev, phi_dev, n, ncols, stream));
}

// ---------------------------------------------------------------------------
// Multi-GPU halo exchange as separate calls (the CPU-side dist layer's path)
// ---------------------------------------------------------------------------
namespace {
int xpack_run(const void* s, const int64_t* ids, int64_t n_ids, int64_t rows, int32_t qr, int32_t f64,
              void* send, void* stream) {
  require(s && send && (ids || n_ids == 0) && rows >= n_ids && qr > 0, "bad exchange pack arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>((rows * qr + 255) / 256, 4096)));
  if (f64)
    xpack_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(s), ids, n_ids, rows, qr,
                                               static_cast<double*>(send));
  else
    xpack_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(s), ids, n_ids, rows, qr,
                                              static_cast<float*>(send));
  CUDA_OK(cudaGetLastError());
  return NESA_OK;
}

int xcombine_run(void* s, const void* recv, const int64_t* imp, const int64_t* contrib, int64_t n_imp,
                 int32_t max_c, int64_t n_recv, int32_t qr, int32_t f64, void* stream) {
  require(s && recv && qr > 0 && max_c >= 1 && (n_imp == 0 || (imp && contrib)), "bad exchange combine arguments");
  if (n_imp == 0) return NESA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>((n_imp * qr + 255) / 256, 4096)));
  if (f64)
    xcombine_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(s), static_cast<const double*>(recv),
                                                  imp, contrib, n_imp, max_c, n_recv, qr);
  else
    xcombine_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(s), static_cast<const float*>(recv),
                                                 imp, contrib, n_imp, max_c, n_recv, qr);
  CUDA_OK(cudaGetLastError());
  return NESA_OK;
}
}  // namespace

NESA_API int nesa_exchange_pack(const void* s_dev, const int64_t* export_ids_dev, int64_t n_export,
                                int64_t send_rows, int32_t qr, int32_t is_f64, void* send_dev,
                                void* stream) {
  NESA_GUARD(return xpack_run(s_dev, export_ids_dev, n_export, send_rows, qr, is_f64, send_dev, stream));
}

NESA_API int nesa_exchange_combine(void* s_dev, const void* recv_dev, const int64_t* import_ids_dev,
                                   const int64_t* contrib_dev, int64_t n_import, int32_t max_contrib,
                                   int64_t n_recv_rows, int32_t qr, int32_t is_f64, void* stream) {
  NESA_GUARD(return xcombine_run(s_dev, recv_dev, import_ids_dev, contrib_dev, n_import, max_contrib,
                                 n_recv_rows, qr, is_f64, stream));
}

NESA_API const char* nesa_last_error(void) { return g_last_error.c_str(); }

NESA_API int nesa_abi_version(void) { return NESA_ABI_VERSION; }

NESA_API int64_t nesa_plan_stat(nesa_plan* P, int32_t which) {
  if (!P) return -1;
  switch (which) {
    case NESA_STAT_NEAR_ENTRIES:
      return P->nearset.entries;
    case NESA_STAT_V_ENTRIES:
      return P->Vset.entries;
    case NESA_STAT_U_ENTRIES:
      return P->Uset.entries;
    case NESA_STAT_D_REFS:
      return P->d_refs;
    case NESA_STAT_N_DTAB:
      return P->n_dtab;
    case NESA_STAT_DEVICE_BYTES: {
      int64_t b = int64_t(P->nearset.blob.n + P->Vset.blob.n + P->Uset.blob.n + P->CT.n +
                          P->BT.n + P->DT.n + P->qt.n + P->phin.n + P->s.n + P->o.n);
      return b;
    }
    case NESA_STAT_NEAR_CTAS:
      return P->nearset.grid;
    case NESA_STAT_KERNELS_PER_MATVEC:
      return P->kernels_per_matvec;
    case NESA_STAT_V_MOMENTS:
      return P->v_mom ? P->v_nm : 0;
    case NESA_STAT_U_TERMS:
      return P->u_mf ? P->u_nt : 0;
    case NESA_STAT_GRAPH_CAPTURES:
      return P->graph_captures;
    case NESA_STAT_GRAPHS_CACHED:
      return int64_t(P->graphs.size());
    case NESA_STAT_NEAR_WIDE:
      return near_wide_ok(P) ? 1 : 0;
    case NESA_STAT_FAR_WIDE:
      return P->wide_far ? 1 : 0;
    default:
      return -1;
  }
}

NESA_API int nesa_profile_reset(nesa_plan* P) {
  NESA_GUARD({
    require(P != nullptr, "null plan");
    CUDA_OK(cudaSetDevice(P->device));
    CUDA_OK(cudaDeviceSynchronize());
    P->prof_used = 0;
    return NESA_OK;
  })
}

// Kernel timeline diagnostics (see KtScope in nesa_kernels.cuh): capacity
// records of {tag, grid, start_ns, end_ns}; capacity 0 turns it off.
namespace {
DevBuf<unsigned long long> g_kt_host_buf;
DevBuf<unsigned int> g_kt_host_cnt;
}  // namespace

NESA_API int nesa_ktrace_enable(nesa_plan* P, int64_t capacity) {
  NESA_GUARD({
    require(P != nullptr && capacity >= 0, "bad argument");
    CUDA_OK(cudaSetDevice(P->device));
    CUDA_OK(cudaDeviceSynchronize());
    unsigned long long* bp = nullptr;
    unsigned int* cp = nullptr;
    unsigned int cap = 0;
    if (capacity > 0) {
      g_kt_host_buf.alloc(size_t(capacity) * 4);
      g_kt_host_cnt.alloc(1);
      bp = g_kt_host_buf.p;
      cp = g_kt_host_cnt.p;
      cap = unsigned(capacity);
    }
    CUDA_OK(cudaMemcpyToSymbol(nesa::g_kt_buf, &bp, sizeof(bp)));
    CUDA_OK(cudaMemcpyToSymbol(nesa::g_kt_cnt, &cp, sizeof(cp)));
    CUDA_OK(cudaMemcpyToSymbol(nesa::g_kt_cap, &cap, sizeof(cap)));
    return NESA_OK;
  })
}

// Copies up to max_records records (4 x uint64 each) and resets the log;
// returns the number of records written (< 0: error).
NESA_API int64_t nesa_ktrace_read(nesa_plan* P, unsigned long long* out, int64_t max_records) {
  try {
    require(P != nullptr && out != nullptr, "null argument");
    CUDA_OK(cudaSetDevice(P->device));
    CUDA_OK(cudaDeviceSynchronize());
    if (!g_kt_host_cnt.p) return 0;
    unsigned int n = 0;
    CUDA_OK(cudaMemcpy(&n, g_kt_host_cnt.p, sizeof(n), cudaMemcpyDeviceToHost));
    const int64_t cnt = std::min<int64_t>({int64_t(n), max_records, int64_t(g_kt_host_buf.n / 4)});
    if (cnt > 0)
      CUDA_OK(cudaMemcpy(out, g_kt_host_buf.p, size_t(cnt) * 4 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemset(g_kt_host_cnt.p, 0, sizeof(unsigned int)));
    return cnt;
  } catch (const NesaError& e) {
    g_last_error = e.what();
    return -e.code;
  }
}

// Diagnostics (NESA_TRACE=1 plans, profiled products): time of the event
// after each traced kernel of the LAST profiled product, in ms from its start.
NESA_API int nesa_trace_read(nesa_plan* P, float* ms, int32_t max) {
  try {
    require(P != nullptr && ms != nullptr, "null argument");
    CUDA_OK(cudaSetDevice(P->device));
    CUDA_OK(cudaDeviceSynchronize());
    if (P->prof_used == 0) return 0;
    const auto& evs = P->prof_events[P->prof_used - 1];
    int n = 0;
    for (size_t i = 0; i < P->trace_names.size() && n < max; ++i) {
      float t = -1.f;
      if (cudaEventElapsedTime(&t, evs[2 * NESA_STAGE_TOTAL], evs[2 * NESA_N_STAGES + i]) != cudaSuccess) {
        cudaGetLastError();
        t = -1.f;
      }
      ms[n++] = t;
    }
    return n;
  } catch (const NesaError& e) {
    g_last_error = e.what();
    return -e.code;
  }
}

NESA_API const char* nesa_trace_name(nesa_plan* P, int32_t i) {
  if (P == nullptr || i < 0 || size_t(i) >= P->trace_names.size()) return "";
  return P->trace_names[size_t(i)].c_str();
}

NESA_API int nesa_profile_read(nesa_plan* P, int32_t stage, float* ms, int32_t max) {
  try {
    require(P != nullptr && ms != nullptr, "null argument");
    require(stage >= 0 && stage < NESA_N_STAGES, "bad stage");
    CUDA_OK(cudaSetDevice(P->device));
    CUDA_OK(cudaDeviceSynchronize());
    int n = 0;
    for (size_t i = 0; i < P->prof_used && n < max; ++i) {
      float t = 0;
      if (cudaEventElapsedTime(&t, P->prof_events[i][2 * stage], P->prof_events[i][2 * stage + 1]) !=
          cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      ms[n++] = t;
    }
    return n;
  } catch (const NesaError& e) {
    g_last_error = e.what();
    return -e.code;
  }
}
