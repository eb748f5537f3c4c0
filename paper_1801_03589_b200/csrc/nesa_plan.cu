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

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
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
  // dynamic launch (n_units > 0): cta_ptr holds n_units claimable ranges,
  // launch_grid CTAs claim them from wq; CTAs on SMs < sm_skip exit at once
  DevBuf<int> wq;
  int n_units = 0;
  int launch_grid = 0;
  int sm_skip = 0;
  size_t smem = 0;  // dynamic shared memory per CTA (0: the layout's own)
  int ncw = kNCW;    // consumer warps of the block-GEMV launch (store mode: 8 or 4)
  int ab = kABytes;  // bytes per ring stage (16 or 32 KB)
  int nst = kStages; // ring stages
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
  int64_t pt_begin = 0, pt_end = 0;      // local tree-order point range
  int n_sm = 148;

  std::vector<int64_t> lvl_first, lvl_count;  // global, index level - l0
  std::vector<int64_t> loc_first, loc_count;  // local (ancestors of local leaves)

  DevBuf<int64_t> perm;        // [N]
  DevBuf<int32_t> iperm;       // [N] original index -> tree index
  bool gather_inv = true;      // gather walked in the original order (gather_inv_kernel; ~same time)
  DevBuf<int32_t> quad;        // [G]
  DevBuf<int64_t> parent;      // [G]
  DevBuf<int64_t> child_first; // [G]
  DevBuf<int32_t> n_child;     // [G]
  DevBuf<unsigned char> CT, BT, DT;  // T tables (transposed)
  int64_t n_dtab = 0, d_refs = 0;

  DevBlockSet nearset, Vset, Uset;

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
  // fused coarse levels l0+1 .. fused_lf (one kernel per pass; see
  // nesa_kernels.cuh "Fused coarse levels"); fused_lf == l0: off
  bool fused = true;
  int fused_lf = 0;
  DevBuf<int2> uchild;                      // [G] local children (first, count)
  DevBuf<int32_t> fused_anc;                // [count(lf)][lf - l0 - 1] ancestors
  DevBuf<int> fused_cnt, fused_state;       // [G] arrival counters / claim states
  // coarse far field as one persistent kernel (coarse_kernel): coarse
  // up + translation + down from a device work queue
  bool coarse_mega = false;                 // (measured slower: items serialise inside CTAs)
  int mega_ctas = 2;                        // persistent CTAs per SM
  bool mega_ready = false;
  DevBuf<int32_t> e_src, e_dt, glevel, mega_tq, mega_lcount;
  DevBuf<int> mega_head, mega_ldone, mega_tdone, mega_ctl;
  int64_t mega_nt = 0;
  int qs = 4;                               // quadrant slots staged per round
  int64_t wide_level = 2048;                // warp-tiled level kernels from this size
  int near_ctas = 2;                        // near-field CTAs per SM (1: 6-stage ring)
  int near_waves = 1;                       // near-field grid = waves x resident CTAs
  int near_units = 0;                       // >0: dynamic near launch over this many ranges
  int near_sm_skip = 0;                     // dynamic: SMs [0, skip) left to the far chain
  size_t near_smem = 0;                     // dynamic: shared memory per near CTA (padding)
  int near_ncw = 4, near_ab = 24576, near_nst = 2;  // near-field kernel variant (NESA_BG_VARIANTS)
  bool priority = true;                     // far-field stream scheduled first
  bool split = true;                        // fine-level translation on a side stream
  int near_after = 0;                       // where the near branch forks (see enqueue_T;
                                            // 0: after the radiation, measured best at C4)
  bool u_mf = false;                        // matrix-free reception (float32 plans)
  bool recv_far = false;                    // reception in the far branch (u_mf only)
  bool pdl = true;                          // programmatic dependent launch in the far chain
  DevBuf<float2> mf_prel;                   // [N] point - leaf center (float32)
  DevBuf<int64_t> gstart, gstop;            // [NL] leaf point ranges
  DevBuf<float> mf_leaf_r;                  // [NL] rho_in_aux * half side (float32)
  // radiation through outgoing moments (float32 plans from geometry)
  bool v_mom = false;
  int v_nm = 0;                             // moments m = 0 .. v_nm - 1
  int u_nt = 0;                             // reception terms m = 1 .. u_nt
  DevBuf<float2> mom_A;                     // [v_nm][Q]: row 0 = (F_k, 0), row m = A_km
  DevBuf<float2> exp_E;                     // [Q][u_nt + 1]: 1, (1/m) e^{-i m theta_k}
  DevBuf<float> mf_leaf_rc;                 // [NL] rho_out_check * half side (float32)
  // Q = 64: s = A^ mu^ as a warp-tiled GEMM over the leaves (KT = mom_kt)
  int mom_kt = 0;
  int mom_buf = 800;                        // staged points per warp in the moment kernel
  int mom_variant = 0;                      // moment kernel instantiation (launch_radiation)
  DevBuf<float> momAT;                      // [mom_kt][Q] transposed real A^
  bool tc = true;                           // translation on the tensor cores (float32, Q = 64)
  bool tc2 = true;                          // ... with the A operand in TMEM (~50 KB smem)
  int tc3_ctas = 2;                         // ... persistent, this many CTAs per SM (0: one CTA per unit)
  DevBuf<float> DTC;                        // [n_dtab + 1][hi | lo][64 x 64] canonical tf32 D (+ zero)
  // target-major translation (float32, Q = 64, tensor cores): units of <= 128
  // targets of one level sharing one interaction pattern (the sorted list of
  // their D matrices); o is written directly, no Y and no reduce
  // (measured 561 vs 527 us at C4: the shared patterns pad the K-loop ~2x and
  // each step's D load is serial in a CTA; NESA_PAT=1 enables it)
  bool pat = false;
  int pat_ctas = 1;                         // persistent CTAs per SM of the pattern kernel
  DevBuf<PUnit> punits;
  DevBuf<int32_t> ptgt, pdid, psrc;
  int n_punits = 0, n_punits_fine = 0;
  DevBuf<TUnit> mom_units;
  DevBuf<TEnt> mom_ents;
  int n_mom_units = 0;
  bool rad_up = false;                      // radiation GEMM also writes the leaf transfers T
  DevBuf<float> radT;                       // [4 quadrants][80][128] stacked [A^; C_q A^]^T
  DevBuf<TUnit> rad_units;
  DevBuf<TEnt> rad_ents;
  int n_rad_units = 0;
  bool beta_tc = false;                     // reception coefficients by tgemm_tc (E^ o)
  bool recv_fused = false;                  // leaf down + beta + reception in one kernel
  bool beta_fused = false;                  // leaf down + beta in one kernel (reception separate)
  DevBuf<float> ET;                         // [64][64] E^ transposed for the warp-tiled GEMM
  DevBuf<float> ETC;                        // [hi | lo][64 x 64] canonical tf32 E^
  DevBuf<unsigned char> beta;               // [NL][64][R] reception coefficients
  DevBuf<unsigned char> mu;                 // [NL][mom_kt][R] moments
  cudaEvent_t ev_mark = nullptr;            // no-op event-record node ahead of the near kernel

  // workspace for R real columns
  int ws_R = 0;
  int ldv = 1;  // row stride of the caller's q / phi (elements) for the current capture
  DevBuf<unsigned char> qt, phin, phif, s, o, Y, Tup;
  DevBuf<unsigned char> farws;              // s | Tup | o, contiguous (one L2 window)
  size_t l2_persist = 0;                    // bytes of L2 set aside for farws (NESA_L2_PERSIST MB)

  cudaStream_t s0 = nullptr, s1 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t s2 = nullptr;                 // fine-level translation branch
  cudaStream_t s3 = nullptr;                 // second near-field launch (near_split)
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  cudaEvent_t ev_gfork = nullptr;           // gather on the near stream (rad_direct)
  bool rad_direct = false;                  // radiation reads q through perm (see enqueue_T;
                                            // measured slower: 556 vs 539 us, random q reads)
  int near_split = 0;                        // far-pass hook position of the 2nd near launch (0: one
                                             // launch; measured slower: half the CTAs stream at
                                             // about half the bandwidth)
  double near_frac = 0.5;                    // share of near-field CTAs in the first launch
  cudaEvent_t ev_sfine = nullptr, ev_tfine = nullptr;
  int split_lv = 0;                          // levels >= split_lv: translated on s2
  int fine_after_up = 0;                     // s2 translation starts after the up pass (1) / coarse translation (2)
  bool fused_spec = false;                   // fused up: speculative parent-matrix prefetch (neutral)
  bool down_ysum = false;                    // wide down kernels sum Y (no fine reduce; measured slower)
  bool node_prio = false;                    // graphs honour the captured stream priorities (measured worse)
  int recv_minb = 6;                         // reception register budget (6 / 8 CTAs per SM; 6: 37 vs 39 us)
  int tc3_minb = 0;                          // tgemm_tc3 register budget (3: <= 168 registers)
  int coarse_tc = 1;                         // coarse translation: 0 FFMA, 1 as fine, 2 one CTA per unit
  int n_tunits_fine = 0;                     // units [0, n_tunits_fine) are fine levels
  int64_t n_red_fine = 0;                    // red_ids [0, n_red_fine) are fine levels
  std::vector<int> tu_start;                 // [lv - l0]: first translation unit of level lv
  std::vector<int64_t> red_start;            // [lv - l0]: first red_ids entry of level lv
  std::vector<cudaEvent_t> ev_lv;            // [lv - l0]: level lv's s is final
  bool split_levels = false;                 // fine levels translated one by one as their s is final
                                             // (NESA_SPLIT_LEVELS=1; measured slower: the translation
                                             // CTAs delay the up chain)

  struct GraphKey {
    const void* q;
    void* phi;
    int R;
    uint32_t flags;
    int stage;
    int ldv;
    bool operator<(const GraphKey& o) const {
      return std::tie(q, phi, R, flags, stage, ldv) <
             std::tie(o.q, o.phi, o.R, o.flags, o.stage, o.ldv);
    }
  };
  struct GraphEntry {
    cudaGraph_t graph = nullptr;  // kept alive: its nodes address the exec's nodes
    cudaGraphExec_t exec = nullptr;
    std::vector<std::pair<cudaGraphNode_t, int>> ev_nodes;  // node, slot (stage*2+end)
  };
  std::map<GraphKey, GraphEntry> graphs;
  int kernels_per_matvec = 0;

  // profiling: per matvec a set of 2*NESA_N_STAGES events
  std::vector<std::vector<cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  cudaEvent_t cap_events[2 * NESA_N_STAGES + kTraceSlots] = {};
  bool trace = false;                       // NESA_TRACE: an event after every kernel
  std::vector<std::string> trace_names;

  ~nesa_plan() {
    cudaSetDevice(device);
    for (auto& kv : graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
    }
    for (auto& v : prof_events)
      for (auto e : v) cudaEventDestroy(e);
    for (auto e : cap_events)
      if (e) cudaEventDestroy(e);
    if (ev_sfine) cudaEventDestroy(ev_sfine);
    if (ev_mark) cudaEventDestroy(ev_mark);
    if (ev_tfine) cudaEventDestroy(ev_tfine);
    if (s2) cudaStreamDestroy(s2);
    if (s3) cudaStreamDestroy(s3);
    if (ev_fork2) cudaEventDestroy(ev_fork2);
    if (ev_gfork) cudaEventDestroy(ev_gfork);
    for (auto e : ev_lv)
      if (e) cudaEventDestroy(e);
    if (ev_join2) cudaEventDestroy(ev_join2);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s0) cudaStreamDestroy(s0);
    if (s1) cudaStreamDestroy(s1);
  }
};

namespace {

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

  // ---- tables
  const int64_t nlt = P->L - P->l0;
  P->mbytes = mat_bytes(Q, sizeof(T));
  if (nlt > 0) {
    upload_table_T<T>(P->CT, d->C, nlt * 4, Q);
    upload_table_T<T>(P->BT, d->B, nlt * 4, Q);
  }
  P->n_dtab = d->n_dtab;
  upload_table_T<T>(P->DT, d->D, d->n_dtab, Q);
  // tensor-core translation (float32, Q = 64): D split into tf32 hi / lo in
  // the canonical K-major core-matrix layout (see tgemm_tc_kernel)
  if (std::is_same<T, float>::value && Q == 64 && P->tc && d->n_dtab > 0) {
    // + one zero matrix at index n_dtab (the pattern of targets without
    // interaction entries, so their translation sum is written as 0)
    std::vector<float> h(size_t(d->n_dtab + 1) * 8192, 0.f);
    auto tf32 = [](float x) {
      uint32_t u;
      std::memcpy(&u, &x, 4);
      u = (u + 0x1000u) & ~0x1FFFu;  // round to nearest (ties away), 10-bit mantissa
      float y;
      std::memcpy(&y, &u, 4);
      return y;
    };
    for (int64_t t = 0; t < d->n_dtab; ++t)
      for (int nn = 0; nn < 64; ++nn)
        for (int k = 0; k < 64; ++k) {
          const float x = float(d->D[(t * 64 + nn) * 64 + k]);
          const float hi = tf32(x), lo = tf32(x - hi);
          const size_t off = size_t(nn / 8) * 512 + size_t(k / 4) * 32 + size_t(nn % 8) * 4 + (k % 4);
          h[size_t(t) * 8192 + off] = hi;
          h[size_t(t) * 8192 + 4096 + off] = lo;
        }
    P->DTC.upload(h);
  } else {
    P->tc = false;
  }
  // quadrant slots per round: keep the level kernels <= ~96 KB so they can
  // co-reside with the persistent near-field CTAs (~110 KB) on one SM
  P->qs = 2;
  while (P->qs > 1 && level_smem_bytes<T>(Q, P->qs) > 96 * 1024) P->qs /= 2;
  require(level_smem_bytes<T>(Q, 1) <= 200 * 1024 && tgemm_smem_bytes<T, 4>(Q) <= 200 * 1024,
          "Q too large for the far-field kernels");
  // per-level gather tables (see nesa_kernels.cuh "Level transfers")
  P->down_order.resize(nlev);
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
        require(cnt[i] <= 4, "more than four children");
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
      const bool wide = Q == 64 && P->loc_count[lv - P->l0] >= P->wide_level;
      if (wide || P->loc_count[lv - P->l0] == 0) break;
      P->fused_lf = lv;
    }
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
    P->fused_cnt.alloc(size_t(G));    // zero-filled
    P->fused_state.alloc(size_t(G));
    if (P->coarse_mega && P->leaf_begin == 0 && P->leaf_end == P->NL) {
      const int64_t nnz = d->int_ptr[G];
      std::vector<int32_t> es(static_cast<size_t>(std::max<int64_t>(nnz, 1)), 0),
          ed(static_cast<size_t>(std::max<int64_t>(nnz, 1)), 0);
      for (int64_t e = 0; e < nnz; ++e) {
        es[size_t(e)] = int32_t(d->int_idx[e]);
        ed[size_t(e)] = int32_t(d->int_dtab[e]);
      }
      P->e_src.upload(es);
      P->e_dt.upload(ed);
      std::vector<int32_t> gl(static_cast<size_t>(G), -1), tq, lc;
      for (int lv = P->l0; lv <= P->L; ++lv) {
        const int lj = lv - P->l0;
        for (int64_t g = P->loc_first[lj]; g < P->loc_first[lj] + P->loc_count[lj]; ++g) gl[size_t(g)] = lv;
      }
      for (int lv = P->fused_lf; lv >= P->l0; --lv) {
        const int lj = lv - P->l0;
        for (int64_t g = P->loc_first[lj]; g < P->loc_first[lj] + P->loc_count[lj]; ++g)
          tq.push_back(int32_t(g));
      }
      for (int lv = P->l0; lv <= P->fused_lf; ++lv) lc.push_back(int32_t(P->loc_count[lv - P->l0]));
      P->glevel.upload(gl);
      P->mega_tq.upload(tq);
      P->mega_lcount.upload(lc);
      P->mega_nt = int64_t(tq.size());
      P->mega_head.alloc(1);
      P->mega_ldone.alloc(lc.size());
      P->mega_tdone.alloc(size_t(G));
      P->mega_ctl.alloc(4);
      P->mega_ready = true;
    }
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
    P->red_start.assign(size_t(nlev) + 1, 0);
    for (int lv = P->L; lv >= P->l0; --lv) {
      const int li = lv - P->l0;
      P->red_start[li] = int64_t(ids.size());
      for (int64_t g = P->loc_first[li]; g < P->loc_first[li] + P->loc_count[li]; ++g)
        ids.push_back(int32_t(g));
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
    P->u_mf = P->u_mf && f32 && !d->U_blob && geom;
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
      P->u_nt = terms(ru, 1e-8);
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
      int64_t W = 0;
      for (int64_t e = d->nbr_ptr[a]; e < d->nbr_ptr[a + 1]; ++e) {
        const int64_t b = d->nbr_idx[e];
        require(b >= 0 && b < NL, "neighbor id out of range");
        W += d->group_stop[b] - d->group_start[b];
      }
      require(W < (int64_t(1) << 31), "near slab too wide");
      if (a >= lb && a < le) {
        // near item(s): panels of <= kMaxRows rows
        const int32_t seg_begin = int32_t(hn.segs.size());
        int32_t col = 0;
        for (int64_t e = d->nbr_ptr[a]; e < d->nbr_ptr[a + 1]; ++e) {
          const int64_t b = d->nbr_idx[e];
          const int64_t bs = d->group_start[b], bn = d->group_stop[b] - bs;
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
                                       int32_t(d->group_start[a] + r0), seg_begin, seg_count, 0, 0});
          near_src_off.push_back(near_off);
          near_src_rows.push_back(int32_t(na));
          near_row0.push_back(int32_t(r0));
          hn.blob_elems += int64_t(ld) * W;
          hn.entries += int64_t(m) * W;
        }
        // V: Q x na, x = qt rows of the leaf, y = s rows of leaf a
        {
          const int32_t sb = int32_t(hv.segs.size());
          hv.segs.push_back(BlockSeg{int32_t(d->group_start[a]), 0});
          const int32_t ld = (Q + 3) / 4 * 4;
          BlockItem it{hv.blob_elems, Q, int32_t(na), ld, int32_t(a * Q), sb, 1,
                       int32_t(d->group_start[a]), 0};
          hv.items.push_back(it);
          v_src_off.push_back(v_off);
          v_src_rows.push_back(Q);
          v_row0.push_back(0);
          v_leaf.push_back(a);
          hv.blob_elems += int64_t(ld) * na;
          hv.entries += int64_t(Q) * na;
        }
        // U: na x Q, x = o rows of leaf a, y = phi rows (stored mode only)
        if (!P->u_mf) {
          const int32_t sb = int32_t(hu.segs.size());
          hu.segs.push_back(BlockSeg{int32_t(a * Q), 0});
          for (int64_t r0 = 0; r0 < na; r0 += kMaxRows) {
            const int32_t m = int32_t(std::min<int64_t>(kMaxRows, na - r0));
            const int32_t ld = (m + 3) / 4 * 4;
            hu.items.push_back(BlockItem{hu.blob_elems, m, Q, ld,
                                         int32_t(d->group_start[a] + r0), sb, 1, 0, 0});
            u_src_off.push_back(u_off);
            u_src_rows.push_back(int32_t(na));
            u_row0.push_back(int32_t(r0));
            u_leaf.push_back(a);
            hu.blob_elems += int64_t(ld) * Q;
            hu.entries += int64_t(m) * Q;
          }
        }
      }
      near_off += na * W;
      v_off += int64_t(Q) * na;
      u_off += na * Q;
    }
    require(int64_t(NL) * Q < (int64_t(1) << 31), "too many groups for int32 rows");
  }
  {
    int ng = P->near_waves * P->near_ctas * P->n_sm;
    if (const char* e = std::getenv("NESA_NEAR_GRID")) ng = std::max(1, std::atoi(e));
    if (P->near_units > 0) ng = P->near_units;
    chunk_and_balance(hn, es, ng, P->near_ab, P->near_ncw * 32);
  }
  chunk_and_balance(hv, es, kBGPerSM * P->n_sm);
  chunk_and_balance(hu, es, kBGPerSM * P->n_sm);
  upload_blockset<T>(P->nearset, hn);
  P->nearset.ncw = P->near_ncw;
  P->nearset.ab = P->near_ab;
  P->nearset.nst = P->near_nst;
  if (P->near_units > 0 && P->near_ctas == 2) {
    P->nearset.n_units = P->nearset.grid;
    P->nearset.launch_grid = kBGPerSM * P->n_sm;
    P->nearset.sm_skip = P->near_sm_skip;
    P->nearset.smem = P->near_smem;
    P->nearset.wq.alloc(2);
  }
  if (!P->v_mom) upload_blockset<T>(P->Vset, hv);
  upload_blockset<T>(P->Uset, hu);

  // ---- fill the blobs: from host operators or assembled on the device
  DevBuf<double> pts;
  const bool need_geom = !d->near_blob || !d->V_blob || !d->U_blob;
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
      // default: A^ applied inside the moment kernel (MU_OUT = false; measured 531 vs
      // 545 us at C4 with FFMA2: one launch less on the critical path);
      // NESA_MOM_INKERNEL=0 selects the separate 64 x 80 moment-map GEMM
      const char* mi = std::getenv("NESA_MOM_INKERNEL");
      if (Q == 64 && mi && std::atoi(mi) == 0) {
        const int need = 2 * P->v_nm - 1;
        P->mom_kt = need <= 80 ? 80 : (need <= 127 ? 128 : 0);  // nm <= 64 (16 per lane)
      }
      if (P->mom_kt) {
        // rows: 0 -> F_k (times -log r mu_0), 2m-1 -> Re A_km, 2m -> -Im A_km
        std::vector<float> AT(size_t(P->mom_kt) * Q, 0.f);
        for (int k = 0; k < Q; ++k) {
          AT[k] = A[k].x;
          for (int m = 1; m < P->v_nm; ++m) {
            AT[size_t(2 * m - 1) * Q + k] = A[size_t(m) * Q + k].x;
            AT[size_t(2 * m) * Q + k] = -A[size_t(m) * Q + k].y;
          }
        }
        P->momAT.upload(AT);
        // leaf level wide (warp-tiled level kernels): fold the leaf transfer
        // into the same GEMM, Y = [A^; C_q A^] mu^ -> s and T in one pass
        // (one stacked 128 x 80 map per child quadrant q, formed in float64)
        const int li = P->L - P->l0;
        const bool leaf_wide = P->L > P->l0 && P->loc_count[li] >= P->wide_level;
        // (measured neutral at C4: the 128-row GEMM costs what the leaf level
        // kernel did; opt in with NESA_RAD_UP=1)
        const char* ru = std::getenv("NESA_RAD_UP");
        if (P->mom_kt == 80 && leaf_wide && ru && std::atoi(ru) != 0) {
          const int kt = 80;
          std::vector<double> ATd(size_t(kt) * Q, 0.0);  // ATd[j][i] = A^[i][j]
          for (int i = 0; i < Q; ++i) {
            ATd[i] = Ad[2 * size_t(i)];
            for (int m = 1; m < P->v_nm; ++m) {
              ATd[size_t(2 * m - 1) * Q + i] = Ad[2 * (size_t(m) * Q + i)];
              ATd[size_t(2 * m) * Q + i] = -Ad[2 * (size_t(m) * Q + i) + 1];
            }
          }
          std::vector<float> RT(size_t(4) * kt * 128, 0.f);
          for (int q = 0; q < 4; ++q) {
            const double* Cq = d->C + (size_t(li - 1) * 4 + q) * Q * Q;
            float* M = RT.data() + size_t(q) * kt * 128;
            for (int j = 0; j < kt; ++j) {
              for (int k = 0; k < Q; ++k) M[size_t(j) * 128 + k] = float(ATd[size_t(j) * Q + k]);
              for (int k = 0; k < Q; ++k) {
                double acc = 0;
                for (int i = 0; i < Q; ++i) acc += Cq[size_t(k) * Q + i] * ATd[size_t(j) * Q + i];
                M[size_t(j) * 128 + Q + k] = float(acc);
              }
            }
          }
          P->radT.upload(RT);
          std::vector<TUnit> units;
          std::vector<TEnt> ents;
          for (int q = 0; q < 4; ++q) {
            std::vector<TEnt> v;
            for (int64_t a = lb; a < le; ++a)
              if (d->quad[a] == q) v.push_back(TEnt{int32_t(a), int32_t(a)});
            for (size_t i = 0; i < v.size(); i += 32) {
              const size_t j = std::min(v.size(), i + 32);
              units.push_back(TUnit{q, int32_t(ents.size()), int32_t(ents.size() + (j - i)), 0});
              ents.insert(ents.end(), v.begin() + i, v.begin() + j);
            }
          }
          P->rad_units.upload(units);
          P->rad_ents.upload(ents);
          P->n_rad_units = int(units.size());
          P->rad_up = true;
        }
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
      // Q = 64 with tensor cores: beta^ = E^ o for all leaves as one GEMM;
      // E^ rows 0 -> 1 (sum of o), 2m-1 / 2m -> Re / Im of (1/m) e^{-i m theta_k}
      const char* ri = std::getenv("NESA_RECV_INKERNEL");
      if (Q == 64 && P->tc && 2 * P->u_nt + 1 <= 64 && !(ri && std::atoi(ri) != 0)) {
        auto tf32 = [](float x) {
          uint32_t u;
          std::memcpy(&u, &x, 4);
          u = (u + 0x1000u) & ~0x1FFFu;
          float y;
          std::memcpy(&y, &u, 4);
          return y;
        };
        std::vector<float> h(8192, 0.f);
        for (int row = 0; row < 64; ++row)
          for (int k = 0; k < 64; ++k) {
            float x = 0.f;
            if (row == 0)
              x = 1.f;
            else if (row <= 2 * P->u_nt)
              x = (row & 1) ? E[size_t(k) * ne + (row + 1) / 2].x : E[size_t(k) * ne + row / 2].y;
            const float hi = tf32(x), lo = tf32(x - hi);
            const size_t off = size_t(row / 8) * 512 + size_t(k / 4) * 32 + size_t(row % 8) * 4 + (k % 4);
            h[off] = hi;
            h[4096 + off] = lo;
          }
        P->ETC.upload(h);
        P->beta_tc = true;
      }
      // leaf level handled by the wide kernels: fuse its downward transfer,
      // beta^ = E^ o and the reception into one kernel (no o / beta round trip)
      const char* rf = std::getenv("NESA_RECV_FUSED");
      const bool leaf_wide = P->L > P->l0 && P->loc_count[P->L - P->l0] >= P->wide_level;
      // (measured slower at C4, 641 vs 627 us: 8 warps per SM cannot hide the
      // point loads the separate 48-warp reception kernel hides; opt in with
      // NESA_RECV_FUSED=1)
      const char* bf = std::getenv("NESA_BETA_FUSED");
      const bool want_recv = rf && std::atoi(rf) != 0;
      const bool want_beta = !want_recv && P->beta_tc && !(bf && std::atoi(bf) == 0);
      if (Q == 64 && leaf_wide && 2 * P->u_nt + 1 <= 64 && (want_recv || want_beta)) {
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
        P->recv_fused = want_recv;
        P->beta_fused = want_beta;
      }
    }
    if (P->mom_kt || P->beta_tc) {
      // one entry per local leaf (src = dst = leaf), 32 leaves per unit
      std::vector<TUnit> units;
      std::vector<TEnt> ents;
      for (int64_t a = lb; a < le; ++a) ents.push_back(TEnt{int32_t(a), int32_t(a)});
      int per = 32;  // one pass of 32 leaves per CTA: the GEMM is latency-bound
      if (const char* e = std::getenv("NESA_MOM_PER")) per = std::max(1, std::atoi(e));
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
    if (P->tc) {
      per = 128;
      if (const char* e = std::getenv("NESA_TC_PER")) per = std::max(32, std::atoi(e));
    }
    std::vector<TEnt> ents;
    std::vector<TUnit> units;
    std::vector<std::vector<TEnt>> by_d(size_t(std::max<int64_t>(d->n_dtab, 1)));
    // levels fine -> coarse; within a level grouped by unique D
    P->tu_start.assign(size_t(P->L - P->l0 + 2), 0);
    for (int lv = P->L; lv >= P->l0; --lv) {
      const int li = lv - P->l0;
      P->tu_start[li] = int(units.size());
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
    }
    P->tunits.upload(units);
    P->tents.upload(ents);
    P->n_tunits = int(units.size());
    if (P->pat && P->tc && std::is_same<T, float>::value && Q == 64 && !P->split_levels) {
      std::vector<PUnit> pu;
      std::vector<int32_t> tg, did, src;
      for (int lv = P->L; lv >= P->l0; --lv) {
        const int li = lv - P->l0;
        std::map<std::vector<int32_t>, std::vector<int64_t>> pats;
        for (int64_t g = P->loc_first[li]; g < P->loc_first[li] + P->loc_count[li]; ++g) {
          std::vector<int32_t> key;
          for (int64_t e = d->int_ptr[g]; e < d->int_ptr[g + 1]; ++e) key.push_back(int32_t(d->int_dtab[e]));
          std::sort(key.begin(), key.end());
          require(std::adjacent_find(key.begin(), key.end()) == key.end(), "repeated D in one interaction list");
          if (key.empty()) key.push_back(int32_t(d->n_dtab));  // zero matrix
          pats[key].push_back(g);
        }
        for (auto& kv : pats) {
          const std::vector<int32_t>& key = kv.first;
          const std::vector<int64_t>& gs = kv.second;
          for (size_t i = 0; i < gs.size(); i += 128) {
            const size_t j = std::min(gs.size(), i + 128);
            PUnit u{};
            u.tgt_begin = int32_t(tg.size());
            u.n_tgt = int32_t(j - i);
            u.off_begin = int32_t(did.size());
            u.n_off = int32_t(key.size());
            u.src_begin = int32_t(src.size());
            for (size_t t = i; t < j; ++t) tg.push_back(int32_t(gs[t]));
            did.insert(did.end(), key.begin(), key.end());
            for (int32_t dt : key)
              for (size_t t = i; t < j; ++t) {
                const int64_t g = gs[t];
                int32_t sg = int32_t(g);  // zero pattern: any valid group
                for (int64_t e = d->int_ptr[g]; e < d->int_ptr[g + 1]; ++e)
                  if (d->int_dtab[e] == dt) sg = int32_t(d->int_idx[e]);
                src.push_back(sg);
              }
            pu.push_back(u);
          }
        }
        if (lv == P->split_lv) P->n_punits_fine = int(pu.size());
      }
      require(src.size() < (size_t(1) << 31), "too many pattern sources");
      P->punits.upload(pu);
      P->ptgt.upload(tg);
      P->pdid.upload(did);
      P->psrc.upload(src);
      P->n_punits = int(pu.size());
    } else {
      P->pat = false;
    }
  }
}



template <typename T>
void ensure_workspace(nesa_plan* P, int R) {
  if (P->ws_R >= R) return;
  const size_t es = sizeof(T);
  P->qt.alloc(size_t(P->N) * R * es);
  P->phin.alloc(size_t(P->N) * R * es);
  if (P->u_mf && P->recv_far) P->phif.alloc(size_t(P->N) * R * es);
  if (P->mom_kt) P->mu.alloc(size_t(P->NL) * P->mom_kt * R * es);
  if (P->beta_tc) P->beta.alloc(size_t(P->NL) * 64 * R * es);
  {
    const size_t fb = (size_t(P->G) * P->Q * R * es + 255) & ~size_t(255);
    P->farws.alloc(3 * fb);
    P->s.view(P->farws.p, fb);
    P->Tup.view(P->farws.p + fb, fb);
    P->o.view(P->farws.p + 2 * fb, fb);
  }
  P->Y.alloc(size_t(P->pat ? 1 : std::max<int64_t>(P->nnz, 1)) * P->Q * R * es);
  P->ws_R = R;
}

inline int grid_for(int64_t n, int threads, int cap) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap)));
}

template <typename T, int R, int MODE, int NST = kStages, int NCW = kNCW, int AB = kABytes>
void launch_blockgemv_v(const DevBlockSet& bs, const T* x, T* y, const T* base, const int64_t* perm,
                      int64_t perm_offset, cudaStream_t st, int cta0 = 0, int ncta = -1) {
  if (bs.n_items == 0) return;
  if (ncta < 0) ncta = bs.grid - cta0;
  if (ncta <= 0) return;
  BlockGemvArgs<T> a{reinterpret_cast<const T*>(bs.blob.p), bs.recs.p, bs.cta_ptr.p + cta0, x, y,
                     base, perm, int(perm_offset), nullptr, 0, 0};
  size_t sm = blockgemv_smem_bytes<T, R, MODE, NST, NCW, AB>();
  if (bs.n_units > 0 && cta0 == 0 && ncta == bs.grid) {
    a.wq = bs.wq.p;
    a.n_units = bs.n_units;
    a.sm_skip = bs.sm_skip;
    ncta = bs.launch_grid;
    sm = std::max(sm, bs.smem);
  }
  blockgemv_kernel<T, R, MODE, NST, NCW, AB><<<ncta, NCW * 32 + 32, sm, st>>>(a);
}

// near-field variants (store mode): (consumer warps, stage bytes, stages)
// (measured in the full C4 product: 4 warps x 24 KB x 2 stages 555 us, 4 x 16 KB x 3 556,
// 4 x 32 KB x 2 580, 8 x 16 KB x 3 (the generic default) 633; fewer consumer threads and
// larger stages amortise the per-chunk consumer overhead that bounds an SM's share)
#define NESA_BG_VARIANTS(X)                                                                 \
  X(4, 24576, 2) X(4, 16384, 3) X(4, 32768, 2) X(8, 32768, 2) X(4, 32768, 3) X(8, 32768, 3) \
  X(4, 49152, 2) X(8, 24576, 4)

bool bg_variant_known(int w, int b, int n) {
  bool known = w == kNCW && b == kABytes && n == kStages;
#define NESA_BG_KNOWN(W, B, S) known = known || (w == W && b == B && n == S);
  NESA_BG_VARIANTS(NESA_BG_KNOWN)
#undef NESA_BG_KNOWN
  return known;
}

template <typename T, int R, int MODE, int NST = kStages>
void launch_blockgemv(const DevBlockSet& bs, const T* x, T* y, const T* base, const int64_t* perm,
                      int64_t perm_offset, cudaStream_t st, int cta0 = 0, int ncta = -1) {
  if constexpr (MODE == kModeStore && NST == kStages) {
#define NESA_BG_CASE(W, B, S)                                                                      \
  if (bs.ncw == W && bs.ab == B && bs.nst == S) {                                                  \
    launch_blockgemv_v<T, R, MODE, S, W, B>(bs, x, y, base, perm, perm_offset, st, cta0, ncta); \
    return;                                                                                        \
  }
    NESA_BG_VARIANTS(NESA_BG_CASE)
#undef NESA_BG_CASE
  }
  launch_blockgemv_v<T, R, MODE, NST>(bs, x, y, base, perm, perm_offset, st, cta0, ncta);
}

template <typename T, int R>
void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  // NESA_CARVEOUT=c (0..100): every kernel asks for the same shared-memory
  // carveout (measured: the driver default is faster for this schedule)
  int carve = -1;
  if (const char* e = std::getenv("NESA_CARVEOUT")) carve = std::atoi(e);
  auto attr = [carve](auto* fn, int smem) {
    if (smem >= 0)
      CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (carve >= 0)
      CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  };
  attr(blockgemv_kernel<T, R, kModeStore>, 113 * 1024);
#define NESA_BG_ATTR(W, B, S) attr(blockgemv_kernel<T, R, kModeStore, S, W, B>, 113 * 1024);
  NESA_BG_VARIANTS(NESA_BG_ATTR)
#undef NESA_BG_ATTR
  attr(blockgemv_kernel<T, R, kModeScatter>, int(blockgemv_smem_bytes<T, R, kModeScatter>()));
  attr(blockgemv_kernel<T, R, kModeStore, 6>, int(blockgemv_smem_bytes<T, R, kModeStore, 6>()));
  const int lim = 220 * 1024;
  attr(tgemm_kernel<T, R>, lim);
  attr(tgemm_wt_kernel<T, R, 64>, lim);
  attr(tgemm_wt_kernel<T, R, 32>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlUpLeaf>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlUpSum>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlDown>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlDownRecv>, lim);
  attr(level_wt_kernel<T, R, 64, kLvlDownBeta>, lim);
  attr(level_kernel<T, R, kLvlUpLeaf>, lim);
  attr(level_kernel<T, R, kLvlUpSum>, lim);
  attr(level_kernel<T, R, kLvlDown>, lim);
  attr(gather_kernel<T, R>, -1);
  attr(scatter_kernel<T, R>, -1);
  attr(reduce_kernel<T, R>, -1);
  attr(sum_children_kernel<T, R>, -1);
  if constexpr (std::is_same<T, float>::value) attr(tgemm_pat_kernel<R>, int(pat_smem_bytes<R>()));
  attr(fused_up_kernel<T, R>, lim);
  attr(fused_down_kernel<T, R>, lim);
  attr(coarse_kernel<T, R>, lim);
  if constexpr (std::is_same<T, float>::value) {
    attr(radiation_mom_kernel<R>, lim);
    attr(radiation_mom_kernel<R, false, 0, 4>, lim);
    attr(radiation_mom_kernel<R, false, 20 / R, 4>, lim);
    attr(radiation_mom_kernel<R, true>, lim);
    attr(tgemm_wt_kernel<float, R, 64, 80>, lim);
    attr(tgemm_wt_kernel<float, R, 128, 80, 64>, lim);
    attr(tgemm_tc_kernel<R>, int(kTcSmem));
    attr(tgemm_tc2_kernel<R>, int(tc2_smem_bytes<R>()));
    attr(tgemm_tc3_kernel<R>, int(tc2_smem_bytes<R>()));
    attr(tgemm_tc3_kernel<R, 3>, int(tc2_smem_bytes<R>()));
    attr(tgemm_wt_kernel<float, R, 64, 128>, lim);
    attr(reception_exp_kernel<R>, lim);
    attr(reception_exp_kernel<R, true>, lim);
    attr(reception_exp_kernel<R, true, 6>, lim);
    attr(reception_exp_kernel<R, true, 8>, lim);
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
void launch_pdl(bool pdl, void (*kernel)(KArgs...), int grid, int block, size_t smem,
                cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CUDA_OK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

constexpr int kExpCtasPerSM = 12;  // reception: leaves are latency-bound, keep many warps
constexpr int kMomCtasPerSM = 4;

// s = V qt: outgoing moments (float32 plans from geometry) or stored V
template <typename T, int R>
int launch_radiation(nesa_plan* P, const T* qt, T* s, cudaStream_t st,
                     const int64_t* qperm = nullptr) {
  if constexpr (std::is_same<T, float>::value) {
    if (P->v_mom) {
      const int64_t nleaf = P->leaf_end - P->leaf_begin;
      const int64_t per_cta = int64_t(kExpWarps) * kMomLeavesPerWarp;
      int mcta = kMomCtasPerSM;
      if (const char* e = std::getenv("NESA_MOM_CTAS")) mcta = std::max(1, std::atoi(e));
      const int grid = int(std::max<int64_t>(
          1, std::min<int64_t>((nleaf + per_cta - 1) / per_cta, int64_t(mcta) * P->n_sm)));
      // point staging (cp.async) helps alone but costs shared memory the
      // concurrent near field needs; NESA_MOM_BUF sets the staged points
      // per warp (0: none)
      int bufpts = P->mom_buf;
      const size_t sm = size_t(kExpWarps) *
                        (size_t(bufpts) * (2 + R) + size_t(kMomLeavesPerWarp) * ((P->v_nm * R + 1) & ~1) * 2) *
                        sizeof(float);
      if (P->mom_kt) {
        float* mu = reinterpret_cast<float*>(P->mu.p);
        radiation_mom_kernel<R, true><<<grid, 32 * kExpWarps, sm, st>>>(
            P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_rc.p, P->mom_A.p, qt, mu, P->leaf_begin,
            nleaf, P->Q, P->v_nm, P->mom_kt, bufpts);
        if (P->rad_up)
          tgemm_wt_kernel<float, R, 128, 80, 64><<<P->n_rad_units, 128, TGW<float, R, 128, 80>::SMEM, st>>>(
              P->rad_units.p, P->rad_ents.p, P->radT.p, mu, s, reinterpret_cast<float*>(P->Tup.p));
        else if (P->mom_kt == 80)
          tgemm_wt_kernel<float, R, 64, 80><<<P->n_mom_units, 128, TGW<float, R, 64, 80>::SMEM, st>>>(
              P->mom_units.p, P->mom_ents.p, P->momAT.p, mu, s, nullptr);
        else
          tgemm_wt_kernel<float, R, 64, 128><<<P->n_mom_units, 128, TGW<float, R, 64, 128>::SMEM, st>>>(
              P->mom_units.p, P->mom_ents.p, P->momAT.p, mu, s, nullptr);
        return 2;
      }
      // register budget for 4 CTAs / SM (<= 128 registers, no spills): at the
      // natural 169 registers only 2 CTAs fit (measured 531 vs 537 us at C4);
      // NESA_MOM_VARIANT=1: uncapped, 3: half the moments per pass (capped)
      auto go = [&](auto kern) {
        kern<<<grid, 32 * kExpWarps, sm, st>>>(P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_rc.p,
                                                P->mom_A.p, qt, s, P->leaf_begin, nleaf, P->Q, P->v_nm, 0,
                                                bufpts, qperm);
      };
      switch (P->mom_variant) {
        case 1: go(radiation_mom_kernel<R>); break;
        case 3: go(radiation_mom_kernel<R, false, 20 / R, 4>); break;
        default: go(radiation_mom_kernel<R, false, 0, 4>); break;
      }
      return 1;
    }
  }
  launch_blockgemv<T, R, kModeStore>(P->Vset, qt, s, nullptr, nullptr, 0, st);
  return 1;
}

// phi[perm] = phin + U o through the incoming expansion (float32 plans)
template <int R>
int launch_reception_exp(nesa_plan* P, const float* o, const float* phin, const int64_t* perm,
                         float* phi, int ldp, cudaStream_t st) {
  const int64_t nleaf = P->leaf_end - P->leaf_begin;
  int rcta = kExpCtasPerSM;
  if (const char* e = std::getenv("NESA_RECV_CTAS")) rcta = std::max(1, std::atoi(e));
  const int grid = int(std::max<int64_t>(
      1, std::min<int64_t>((nleaf + kExpWarps - 1) / kExpWarps, int64_t(rcta) * P->n_sm)));
  const int Q = P->Q, nt = P->u_nt;
  const size_t nb = ((size_t(nt) + 1) * R + 1) & ~size_t(1);
  const size_t sm = size_t(kExpWarps) * (nb + ((size_t(Q) * R + 3) & ~size_t(3)) / 2) * sizeof(float2);
  if (P->beta_tc) {
    // beta^ = E^ o for every leaf on the tensor cores (or already by the fused
    // leaf-level kernel), then the per-point series
    float* beta = reinterpret_cast<float*>(P->beta.p);
    if (P->beta_fused)
      ;
    else if (P->tc2)
      tgemm_tc2_kernel<R><<<P->n_mom_units, 128, tc2_smem_bytes<R>(), st>>>(P->mom_units.p, P->mom_ents.p,
                                                                           P->ETC.p, o, beta);
    else
      tgemm_tc_kernel<R><<<P->n_mom_units, 128, kTcSmem, st>>>(P->mom_units.p, P->mom_ents.p,
                                                              P->ETC.p, o, beta);
    if (P->recv_minb >= 8)
      reception_exp_kernel<R, true, 8><<<grid, 32 * kExpWarps, sm, st>>>(
          P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_r.p, P->exp_E.p, beta, phin, perm, phi,
          P->leaf_begin, nleaf, Q, nt, ldp);
    else if (P->recv_minb >= 6)
      reception_exp_kernel<R, true, 6><<<grid, 32 * kExpWarps, sm, st>>>(
          P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_r.p, P->exp_E.p, beta, phin, perm, phi,
          P->leaf_begin, nleaf, Q, nt, ldp);
    else
      reception_exp_kernel<R, true><<<grid, 32 * kExpWarps, sm, st>>>(
          P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_r.p, P->exp_E.p, beta, phin, perm, phi,
          P->leaf_begin, nleaf, Q, nt, ldp);
    return P->beta_fused ? 1 : 2;
  }
  reception_exp_kernel<R><<<grid, 32 * kExpWarps, sm, st>>>(
      P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_r.p, P->exp_E.p, o, phin, perm, phi,
      P->leaf_begin, nleaf, Q, nt, ldp);
  return 1;
}

// Enqueue one product, or one of its two stages (multi-GPU), on P->s0/P->s1.
//   stage 0: gather, fork{near | V, up, translate, down}, join, reception
//   stage 1: gather, V, up                  (before the s halo exchange)
//   stage 2: fork{near | translate, down}, join, reception
template <typename T, int R>
int enqueue_T(nesa_plan* P, const T* q, T* phi, uint32_t flags, int stage) {
  const bool near = flags & NESA_NEAR, far = flags & NESA_FAR, profn = flags & NESA_PROFILE;
  const bool prof = profn && !(flags & NESA_PROFILE_NEAR);  // stage marks on the far path
  cudaStream_t s0 = P->s0, s1 = P->s1;
  cudaStream_t join_stream = s1;  // the near branch's last stream (s3 with a split near launch)
  T* qt = reinterpret_cast<T*>(P->qt.p);
  T* phin = reinterpret_cast<T*>(P->phin.p);
  T* s = reinterpret_cast<T*>(P->s.p);
  T* o = reinterpret_cast<T*>(P->o.p);
  const T* CT = reinterpret_cast<const T*>(P->CT.p);
  const T* BT = reinterpret_cast<const T*>(P->BT.p);
  const int Q = P->Q;
  const int cap = P->n_sm * 8;
  const int64_t nloc = P->pt_end - P->pt_begin;
  int nk = 0;
  if (prof) P->trace_names.clear();
  // NESA_TRACE diagnostics: an event-record node after each kernel
  auto tr = [&](const char* name, cudaStream_t st) {
    if (!prof || !P->trace || P->trace_names.size() >= size_t(kTraceSlots)) return;
    prof_mark(P, true, 2 * NESA_N_STAGES + int(P->trace_names.size()), st);
    P->trace_names.emplace_back(name);
  };

  const size_t mstride = P->mbytes / sizeof(T);
  const FarGeom FG = far_geom(Q);
  const size_t lvl_sm = level_smem_bytes<T>(Q, P->qs);
  // groups per CTA: fill the column tile only when the level is big enough to
  // occupy every SM twice; coarse levels get one group per CTA
  auto tile_for = [&](int64_t count) {
    const int64_t want = (count + 2 * P->n_sm - 1) / (2 * P->n_sm);
    return int(std::max<int64_t>(1, std::min<int64_t>(FG.NC / R, want)));
  };
  T* Tup = reinterpret_cast<T*>(P->Tup.p);
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
    la.QS = P->qs;
    la.TC = tile_for(la.count);
    return la;
  };
  auto up_level = [&](int lv) {
    // children-major: T[c] = C s[c]; s[parent] = sum of its children's T
    const int ci = lv - P->l0;
    if (P->loc_count[ci] == 0) return;
    if (lv == P->L && P->rad_up) return;  // the radiation GEMM wrote the leaf T
    const LevelArgs<T, R> la = level_args(ci, CT + size_t(ci - 1) * 4 * mstride);
    const int grid = int((la.count + la.TC - 1) / la.TC);
    if (Q == 64 && la.count >= P->wide_level) {
      const int gw = int((la.count + TGW<T, R, 64>::PER - 1) / TGW<T, R, 64>::PER);
      if (lv == P->L)
        launch_pdl(P->pdl, level_wt_kernel<T, R, 64, kLvlUpLeaf>, gw, 128, LVW<T, R, 64, kLvlUpLeaf>::SMEM, s0, la, RecvArgs{});
      else
        launch_pdl(P->pdl, level_wt_kernel<T, R, 64, kLvlUpSum>, gw, 128, LVW<T, R, 64, kLvlUpSum>::SMEM, s0, la, RecvArgs{});
    } else if (lv == P->L) {
      launch_pdl(P->pdl, level_kernel<T, R, kLvlUpLeaf>, grid, kFarThreads, lvl_sm, s0, la);
    } else {
      launch_pdl(P->pdl, level_kernel<T, R, kLvlUpSum>, grid, kFarThreads, lvl_sm, s0, la);
    }
    nk++;
    tr(la.count >= P->wide_level && Q == 64 ? "up_wt" : "up", s0);
  };
  auto top_sum = [&]() {
    if (P->L > P->l0 && P->loc_count[0] > 0) {
      const int64_t n = P->loc_count[0] * Q * R;
      launch_pdl(P->pdl, sum_children_kernel<T, R>, grid_for(n, 256, cap), 256, 0, s0,
                 (const int64_t*)P->child_first.p, (const int32_t*)P->n_child.p, P->loc_first[0],
                 P->loc_count[0], P->loc_first[1], P->loc_first[1] + P->loc_count[1],
                 (const T*)Tup, s, Q);
      nk++;
      tr("top_sum", s0);
    }
  };
  T* Y = reinterpret_cast<T*>(P->Y.p);
  auto translate = [&](int u0, int u1, cudaStream_t st) {
    if (u1 <= u0) return;
    if constexpr (std::is_same<T, float>::value) {
      if (P->pat) {
        // unit ranges map to the fine / coarse pattern units
        const int p0 = u0 == 0 ? 0 : P->n_punits_fine;
        const int p1 = u1 == P->n_tunits ? P->n_punits : P->n_punits_fine;
        if (p1 > p0)
          launch_pdl(P->pdl && st == s0, tgemm_pat_kernel<R>, std::min(p1 - p0, P->pat_ctas * P->n_sm), 128,
                     pat_smem_bytes<R>(), st, (const PUnit*)(P->punits.p + p0), p1 - p0,
                     (const int32_t*)P->ptgt.p, (const int32_t*)P->pdid.p, (const int32_t*)P->psrc.p,
                     (const float*)P->DTC.p, (const float*)s, o);
        nk++;
        tr("translate", st);
        return;
      }
    }
    const T* DTp = reinterpret_cast<const T*>(P->DT.p);
    const TUnit* up = P->tunits.p + u0;
    const bool coarse = u0 >= P->n_tunits_fine && P->split_lv <= P->L;
    if (P->tc && !(coarse && P->coarse_tc == 0)) {
      if constexpr (std::is_same<T, float>::value) {
        if (P->tc2 && P->tc3_ctas > 0 && !(coarse && P->coarse_tc == 2) && P->tc3_minb >= 3)
          launch_pdl(P->pdl && st == s0, tgemm_tc3_kernel<R, 3>,
                     std::min(u1 - u0, P->tc3_ctas * P->n_sm), 128, tc2_smem_bytes<R>(), st, up, u1 - u0,
                     (const TEnt*)P->tents.p, (const float*)P->DTC.p, (const float*)s, Y);
        else if (P->tc2 && P->tc3_ctas > 0 && !(coarse && P->coarse_tc == 2))
          launch_pdl(P->pdl && st == s0, tgemm_tc3_kernel<R>,
                     std::min(u1 - u0, P->tc3_ctas * P->n_sm), 128, tc2_smem_bytes<R>(), st, up, u1 - u0,
                     (const TEnt*)P->tents.p, (const float*)P->DTC.p, (const float*)s, Y);
        else if (P->tc2)
          launch_pdl(P->pdl && st == s0, tgemm_tc2_kernel<R>, u1 - u0, 128, tc2_smem_bytes<R>(), st, up,
                     (const TEnt*)P->tents.p, (const float*)P->DTC.p, (const float*)s, Y);
        else
          launch_pdl(P->pdl && st == s0, tgemm_tc_kernel<R>, u1 - u0, 128, kTcSmem, st, up,
                     (const TEnt*)P->tents.p, (const float*)P->DTC.p, (const float*)s, Y);
      }
    } else if (Q == 64)
      launch_pdl(P->pdl && st == s0, tgemm_wt_kernel<T, R, 64>, u1 - u0, 128, TGW<T, R, 64>::SMEM, st,
                 up, (const TEnt*)P->tents.p, DTp, (const T*)s, Y, (T*)nullptr);
    else if (Q == 32)
      launch_pdl(P->pdl && st == s0, tgemm_wt_kernel<T, R, 32>, u1 - u0, 128, TGW<T, R, 32>::SMEM, st,
                 up, (const TEnt*)P->tents.p, DTp, (const T*)s, Y, (T*)nullptr);
    else
      tgemm_kernel<T, R><<<u1 - u0, kTGThreads, tgemm_smem_bytes<T, R>(Q), st>>>(up, P->tents.p, DTp,
                                                                                s, Y, Q);
    nk++;
    tr("translate", st);
  };
  auto reduce = [&](int64_t i0, int64_t i1, cudaStream_t st) {
    // o[g] = translation sum of the listed local groups
    if (i1 <= i0 || P->pat) return;
    launch_pdl(P->pdl && st == s0, reduce_kernel<T, R>, grid_for((i1 - i0) * 32, 256, cap), 256, 0,
               st, (const int32_t*)(P->red_ids.p + i0), i1 - i0, (const int64_t*)P->int_ptr.p,
               (const T*)Y, o, Q);
    nk++;
    tr("reduce", st);
  };
  // the near field's completion joins the far stream once: before the fused
  // leaf-level reception (recv_fused) or before finish()
  bool near_joined = false, recv_done = false;
  const bool far_recv = far && (stage == 0 || stage == 2);
  auto join_near = [&]() {
    if (near_joined) return;
    near_joined = true;
    CUDA_OK(cudaEventRecord(P->ev_join, join_stream));
    CUDA_OK(cudaStreamWaitEvent(s0, P->ev_join, 0));
  };
  // fine levels: the wide downward kernels sum the translation partials Y
  // themselves (no fine reduce pass; NESA_DOWN_YSUM=0 restores it)
  bool ysum_down = false;
  auto down_level = [&](int lv) {
    const int ci = lv - P->l0;
    if (P->loc_count[ci] == 0) return;
    LevelArgs<T, R> la = level_args(ci, BT + size_t(ci - 1) * 4 * mstride);
    if (ysum_down && lv >= P->split_lv) {  // translation sums formed in the down kernel
      la.Y = Y;
      la.yptr = P->int_ptr.p;
    }
    if (Q == 64 && la.count >= P->wide_level) {
      const int gw = int((la.count + TGW<T, R, 64>::PER - 1) / TGW<T, R, 64>::PER);
      if (lv == P->L && P->beta_fused && far_recv) {
        // leaf level + reception coefficients beta^ = E^ o in one kernel
        if constexpr (std::is_same<T, float>::value) {
          RecvArgs rv{};
          rv.ET = P->ET.p;
          rv.beta = reinterpret_cast<float*>(P->beta.p);
          launch_pdl(P->pdl, level_wt_kernel<T, R, 64, kLvlDownBeta>, gw, 128,
                     LVW<T, R, 64, kLvlDownBeta>::SMEM, s0, la, rv);
        }
      } else if (lv == P->L && P->recv_fused && far_recv) {
        // leaf level + reception coefficients + reception in one kernel: the
        // near field must be complete (phin)
        join_near();
        if constexpr (std::is_same<T, float>::value) {
          RecvArgs rv{P->ET.p, P->mf_prel.p, P->gstart.p, P->gstop.p, P->mf_leaf_r.p,
                      near ? reinterpret_cast<const float*>(phin) : nullptr, P->perm.p,
                      reinterpret_cast<float*>(phi), P->ldv, P->u_nt};
          launch_pdl(false, level_wt_kernel<T, R, 64, kLvlDownRecv>, gw, 128,
                     LVW<T, R, 64, kLvlDownRecv>::SMEM, s0, la, rv);
        }
        recv_done = true;
      } else {
        launch_pdl(P->pdl, level_wt_kernel<T, R, 64, kLvlDown>, gw, 128, LVW<T, R, 64, kLvlDown>::SMEM, s0, la,
                   RecvArgs{});
      }
    } else {
      launch_pdl(P->pdl, level_kernel<T, R, kLvlDown>, int((la.count + la.TC - 1) / la.TC),
                 kFarThreads, lvl_sm, s0, la);
    }
    nk++;
    tr(la.count >= P->wide_level && Q == 64 ? "down_wt" : "down", s0);
  };
  auto fused_args = [&](const T* MT) {
    FusedArgs<T> fa{};
    fa.MT = MT;
    fa.mstride = mstride;
    fa.quad = P->quad.p;
    fa.parent = P->parent.p;
    fa.uchild = P->uchild.p;
    fa.anc = P->fused_anc.p;
    fa.cnt = P->fused_cnt.p;
    fa.state = P->fused_state.p;
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
    fa.spec = P->fused_spec ? 1 : 0;
    return fa;
  };
  const bool fused = P->fused_lf > P->l0;
  const size_t fsm = fused_smem_bytes<T>(Q, R);
  // upward transfers of the fused coarse levels + the top-level sum
  auto fused_up = [&]() {
    const FusedArgs<T> fa = fused_args(CT);
    launch_pdl(P->pdl, fused_up_kernel<T, R>, int(fa.count), kFusedThreads, fsm, s0, fa);
    nk++;
    tr("up_fused", s0);
  };
  auto fused_down = [&]() {
    const FusedArgs<T> fa = fused_args(BT);
    launch_pdl(P->pdl, fused_down_kernel<T, R>, int(fa.count), kFusedThreads, fsm, s0, fa);
    nk++;
    tr("down_fused", s0);
  };
  auto coarse_mega = [&]() {
    CoarseArgs<T> ca{};
    ca.f = fused_args(CT);
    ca.BT = BT;
    ca.DT = reinterpret_cast<const T*>(P->DT.p);
    ca.int_ptr = P->int_ptr.p;
    ca.e_src = P->e_src.p;
    ca.e_dt = P->e_dt.p;
    ca.glevel = P->glevel.p;
    ca.tq = P->mega_tq.p;
    ca.n_t = P->mega_nt;
    ca.lvl_count = P->mega_lcount.p;
    ca.head = P->mega_head.p;
    ca.lvl_done = P->mega_ldone.p;
    ca.tdone = P->mega_tdone.p;
    ca.ctl = P->mega_ctl.p;
    const int items = int(2 * ca.f.count + ca.n_t);
    launch_pdl(P->pdl, coarse_kernel<T, R>, std::max(1, std::min(items, P->mega_ctas * P->n_sm)),
               kFusedThreads, coarse_smem_bytes<T>(Q, R), s0, ca);
    nk++;
    tr("coarse", s0);
  };
  // Far field.  The wide (fine) levels' translation + reduce run on s2 as
  // soon as their s is final, concurrently with the coarse end of the
  // upward chain, the coarse translations and the coarse downward levels.
  auto far_pass = [&](bool split, const std::function<void(int)>& hook) {
    const bool fine = split && P->split_lv <= P->L;
    // per-level split: each fine level's translation + reduce goes to s2 as
    // soon as that level's s is final (overlapping the rest of the up pass);
    // units / red_ids are ordered fine -> coarse, level lv's range ends where
    // level lv - 1's begins (or at the fine / total boundary)
    const bool per_level = fine && P->split_levels;
    auto unit_end = [&](int lv) {
      return lv == P->split_lv ? P->n_tunits_fine : P->tu_start[lv - 1 - P->l0];
    };
    auto red_end = [&](int lv) {
      return lv == P->split_lv ? P->n_red_fine : P->red_start[lv - 1 - P->l0];
    };
    for (int lv = P->L; lv > P->l0; --lv) {
      if (fused && lv <= P->fused_lf) break;
      up_level(lv);
      if (lv == P->L) hook(2);
      if (per_level && lv >= P->split_lv) {
        const int li = lv - P->l0;
        CUDA_OK(cudaEventRecord(P->ev_lv[li], s0));
        CUDA_OK(cudaStreamWaitEvent(P->s2, P->ev_lv[li], 0));
        translate(P->tu_start[li], unit_end(lv), P->s2);
        reduce(P->red_start[li], red_end(lv), P->s2);
      } else if (fine && lv == P->split_lv && !P->fine_after_up) {
        CUDA_OK(cudaEventRecord(P->ev_sfine, s0));
      }
    }
    if (P->L == P->split_lv && fine && P->L == P->l0) CUDA_OK(cudaEventRecord(P->ev_sfine, s0));
    // the coarse levels' up, translation and down in one persistent kernel
    const bool mega = fused && fine && !per_level && P->fine_after_up == 0 && P->coarse_mega && P->mega_ready &&
                      P->split_lv == P->fused_lf + 1 && Q * R <= 256;
    if (mega) {
      coarse_mega();
    } else if (fused) {
      fused_up();
      if (P->fused_lf == P->L) hook(2);
    } else {
      top_sum();
    }
    hook(3);
    if (fine && ((P->split_lv == P->l0 && P->L > P->l0) || (P->fine_after_up == 1 && !per_level)))
      CUDA_OK(cudaEventRecord(P->ev_sfine, s0));
    if (fine) {
      if (P->fine_after_up >= 2 && !per_level) {
        // coarse translation first (it is on the critical path and needs
        // the SM slots the fine one would hold), then the fine one on s2
        translate(P->n_tunits_fine, P->n_tunits, s0);
        reduce(P->n_red_fine, P->n_red, s0);
        CUDA_OK(cudaEventRecord(P->ev_sfine, s0));
        CUDA_OK(cudaStreamWaitEvent(P->s2, P->ev_sfine, 0));
        translate(0, P->n_tunits_fine, P->s2);
        reduce(0, P->n_red_fine, P->s2);
        CUDA_OK(cudaEventRecord(P->ev_tfine, P->s2));
      } else {
        if (!per_level) {
          CUDA_OK(cudaStreamWaitEvent(P->s2, P->ev_sfine, 0));
          translate(0, P->n_tunits_fine, P->s2);
          ysum_down = P->down_ysum && Q == 64 && !P->pat && P->split_lv >= P->l0 + 1;
          if (!ysum_down) reduce(0, P->n_red_fine, P->s2);
        }
        CUDA_OK(cudaEventRecord(P->ev_tfine, P->s2));
        if (!mega) {
          translate(P->n_tunits_fine, P->n_tunits, s0);
          reduce(P->n_red_fine, P->n_red, s0);
        }
      }
    } else {
      translate(0, P->n_tunits, s0);
      reduce(0, P->n_red, s0);
    }
    hook(4);
    bool joined = !fine;
    if (fused && !mega) fused_down();
    for (int lv = P->l0 + 1; lv <= P->L; ++lv) {
      if (fused && lv <= P->fused_lf) continue;
      if (!joined && lv >= P->split_lv) {
        CUDA_OK(cudaStreamWaitEvent(s0, P->ev_tfine, 0));
        joined = true;
      }
      down_level(lv);
    }
    if (!joined) CUDA_OK(cudaStreamWaitEvent(s0, P->ev_tfine, 0));
  };
  auto up_pass = [&]() {
    for (int lv = P->L; lv > P->l0; --lv) {
      if (fused && lv <= P->fused_lf) break;
      up_level(lv);
    }
    if (fused)
      fused_up();
    else
      top_sum();
  };
  auto down_pass = [&]() {
    translate(0, P->n_tunits, s0);
    reduce(0, P->n_red, s0);
    if (fused) fused_down();
    for (int lv = P->l0 + 1; lv <= P->L; ++lv)
      if (!fused || lv > P->fused_lf) down_level(lv);
  };
  auto gather = [&]() {
    if (P->gather_inv)
      gather_inv_kernel<T, R><<<grid_for(P->N, 256, cap), 256, 0, s0>>>(q, P->iperm.p, qt, P->N, P->ldv);
    else
      gather_kernel<T, R><<<grid_for(P->N, 256, cap), 256, 0, s0>>>(q, P->perm.p, qt, P->N, P->ldv);
    nk++;
    tr("gather", s0);
  };
  auto finish = [&]() {
    if (recv_done) return;  // the fused leaf-level kernel wrote phi
    prof_mark(P, prof, 2 * NESA_STAGE_RECEPTION, s0);
    if (far && P->u_mf) {
      if constexpr (std::is_same<T, float>::value)
        nk += launch_reception_exp<R>(P, o, near ? phin : nullptr, P->perm.p, phi, P->ldv, s0);
    } else if (far) {
      launch_blockgemv<T, R, kModeScatter>(P->Uset, o, phi, near ? phin : nullptr, P->perm.p,
                                           P->ldv, s0);
      nk++;
    } else if (near) {
      scatter_kernel<T, R><<<grid_for(nloc, 256, cap), 256, 0, s0>>>(
          phin, nullptr, P->perm.p, phi, P->pt_begin, nloc, P->ldv);
      nk++;
    } else {
      scatter_kernel<T, R><<<grid_for(nloc, 256, cap), 256, 0, s0>>>(
          nullptr, nullptr, P->perm.p, phi, P->pt_begin, nloc, P->ldv);
      nk++;
    }
    tr("finish", s0);
    prof_mark(P, prof, 2 * NESA_STAGE_RECEPTION + 1, s0);
  };

  if (stage == 0) {
    // gather -> radiation (full bandwidth) -> fork {near | up, translate,
    // down: compute-bound, overlaps the memory-bound near field} -> join ->
    // reception + scatter
    prof_mark(P, prof, 2 * NESA_STAGE_TOTAL, s0);
    // Near branch: forks from s0 at position `near_after` (-1/-2: before the
    // radiation; 0/1: after it; -1 and 1 add a no-op event node so the
    // far-field kernel is launched -- and resident -- before the persistent
    // near-field CTAs; 2: after the leaf-level upward kernel; 3: after the
    // upward pass; 4: after translation).
    bool forked = false;
    const bool nsplit = near && far && P->near_split > 0 && P->near_ctas != 1 && P->nearset.grid > 1;
    const int n_a = nsplit ? std::max(1, std::min(P->nearset.grid - 1,
                                                   int(P->near_frac * P->nearset.grid + 0.5)))
                           : P->nearset.grid;
    if (nsplit) join_stream = P->s3;
    auto launch_near = [&]() {
      if (forked) return;
      forked = true;
      CUDA_OK(cudaEventRecord(P->ev_fork, s0));
      CUDA_OK(cudaStreamWaitEvent(s1, P->ev_fork, 0));
      if (!near) return;
      if (profn)
        prof_mark(P, profn, 2 * NESA_STAGE_NEAR, s1);
      else if (P->near_after == 1 || P->near_after == -1)
        CUDA_OK(cudaEventRecordWithFlags(P->ev_mark, s1, cudaEventRecordExternal));
      if (P->near_ctas == 1 && P->near_nst == kStages && P->near_ncw == kNCW && P->near_ab == kABytes)
        launch_blockgemv<T, R, kModeStore, 6>(P->nearset, qt, phin, nullptr, nullptr, 0, s1);
      else if (nsplit)
        launch_blockgemv<T, R, kModeStore>(P->nearset, qt, phin, nullptr, nullptr, 0, s1, 0, n_a);
      else
        launch_blockgemv<T, R, kModeStore>(P->nearset, qt, phin, nullptr, nullptr, 0, s1);
      nk++;
      if (!nsplit) prof_mark(P, profn, 2 * NESA_STAGE_NEAR + 1, s1);
      tr("near", s1);
    };
    // optional second near-field launch (the remaining CTAs' items) forked
    // from the far chain at hook position near_split, on its own stream
    bool forked2 = false;
    auto launch_near2 = [&]() {
      if (!nsplit || forked2) return;
      forked2 = true;
      CUDA_OK(cudaEventRecord(P->ev_fork2, s0));
      CUDA_OK(cudaStreamWaitEvent(P->s3, P->ev_fork2, 0));
      launch_blockgemv<T, R, kModeStore>(P->nearset, qt, phin, nullptr, nullptr, 0, P->s3, n_a);
      nk++;
      CUDA_OK(cudaEventRecord(P->ev_join2, P->s1));
      CUDA_OK(cudaStreamWaitEvent(P->s3, P->ev_join2, 0));
      prof_mark(P, profn, 2 * NESA_STAGE_NEAR + 1, P->s3);
    };
    // float32 moment radiation reading q in the original order: the gather
    // (only the near field needs tree-ordered q) moves to the near stream
    const bool rad_direct = std::is_same<T, float>::value && far && near && P->v_mom && P->rad_direct &&
                            P->near_after == 0 && !nsplit && P->ldv == R && P->mom_kt == 0;
    if (rad_direct) {
      CUDA_OK(cudaEventRecord(P->ev_gfork, s0));
      CUDA_OK(cudaStreamWaitEvent(s1, P->ev_gfork, 0));
      if (P->gather_inv)
        gather_inv_kernel<T, R><<<grid_for(P->N, 256, cap), 256, 0, s1>>>(q, P->iperm.p, qt, P->N, P->ldv);
      else
        gather_kernel<T, R><<<grid_for(P->N, 256, cap), 256, 0, s1>>>(q, P->perm.p, qt, P->N, P->ldv);
      nk++;
    } else {
      gather();
    }
    if (far && P->near_after < 0) launch_near();
    if (far) {
      prof_mark(P, prof, 2 * NESA_STAGE_FAR, s0);
      nk += rad_direct ? launch_radiation<T, R>(P, q, s, s0, P->perm.p) : launch_radiation<T, R>(P, qt, s, s0);
      tr("radiation", s0);
    }
    if (!far || P->near_after <= 1) launch_near();
    // float32 + near + far: the (compute-bound) matrix-free reception runs at
    // the end of the far branch into phif, overlapping the near field; the
    // join is followed by one combining scatter phi[perm] = phin + phif.
    const bool rfar = far && near && P->u_mf && P->recv_far && !P->recv_fused && std::is_same<T, float>::value;
    if (far) {
      far_pass(P->split, [&](int pos) {
        if (pos == P->near_after) launch_near();
        if (pos == P->near_split) launch_near2();
      });
      launch_near2();
      launch_near();
      prof_mark(P, prof, 2 * NESA_STAGE_FAR + 1, s0);
      if (rfar) {
        if constexpr (std::is_same<T, float>::value) {
          prof_mark(P, prof, 2 * NESA_STAGE_RECEPTION, s0);
          nk += launch_reception_exp<R>(P, o, nullptr, nullptr, reinterpret_cast<float*>(P->phif.p), R, s0);
          tr("reception", s0);
          prof_mark(P, prof, 2 * NESA_STAGE_RECEPTION + 1, s0);
        }
      }
    }
    join_near();
    if (rfar) {
      scatter_kernel<T, R><<<grid_for(nloc, 256, cap), 256, 0, s0>>>(
          phin, reinterpret_cast<const T*>(P->phif.p), P->perm.p, phi, P->pt_begin, nloc, P->ldv);
      nk++;
      tr("combine", s0);
    } else {
      finish();
    }
    prof_mark(P, prof, 2 * NESA_STAGE_TOTAL + 1, s0);
  } else if (stage == 1) {
    // multi-GPU stage 1: the near field (local leaves) runs beside the
    // radiation and the upward pass, before the halo exchange; stage 2 is
    // the far field's second half and the reception
    gather();
    CUDA_OK(cudaEventRecord(P->ev_fork, s0));
    CUDA_OK(cudaStreamWaitEvent(s1, P->ev_fork, 0));
    if (near) {
      launch_blockgemv<T, R, kModeStore>(P->nearset, qt, phin, nullptr, nullptr, 0, s1);
      nk++;
    }
    if (far) {
      nk += launch_radiation<T, R>(P, qt, s, s0);
      up_pass();
    }
    join_near();
  } else {
    near_joined = true;  // phin was completed in stage 1
    if (far) down_pass();
    finish();
  }
  return nk;
}

template <typename T>
int enqueue_dispatch(nesa_plan* P, const void* q, void* phi, int R, uint32_t flags, int stage) {
  switch (R) {
    case 1:
      set_smem_attrs<T, 1>();
      return enqueue_T<T, 1>(P, static_cast<const T*>(q), static_cast<T*>(phi), flags, stage);
    case 2:
      set_smem_attrs<T, 2>();
      return enqueue_T<T, 2>(P, static_cast<const T*>(q), static_cast<T*>(phi), flags, stage);
    case 4:
      set_smem_attrs<T, 4>();
      return enqueue_T<T, 4>(P, static_cast<const T*>(q), static_cast<T*>(phi), flags, stage);
    default:
      throw NesaError(NESA_ERR_UNSUPPORTED, "nrhs * (1 + is_complex) must be 1, 2 or 4");
  }
}

int run_block(nesa_plan* P, const void* q, void* phi, int R, int ldv, uint32_t flags, void* stream,
              int stage);

// One product of nrhs right-hand sides: real columns are processed in blocks
// of <= 4 (one captured graph per block; rows of q / phi keep their stride).
int run_matvec(nesa_plan* P, const void* q, void* phi, int32_t nrhs, int32_t is_complex,
               uint32_t flags, void* stream, int stage) {
  require(P != nullptr, "null plan");
  require(nrhs >= 1, "nrhs must be >= 1");
  require(q != nullptr && phi != nullptr, "null vector");
  require(stage == 0 || !(flags & NESA_PROFILE), "profiling needs a full product");
  const int Rt = nrhs * (is_complex ? 2 : 1);
  if (Rt == 1 || Rt == 2 || Rt == 4) return run_block(P, q, phi, Rt, Rt, flags, stream, stage);
  require(stage == 0, "the staged (multi-GPU) product takes at most 4 real columns");
  require(!(flags & NESA_PROFILE), "profiling takes at most 4 real columns");
  const size_t es = P->esz;
  for (int c0 = 0; c0 < Rt;) {
    const int Rb = Rt - c0 >= 4 ? 4 : (Rt - c0 >= 2 ? 2 : 1);
    run_block(P, static_cast<const char*>(q) + c0 * es, static_cast<char*>(phi) + c0 * es, Rb, Rt,
              flags, stream, stage);
    c0 += Rb;
  }
  return NESA_OK;
}

int run_block(nesa_plan* P, const void* q, void* phi, int R, int ldv, uint32_t flags, void* stream,
              int stage) {
  CUDA_OK(cudaSetDevice(P->device));
  if (P->dtype == NESA_F64)
    ensure_workspace<double>(P, R);
  else
    ensure_workspace<float>(P, R);
  nesa_plan::GraphKey key{q, phi, R, flags & (NESA_NEAR | NESA_FAR | NESA_PROFILE | NESA_PROFILE_NEAR),
                          stage, ldv};
  P->ldv = ldv;
  auto itg = P->graphs.find(key);
  if (itg == P->graphs.end()) {
    cudaGraph_t g = nullptr;
    CUDA_OK(cudaStreamBeginCapture(P->s0, cudaStreamCaptureModeThreadLocal));
    int nk = 0;
    try {
      nk = P->dtype == NESA_F64 ? enqueue_dispatch<double>(P, q, phi, R, flags, stage)
                                : enqueue_dispatch<float>(P, q, phi, R, flags, stage);
    } catch (...) {
      cudaStreamEndCapture(P->s0, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CUDA_OK(cudaStreamEndCapture(P->s0, &g));
    if (P->l2_persist > 0) {
      // s / T / o stay L2-resident while the near field streams past them
      cudaKernelNodeAttrValue av = {};
      av.accessPolicyWindow.base_ptr = P->farws.p;
      av.accessPolicyWindow.num_bytes = P->farws.n;
      av.accessPolicyWindow.hitRatio =
          float(std::min(1.0, double(P->l2_persist) / double(std::max<size_t>(P->farws.n, 1))));
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      size_t nn = 0;
      CUDA_OK(cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      CUDA_OK(cudaGraphGetNodes(g, nodes.data(), &nn));
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        CUDA_OK(cudaGraphNodeGetType(nd, &ty));
        if (ty == cudaGraphNodeTypeKernel)
          CUDA_OK(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &av));
      }
    }
    nesa_plan::GraphEntry ent;
    // node priorities: the captured kernels keep their streams' priorities
    // (far chain above the near field) only with this flag
    CUDA_OK(cudaGraphInstantiate(&ent.exec, g, P->node_prio ? cudaGraphInstantiateFlagUseNodePriority : 0));
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
    ent.graph = g;
    if (stage == 0 && (flags & NESA_NEAR) && (flags & NESA_FAR)) P->kernels_per_matvec = nk;  // full product
    itg = P->graphs.emplace(key, ent).first;
  }
  if (flags & NESA_PROFILE) {
    if (P->prof_used == P->prof_events.size()) {
      std::vector<cudaEvent_t> evs(2 * NESA_N_STAGES + kTraceSlots);
      for (auto& e : evs) CUDA_OK(cudaEventCreate(&e));
      P->prof_events.push_back(evs);
    }
    auto& evs = P->prof_events[P->prof_used++];
    for (auto& pr : itg->second.ev_nodes)
      CUDA_OK(cudaGraphExecEventRecordNodeSetEvent(itg->second.exec, pr.first, evs[pr.second]));
  }
  CUDA_OK(cudaGraphLaunch(itg->second.exec, static_cast<cudaStream_t>(stream)));
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

NESA_API int nesa_plan_create(const nesa_plan_desc* d, int device, nesa_plan** out) {
  NESA_GUARD({
    require(d != nullptr && out != nullptr, "null argument");
    *out = nullptr;
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
    if (const char* nc = std::getenv("NESA_NEAR_CTAS")) P->near_ctas = std::atoi(nc) == 1 ? 1 : 2;
    if (const char* e = std::getenv("NESA_NEAR_UNITS")) P->near_units = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("NESA_NEAR_SKIP")) P->near_sm_skip = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("NESA_NEAR_SMEM")) P->near_smem = size_t(std::max(0, std::atoi(e)));
    if (const char* e = std::getenv("NESA_NEAR_VARIANT")) {  // "warps,stage_bytes,stages"
      int w = kNCW;
      int b = kABytes;
      int n = kStages;
      if (std::sscanf(e, "%d,%d,%d", &w, &b, &n) == 3 && bg_variant_known(w, b, n)) {
        P->near_ncw = w;
        P->near_ab = b;
        P->near_nst = n;
      }
    }
    if (P->near_ctas == 1 && !std::getenv("NESA_NEAR_VARIANT")) {
      // one CTA per SM: the generic geometry with a 6-stage ring
      P->near_ncw = kNCW;
      P->near_ab = kABytes;
      P->near_nst = kStages;
    }
    if (const char* lp = std::getenv("NESA_L2_PERSIST")) {
      int maxp = 0;
      CUDA_OK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device));
      P->l2_persist = std::min<size_t>(size_t(std::max(0, std::atoi(lp))) << 20, size_t(maxp));
      if (P->l2_persist > 0) CUDA_OK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, P->l2_persist));
    }
    if (const char* mb = std::getenv("NESA_MOM_BUF")) P->mom_buf = std::max(0, std::atoi(mb));
    if (const char* mv = std::getenv("NESA_MOM_VARIANT")) P->mom_variant = std::atoi(mv);
    if (const char* tc = std::getenv("NESA_TC")) P->tc = std::atoi(tc) != 0;
    if (const char* tc2 = std::getenv("NESA_TC2")) P->tc2 = std::atoi(tc2) != 0;
    if (const char* t3 = std::getenv("NESA_TC3_CTAS")) P->tc3_ctas = std::max(0, std::atoi(t3));
    if (const char* fu = std::getenv("NESA_FUSED")) P->fused = std::atoi(fu) != 0;
    if (const char* ns = std::getenv("NESA_NEAR_SPLIT")) P->near_split = std::atoi(ns);
    if (const char* nf = std::getenv("NESA_NEAR_FRAC")) P->near_frac = std::atof(nf);
    if (const char* nw = std::getenv("NESA_NEAR_WAVES")) P->near_waves = std::max(1, std::atoi(nw));
    if (const char* pr = std::getenv("NESA_PRIORITY")) P->priority = std::atoi(pr) != 0;
    if (const char* sp = std::getenv("NESA_SPLIT")) P->split = std::atoi(sp) != 0;
    if (const char* sl = std::getenv("NESA_SPLIT_LEVELS")) P->split_levels = std::atoi(sl) != 0;
    if (const char* fa = std::getenv("NESA_FINE_AFTER_UP")) P->fine_after_up = std::atoi(fa);
    if (const char* ct = std::getenv("NESA_COARSE_TC")) P->coarse_tc = std::atoi(ct);
    if (const char* tm = std::getenv("NESA_TC3_MINB")) P->tc3_minb = std::atoi(tm);
    if (const char* rm = std::getenv("NESA_RECV_MINB")) P->recv_minb = std::atoi(rm);
    if (const char* np = std::getenv("NESA_NODE_PRIO")) P->node_prio = std::atoi(np) != 0;
    if (const char* dy = std::getenv("NESA_DOWN_YSUM")) P->down_ysum = std::atoi(dy) != 0;
    if (const char* pt = std::getenv("NESA_PAT")) P->pat = std::atoi(pt) != 0;
    if (const char* gi = std::getenv("NESA_GATHER_INV")) P->gather_inv = std::atoi(gi) != 0;
    if (const char* rd = std::getenv("NESA_RAD_DIRECT")) P->rad_direct = std::atoi(rd) != 0;
    if (const char* fs = std::getenv("NESA_FUSED_SPEC")) P->fused_spec = std::atoi(fs) != 0;
    if (const char* cm = std::getenv("NESA_COARSE_MEGA")) P->coarse_mega = std::atoi(cm) != 0;
    if (const char* mc = std::getenv("NESA_MEGA_CTAS")) P->mega_ctas = std::max(1, std::atoi(mc));
    if (const char* pc = std::getenv("NESA_PAT_CTAS")) P->pat_ctas = std::max(1, std::atoi(pc));
    if (const char* na = std::getenv("NESA_NEAR_AFTER")) P->near_after = std::atoi(na);
    if (const char* pd = std::getenv("NESA_PDL")) P->pdl = std::atoi(pd) != 0;
    P->u_mf = d->op_dtype == NESA_F32 && !d->U_blob;
    if (const char* us = std::getenv("NESA_U_STORED")) P->u_mf = P->u_mf && std::atoi(us) == 0;
    P->v_mom = d->op_dtype == NESA_F32 && !d->V_blob;
    if (const char* vs = std::getenv("NESA_V_STORED")) P->v_mom = P->v_mom && std::atoi(vs) == 0;
    if (const char* tr = std::getenv("NESA_TRACE")) P->trace = std::atoi(tr) != 0;
    if (const char* rf = std::getenv("NESA_RECV_FAR")) P->recv_far = std::atoi(rf) != 0;
    P->leaf_begin = d->leaf_begin;
    P->leaf_end = d->leaf_end;
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
    {
      int lo = 0;  // numerically lower = higher priority
      int hi = 0;
      CUDA_OK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      // NESA_NEAR_PRIO=1: the near-field stream above the far chain
      const bool nprio = std::getenv("NESA_NEAR_PRIO") && std::atoi(std::getenv("NESA_NEAR_PRIO")) != 0;
      CUDA_OK(cudaStreamCreateWithPriority(&P->s0, cudaStreamNonBlocking, P->priority && !nprio ? hi : lo));
      CUDA_OK(cudaStreamCreateWithPriority(&P->s1, cudaStreamNonBlocking, nprio ? hi : lo));
      // s2 (side-stream translation) one step below the far chain so the
      // latency-bound level kernels are scheduled first (NESA_S2_PRIO:
      // 0 = same as the chain, 1 = middle, 2 = lowest)
      int s2p = P->priority ? hi : lo;
      if (const char* e = std::getenv("NESA_S2_PRIO")) {
        const int v = std::atoi(e);
        if (v == 1) s2p = (hi + lo) / 2 == hi ? std::min(lo, hi + 1) : (hi + lo) / 2;
        if (v >= 2) s2p = lo;
      }
      CUDA_OK(cudaStreamCreateWithPriority(&P->s2, cudaStreamNonBlocking, s2p));
      CUDA_OK(cudaStreamCreateWithPriority(&P->s3, cudaStreamNonBlocking, lo));
    }
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_fork2, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_gfork, cudaEventDisableTiming));
    P->ev_lv.assign(size_t(P->L - P->l0 + 1), nullptr);
    for (auto& e : P->ev_lv) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_join2, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_sfine, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_mark, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_tfine, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming));
    for (auto& e : P->cap_events) CUDA_OK(cudaEventCreate(&e));
    *out = P.release();
    return NESA_OK;
  })
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
// Multi-GPU halo exchange (paper_1801_03589_b200/dist.py):
// pack this rank's partial source amplitudes that other ranks need into the
// all_gather send buffer, and complete the needed groups' amplitudes as the
// rank-ordered sum of their contributors' partials (contrib rows < n_recv
// index the gathered buffer, rows >= n_recv this rank's own s[row - n_recv]).
// One kernel each instead of a dozen torch ops per product.
// ---------------------------------------------------------------------------
namespace {
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
