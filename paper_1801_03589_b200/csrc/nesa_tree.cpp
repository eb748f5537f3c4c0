// nesa_tree.cpp -- native, bit-exact build of the sparse quadtree and its
// neighbor / interaction lists (reference: quadtree.py:96-245; the numpy
// restatement paper_1801_03589_b200/quadtree.py is the same algorithm).
//
// Exactness: cell coordinates are floor((p - origin) / (side / 2^l)),
// clipped, as the reference computes them.  They are formed once at level
// 30 and shifted: side / 2^(l+1) = (side / 2^l) / 2 exactly, so
// fl(d / c_(l+1)) = 2 fl(d / c_l) and floor(2y) >> 1 = floor(y) for y >= 0;
// clipping commutes with the shift.  Hence the Morton key of a point at
// level l is its level-30 key >> 2 (30 - l), bit for bit, and one sort of
// the level-30 keys gives every level's distinct-cell count.  The leaf
// order is a stable sort by the level-L key (ties in input order), group
// ids are leaves first then coarser levels, each in Morton order, and every
// list is sorted by id, as quadtree.py:151-245 does.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

constexpr int kMaxLevel = 30;

uint64_t dilate(uint64_t v) {
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
uint64_t morton(int64_t ix, int64_t iy) { return dilate(uint64_t(ix)) | (dilate(uint64_t(iy)) << 1); }

struct TreeOut {
  int32_t l0 = 0, L = 0;
  double origin[2] = {0, 0}, side = 0;
  std::vector<int32_t> level;
  std::vector<int64_t> ix, iy, start, stop, parent, child_first, n_children;
  std::vector<double> box;  // G x 4
  std::vector<int64_t> level_first, level_count;  // index lv - l0
  std::vector<int64_t> nbr_ptr, nbr_idx, int_ptr, int_idx, perm;
  std::string err;
};

struct TreeErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void build(const double* pts, int64_t n, double P, int l0_longest, TreeOut& T) {
  if (n < l0_longest) throw TreeErr("too few points for the coarsest level");
  double xmin = pts[0], ymin = pts[1], xmax = pts[0], ymax = pts[1];
  for (int64_t i = 1; i < n; ++i) {
    xmin = std::min(xmin, pts[2 * i]);
    xmax = std::max(xmax, pts[2 * i]);
    ymin = std::min(ymin, pts[2 * i + 1]);
    ymax = std::max(ymax, pts[2 * i + 1]);
  }
  const double ex = xmax - xmin, ey = ymax - ymin;
  const double side = ex >= ey ? ex : ey;  // max((ex, ey)) keeps the first of equals
  // zero extent with n >= 2 means repeated points (the reference's
  // distinctness check fires first)
  if (!(side > 0)) throw TreeErr("points must be pairwise distinct");
  int l0 = 0;
  while ((int64_t(1) << (l0 + 1)) <= l0_longest) ++l0;  // bit_length - 1
  // level-30 cell coordinates and keys
  const double cell30 = side / double(int64_t(1) << kMaxLevel);
  const int64_t top = (int64_t(1) << kMaxLevel) - 1;
  std::vector<uint64_t> key(n);
  for (int64_t i = 0; i < n; ++i) {
    const double dx = pts[2 * i] - xmin, dy = pts[2 * i + 1] - ymin;
    int64_t a = int64_t(std::floor(dx / cell30)), b = int64_t(std::floor(dy / cell30));
    a = a < 0 ? 0 : (a > top ? top : a);
    b = b < 0 ? 0 : (b > top ? top : b);
    key[i] = morton(a, b);
  }
  // one sort of (level-30 key, index) pairs serves the distinct-point check,
  // every level's cell count and (run by run) the stable leaf order
  std::vector<std::pair<uint64_t, int64_t>> kp(n);
  for (int64_t i = 0; i < n; ++i) kp[i] = {key[i], i};
  std::sort(kp.begin(), kp.end());
  std::vector<uint64_t> sk(n);
  for (int64_t i = 0; i < n; ++i) sk[i] = kp[i].first;
  // distinct points: equal points share the level-30 key
  for (int64_t i0 = 0; i0 < n;) {
    int64_t i1 = i0 + 1;
    while (i1 < n && sk[i1] == sk[i0]) ++i1;
    for (int64_t u = i0; u < i1; ++u)
      for (int64_t v = u + 1; v < i1; ++v) {
        const int64_t a = kp[u].second, b = kp[v].second;
        if (pts[2 * a] == pts[2 * b] && pts[2 * a + 1] == pts[2 * b + 1])
          throw TreeErr("points must be pairwise distinct");
      }
    i0 = i1;
  }
  auto cells = [&](int lv) {
    const int sh = 2 * (kMaxLevel - lv);
    int64_t c = 1;
    for (int64_t i = 1; i < n; ++i) c += (sk[i] >> sh) != (sk[i - 1] >> sh);
    return c;
  };
  // stopping rule (quadtree.py:140-149)
  int L = l0;
  int64_t count = cells(l0);
  while (L < kMaxLevel) {
    const int64_t nxt = cells(L + 1);
    if (nxt <= count || double(n) / double(nxt) < P) break;
    ++L;
    count = nxt;
  }
  // leaf order: stable sort by the level-L key
  const int shL = 2 * (kMaxLevel - L);
  // level-L cells are runs of the level-30 order; inside a run the stable
  // order is the input order
  std::vector<int64_t> perm(n);
  for (int64_t i0 = 0; i0 < n;) {
    int64_t i1 = i0 + 1;
    while (i1 < n && (sk[i1] >> shL) == (sk[i0] >> shL)) ++i1;
    for (int64_t i = i0; i < i1; ++i) perm[i] = kp[i].second;
    std::sort(perm.begin() + i0, perm.begin() + i1);
    i0 = i1;
  }
  const int nlev = L - l0 + 1;
  std::vector<std::vector<uint64_t>> lkeys(nlev);
  std::vector<std::vector<int64_t>> lstart(nlev), lstop(nlev), lix(nlev), liy(nlev), lpar(nlev);
  {
    auto& k = lkeys[L - l0];
    auto& s = lstart[L - l0];
    for (int64_t i = 0; i < n; ++i) {
      const uint64_t kk = key[perm[i]] >> shL;
      if (i == 0 || kk != k.back()) {
        k.push_back(kk);
        s.push_back(i);
      }
    }
    auto& e = lstop[L - l0];
    e.resize(s.size());
    for (size_t j = 0; j < s.size(); ++j) e[j] = j + 1 < s.size() ? s[j + 1] : n;
    // ij at level L: the division at level L itself, as quadtree.py:111-120
    lix[L - l0].resize(s.size());
    liy[L - l0].resize(s.size());
    for (size_t j = 0; j < s.size(); ++j) {
      const int64_t p = perm[s[j]];
      const double dx = pts[2 * p] - xmin, dy = pts[2 * p + 1] - ymin;
      int64_t a = int64_t(std::floor(dx / (side / double(int64_t(1) << L))));
      int64_t b = int64_t(std::floor(dy / (side / double(int64_t(1) << L))));
      const int64_t tl = (int64_t(1) << L) - 1;
      lix[L - l0][j] = a < 0 ? 0 : (a > tl ? tl : a);
      liy[L - l0][j] = b < 0 ? 0 : (b > tl ? tl : b);
    }
  }
  for (int lv = L - 1; lv >= l0; --lv) {
    const auto& ck = lkeys[lv + 1 - l0];
    auto& k = lkeys[lv - l0];
    auto& par = lpar[lv + 1 - l0];
    par.resize(ck.size());
    std::vector<size_t> pos;
    for (size_t j = 0; j < ck.size(); ++j) {
      const uint64_t pk = ck[j] >> 2;
      if (j == 0 || pk != (ck[j - 1] >> 2)) {
        k.push_back(pk);
        pos.push_back(j);
      }
      par[j] = int64_t(k.size()) - 1;
    }
    auto& s = lstart[lv - l0];
    auto& e = lstop[lv - l0];
    s.resize(pos.size());
    e.resize(pos.size());
    lix[lv - l0].resize(pos.size());
    liy[lv - l0].resize(pos.size());
    for (size_t j = 0; j < pos.size(); ++j) {
      s[j] = lstart[lv + 1 - l0][pos[j]];
      e[j] = j + 1 < pos.size() ? lstart[lv + 1 - l0][pos[j + 1]] : n;
      lix[lv - l0][j] = lix[lv + 1 - l0][pos[j]] >> 1;
      liy[lv - l0][j] = liy[lv + 1 - l0][pos[j]] >> 1;
    }
  }
  // ids: leaves first, then coarser levels
  T.l0 = l0;
  T.L = L;
  T.origin[0] = xmin;
  T.origin[1] = ymin;
  T.side = side;
  T.level_first.assign(nlev, 0);
  T.level_count.assign(nlev, 0);
  int64_t G = 0;
  for (int lv = L; lv >= l0; --lv) {
    T.level_first[lv - l0] = G;
    T.level_count[lv - l0] = int64_t(lkeys[lv - l0].size());
    G += T.level_count[lv - l0];
  }
  T.level.assign(G, 0);
  T.ix.assign(G, 0);
  T.iy.assign(G, 0);
  T.start.assign(G, 0);
  T.stop.assign(G, 0);
  T.parent.assign(G, -1);
  T.child_first.assign(G, -1);
  T.n_children.assign(G, 0);
  T.box.assign(size_t(G) * 4, 0.0);
  for (int lv = L; lv >= l0; --lv) {
    const int li = lv - l0;
    const int64_t f = T.level_first[li], c = T.level_count[li];
    const double h = side / double(int64_t(1) << lv);
    for (int64_t j = 0; j < c; ++j) {
      const int64_t g = f + j;
      T.level[g] = lv;
      T.ix[g] = lix[li][j];
      T.iy[g] = liy[li][j];
      T.start[g] = lstart[li][j];
      T.stop[g] = lstop[li][j];
      T.box[4 * g + 0] = xmin + double(T.ix[g]) * h;
      T.box[4 * g + 1] = ymin + double(T.iy[g]) * h;
      T.box[4 * g + 2] = xmin + double(T.ix[g] + 1) * h;
      T.box[4 * g + 3] = ymin + double(T.iy[g] + 1) * h;
      if (lv > l0) {
        const int64_t pid = T.level_first[li - 1] + lpar[li][j];
        T.parent[g] = pid;
        if (T.child_first[pid] < 0) T.child_first[pid] = g;
        T.n_children[pid] += 1;
      }
    }
  }
  // group id at integer coords (qx, qy) of level lv, -1 if absent
  auto lookup = [&](int lv, int64_t qx, int64_t qy) -> int64_t {
    if (qx < 0 || qy < 0) return -1;
    const auto& k = lkeys[lv - l0];
    const uint64_t q = morton(qx, qy);
    auto it = std::lower_bound(k.begin(), k.end(), q);
    if (it == k.end() || *it != q) return -1;
    return T.level_first[lv - l0] + int64_t(it - k.begin());
  };
  // leaf neighbor lists (3 x 3 stencil, sorted ids)
  {
    const int64_t f = T.level_first[L - l0], c = T.level_count[L - l0];
    T.nbr_ptr.assign(c + 1, 0);
    int64_t cand[9];
    for (int64_t j = 0; j < c; ++j) {
      const int64_t g = f + j;
      int m = 0;
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy) {
          const int64_t id = lookup(L, T.ix[g] + dx, T.iy[g] + dy);
          if (id >= 0) cand[m++] = id;
        }
      std::sort(cand, cand + m);
      T.nbr_idx.insert(T.nbr_idx.end(), cand, cand + m);
      T.nbr_ptr[j + 1] = int64_t(T.nbr_idx.size());
    }
  }
  // interaction lists (children of the parent's neighbors, Chebyshev >= 2)
  std::vector<int64_t> cnt(G, 0);
  std::vector<std::vector<int64_t>> rows(nlev);
  for (int lv = l0; lv <= L; ++lv) {
    const int li = lv - l0;
    const int64_t f = T.level_first[li], c = T.level_count[li];
    auto& out = rows[li];
    std::vector<int64_t> cand;
    for (int64_t j = 0; j < c; ++j) {
      const int64_t g = f + j;
      cand.clear();
      if (lv == l0) {
        for (int64_t k = 0; k < c; ++k) cand.push_back(f + k);
      } else {
        const int64_t p = T.parent[g];
        for (int dx = -1; dx <= 1; ++dx)
          for (int dy = -1; dy <= 1; ++dy) {
            const int64_t pn = lookup(lv - 1, T.ix[p] + dx, T.iy[p] + dy);
            if (pn < 0) continue;
            for (int64_t k = 0; k < T.n_children[pn]; ++k) cand.push_back(T.child_first[pn] + k);
          }
      }
      size_t w = 0;
      for (size_t r = 0; r < cand.size(); ++r) {
        const int64_t b = cand[r];
        const int64_t ch = std::max(std::llabs(T.ix[b] - T.ix[g]), std::llabs(T.iy[b] - T.iy[g]));
        if (ch >= 2) cand[w++] = b;
      }
      cand.resize(w);
      std::sort(cand.begin(), cand.end());
      out.insert(out.end(), cand.begin(), cand.end());
      cnt[g] = int64_t(w);
    }
  }
  T.int_ptr.assign(G + 1, 0);
  for (int64_t g = 0; g < G; ++g) T.int_ptr[g + 1] = T.int_ptr[g] + cnt[g];
  T.int_idx.reserve(T.int_ptr[G]);
  for (int lv = L; lv >= l0; --lv) T.int_idx.insert(T.int_idx.end(), rows[lv - l0].begin(), rows[lv - l0].end());
  T.perm = std::move(perm);
}

}  // namespace

#define NESA_TREE_API extern "C" __attribute__((visibility("default")))

struct nesa_tree {
  TreeOut t;
};

// 0 = OK; 1 = invalid input (message in nesa_tree_error); 2 = internal
NESA_TREE_API int nesa_tree_build(const double* points, int64_t n, double P, int32_t l0_groups_longest,
                                  nesa_tree** out) {
  *out = nullptr;
  nesa_tree* T = new nesa_tree;
  try {
    build(points, n, P, l0_groups_longest, T->t);
  } catch (const TreeErr& e) {
    T->t.err = e.what();
    *out = T;
    return 1;
  } catch (const std::exception& e) {
    T->t.err = e.what();
    *out = T;
    return 2;
  }
  *out = T;
  return 0;
}

NESA_TREE_API const char* nesa_tree_error(nesa_tree* T) { return T ? T->t.err.c_str() : "null tree"; }

// sizes: 0 G, 1 n_leaves, 2 nbr_idx length, 3 int_idx length, 4 l0, 5 L, 6 n (perm length)
NESA_TREE_API int64_t nesa_tree_size(nesa_tree* T, int32_t what) {
  const TreeOut& t = T->t;
  switch (what) {
    case 0: return int64_t(t.level.size());
    case 1: return t.level_count.empty() ? 0 : t.level_count[t.L - t.l0];
    case 2: return int64_t(t.nbr_idx.size());
    case 3: return int64_t(t.int_idx.size());
    case 4: return t.l0;
    case 5: return t.L;
    case 6: return int64_t(t.perm.size());
    default: return -1;
  }
}

// fields: 0 level (int32), 1 ix, 2 iy, 3 start, 4 stop, 5 parent, 6 child_first,
// 7 n_children, 8 box (double G x 4), 9 level_first, 10 level_count (L - l0 + 1,
// index lv - l0), 11 nbr_ptr, 12 nbr_idx, 13 int_ptr, 14 int_idx, 15 perm (int64),
// 16 origin + side (3 doubles)
NESA_TREE_API int nesa_tree_copy(nesa_tree* T, int32_t field, void* dst) {
  const TreeOut& t = T->t;
  auto cp = [&](const auto& v) {
    std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    return 0;
  };
  switch (field) {
    case 0: return cp(t.level);
    case 1: return cp(t.ix);
    case 2: return cp(t.iy);
    case 3: return cp(t.start);
    case 4: return cp(t.stop);
    case 5: return cp(t.parent);
    case 6: return cp(t.child_first);
    case 7: return cp(t.n_children);
    case 8: return cp(t.box);
    case 9: return cp(t.level_first);
    case 10: return cp(t.level_count);
    case 11: return cp(t.nbr_ptr);
    case 12: return cp(t.nbr_idx);
    case 13: return cp(t.int_ptr);
    case 14: return cp(t.int_idx);
    case 15: return cp(t.perm);
    case 16: {
      const double v[3] = {t.origin[0], t.origin[1], t.side};
      std::memcpy(dst, v, sizeof(v));
      return 0;
    }
    default: return 1;
  }
}

NESA_TREE_API void nesa_tree_free(nesa_tree* T) { delete T; }
