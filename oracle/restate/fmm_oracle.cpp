// oracle/restate — CPU restatement of the reference black-box FMM evaluation path.
//
// TEST INFRASTRUCTURE ONLY. This is the checker the GPU path is compared against:
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
// oracle/_build/liboracle.so. It is never part of the product path.
//
// It restates, in our own code and in plain scalar C++, the algorithm of the
// reference ("taskfmm", /root/reference/proj) for exactly the hot path of
// each function cites the reference file:line it follows. Loop
// orders follow the reference so the integer outputs are bit-exact and the FP64
// outputs agree to rounding. The one deliberate difference: the truncated SVD of
// the 16 canonical M2L operators (reference: Eigen BDCSVD, m2l.cpp:113-129) is a
// one-sided Jacobi SVD here; the rank rule is identical and the operator can also
// be loaded from the reference's binary cache (m2l.cpp:212-288) so that both sides
// use identical factors. Pinned against the reference's KATs and against
// oracle/_ref (the reference itself, built by oracle/build_ref.sh) in
// tests/test_oracle_*.py.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
constexpr u32 npos = 0xffffffffu;

thread_local std::string g_err;

// ---------------------------------------------------------------- geometry
struct Cube {
  double c[3] = {0.5, 0.5, 0.5};
  double w = 1.0;
};

// geometry.cpp:18-36
Cube bounding_cube(const double* xyzw, u64 n) {
  if (n == 0) throw std::invalid_argument("bounding_cube: empty particle set");
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = xyzw[a];
  for (u64 p = 0; p < n; ++p)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], xyzw[4 * p + a]);
      hi[a] = std::max(hi[a], xyzw[4 * p + a]);
    }
  double extent = 0;
  Cube cube;
  for (int a = 0; a < 3; ++a) {
    cube.c[a] = 0.5 * (lo[a] + hi[a]);
    extent = std::max(extent, hi[a] - lo[a]);
  }
  cube.w = extent > 0 ? extent * (1.0 + 1e-6) : 1.0;
  return cube;
}

// geometry.cpp:38-57: bit b of i -> 3b+2, j -> 3b+1, k -> 3b
u64 morton_encode(u32 i, u32 j, u32 k, int level) {
  u64 code = 0;
  for (int b = 0; b < level; ++b) {
    code |= u64((i >> b) & 1) << (3 * b + 2);
    code |= u64((j >> b) & 1) << (3 * b + 1);
    code |= u64((k >> b) & 1) << (3 * b);
  }
  return code;
}
void morton_decode(u64 code, int level, u32 out[3]) {
  out[0] = out[1] = out[2] = 0;
  for (int b = 0; b < level; ++b) {
    out[0] |= u32((code >> (3 * b + 2)) & 1) << b;
    out[1] |= u32((code >> (3 * b + 1)) & 1) << b;
    out[2] |= u32((code >> (3 * b)) & 1) << b;
  }
}

struct Level {
  std::vector<u64> code;
  std::vector<u32> first_particle, particle_count, parent, first_child, child_count;
  std::vector<u32> block_offsets;
  std::vector<double> multipole, local_own, local_down;
  u64 size() const { return code.size(); }
};

struct Tree {
  int height = 0, group = 0;
  Cube root;
  std::vector<Level> lv;
  std::vector<double> x, y, z, w, pot, fx, fy, fz;
  std::vector<u32> id;
  int leaf() const { return height - 1; }
  double cell_width(int v) const { return root.w / static_cast<double>(u64{1} << v); }
  // geometry.cpp:165-175
  Cube cell_cube(int v, u32 c) const {
    const double cw = cell_width(v);
    u32 ijk[3];
    morton_decode(lv[v].code[c], v, ijk);
    Cube cube;
    for (int a = 0; a < 3; ++a) cube.c[a] = root.c[a] - 0.5 * root.w + (ijk[a] + 0.5) * cw;
    cube.w = cw;
    return cube;
  }
  // geometry.cpp:177-186
  u32 find_cell(int v, u64 code) const {
    const Level& L = lv[v];
    if (code >= (u64{1} << (3 * v))) return npos;
    if (L.size() == (u64{1} << (3 * v))) return static_cast<u32>(code);
    auto it = std::lower_bound(L.code.begin(), L.code.end(), code);
    if (it == L.code.end() || *it != code) return npos;
    return static_cast<u32>(it - L.code.begin());
  }
  u32 block_of_cell(u32 c) const { return c / static_cast<u32>(group); }
  std::pair<u32, u32> block_particles(u32 b) const {  // geometry.cpp:192-197
    const Level& L = lv[leaf()];
    const u32 f = L.block_offsets[b], l = L.block_offsets[b + 1] - 1;
    return {L.first_particle[f], L.first_particle[l] + L.particle_count[l]};
  }
};

// geometry.cpp:59-161
Tree* build_tree(const double* xyzw, u64 n, int height, int group, const Cube* root_in) {
  if (height < 3 || height > 21) throw std::invalid_argument("GroupTree: height must be in [3, 21]");
  if (group < 1) throw std::invalid_argument("GroupTree: group size must be positive");
  if (n == 0) throw std::invalid_argument("GroupTree: empty particle set");
  Cube root = root_in ? *root_in : bounding_cube(xyzw, n);
  if (!(root.w > 0)) throw std::invalid_argument("GroupTree: root cube width must be positive");
  auto* t = new Tree;
  t->height = height;
  t->group = group;
  t->root = root;
  const int leaf = height - 1;
  const u32 grid = u32{1} << leaf;
  const double cw = root.w / static_cast<double>(grid);
  double lo[3];
  for (int a = 0; a < 3; ++a) lo[a] = root.c[a] - 0.5 * root.w;
  std::vector<std::pair<u64, u32>> order(n);
  for (u64 p = 0; p < n; ++p) {
    u32 ijk[3];
    for (int a = 0; a < 3; ++a) {
      const double c = xyzw[4 * p + a];
      if (c < lo[a] || c > lo[a] + root.w) {
        delete t;
        throw std::domain_error("GroupTree: particle outside the root cube");
      }
      double u = std::floor((c - lo[a]) / cw);
      if (u < 0) u = 0;
      if (u >= grid) u = grid - 1;
      ijk[a] = static_cast<u32>(u);
    }
    order[p] = {morton_encode(ijk[0], ijk[1], ijk[2], leaf), static_cast<u32>(p)};
  }
  std::sort(order.begin(), order.end());  // ties by input index (geometry.cpp:95)
  t->x.resize(n); t->y.resize(n); t->z.resize(n); t->w.resize(n); t->id.resize(n);
  for (u64 s = 0; s < n; ++s) {
    const double* p = xyzw + 4 * order[s].second;
    t->x[s] = p[0]; t->y[s] = p[1]; t->z[s] = p[2]; t->w[s] = p[3];
    t->id[s] = order[s].second;
  }
  t->lv.resize(height);
  Level& L = t->lv[leaf];
  for (u64 s = 0; s < n;) {  // geometry.cpp:113-122
    u64 e = s;
    while (e < n && order[e].first == order[s].first) ++e;
    L.code.push_back(order[s].first);
    L.first_particle.push_back(static_cast<u32>(s));
    L.particle_count.push_back(static_cast<u32>(e - s));
    s = e;
  }
  L.parent.assign(L.size(), 0); L.first_child.assign(L.size(), 0); L.child_count.assign(L.size(), 0);
  // geometry.cpp:126-136: coincident distinct particles
  std::vector<std::array<double, 3>> pos;
  for (u64 c = 0; c < L.size(); ++c) {
    pos.clear();
    for (u32 s = L.first_particle[c]; s < L.first_particle[c] + L.particle_count[c]; ++s)
      pos.push_back({t->x[s], t->y[s], t->z[s]});
    std::sort(pos.begin(), pos.end());
    for (size_t s = 1; s < pos.size(); ++s)
      if (pos[s] == pos[s - 1]) {
        delete t;
        throw std::domain_error("GroupTree: coincident particles");
      }
  }
  for (int v = leaf - 1; v >= 0; --v) {  // geometry.cpp:138-153
    Level& P = t->lv[v];
    Level& C = t->lv[v + 1];
    for (u32 c = 0; c < C.size();) {
      const u64 pc = C.code[c] >> 3;
      const u32 first = c;
      while (c < C.size() && (C.code[c] >> 3) == pc) C.parent[c++] = static_cast<u32>(P.size());
      P.code.push_back(pc);
      P.first_particle.push_back(0);
      P.particle_count.push_back(0);
      P.parent.push_back(0);
      P.first_child.push_back(first);
      P.child_count.push_back(c - first);
    }
  }
  for (int v = 0; v < height; ++v) {  // geometry.cpp:155-160
    Level& V = t->lv[v];
    const u32 cells = static_cast<u32>(V.size());
    for (u32 b = 0; b < cells; b += static_cast<u32>(group)) V.block_offsets.push_back(b);
    V.block_offsets.push_back(cells);
  }
  return t;
}

// geometry.cpp:222-242
std::vector<u32> near_field_list(const Tree& t, int v, u32 c) {
  u32 ijk[3];
  morton_decode(t.lv[v].code[c], v, ijk);
  const std::int64_t grid = std::int64_t{1} << v;
  std::vector<u32> out;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        if (!di && !dj && !dk) continue;
        const std::int64_t i = std::int64_t{ijk[0]} + di, j = std::int64_t{ijk[1]} + dj,
                           k = std::int64_t{ijk[2]} + dk;
        if (i < 0 || j < 0 || k < 0 || i >= grid || j >= grid || k >= grid) continue;
        const u32 f = t.find_cell(v, morton_encode(u32(i), u32(j), u32(k), v));
        if (f != npos) out.push_back(f);
      }
  std::sort(out.begin(), out.end());
  return out;
}

struct FarPair {
  u32 source;
  int tv[3];
};
// geometry.cpp:244-280
std::vector<FarPair> far_field_list(const Tree& t, int v, u32 c) {
  const Level& L = t.lv[v];
  const Level& P = t.lv[v - 1];
  u32 ijk[3], pijk[3];
  morton_decode(L.code[c], v, ijk);
  morton_decode(P.code[L.parent[c]], v - 1, pijk);
  const std::int64_t pgrid = std::int64_t{1} << (v - 1);
  std::vector<FarPair> out;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        const std::int64_t i = std::int64_t{pijk[0]} + di, j = std::int64_t{pijk[1]} + dj,
                           k = std::int64_t{pijk[2]} + dk;
        if (i < 0 || j < 0 || k < 0 || i >= pgrid || j >= pgrid || k >= pgrid) continue;
        const u32 np = t.find_cell(v - 1, morton_encode(u32(i), u32(j), u32(k), v - 1));
        if (np == npos) continue;
        for (u32 ch = P.first_child[np]; ch < P.first_child[np] + P.child_count[np]; ++ch) {
          u32 cijk[3];
          morton_decode(L.code[ch], v, cijk);
          FarPair fp{ch, {int(cijk[0]) - int(ijk[0]), int(cijk[1]) - int(ijk[1]), int(cijk[2]) - int(ijk[2])}};
          const int d = std::max({std::abs(fp.tv[0]), std::abs(fp.tv[1]), std::abs(fp.tv[2])});
          if (d <= 1) continue;
          out.push_back(fp);
        }
      }
  std::sort(out.begin(), out.end(), [](const FarPair& a, const FarPair& b) { return a.source < b.source; });
  return out;
}

// ---------------------------------------------------------------- chebyshev
// chebyshev.cpp:15-55
double cheb_t(int n, double x) {
  double tp = 1.0, tc = x;
  if (n == 0) return tp;
  for (int i = 1; i < n; ++i) {
    const double nx = 2.0 * x * tc - tp;
    tp = tc;
    tc = nx;
  }
  return tc;
}
std::vector<double> roots(int l) {
  std::vector<double> r(l);
  for (int m = 0; m < l; ++m) r[m] = std::cos((2 * m + 1) * std::numbers::pi / (2 * l));
  return r;
}
double s_eval(double root, double x, int l) {
  double acc = 1.0 / l;
  for (int n = 1; n < l; ++n) acc += (2.0 / l) * cheb_t(n, root) * cheb_t(n, x);
  return acc;
}

struct Interp {  // chebyshev.cpp:57-114
  int l = 0;
  std::vector<double> r, tn;  // tn[m*(l-1)+n-1] = T_n(root_m)
  std::vector<double> child[2], child_t[2];
  explicit Interp(int order) : l(order) {
    if (order < 2 || order > 10) throw std::invalid_argument("InterpolationEngine: order must be in [2, 10]");
    r = roots(l);
    tn.resize(size_t(l) * (l - 1));
    for (int m = 0; m < l; ++m)
      for (int n = 1; n < l; ++n) tn[m * (l - 1) + n - 1] = cheb_t(n, r[m]);
    for (int s = 0; s < 2; ++s) {
      child[s].resize(l * l);
      child_t[s].resize(l * l);
      for (int m = 0; m < l; ++m)
        for (int k = 0; k < l; ++k) {
          const double v = s_eval(r[m], 0.5 * r[k] + (s ? 0.5 : -0.5), l);
          child[s][m * l + k] = v;
          child_t[s][k * l + m] = v;
        }
    }
  }
  void eval_all(double x, double* out) const {
    double t[10];
    double tp = 1.0, tc = x;
    for (int n = 1; n < l; ++n) {
      t[n - 1] = tc;
      const double nx = 2.0 * x * tc - tp;
      tp = tc;
      tc = nx;
    }
    for (int m = 0; m < l; ++m) {
      double acc = 0;
      for (int n = 0; n < l - 1; ++n) acc += tn[m * (l - 1) + n] * t[n];
      out[m] = 1.0 / l + 2.0 / l * acc;
    }
  }
  void grad_all(double x, double* out) const {
    double dt[10];
    double up = 1.0, uc = 2.0 * x;
    for (int n = 1; n < l; ++n) {
      dt[n - 1] = n * up;
      const double nx = 2.0 * x * uc - up;
      up = uc;
      uc = nx;
    }
    for (int m = 0; m < l; ++m) {
      double acc = 0;
      for (int n = 0; n < l - 1; ++n) acc += tn[m * (l - 1) + n] * dt[n];
      out[m] = 2.0 / l * acc;
    }
  }
  // chebyshev.cpp:116-136
  void p2m(const Cube& cell, const double* px, const double* py, const double* pz, const double* pw,
           u64 n, double* mp) const {
    const double inv = 2.0 / cell.w;
    double sx[10], sy[10], sz[10];
    for (u64 j = 0; j < n; ++j) {
      eval_all((px[j] - cell.c[0]) * inv, sx);
      eval_all((py[j] - cell.c[1]) * inv, sy);
      eval_all((pz[j] - cell.c[2]) * inv, sz);
      double* o = mp;
      for (int a = 0; a < l; ++a) {
        const double wx = pw[j] * sx[a];
        for (int b = 0; b < l; ++b) {
          const double wxy = wx * sy[b];
          for (int c = 0; c < l; ++c) *o++ += wxy * sz[c];
        }
      }
    }
  }
  // chebyshev.cpp:138-179
  void l2p(const Cube& cell, const double* loc, const double* px, const double* py, const double* pz,
           u64 n, double* pot, double* fx, double* fy, double* fz) const {
    const double inv = 2.0 / cell.w;
    double sx[10], sy[10], sz[10], gx[10], gy[10], gz[10];
    for (u64 j = 0; j < n; ++j) {
      const double rx = (px[j] - cell.c[0]) * inv, ry = (py[j] - cell.c[1]) * inv,
                   rz = (pz[j] - cell.c[2]) * inv;
      eval_all(rx, sx); eval_all(ry, sy); eval_all(rz, sz);
      grad_all(rx, gx); grad_all(ry, gy); grad_all(rz, gz);
      double p = 0, dx = 0, dy = 0, dz = 0;
      const double* in = loc;
      for (int a = 0; a < l; ++a)
        for (int b = 0; b < l; ++b) {
          const double ss = sx[a] * sy[b], gs = gx[a] * sy[b], sg = sx[a] * gy[b];
          for (int c = 0; c < l; ++c) {
            const double v = *in++;
            p += v * ss * sz[c];
            dx += v * gs * sz[c];
            dy += v * sg * sz[c];
            dz += v * ss * gz[c];
          }
        }
      pot[j] += p;
      fx[j] -= inv * dx;
      fy[j] -= inv * dy;
      fz[j] -= inv * dz;
    }
  }
  // chebyshev.cpp:186-229 (three 1-D passes, axes cycle back into place)
  void tensor_step(const double* mt, const double* src, double* dst) const {
    const int rest = l * l;
    for (int i = 0; i < rest * l; ++i) dst[i] = 0;
    for (int k = 0; k < l; ++k)
      for (int rr = 0; rr < rest; ++rr) {
        const double s = src[k * rest + rr];
        for (int n = 0; n < l; ++n) dst[rr * l + n] += mt[k * l + n] * s;
      }
  }
  void tensor_apply(const double* m0, const double* m1, const double* m2, const double* in, double* out) const {
    double t1[1000], t2[1000];
    tensor_step(m0, in, t1);
    tensor_step(m1, t1, t2);
    tensor_step(m2, t2, out);
  }
  void m2m(int oct, const double* child_mp, double* parent) const {
    double res[1000];
    tensor_apply(child_t[(oct >> 2) & 1].data(), child_t[(oct >> 1) & 1].data(), child_t[oct & 1].data(), child_mp, res);
    for (int i = 0; i < l * l * l; ++i) parent[i] += res[i];
  }
  void l2l(int oct, const double* parent, double* child_loc) const {
    double res[1000];
    tensor_apply(child[(oct >> 2) & 1].data(), child[(oct >> 1) & 1].data(), child[oct & 1].data(), parent, res);
    for (int i = 0; i < l * l * l; ++i) child_loc[i] += res[i];
  }
};

// ---------------------------------------------------------------- m2l
struct Sym {
  int perm[3], sign[3];
};
// m2l.cpp:12-25 (perm-major, sign bits a=0 most significant)
std::array<Sym, 48> cube_symmetries() {
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  std::array<Sym, 48> ops{};
  int idx = 0;
  for (auto& p : perms)
    for (int bits = 0; bits < 8; ++bits) {
      Sym s;
      for (int a = 0; a < 3; ++a) {
        s.perm[a] = p[a];
        s.sign[a] = (bits >> (2 - a)) & 1 ? -1 : 1;
      }
      ops[idx++] = s;
    }
  return ops;
}
// m2l.cpp:45-55
std::array<std::array<int, 3>, 16> canonical_vectors() {
  std::array<std::array<int, 3>, 16> out{};
  int idx = 0;
  for (int i = 2; i <= 3; ++i)
    for (int j = 0; j <= i; ++j)
      for (int k = 0; k <= j; ++k) out[idx++] = {i, j, k};
  return out;
}
// m2l.cpp:57-70: first op (in cube_symmetries order) mapping v into the cone
int canonicalize(const int v[3], Sym* op_out) {
  const int d = std::max({std::abs(v[0]), std::abs(v[1]), std::abs(v[2])});
  if (d < 2 || d > 3) throw std::invalid_argument("canonicalize_m2l_vector: max-norm must be 2 or 3");
  static const auto ops = cube_symmetries();
  static const auto canon = canonical_vectors();
  for (const Sym& op : ops) {
    int u[3];
    for (int a = 0; a < 3; ++a) u[a] = op.sign[a] * v[op.perm[a]];
    if (!(u[0] >= u[1] && u[1] >= u[2] && u[2] >= 0 && u[0] >= 2 && u[0] <= 3)) continue;
    for (int c = 0; c < 16; ++c)
      if (canon[c][0] == u[0] && canon[c][1] == u[1] && canon[c][2] == u[2]) {
        if (op_out) *op_out = op;
        return c;
      }
  }
  throw std::logic_error("canonicalize_m2l_vector: no symmetry found");
}
// m2l.cpp:72-88
std::vector<u32> grid_permutation(const Sym& op, int l) {
  std::vector<u32> p(size_t(l) * l * l);
  int m[3];
  for (m[0] = 0; m[0] < l; ++m[0])
    for (m[1] = 0; m[1] < l; ++m[1])
      for (m[2] = 0; m[2] < l; ++m[2]) {
        u32 flat = 0;
        for (int a = 0; a < 3; ++a) {
          const int c = op.sign[a] > 0 ? m[op.perm[a]] : l - 1 - m[op.perm[a]];
          flat = flat * l + c;
        }
        p[(m[0] * l + m[1]) * l + m[2]] = flat;
      }
  return p;
}
inline int vec_slot(int i, int j, int k) { return (i + 3) * 49 + (j + 3) * 7 + (k + 3); }

// m2l.cpp:90-111, row-major n3 x n3
std::vector<double> assemble_m2l(const int v[3], int l, double width) {
  const auto r = roots(l);
  const int n3 = l * l * l;
  std::vector<std::array<double, 3>> nodes(n3);
  int idx = 0;
  for (int a = 0; a < l; ++a)
    for (int b = 0; b < l; ++b)
      for (int c = 0; c < l; ++c) nodes[idx++] = {r[a] * 0.5 * width, r[b] * 0.5 * width, r[c] * 0.5 * width};
  std::vector<double> k(size_t(n3) * n3);
  for (int m = 0; m < n3; ++m)
    for (int n = 0; n < n3; ++n) {
      const double dx = nodes[m][0] - v[0] * width - nodes[n][0];
      const double dy = nodes[m][1] - v[1] * width - nodes[n][1];
      const double dz = nodes[m][2] - v[2] * width - nodes[n][2];
      k[size_t(m) * n3 + n] = 1.0 / std::sqrt(dx * dx + dy * dy + dz * dz);
    }
  return k;
}

// One-sided Jacobi SVD of a square n x n row-major matrix: A = U diag(s) V^T,
// singular values descending. (Replaces Eigen::BDCSVD, m2l.cpp:114.)
void jacobi_svd(const std::vector<double>& a, int n, std::vector<double>& u, std::vector<double>& s,
                std::vector<double>& v) {
  // work on columns of A: W = A (col-major copy), V = I
  std::vector<double> w(size_t(n) * n), vv(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) w[size_t(j) * n + i] = a[size_t(i) * n + j];
  for (int i = 0; i < n; ++i) vv[size_t(i) * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double* wp = &w[size_t(p) * n];
        double* wq = &w[size_t(q) * n];
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < n; ++i) {
          alpha += wp[i] * wp[i];
          beta += wq[i] * wq[i];
          gamma += wp[i] * wq[i];
        }
        if (gamma == 0) continue;
        const double conv = std::abs(gamma) / std::sqrt(alpha * beta);
        off = std::max(off, conv);
        if (conv < 1e-17) continue;
        const double zeta = (beta - alpha) / (2 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
        const double c = 1 / std::sqrt(1 + t * t), sn = c * t;
        for (int i = 0; i < n; ++i) {
          const double x = wp[i], y = wq[i];
          wp[i] = c * x - sn * y;
          wq[i] = sn * x + c * y;
        }
        double* vp = &vv[size_t(p) * n];
        double* vq = &vv[size_t(q) * n];
        for (int i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - sn * y;
          vq[i] = sn * x + c * y;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> norms(n);
  std::vector<int> ord(n);
  for (int j = 0; j < n; ++j) {
    double s2 = 0;
    for (int i = 0; i < n; ++i) s2 += w[size_t(j) * n + i] * w[size_t(j) * n + i];
    norms[j] = std::sqrt(s2);
    ord[j] = j;
  }
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return norms[x] > norms[y]; });
  u.assign(size_t(n) * n, 0.0);
  v.assign(size_t(n) * n, 0.0);
  s.assign(n, 0.0);
  for (int jj = 0; jj < n; ++jj) {
    const int j = ord[jj];
    s[jj] = norms[j];
    for (int i = 0; i < n; ++i) {
      u[size_t(i) * n + jj] = norms[j] > 0 ? w[size_t(j) * n + i] / norms[j] : 0.0;
      v[size_t(i) * n + jj] = vv[size_t(j) * n + i];
    }
  }
}

struct M2LOps {  // m2l.cpp:136-204
  int l = 0;
  double eps = 0;
  int rank[16] = {};
  std::vector<double> u[16], sigma[16], v[16];  // u,v row-major n3 x rank
  int canonical[343];
  std::vector<u32> perm[343];
  int mult[16] = {};
  void build_transport() {
    std::fill(mult, mult + 16, 0);
    for (int s = 0; s < 343; ++s) canonical[s] = -1;
    for (int i = -3; i <= 3; ++i)
      for (int j = -3; j <= 3; ++j)
        for (int k = -3; k <= 3; ++k) {
          if (std::max({std::abs(i), std::abs(j), std::abs(k)}) < 2) continue;
          const int vv[3] = {i, j, k};
          Sym op;
          const int c = canonicalize(vv, &op);
          canonical[vec_slot(i, j, k)] = c;
          perm[vec_slot(i, j, k)] = grid_permutation(op, l);
          ++mult[c];
        }
  }
  void compute(int order, double e) {
    l = order;
    eps = e;
    const int n3 = l * l * l;
    const auto cv = canonical_vectors();
    for (int c = 0; c < 16; ++c) {
      const int vv[3] = {cv[c][0], cv[c][1], cv[c][2]};
      const auto k = assemble_m2l(vv, l, 1.0);
      std::vector<double> uu, ss, vvv;
      jacobi_svd(k, n3, uu, ss, vvv);
      int r = n3;  // m2l.cpp:116-122
      for (int i = 1; i < n3; ++i)
        if (ss[i] <= e * ss[0]) {
          r = i;
          break;
        }
      rank[c] = r;
      u[c].resize(size_t(n3) * r);
      v[c].resize(size_t(n3) * r);
      sigma[c].assign(ss.begin(), ss.begin() + r);
      for (int i = 0; i < n3; ++i)
        for (int s = 0; s < r; ++s) {
          u[c][size_t(i) * r + s] = uu[size_t(i) * n3 + s];
          v[c][size_t(i) * r + s] = vvv[size_t(i) * n3 + s];
        }
    }
    build_transport();
  }
  // m2l.cpp:247-288 (binary cache; row-major U, sigma, V per class)
  bool load(const char* path, int order, double e) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    u64 magic = 0;
    std::int32_t o = 0;
    double fe = 0;
    bool ok = std::fread(&magic, 8, 1, f) == 1 && std::fread(&o, 4, 1, f) == 1 && std::fread(&fe, 8, 1, f) == 1;
    if (!ok || magic != 0x4c324d4d4d465400ull || o != order || fe != e) {
      std::fclose(f);
      return false;
    }
    l = order;
    eps = e;
    const int n3 = l * l * l;
    std::int32_t rk[16];
    ok = std::fread(rk, 4, 16, f) == 16;
    for (int c = 0; c < 16 && ok; ++c) {
      rank[c] = rk[c];
      if (rk[c] < 1 || rk[c] > n3) { ok = false; break; }
      u[c].resize(size_t(n3) * rk[c]);
      sigma[c].resize(rk[c]);
      v[c].resize(size_t(n3) * rk[c]);
      ok = ok && std::fread(u[c].data(), 8, u[c].size(), f) == u[c].size();
      ok = ok && std::fread(sigma[c].data(), 8, sigma[c].size(), f) == sigma[c].size();
      ok = ok && std::fread(v[c].data(), 8, v[c].size(), f) == v[c].size();
    }
    std::fclose(f);
    if (ok) build_transport();
    return ok;
  }
  // m2l.cpp:182-204, one pair at a time (same arithmetic as the batched GEMMs)
  void apply_pair(int slot, const double* w, double* out, double scale) const {
    const int c = canonical[slot];
    const int n3 = l * l * l, r = rank[c];
    const u32* p = perm[slot].data();
    std::vector<double> z(n3), t(r), y(n3);
    for (int n = 0; n < n3; ++n) z[p[n]] = w[n];
    for (int s = 0; s < r; ++s) {
      double acc = 0;
      for (int i = 0; i < n3; ++i) acc += v[c][size_t(i) * r + s] * z[i];
      t[s] = sigma[c][s] * acc;
    }
    for (int i = 0; i < n3; ++i) {
      double acc = 0;
      for (int s = 0; s < r; ++s) acc += u[c][size_t(i) * r + s] * t[s];
      y[i] = acc;
    }
    for (int m = 0; m < n3; ++m) out[m] += scale * y[p[m]];
  }
};

// ---------------------------------------------------------------- plans
struct NearPlan {  // direct.cpp:22-61
  std::vector<u32> off, cells;
  std::vector<std::vector<u32>> above, below;
  std::vector<u64> task_inter;
  u64 total = 0;
};
NearPlan near_plan(const Tree& t) {
  const int leaf = t.leaf();
  const Level& L = t.lv[leaf];
  NearPlan p;
  p.off.assign(L.size() + 1, 0);
  for (u64 c = 0; c < L.size(); ++c) {
    const auto nl = near_field_list(t, leaf, u32(c));
    p.off[c + 1] = p.off[c] + u32(nl.size());
    p.cells.insert(p.cells.end(), nl.begin(), nl.end());
  }
  const u64 nb = L.block_offsets.size() - 1;
  p.above.resize(nb);
  p.below.resize(nb);
  p.task_inter.assign(nb, 0);
  for (u32 b = 0; b < nb; ++b) {
    std::vector<u32> partners;
    u64 owned = 0;
    for (u32 c = L.block_offsets[b]; c < L.block_offsets[b + 1]; ++c) {
      const u64 nc = L.particle_count[c];
      owned += nc * (nc - 1);
      for (u32 k = p.off[c]; k < p.off[c + 1]; ++k) {
        const u32 o = p.cells[k];
        const u32 ob = t.block_of_cell(o);
        if (ob < b || (ob == b && o < c)) continue;
        if (ob != b) partners.push_back(ob);
        owned += 2 * nc * L.particle_count[o];
      }
    }
    std::sort(partners.begin(), partners.end());
    partners.erase(std::unique(partners.begin(), partners.end()), partners.end());
    p.above[b] = partners;
    p.task_inter[b] = owned;
    p.total += owned;
  }
  for (u32 b = 0; b < nb; ++b)
    for (u32 q : p.above[b]) p.below[q].push_back(b);
  return p;
}

struct FarPlan {  // taskflow.cpp:67-105 (one level)
  std::vector<u32> target, source;
  std::vector<std::uint16_t> vec;
  std::vector<u64> group_off;
  std::vector<std::vector<u32>> source_blocks;
};
FarPlan far_plan(const Tree& t, int v, const M2LOps* canon_src) {
  const Level& L = t.lv[v];
  const u64 nb = L.block_offsets.size() - 1;
  std::vector<std::vector<std::array<u32, 3>>> groups(nb * 16);
  std::vector<std::vector<u32>> sources(nb);
  for (u32 c = 0; c < L.size(); ++c) {
    const u32 tb = t.block_of_cell(c);
    for (const FarPair& fp : far_field_list(t, v, c)) {
      const int slot = vec_slot(fp.tv[0], fp.tv[1], fp.tv[2]);
      const int cl = canon_src ? canon_src->canonical[slot] : canonicalize(fp.tv, nullptr);
      groups[tb * 16 + cl].push_back({c, fp.source, u32(slot)});
      sources[tb].push_back(t.block_of_cell(fp.source));
    }
  }
  FarPlan f;
  f.group_off.assign(nb * 16 + 1, 0);
  for (u64 g = 0; g < groups.size(); ++g) f.group_off[g + 1] = f.group_off[g] + groups[g].size();
  for (auto& g : groups)
    for (auto& pr : g) {
      f.target.push_back(pr[0]);
      f.source.push_back(pr[1]);
      f.vec.push_back(std::uint16_t(pr[2]));
    }
  f.source_blocks.resize(nb);
  for (u64 b = 0; b < nb; ++b) {
    auto& s = sources[b];
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    f.source_blocks[b] = s;
  }
  return f;
}

// ---------------------------------------------------------------- evaluation
// p2p_block(mutual=true) + P2PBuffers + p2p_reduce (direct.cpp:63-200), all blocks
void p2p_mutual(Tree& t, const NearPlan& np) {
  const int leaf = t.leaf();
  const Level& L = t.lv[leaf];
  const u64 nb = L.block_offsets.size() - 1;
  // slots: per block, contributors = below + self, ascending
  std::vector<std::vector<u32>> contrib(nb);
  std::vector<std::vector<double>> data(nb);
  std::vector<u32> base(nb), pc(nb);
  for (u32 b = 0; b < nb; ++b) {
    contrib[b] = np.below[b];
    contrib[b].push_back(b);
    auto [p0, p1] = t.block_particles(b);
    base[b] = p0;
    pc[b] = p1 - p0;
    data[b].assign(contrib[b].size() * 4 * pc[b], 0.0);
  }
  auto slot = [&](u32 b, u32 who) -> double* {
    auto it = std::lower_bound(contrib[b].begin(), contrib[b].end(), who);
    if (it == contrib[b].end() || *it != who) throw std::out_of_range("P2PBuffers::slot: unknown contributor");
    return data[b].data() + (it - contrib[b].begin()) * 4 * pc[b];
  };
  const double *px = t.x.data(), *py = t.y.data(), *pz = t.z.data(), *pw = t.w.data();
  for (u32 b = 0; b < nb; ++b) {
    double* own = slot(b, b);
    for (u32 c = L.block_offsets[b]; c < L.block_offsets[b + 1]; ++c) {
      const u32 a0 = L.first_particle[c], a1 = a0 + L.particle_count[c];
      auto pair = [&](u32 i, u32 j, double* sj, u32 jb) {
        const double dx = px[i] - px[j], dy = py[i] - py[j], dz = pz[i] - pz[j];
        const double inv = 1.0 / std::sqrt(dx * dx + dy * dy + dz * dz);
        const double inv3 = inv * inv * inv;
        const u32 a = i - base[b], bb = j - base[jb];
        const u32 na = pc[b], nbb = pc[jb];
        own[a] += pw[j] * inv;
        own[na + a] += pw[j] * inv3 * dx;
        own[2 * na + a] += pw[j] * inv3 * dy;
        own[3 * na + a] += pw[j] * inv3 * dz;
        sj[bb] += pw[i] * inv;
        sj[nbb + bb] -= pw[i] * inv3 * dx;
        sj[2 * nbb + bb] -= pw[i] * inv3 * dy;
        sj[3 * nbb + bb] -= pw[i] * inv3 * dz;
      };
      for (u32 i = a0; i < a1; ++i)
        for (u32 j = i + 1; j < a1; ++j) pair(i, j, own, b);
      for (u32 k = np.off[c]; k < np.off[c + 1]; ++k) {
        const u32 o = np.cells[k];
        const u32 ob = t.block_of_cell(o);
        if (ob < b || (ob == b && o < c)) continue;
        double* side = ob == b ? own : slot(ob, b);
        for (u32 i = a0; i < a1; ++i)
          for (u32 j = L.first_particle[o]; j < L.first_particle[o] + L.particle_count[o]; ++j)
            pair(i, j, side, ob);
      }
    }
  }
  for (u32 b = 0; b < nb; ++b)  // direct.cpp:187-200
    for (u32 who : contrib[b]) {
      const double* s = slot(b, who);
      for (u32 k = 0; k < pc[b]; ++k) {
        t.pot[base[b] + k] += s[k];
        t.fx[base[b] + k] += s[pc[b] + k];
        t.fy[base[b] + k] += s[2 * pc[b] + k];
        t.fz[base[b] + k] += s[3 * pc[b] + k];
      }
    }
}

// One-sided near field (p2p_block mutual=false, direct.cpp:117-149), all cells.
void p2p_onesided(Tree& t, const NearPlan& np) {
  const Level& L = t.lv[t.leaf()];
  for (u32 c = 0; c < L.size(); ++c) {
    const u32 a0 = L.first_particle[c], a1 = a0 + L.particle_count[c];
    auto in = [&](u32 i, u32 j) {
      const double dx = t.x[i] - t.x[j], dy = t.y[i] - t.y[j], dz = t.z[i] - t.z[j];
      const double inv = 1.0 / std::sqrt(dx * dx + dy * dy + dz * dz);
      const double s = t.w[j] * inv * inv * inv;
      t.pot[i] += t.w[j] * inv;
      t.fx[i] += s * dx;
      t.fy[i] += s * dy;
      t.fz[i] += s * dz;
    };
    for (u32 i = a0; i < a1; ++i)
      for (u32 j = a0; j < a1; ++j)
        if (j != i) in(i, j);
    for (u32 k = np.off[c]; k < np.off[c + 1]; ++k) {
      const u32 o = np.cells[k];
      for (u32 i = a0; i < a1; ++i)
        for (u32 j = L.first_particle[o]; j < L.first_particle[o] + L.particle_count[o]; ++j) in(i, j);
    }
  }
}

enum : unsigned { K_P2M = 1, K_M2M = 2, K_M2L = 4, K_L2L = 8, K_L2P = 16, K_P2P = 32, K_ALL = 63 };

// The payloads of bench.cpp:255-344 in a topological order (level-synchronous).
void evaluate(Tree& t, const Interp& I, const M2LOps& ops, unsigned mask, bool mutual_p2p) {
  const int leaf = t.leaf();
  const size_t n3 = size_t(I.l) * I.l * I.l;
  const u64 n = t.x.size();
  t.pot.assign(n, 0); t.fx.assign(n, 0); t.fy.assign(n, 0); t.fz.assign(n, 0);
  for (auto& L : t.lv) {
    L.multipole.assign(L.size() * n3, 0);
    L.local_own.assign(L.size() * n3, 0);
    L.local_down.assign(L.size() * n3, 0);
  }
  Level& LL = t.lv[leaf];
  if (mask & K_P2M)
    for (u32 c = 0; c < LL.size(); ++c) {
      const u32 f = LL.first_particle[c];
      I.p2m(t.cell_cube(leaf, c), &t.x[f], &t.y[f], &t.z[f], &t.w[f], LL.particle_count[c], &LL.multipole[c * n3]);
    }
  if (mask & K_M2M)
    for (int v = leaf - 1; v >= 2; --v) {
      Level& P = t.lv[v];
      Level& C = t.lv[v + 1];
      for (u32 c = 0; c < P.size(); ++c)
        for (u32 ch = P.first_child[c]; ch < P.first_child[c] + P.child_count[c]; ++ch)
          I.m2m(int(C.code[ch] & 7), &C.multipole[ch * n3], &P.multipole[c * n3]);
    }
  if (mask & K_M2L)
    for (int v = 2; v <= leaf; ++v) {
      const FarPlan f = far_plan(t, v, &ops);
      Level& L = t.lv[v];
      const double scale = 1.0 / t.cell_width(v);
      for (u64 i = 0; i < f.target.size(); ++i)
        ops.apply_pair(f.vec[i], &L.multipole[f.source[i] * n3], &L.local_own[f.target[i] * n3], scale);
    }
  if (mask & K_L2L)
    for (int v = 2; v < leaf; ++v) {
      Level& P = t.lv[v];
      Level& C = t.lv[v + 1];
      std::vector<double> total(n3);
      for (u32 c = 0; c < P.size(); ++c) {
        if (P.child_count[c] == 0) continue;
        for (size_t i = 0; i < n3; ++i) total[i] = P.local_own[c * n3 + i] + P.local_down[c * n3 + i];
        for (u32 ch = P.first_child[c]; ch < P.first_child[c] + P.child_count[c]; ++ch)
          I.l2l(int(C.code[ch] & 7), total.data(), &C.local_down[ch * n3]);
      }
    }
  if (mask & K_L2P) {
    std::vector<double> total(n3);
    for (u32 c = 0; c < LL.size(); ++c) {
      for (size_t i = 0; i < n3; ++i) total[i] = LL.local_own[c * n3 + i] + LL.local_down[c * n3 + i];
      const u32 f = LL.first_particle[c];
      I.l2p(t.cell_cube(leaf, c), total.data(), &t.x[f], &t.y[f], &t.z[f], LL.particle_count[c], &t.pot[f],
            &t.fx[f], &t.fy[f], &t.fz[f]);
    }
  }
  if (mask & K_P2P) {
    const NearPlan np = near_plan(t);
    if (mutual_p2p)
      p2p_mutual(t, np);
    else
      p2p_onesided(t, np);
  }
}

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::domain_error*>(&e)) return 2;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
  if (dynamic_cast<const std::logic_error*>(&e)) return 4;
  return 5;
}

}  // namespace orc

using namespace orc;

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// bench.cpp:19-61
void orc_generate_particles(u64 n, int dist, u64 seed, double* xyzw) {
  std::mt19937_64 rng(seed);
  auto u01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  if (dist == 0) {
    for (u64 i = 0; i < n; ++i) {
      const double x = u01(), y = u01(), z = u01();
      xyzw[4 * i] = x; xyzw[4 * i + 1] = y; xyzw[4 * i + 2] = z; xyzw[4 * i + 3] = 1.0;
    }
    return;
  }
  constexpr double two_pi = 6.283185307179586476925286766559;
  auto normal_pair = [&](double& a, double& b) {
    const double u1 = static_cast<double>((rng() >> 11) + 1) * 0x1.0p-53;
    const double u2 = u01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    a = r * std::cos(two_pi * u2);
    b = r * std::sin(two_pi * u2);
  };
  for (u64 i = 0; i < n; ++i) {
    double gx, gy, gz, spare, norm = 0;
    do {
      normal_pair(gx, gy);
      normal_pair(gz, spare);
      norm = std::sqrt(gx * gx + gy * gy + gz * gz);
    } while (norm < 1e-12);
    // dist 1: the reference's sphere (bench.cpp:40-59); dist 2: BASELINE.json config D's
    // "ellipsoid surface", defined as the same directions on semi-axes
    // (0.5, 0.35, 0.2) about (1/2, 1/2, 1/2)
    const double ax = 0.5, ay = dist == 2 ? 0.35 : 0.5, az = dist == 2 ? 0.2 : 0.5;
    xyzw[4 * i] = 0.5 + ax * gx / norm;
    xyzw[4 * i + 1] = 0.5 + ay * gy / norm;
    xyzw[4 * i + 2] = 0.5 + az * gz / norm;
    xyzw[4 * i + 3] = 1.0;
  }
}

u64 orc_morton_encode(u32 i, u32 j, u32 k, int level) { return morton_encode(i, j, k, level); }
int orc_bounding_cube(const double* xyzw, u64 n, double* out4) {
  try {
    const Cube c = bounding_cube(xyzw, n);
    out4[0] = c.c[0]; out4[1] = c.c[1]; out4[2] = c.c[2]; out4[3] = c.w;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_tree_create(const double* xyzw, u64 n, int height, int group, const double* root4, void** out) {
  try {
    Cube r;
    if (root4) { r.c[0] = root4[0]; r.c[1] = root4[1]; r.c[2] = root4[2]; r.w = root4[3]; }
    *out = build_tree(xyzw, n, height, group, root4 ? &r : nullptr);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
void orc_tree_destroy(void* h) { delete static_cast<Tree*>(h); }
void orc_root_cube(void* h, double* out4) {
  const Cube& c = static_cast<Tree*>(h)->root;
  out4[0] = c.c[0]; out4[1] = c.c[1]; out4[2] = c.c[2]; out4[3] = c.w;
}
u64 orc_level_cells(void* h, int v) { return static_cast<Tree*>(h)->lv[v].size(); }
// Cell AoS exactly as geometry.hpp:34-41 (32 B)
void orc_level_dump(void* h, int v, void* cells, u32* block_offsets) {
  const Level& L = static_cast<Tree*>(h)->lv[v];
  auto* out = static_cast<unsigned char*>(cells);
  for (u64 c = 0; c < L.size(); ++c) {
    unsigned char* p = out + 32 * c;
    std::memcpy(p, &L.code[c], 8);
    std::memcpy(p + 8, &L.first_particle[c], 4);
    std::memcpy(p + 12, &L.particle_count[c], 4);
    std::memcpy(p + 16, &L.parent[c], 4);
    std::memcpy(p + 20, &L.first_child[c], 4);
    std::memcpy(p + 24, &L.child_count[c], 4);
    std::memset(p + 28, 0, 4);
  }
  std::memcpy(block_offsets, L.block_offsets.data(), 4 * L.block_offsets.size());
}
void orc_sorted_particles(void* h, double* x, double* y, double* z, double* w, u32* id) {
  const Tree& t = *static_cast<Tree*>(h);
  const u64 n = t.x.size();
  std::memcpy(x, t.x.data(), 8 * n); std::memcpy(y, t.y.data(), 8 * n);
  std::memcpy(z, t.z.data(), 8 * n); std::memcpy(w, t.w.data(), 8 * n);
  std::memcpy(id, t.id.data(), 4 * n);
}

u64 orc_near_entries(void* h) { return near_plan(*static_cast<Tree*>(h)).cells.size(); }
u64 orc_near_dump(void* h, u32* off, u32* cells, u64* task_inter) {
  const NearPlan p = near_plan(*static_cast<Tree*>(h));
  std::memcpy(off, p.off.data(), 4 * p.off.size());
  std::memcpy(cells, p.cells.data(), 4 * p.cells.size());
  if (task_inter) std::memcpy(task_inter, p.task_inter.data(), 8 * p.task_inter.size());
  return p.total;
}
u64 orc_far_pairs(void* h, int v) { return far_plan(*static_cast<Tree*>(h), v, nullptr).target.size(); }
void orc_far_dump(void* h, int v, u32* target, u32* source, std::uint16_t* vec, u64* group_off) {
  const FarPlan f = far_plan(*static_cast<Tree*>(h), v, nullptr);
  std::memcpy(target, f.target.data(), 4 * f.target.size());
  std::memcpy(source, f.source.data(), 4 * f.source.size());
  std::memcpy(vec, f.vec.data(), 2 * f.vec.size());
  std::memcpy(group_off, f.group_off.data(), 8 * f.group_off.size());
}

// M2L operator set: computed (Jacobi SVD) or loaded from the reference cache.
int orc_ops_create(int order, double eps, const char* cache_path, void** out) {
  try {
    auto* o = new M2LOps;
    if (cache_path && *cache_path) {
      if (!o->load(cache_path, order, eps)) {
        delete o;
        g_err = "cannot load M2L cache";
        return 5;
      }
    } else {
      if (order < 2 || order > 10) throw std::invalid_argument("order must be in [2, 10]");
      o->compute(order, eps);
    }
    *out = o;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
void orc_ops_destroy(void* h) { delete static_cast<M2LOps*>(h); }
void orc_ops_ranks(void* h, int* ranks16, int* mult16) {
  const M2LOps& o = *static_cast<M2LOps*>(h);
  for (int c = 0; c < 16; ++c) {
    ranks16[c] = o.rank[c];
    if (mult16) mult16[c] = o.mult[c];
  }
}
// reconstructed dense operator U diag(s) V^T for canonical class c (row-major n3 x n3)
void orc_ops_dense(void* h, int c, double* out) {
  const M2LOps& o = *static_cast<M2LOps*>(h);
  const int n3 = o.l * o.l * o.l, r = o.rank[c];
  for (int m = 0; m < n3; ++m)
    for (int n = 0; n < n3; ++n) {
      double acc = 0;
      for (int s = 0; s < r; ++s) acc += o.u[c][size_t(m) * r + s] * o.sigma[c][s] * o.v[c][size_t(n) * r + s];
      out[size_t(m) * n3 + n] = acc;
    }
}
int orc_canonicalize(int i, int j, int k, int* perm3, int* sign3) {
  try {
    const int v[3] = {i, j, k};
    Sym op;
    const int c = canonicalize(v, &op);
    for (int a = 0; a < 3; ++a) { perm3[a] = op.perm[a]; sign3[a] = op.sign[a]; }
    return c;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}
void orc_grid_permutation(const int* perm3, const int* sign3, int order, u32* out) {
  Sym s;
  for (int a = 0; a < 3; ++a) { s.perm[a] = perm3[a]; s.sign[a] = sign3[a]; }
  const auto p = grid_permutation(s, order);
  std::memcpy(out, p.data(), 4 * p.size());
}
void orc_assemble_m2l(int i, int j, int k, int order, double width, double* out_rowmajor) {
  const int v[3] = {i, j, k};
  const auto m = assemble_m2l(v, order, width);
  std::memcpy(out_rowmajor, m.data(), 8 * m.size());
}
void orc_roots(int order, double* out) {
  const auto r = roots(order);
  std::memcpy(out, r.data(), 8 * order);
}
void orc_child_matrix(int order, int side, double* out) {
  Interp I(order);
  std::memcpy(out, I.child[side].data(), 8 * order * order);
}
double orc_s_eval(double root, double x, int order) { return s_eval(root, x, order); }
void orc_p2m(int order, const double* cube4, const double* px, const double* py, const double* pz, const double* pw,
             u64 n, double* mp) {
  Interp I(order);
  Cube c;
  c.c[0] = cube4[0]; c.c[1] = cube4[1]; c.c[2] = cube4[2]; c.w = cube4[3];
  I.p2m(c, px, py, pz, pw, n, mp);
}
void orc_l2p(int order, const double* cube4, const double* loc, const double* px, const double* py, const double* pz,
             u64 n, double* pot, double* fx, double* fy, double* fz) {
  Interp I(order);
  Cube c;
  c.c[0] = cube4[0]; c.c[1] = cube4[1]; c.c[2] = cube4[2]; c.w = cube4[3];
  I.l2p(c, loc, px, py, pz, n, pot, fx, fy, fz);
}
void orc_m2m(int order, int oct, const double* child, double* parent) { Interp(order).m2m(oct, child, parent); }
void orc_l2l(int order, int oct, const double* parent, double* child) { Interp(order).l2l(oct, parent, child); }

// Full (or masked) evaluation; fields returned in Morton order and in input order.
int orc_evaluate(void* tree, void* ops, unsigned mask, int mutual_p2p, double* pot, double* fx, double* fy,
                 double* fz) {
  try {
    Tree& t = *static_cast<Tree*>(tree);
    const M2LOps& o = *static_cast<M2LOps*>(ops);
    Interp I(o.l);
    evaluate(t, I, o, mask, mutual_p2p != 0);
    for (u64 i = 0; i < t.x.size(); ++i) {  // FmmContext::gather, bench.cpp:350-365
      pot[t.id[i]] = t.pot[i];
      fx[t.id[i]] = t.fx[i];
      fy[t.id[i]] = t.fy[i];
      fz[t.id[i]] = t.fz[i];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
// expansions after orc_evaluate; which: 0 multipole, 1 local_own, 2 local_down
void orc_level_expansion(void* tree, int v, int which, double* out) {
  const Level& L = static_cast<Tree*>(tree)->lv[v];
  const auto& a = which == 0 ? L.multipole : which == 1 ? L.local_own : L.local_down;
  std::memcpy(out, a.data(), 8 * a.size());
}

// direct.cpp:202-226
void orc_direct(const double* xyzw, u64 n, const u32* targets, u64 nt, double* pot, double* fx, double* fy,
                double* fz) {
  for (u64 t = 0; t < nt; ++t) {
    const double* a = xyzw + 4 * u64(targets[t]);
    double p = 0, x = 0, y = 0, z = 0;
    for (u64 j = 0; j < n; ++j) {
      if (j == targets[t]) continue;
      const double* b = xyzw + 4 * j;
      const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
      const double inv = 1.0 / std::sqrt(dx * dx + dy * dy + dz * dz);
      const double s = b[3] * inv * inv * inv;
      p += b[3] * inv;
      x += s * dx;
      y += s * dy;
      z += s * dz;
    }
    pot[t] = p; fx[t] = x; fy[t] = y; fz[t] = z;
  }
}

// count_interactions + flop_cost (taskflow.cpp:113-135, bench.cpp:102-122, 151-181):
// out: [0] near_directional, [1..height] M2L pairs per level, flops per kind in flops7
u64 orc_count(void* tree, void* ops, u64* m2l_pairs_per_level, u64* flops7) {
  const Tree& t = *static_cast<Tree*>(tree);
  const M2LOps& o = *static_cast<M2LOps*>(ops);
  const int leaf = t.leaf();
  const Level& L = t.lv[leaf];
  u64 near = 0;
  for (u32 c = 0; c < L.size(); ++c) {
    const u64 nc = L.particle_count[c];
    near += nc * (nc - 1);
    for (u32 nb : near_field_list(t, leaf, c)) near += nc * L.particle_count[nb];
  }
  const u64 l = u64(o.l), n = t.x.size();
  u64 m2l_flops = 0, transfers = 0;
  for (int v = 0; v < t.height; ++v) m2l_pairs_per_level[v] = 0;
  for (int v = 2; v <= leaf; ++v)
    for (u32 c = 0; c < t.lv[v].size(); ++c)
      for (const FarPair& fp : far_field_list(t, v, c)) {
        const u64 r = u64(o.rank[o.canonical[vec_slot(fp.tv[0], fp.tv[1], fp.tv[2])]]);
        ++m2l_pairs_per_level[v];
        m2l_flops += 4 * l * l * l * r + r * r;
      }
  for (int v = 2; v < leaf; ++v) transfers += t.lv[v + 1].size();
  flops7[0] = n * (4 * l * l * l + 15 * l);      // P2M
  flops7[1] = transfers * 6 * l * l * l * l;     // M2M
  flops7[2] = m2l_flops;                         // M2L
  flops7[3] = transfers * 6 * l * l * l * l;     // L2L
  flops7[4] = n * (16 * l * l * l + 30 * l);     // L2P
  flops7[5] = near * 15;                         // P2P
  flops7[6] = 0;                                 // P2PREDUCE
  return near;
}

}  // extern "C"
