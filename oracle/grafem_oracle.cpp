// grafem_oracle.cpp — CPU ORACLE for the grafem per-timestep hot path.
//
// TEST INFRASTRUCTURE, NOT PRODUCT. A plain-C++ (no Eigen) restatement of the reference's
// algorithm, used (a) as the parity checker for the CUDA product and (b) as the CPU
// baseline that bench.py times. Nothing under paper_2103_14870_b200/ links or calls it.
//
// Each function cites the reference file:line it restates (paths relative to
// /root/reference/proj). The reference itself cannot be compiled here (Eigen3 and the
// vendored doctest/json/CLI11 are absent), so bit-parity of this oracle
// against the real Eigen build is UNPINNED; it is pinned to the reference's own unit-test
// known answers (tests/test_oracle_kat.py). The floating-point evaluation orders below
// are the documented reading of Eigen 3.4 / SSE2 / no-FMA and are
// the contract the CUDA damage kernels reproduce bit-for-bit:
//   R1  3x3 product A*B (A a plain column-major matrix): rows 0,1 -> (a0b0+a1b1)+a2b2,
//       row 2 -> a0b0+(a1b1+a2b2)   (slice-vectorised packet rows + scalar tail row)
//   R2  A^T*B (lhs is a transpose): every entry (a0b0+a1b1)+a2b2
//   R3  6x6*6 and the non-local accumulation: strictly sequential in k / table order
//   S9  sum of 9 coefficients (squaredNorm, cwiseProduct().sum()), column-major x0..x8:
//       ((x0+x2)+(x4+x6)) + ((x1+x3)+(x5+x7)), then + x8
//   N3  Vector3 norm: sqrt((x^2+y^2)+z^2);  trace: d0+(d1+d2);  det: (h0-h1)+h2 (Eigen
//       bruteforce_det3_helper)
//   material.cpp:128 `sigma = 0.5*(sigma+sigma.transpose())` has no .eval(): in a Release
//       (NDEBUG) build Eigen evaluates it in place in column-major order, so the upper
//       triangle reads already-symmetrised lower entries. Restated as such (cauchy()).
// Compile with -ffp-contract=off (no FMA contraction), IEEE div/sqrt, no -ffast-math.

#include "oracle.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolveError : std::runtime_error { using std::runtime_error::runtime_error; };

using V3 = std::array<double, 3>;
using V6 = std::array<double, 6>;
struct M3 {
  double a[3][3];  // a[row][col]
};
static M3 zero3() { M3 m; std::memset(&m, 0, sizeof m); return m; }
static M3 eye3() { M3 m = zero3(); m.a[0][0] = m.a[1][1] = m.a[2][2] = 1.0; return m; }

// ---------------------------------------------------------------- FP-order primitives
static inline M3 prod_r1(const M3& A, const M3& B) {  // R1
  M3 C;
  for (int c = 0; c < 3; ++c) {
    for (int r = 0; r < 2; ++r)
      C.a[r][c] = (A.a[r][0] * B.a[0][c] + A.a[r][1] * B.a[1][c]) + A.a[r][2] * B.a[2][c];
    C.a[2][c] = A.a[2][0] * B.a[0][c] + (A.a[2][1] * B.a[1][c] + A.a[2][2] * B.a[2][c]);
  }
  return C;
}
static inline M3 prod_r1_bt(const M3& A, const M3& B) {  // A * B^T, R1
  M3 C;
  for (int c = 0; c < 3; ++c) {
    for (int r = 0; r < 2; ++r)
      C.a[r][c] = (A.a[r][0] * B.a[c][0] + A.a[r][1] * B.a[c][1]) + A.a[r][2] * B.a[c][2];
    C.a[2][c] = A.a[2][0] * B.a[c][0] + (A.a[2][1] * B.a[c][1] + A.a[2][2] * B.a[c][2]);
  }
  return C;
}
static inline M3 prod_r2_at(const M3& A, const M3& B) {  // A^T * B, R2
  M3 C;
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r)
      C.a[r][c] = (A.a[0][r] * B.a[0][c] + A.a[1][r] * B.a[1][c]) + A.a[2][r] * B.a[2][c];
  return C;
}
static inline double sum9(const double x[9]) {  // S9 over column-major linear order
  const double l0 = (x[0] + x[2]) + (x[4] + x[6]);
  const double l1 = (x[1] + x[3]) + (x[5] + x[7]);
  return (l0 + l1) + x[8];
}
static inline void colmajor(const M3& m, double x[9]) {
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) x[3 * c + r] = m.a[r][c];
}
static inline double sqnorm9(const M3& F) {
  double x[9];
  colmajor(F, x);
  for (double& v : x) v = v * v;
  return sum9(x);
}
static inline double cwise_dot9(const M3& A, const M3& B) {
  double x[9], y[9];
  colmajor(A, x);
  colmajor(B, y);
  for (int i = 0; i < 9; ++i) x[i] = x[i] * y[i];
  return sum9(x);
}
static inline double det3(const M3& m) {  // Eigen bruteforce_det3_helper, first-row expansion
  const double h0 = m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]);
  const double h1 = m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]);
  const double h2 = m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
  return (h0 - h1) + h2;
}
static inline double trace3(const M3& m) { return m.a[0][0] + (m.a[1][1] + m.a[2][2]); }
static inline double norm3(const V3& v) { return std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]); }
static inline V3 sub3(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
static inline V3 add3(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
static inline V3 cross3(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
static inline V3 col3(const M3& m, int c) { return {m.a[0][c], m.a[1][c], m.a[2][c]}; }
static inline void setcol3(M3& m, int c, const V3& v) {
  m.a[0][c] = v[0]; m.a[1][c] = v[1]; m.a[2][c] = v[2];
}
static M3 scale3(double s, const M3& m) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = s * m.a[i][j];
  return r;
}
static M3 addm3(const M3& x, const M3& y) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = x.a[i][j] + y.a[i][j];
  return r;
}
static M3 transpose3(const M3& m) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = m.a[j][i];
  return r;
}

// ---------------------------------------------------------------- splitmix64 jitter RNG
// Not in the reference (BASELINE configs ask for seeded interior-node jitter);
// the product implements the same counter-based generator bit-for-bit.
static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline double jitter_unit(uint64_t seed, uint64_t node, int comp) {
  const uint64_t r = splitmix64(splitmix64(seed) + 3ull * node + static_cast<uint64_t>(comp));
  const double u = static_cast<double>(r >> 11) * (1.0 / 9007199254740992.0);  // [0,1)
  return 2.0 * u - 1.0;                                                        // [-1,1)
}

// ---------------------------------------------------------------- mesh (mesh.hpp:15-43)
struct Mesh {
  std::vector<V3> X;
  std::vector<std::array<int, 4>> tets;
  std::vector<std::array<int, 2>> edges;
  std::vector<std::array<int, 6>> tet_edges;
  std::vector<std::vector<int>> edge_tets;
  std::vector<double> vol;
  std::vector<M3> binv;
  std::vector<V3> centroid;
  std::vector<double> rest_len;
  int nn() const { return (int)X.size(); }
  int nt() const { return (int)tets.size(); }
  int ne() const { return (int)edges.size(); }
};
static constexpr int kLocalEdges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

// induce_edge_graph (mesh.cpp:34-70): canonical sorted unique edges; tet_edges in local
// order; edge_tets appended in ascending tet order. sort+unique == std::set iteration order.
static void induce_edge_graph(Mesh& m) {
  if (m.tets.empty()) throw GeometryError("mesh has no tetrahedra");
  const int n = m.nn();
  for (size_t e = 0; e < m.tets.size(); ++e) {
    const auto& t = m.tets[e];
    for (int i = 0; i < 4; ++i) {
      if (t[i] < 0 || t[i] >= n)
        throw GeometryError("tet " + std::to_string(e) + " references node " + std::to_string(t[i]) +
                            " out of range");
      for (int j = i + 1; j < 4; ++j)
        if (t[i] == t[j])
          throw GeometryError("tet " + std::to_string(e) + " repeats node " + std::to_string(t[i]));
    }
  }
  std::vector<uint64_t> keys;
  keys.reserve(m.tets.size() * 6);
  for (const auto& t : m.tets)
    for (const auto& le : kLocalEdges) {
      const uint64_t a = (uint64_t)std::min(t[le[0]], t[le[1]]);
      const uint64_t b = (uint64_t)std::max(t[le[0]], t[le[1]]);
      keys.push_back((a << 32) | b);
    }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  m.edges.resize(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) m.edges[i] = {(int)(keys[i] >> 32), (int)(keys[i] & 0xffffffffu)};
  m.tet_edges.resize(m.tets.size());
  m.edge_tets.assign(keys.size(), {});
  for (size_t e = 0; e < m.tets.size(); ++e) {
    const auto& t = m.tets[e];
    for (int k = 0; k < 6; ++k) {
      const uint64_t a = (uint64_t)std::min(t[kLocalEdges[k][0]], t[kLocalEdges[k][1]]);
      const uint64_t b = (uint64_t)std::max(t[kLocalEdges[k][0]], t[kLocalEdges[k][1]]);
      const int id = (int)(std::lower_bound(keys.begin(), keys.end(), (a << 32) | b) - keys.begin());
      m.tet_edges[e][k] = id;
      m.edge_tets[id].push_back((int)e);
    }
  }
}

// Eigen compute_inverse<3> (cofactor column 0, det by vectorised 3-redux, times 1/det)
static M3 inverse3(const M3& m) {
  auto cof = [&](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return m.a[i1][j1] * m.a[i2][j2] - m.a[i1][j2] * m.a[i2][j1];
  };
  const double c00 = cof(0, 0), c10 = cof(1, 0), c20 = cof(2, 0);
  const double det = (c00 * m.a[0][0] + c10 * m.a[1][0]) + c20 * m.a[2][0];
  const double invdet = 1.0 / det;
  M3 r;  // result(r,c) = cofactor<c,r> * invdet; result.row(0) = cofactors_col0 * invdet
  r.a[0][0] = c00 * invdet;
  r.a[0][1] = c10 * invdet;
  r.a[0][2] = c20 * invdet;
  r.a[1][0] = cof(0, 1) * invdet;
  r.a[1][1] = cof(1, 1) * invdet;
  r.a[1][2] = cof(2, 1) * invdet;
  r.a[2][0] = cof(0, 2) * invdet;
  r.a[2][1] = cof(1, 2) * invdet;
  r.a[2][2] = cof(2, 2) * invdet;
  return r;
}

// rest_quantities (mesh.cpp:72-100)
static void rest_quantities(Mesh& m) {
  const size_t nt = m.tets.size();
  m.vol.resize(nt);
  m.binv.resize(nt);
  m.centroid.resize(nt);
  for (size_t e = 0; e < nt; ++e) {
    const auto& t = m.tets[e];
    const V3& p0 = m.X[t[0]];
    M3 dm;
    setcol3(dm, 0, sub3(m.X[t[1]], p0));
    setcol3(dm, 1, sub3(m.X[t[2]], p0));
    setcol3(dm, 2, sub3(m.X[t[3]], p0));
    const double det = det3(dm);
    if (!(det > 0.0)) {
      std::ostringstream s;
      s << "tet " << e << " is degenerate or inverted (det = " << std::to_string(det) << ")";
      throw GeometryError(s.str());
    }
    m.vol[e] = det / 6.0;
    m.binv[e] = inverse3(dm);
    const V3 s = add3(add3(add3(p0, m.X[t[1]]), m.X[t[2]]), m.X[t[3]]);
    m.centroid[e] = {0.25 * s[0], 0.25 * s[1], 0.25 * s[2]};
  }
  m.rest_len.resize(m.edges.size());
  for (size_t i = 0; i < m.edges.size(); ++i)
    m.rest_len[i] = norm3(sub3(m.X[m.edges[i][1]], m.X[m.edges[i][0]]));
}

static Mesh make_mesh(std::vector<V3> nodes, std::vector<std::array<int, 4>> tets) {  // mesh.cpp:102-109
  Mesh m;
  m.X = std::move(nodes);
  m.tets = std::move(tets);
  induce_edge_graph(m);
  rest_quantities(m);
  return m;
}

// make_box_mesh / structured_mesh (primitives.cpp:13-79) plus seeded interior jitter
// (BASELINE configs; amplitude in cell units, applied inside node_at before rest_quantities).
static Mesh make_box(const V3& size, const std::array<int, 3>& cells, const V3& origin, double jitter,
                     uint64_t seed) {
  static constexpr int kCubeTets[6][4] = {{0, 1, 3, 7}, {0, 3, 2, 7}, {0, 2, 6, 7},
                                          {0, 6, 4, 7}, {0, 4, 5, 7}, {0, 5, 1, 7}};
  const int nx = cells[0], ny = cells[1], nz = cells[2];
  if (nx < 1 || ny < 1 || nz < 1) throw GeometryError("cell counts must be positive");
  const V3 h = {size[0] / cells[0], size[1] / cells[1], size[2] / cells[2]};
  auto node_id = [&](int i, int j, int k) { return (i * (ny + 1) + j) * (nz + 1) + k; };
  std::vector<std::array<int, 4>> tets;
  tets.reserve((size_t)nx * ny * nz * 6);
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < nz; ++k) {
        int corner[8];
        for (int b = 0; b < 8; ++b) corner[b] = node_id(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1));
        for (const auto& t : kCubeTets) tets.push_back({corner[t[0]], corner[t[1]], corner[t[2]], corner[t[3]]});
      }
  // every node is referenced by a full box, so the compaction remap is the identity
  std::vector<V3> nodes;
  nodes.reserve((size_t)(nx + 1) * (ny + 1) * (nz + 1));
  for (int i = 0; i <= nx; ++i)
    for (int j = 0; j <= ny; ++j)
      for (int k = 0; k <= nz; ++k) {
        V3 p = {origin[0] + i * h[0], origin[1] + j * h[1], origin[2] + k * h[2]};
        if (jitter != 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz) {
          const uint64_t g = (uint64_t)node_id(i, j, k);
          for (int c = 0; c < 3; ++c) p[c] = p[c] + (jitter * h[c]) * jitter_unit(seed, g, c);
        }
        nodes.push_back(p);
      }
  for (auto& t : tets) {  // orientation fix (primitives.cpp:56-62)
    M3 dm;
    setcol3(dm, 0, sub3(nodes[t[1]], nodes[t[0]]));
    setcol3(dm, 1, sub3(nodes[t[2]], nodes[t[0]]));
    setcol3(dm, 2, sub3(nodes[t[3]], nodes[t[0]]));
    if (det3(dm) < 0.0) std::swap(t[2], t[3]);
  }
  return make_mesh(std::move(nodes), std::move(tets));
}

// load_tetgen (mesh.cpp:157-221)
static std::vector<std::pair<int, std::vector<std::string>>> tokenize(const std::string& text) {
  std::vector<std::pair<int, std::vector<std::string>>> lines;
  std::istringstream in(text);
  std::string line;
  int number = 0;
  while (std::getline(in, line)) {
    ++number;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    std::istringstream ls(line);
    std::vector<std::string> tokens;
    std::string tok;
    while (ls >> tok) tokens.push_back(tok);
    if (!tokens.empty()) lines.emplace_back(number, std::move(tokens));
  }
  return lines;
}
static long parse_long(const std::string& tok, int line) {
  try {
    size_t pos = 0;
    const long v = std::stol(tok, &pos);
    if (pos != tok.size()) throw std::invalid_argument(tok);
    return v;
  } catch (const std::exception&) {
    throw FormatError("line " + std::to_string(line) + ": expected integer, got '" + tok + "'");
  }
}
static double parse_double(const std::string& tok, int line) {
  try {
    size_t pos = 0;
    const double v = std::stod(tok, &pos);
    if (pos != tok.size()) throw std::invalid_argument(tok);
    return v;
  } catch (const std::exception&) {
    throw FormatError("line " + std::to_string(line) + ": expected number, got '" + tok + "'");
  }
}
static Mesh load_tetgen(const std::string& node_text, const std::string& ele_text) {
  const auto nl = tokenize(node_text);
  if (nl.empty()) throw FormatError(".node: file is empty");
  const int hl = nl.front().first;
  const auto& ht = nl.front().second;
  if (ht.size() < 2) throw FormatError("line " + std::to_string(hl) + ": .node header needs '<count> <dim> [attrs] [markers]'");
  const long np = parse_long(ht[0], hl), dim = parse_long(ht[1], hl);
  if (dim != 3) throw FormatError("line " + std::to_string(hl) + ": only 3-dimensional .node files are supported");
  if (np <= 0) throw FormatError("line " + std::to_string(hl) + ": point count must be positive");
  if ((long)nl.size() - 1 < np)
    throw FormatError(".node: expected " + std::to_string(np) + " point lines, found " + std::to_string(nl.size() - 1));
  long base = -1;
  std::vector<V3> pts(np);
  for (long i = 0; i < np; ++i) {
    const int line = nl[i + 1].first;
    const auto& tok = nl[i + 1].second;
    if (tok.size() < 4) throw FormatError("line " + std::to_string(line) + ": point record needs '<index> x y z'");
    const long idx = parse_long(tok[0], line);
    if (base < 0) base = (idx == 0) ? 0 : 1;
    const long at = idx - base;
    if (at < 0 || at >= np)
      throw FormatError("line " + std::to_string(line) + ": point index " + std::to_string(idx) + " out of range");
    pts[at] = {parse_double(tok[1], line), parse_double(tok[2], line), parse_double(tok[3], line)};
  }
  const auto el = tokenize(ele_text);
  if (el.empty()) throw FormatError(".ele: file is empty");
  const int ehl = el.front().first;
  const auto& eht = el.front().second;
  if (eht.size() < 2) throw FormatError("line " + std::to_string(ehl) + ": .ele header needs '<count> <nodes-per-tet> [attrs]'");
  const long ntet = parse_long(eht[0], ehl), per = parse_long(eht[1], ehl);
  if (per != 4) throw FormatError("line " + std::to_string(ehl) + ": only 4-node tetrahedra are supported");
  if (ntet <= 0) throw FormatError("line " + std::to_string(ehl) + ": element count must be positive");
  if ((long)el.size() - 1 < ntet)
    throw FormatError(".ele: expected " + std::to_string(ntet) + " element lines, found " + std::to_string(el.size() - 1));
  long ebase = -1;
  std::vector<std::array<int, 4>> tets(ntet);
  for (long i = 0; i < ntet; ++i) {
    const int line = el[i + 1].first;
    const auto& tok = el[i + 1].second;
    if (tok.size() < 5) throw FormatError("line " + std::to_string(line) + ": element record needs '<index> n1 n2 n3 n4'");
    const long idx = parse_long(tok[0], line);
    if (ebase < 0) ebase = (idx == 0) ? 0 : 1;
    const long at = idx - ebase;
    if (at < 0 || at >= ntet)
      throw FormatError("line " + std::to_string(line) + ": element index " + std::to_string(idx) + " out of range");
    for (int k = 0; k < 4; ++k) {
      const long node = parse_long(tok[1 + k], line) - base;
      if (node < 0 || node >= np)
        throw FormatError("line " + std::to_string(line) + ": node index " + std::to_string(node + base) +
                          " out of range (have " + std::to_string(np) + " points)");
      tets[at][k] = (int)node;
    }
  }
  return make_mesh(std::move(pts), std::move(tets));
}

static double mean_face_area(const Mesh& m) {  // mesh.cpp:18-32
  double sum = 0.0;
  long count = 0;
  static constexpr int fl[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
  for (const auto& t : m.tets)
    for (const auto& f : fl) {
      const V3 c = cross3(sub3(m.X[t[f[1]]], m.X[t[f[0]]]), sub3(m.X[t[f[2]]], m.X[t[f[0]]]));
      sum += 0.5 * norm3(c);
      ++count;
    }
  return count ? sum / (double)count : 0.0;
}

// ---------------------------------------------------------------- material (material.cpp)
struct Material {
  double youngs = 1e6, poisson = 0.3, density = 1000.0, mu = 0.0, lambda = 0.0, sigma_thres = 1e5,
         r_d = 0.0, damp_mass = 0.0, damp_stiff = 0.0;
  int model = 0;  // 0 stable neo-hookean, 1 stvk
};
static Material mat_from(const or_material* p) {
  Material m;
  m.youngs = p->youngs; m.poisson = p->poisson; m.density = p->density; m.mu = p->mu; m.lambda = p->lambda;
  m.sigma_thres = p->sigma_thres; m.r_d = p->r_d; m.damp_mass = p->damp_mass_coeff;
  m.damp_stiff = p->damp_stiff_coeff; m.model = p->energy_model;
  return m;
}
static void validate(const Material& p) {  // material.cpp:37-43
  if (!(p.youngs > 0.0)) throw FormatError("youngs modulus must be positive");
  if (!(p.poisson >= 0.0 && p.poisson < 0.5)) throw FormatError("poisson ratio must be in [0, 0.5)");
  if (!(p.density > 0.0)) throw FormatError("density must be positive");
  if (!(p.sigma_thres > 0.0)) throw FormatError("sigma_thres must be positive");
  if (!(p.r_d >= 0.0)) throw FormatError("r_d must be non-negative");
}
static M3 cofactor(const M3& f) {  // material.cpp:48-54
  M3 c;
  setcol3(c, 0, cross3(col3(f, 1), col3(f, 2)));
  setcol3(c, 1, cross3(col3(f, 2), col3(f, 0)));
  setcol3(c, 2, cross3(col3(f, 0), col3(f, 1)));
  return c;
}
static M3 cofactor_differential(const M3& f, const M3& df) {  // material.cpp:56-62
  M3 c;
  setcol3(c, 0, add3(cross3(col3(df, 1), col3(f, 2)), cross3(col3(f, 1), col3(df, 2))));
  setcol3(c, 1, add3(cross3(col3(df, 2), col3(f, 0)), cross3(col3(f, 2), col3(df, 0))));
  setcol3(c, 2, add3(cross3(col3(df, 0), col3(f, 1)), cross3(col3(f, 0), col3(df, 1))));
  return c;
}
static inline double nh_alpha(const Material& p) { return 1.0 + p.mu / p.lambda - p.mu / (4.0 * p.lambda); }

static double energy_density(const M3& F, const Material& p) {  // material.cpp:71-84
  if (p.model == 1) {
    const M3 C = prod_r2_at(F, F);
    const double ic = trace3(C);
    const double iic = cwise_dot9(C, C);
    return 0.125 * p.lambda * (ic - 3.0) * (ic - 3.0) + 0.25 * p.mu * (iic - 2.0 * ic + 3.0);
  }
  const double ic = sqnorm9(F);
  const double j = det3(F);
  const double a = nh_alpha(p);
  return 0.5 * p.mu * (ic - 3.0) + 0.5 * p.lambda * (j - a) * (j - a) - 0.5 * p.mu * std::log(ic + 1.0);
}

static M3 stvk_S(const M3& E, const Material& p) {  // 2 mu E + lambda tr(E) I
  const double s2mu = 2.0 * p.mu;
  const double lt = p.lambda * trace3(E);
  M3 S;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) S.a[r][c] = s2mu * E.a[r][c] + lt * (r == c ? 1.0 : 0.0);
  return S;
}
static M3 stvk_E(const M3& F) {  // 0.5 (F^T F - I)
  const M3 C = prod_r2_at(F, F);
  M3 E;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) E.a[r][c] = 0.5 * (C.a[r][c] - (r == c ? 1.0 : 0.0));
  return E;
}

static M3 pk1(const M3& F, const Material& p) {  // material.cpp:86-95
  if (p.model == 1) return prod_r1(F, stvk_S(stvk_E(F), p));
  const double ic = sqnorm9(F);
  const double j = det3(F);
  const double a = nh_alpha(p);
  const double s1 = p.mu * (1.0 - 1.0 / (ic + 1.0));
  const double s2 = p.lambda * (j - a);
  const M3 cof = cofactor(F);
  M3 P;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) P.a[r][c] = s1 * F.a[r][c] + s2 * cof.a[r][c];
  return P;
}

static M3 pk1_differential(const M3& F, const M3& dF, const Material& p) {  // material.cpp:97-113
  if (p.model == 1) {
    const M3 E = stvk_E(F);
    const M3 A = prod_r2_at(dF, F), B = prod_r2_at(F, dF);
    M3 dE;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) dE.a[r][c] = 0.5 * (A.a[r][c] + B.a[r][c]);
    return addm3(prod_r1(dF, stvk_S(E, p)), prod_r1(F, stvk_S(dE, p)));
  }
  const double ic = sqnorm9(F);
  const double dic = 2.0 * cwise_dot9(F, dF);
  const double j = det3(F);
  const M3 cof = cofactor(F);
  const double dj = cwise_dot9(cof, dF);
  const double a = nh_alpha(p);
  const double c1 = p.mu * (1.0 - 1.0 / (ic + 1.0));
  const double c2 = p.mu * dic / ((ic + 1.0) * (ic + 1.0));
  const double c3 = p.lambda * dj;
  const double c4 = p.lambda * (j - a);
  const M3 dcof = cofactor_differential(F, dF);
  M3 out;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      out.a[r][c] = ((c1 * dF.a[r][c] + c2 * F.a[r][c]) + c3 * cof.a[r][c]) + c4 * dcof.a[r][c];
  return out;
}

// cartesian_stress_sixvector (material.cpp:115-135), with the Release-build in-place
// symmetrisation of material.cpp:128 (see file header).
static V6 cauchy(const M3& F, const Material& p, bool* fallback) {
  const M3 P = pk1(F, p);
  const double j = det3(F);
  M3 s;
  if (j > 0.0) {
    s = prod_r1_bt(P, F);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) s.a[r][c] = s.a[r][c] / j;
    // column-major in-place traversal of sigma = 0.5*(sigma + sigma^T)
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) s.a[r][c] = 0.5 * (s.a[r][c] + s.a[c][r]);
    if (fallback) *fallback = false;
  } else {
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) s.a[r][c] = 0.5 * (P.a[r][c] + P.a[c][r]);
    if (fallback) *fallback = true;
  }
  return {s.a[0][0], s.a[1][1], s.a[2][2], 2.0 * s.a[0][1], 2.0 * s.a[0][2], 2.0 * s.a[1][2]};
}

// ---------------------------------------------------------------- fem (fem.cpp)
struct State {
  std::vector<V3> u, v;
  std::vector<uint8_t> zeta;
  std::vector<double> chi;
  double time = 0.0;
};
static State rest_state(const Mesh& m) {  // fem.cpp:7-14
  State s;
  s.u.assign(m.nn(), V3{0, 0, 0});
  s.v.assign(m.nn(), V3{0, 0, 0});
  s.zeta.assign(m.ne(), 0);
  s.chi.assign(m.nt(), 1.0);
  return s;
}

static M3 deformation_gradient(const Mesh& m, const std::vector<V3>& u, int tet) {  // fem.cpp:22-31
  const auto& t = m.tets[tet];
  const V3& u0 = u[t[0]];
  M3 du;
  setcol3(du, 0, sub3(u[t[1]], u0));
  setcol3(du, 1, sub3(u[t[2]], u0));
  setcol3(du, 2, sub3(u[t[3]], u0));
  const M3 prod = prod_r1(du, m.binv[tet]);
  M3 F;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) F.a[r][c] = (r == c ? 1.0 : 0.0) + prod.a[r][c];
  return F;
}

using NodalForces = std::array<V3, 4>;
static NodalForces forces_from_gradient(const M3& g) {  // fem.cpp:37-44
  NodalForces f;
  for (int c = 0; c < 3; ++c) {
    const V3 col = col3(g, c);
    f[c + 1] = {-col[0], -col[1], -col[2]};
  }
  f[0] = add3(add3(col3(g, 0), col3(g, 1)), col3(g, 2));
  return f;
}

static NodalForces element_internal_force(const Mesh& m, const State& s, const Material& p, int tet) {  // fem.cpp:48-55
  const double scale = s.chi[tet] * m.vol[tet];
  if (scale == 0.0) return {V3{0, 0, 0}, V3{0, 0, 0}, V3{0, 0, 0}, V3{0, 0, 0}};
  const M3 F = deformation_gradient(m, s.u, tet);
  const M3 g = prod_r1_bt(scale3(scale, pk1(F, p)), m.binv[tet]);
  return forces_from_gradient(g);
}

// pinv_small (sparse.cpp:190-204): pseudo-inverse through an SVD with the 1e-12 * sigma_max cutoff. Eigen's JacobiSVD
// is restated as a one-sided (Hestenes) Jacobi SVD: column pairs of A (m x n, m >= n) are rotated until mutually
// orthogonal, V accumulates the rotations, sigma_j = |a_j|, U = a_j / sigma_j. Bits may differ from Eigen's two-sided
// sweep; the reference pins this path to tolerance only (test_fem.cpp:98-139: 1e-8, 1e-12).
static std::vector<double> pinv_small(const std::vector<double>& a_in, int m, int n, bool* rank_deficient) {
  std::vector<double> a(a_in), v((size_t)n * n, 0.0);  // a row-major m x n
  for (int j = 0; j < n; ++j) v[(size_t)j * n + j] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int i = 0; i < m; ++i) {
          const double ap = a[(size_t)i * n + p], aq = a[(size_t)i * n + q];
          alpha += ap * ap;
          beta += aq * aq;
          gamma += ap * aq;
        }
        if (gamma == 0.0) continue;
        off = std::max(off, std::abs(gamma) / std::sqrt(alpha * beta));
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < m; ++i) {
          const double ap = a[(size_t)i * n + p], aq = a[(size_t)i * n + q];
          a[(size_t)i * n + p] = c * ap - sn * aq;
          a[(size_t)i * n + q] = sn * ap + c * aq;
        }
        for (int i = 0; i < n; ++i) {
          const double vp = v[(size_t)i * n + p], vq = v[(size_t)i * n + q];
          v[(size_t)i * n + p] = c * vp - sn * vq;
          v[(size_t)i * n + q] = sn * vp + c * vq;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> sig(n);
  double smax = 0.0;
  for (int j = 0; j < n; ++j) {
    double ss = 0.0;
    for (int i = 0; i < m; ++i) ss += a[(size_t)i * n + j] * a[(size_t)i * n + j];
    sig[j] = std::sqrt(ss);
    smax = std::max(smax, sig[j]);
  }
  const double cutoff = 1e-12 * smax;
  int rank = 0;
  std::vector<double> out((size_t)n * m, 0.0);  // n x m
  for (int j = 0; j < n; ++j) {
    if (!(sig[j] > cutoff && sig[j] > 0.0)) continue;
    ++rank;
    for (int r = 0; r < n; ++r)
      for (int i = 0; i < m; ++i) out[(size_t)r * m + i] += v[(size_t)r * n + j] * (a[(size_t)i * n + j] / sig[j]) / sig[j];
  }
  if (rank_deficient) *rank_deficient = rank < std::min(m, n);
  return out;
}

struct EdgeDecomposition {  // EdgeForceDecomposition (fem.hpp:44-48)
  std::array<double, 6> coeff{};
  double residual = 0.0;
  bool ok = false;
};

// edge_decomposed_forces (fem.cpp:57-94): least-squares edge-force magnitudes of the element's nodal forces (rest
// volume, no chi), f_i = sum_k c_k s_ik dir_k (s = +1 where the edge leaves node i); ok = false on a current edge
// shorter than 1e-14 or a rank-deficient system
static EdgeDecomposition edge_decomposed_forces(const Mesh& m, const State& s, const Material& p, int tet) {
  EdgeDecomposition out;
  const auto& t = m.tets[tet];
  const M3 F = deformation_gradient(m, s.u, tet);
  const M3 g = prod_r1_bt(scale3(m.vol[tet], pk1(F, p)), m.binv[tet]);
  const NodalForces f = forces_from_gradient(g);
  std::array<V3, 6> dir;
  for (int k = 0; k < 6; ++k) {
    const int a = kLocalEdges[k][0], b = kLocalEdges[k][1];
    const V3 xa = add3(m.X[t[a]], s.u[t[a]]), xb = add3(m.X[t[b]], s.u[t[b]]);
    const V3 d = sub3(xb, xa);
    const double len = std::sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    if (len < 1e-14) return out;
    dir[k] = {d[0] / len, d[1] / len, d[2] / len};
  }
  std::vector<double> A(12 * 6, 0.0), b(12);
  for (int i = 0; i < 4; ++i)
    for (int a = 0; a < 3; ++a) b[3 * i + a] = f[i][a];
  for (int k = 0; k < 6; ++k)
    for (int a = 0; a < 3; ++a) {
      A[(size_t)(3 * kLocalEdges[k][0] + a) * 6 + k] = dir[k][a];
      A[(size_t)(3 * kLocalEdges[k][1] + a) * 6 + k] = -dir[k][a];
    }
  bool deficient = false;
  const std::vector<double> Ai = pinv_small(A, 12, 6, &deficient);
  double res = 0.0;
  for (int k = 0; k < 6; ++k) {
    double c = 0.0;
    for (int i = 0; i < 12; ++i) c += Ai[(size_t)k * 12 + i] * b[i];
    out.coeff[k] = c;
  }
  for (int i = 0; i < 12; ++i) {
    double r = -b[i];
    for (int k = 0; k < 6; ++k) r += A[(size_t)i * 6 + k] * out.coeff[k];
    res += r * r;
  }
  out.residual = std::sqrt(res);
  out.ok = !deficient;
  return out;
}

static std::vector<double> assemble_forces(const Mesh& m, const State& s, const Material& p) {  // fem.cpp:96-108
  const int nt = m.nt();
  std::vector<NodalForces> per(nt);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < nt; ++e) per[e] = element_internal_force(m, s, p, e);
  std::vector<double> f(3 * (size_t)m.nn(), 0.0);
  for (int e = 0; e < nt; ++e)
    for (int i = 0; i < 4; ++i)
      for (int a = 0; a < 3; ++a) f[3 * (size_t)m.tets[e][i] + a] += per[e][i][a];
  return f;
}

using Block12 = std::array<double, 144>;  // row-major 12x12
static void element_stiffness(const Mesh& m, const State& s, const Material& p, int tet, Block12& k) {  // fem.cpp:110-138
  k.fill(0.0);
  const double scale = s.chi[tet] * m.vol[tet];
  if (scale == 0.0) return;
  const M3 F = deformation_gradient(m, s.u, tet);
  const M3& binv = m.binv[tet];
  for (int c = 0; c < 4; ++c)
    for (int ax = 0; ax < 3; ++ax) {
      M3 dds = zero3();
      if (c == 0) {
        dds.a[ax][0] = -1.0; dds.a[ax][1] = -1.0; dds.a[ax][2] = -1.0;
      } else {
        dds.a[ax][c - 1] = 1.0;
      }
      const M3 dF = prod_r1(dds, binv);
      const M3 dg = prod_r1_bt(scale3(scale, pk1_differential(F, dF, p)), binv);
      const NodalForces df = forces_from_gradient(dg);
      for (int i = 0; i < 4; ++i)
        for (int a = 0; a < 3; ++a) k[(3 * i + a) * 12 + 3 * c + ax] = -df[i][a];
    }
  Block12 sym;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) sym[i * 12 + j] = 0.5 * (k[i * 12 + j] + k[j * 12 + i]);
  k = sym;
}

// ---------------------------------------------------------------- sparse (sparse.cpp)
struct Csr {
  int n = 0;
  std::vector<int> row_ptr, col;
  std::vector<double> val;
  int find(int i, int j) const {  // sparse.cpp:29-35
    const auto b = col.begin() + row_ptr[i], e = col.begin() + row_ptr[i + 1];
    const auto it = std::lower_bound(b, e, j);
    if (it == e || *it != j) return -1;
    return (int)(it - col.begin());
  }
  void add(int i, int j, double v) {  // sparse.cpp:37-42
    const int k = find(i, j);
    if (k < 0) throw SolveError("entry (" + std::to_string(i) + "," + std::to_string(j) + ") not in the fixed pattern");
    val[k] += v;
  }
  std::vector<double> multiply(const std::vector<double>& x) const {  // sparse.cpp:49-60
    std::vector<double> y(n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) acc += val[k] * x[col[k]];
      y[i] = acc;
    }
    return y;
  }
  std::vector<double> diagonal() const {  // sparse.cpp:62-69
    std::vector<double> d(n, 0.0);
    for (int i = 0; i < n; ++i) {
      const int k = find(i, i);
      if (k >= 0) d[i] = val[k];
    }
    return d;
  }
  uint64_t structure_hash() const {  // sparse.cpp:71-81
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t v) { h ^= v; h *= 1099511628211ull; };
    mix((uint64_t)n);
    for (int v : row_ptr) mix((uint64_t)v);
    for (int v : col) mix((uint64_t)v);
    return h;
  }
  void project_dirichlet(const std::vector<int>& dofs, const std::vector<double>& values, std::vector<double>& rhs) {  // sparse.cpp:98-120
    std::vector<char> fixed(n, 0);
    for (int d : dofs) fixed[d] = 1;
    for (int d : dofs) {
      const double v = values[d];
      for (int k = row_ptr[d]; k < row_ptr[d + 1]; ++k) {
        const int j = col[k];
        if (!fixed[j]) {
          const int k2 = find(j, d);
          if (k2 >= 0) {
            rhs[j] -= val[k2] * v;
            val[k2] = 0.0;
          }
        }
        val[k] = 0.0;
      }
      const int kd = find(d, d);
      if (kd >= 0) val[kd] = 1.0;
      rhs[d] = v;
    }
  }
  void shift_diagonal(const std::vector<double>& m, double s) {  // sparse.cpp:122-127
    for (int i = 0; i < n; ++i) {
      const int k = find(i, i);
      if (k >= 0) val[k] += s * m[i];
    }
  }
};

// make_system_pattern + finalize (fem.cpp:140-149, sparse.cpp:13-25): sorted unique
// scalar entries of every 3x3 node-pair block of every tet.
static Csr make_system_pattern(const Mesh& m) {
  const int nn = m.nn();
  std::vector<std::vector<int>> adj(nn);
  for (const auto& t : m.tets)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) adj[t[i]].push_back(t[j]);
  Csr K;
  K.n = 3 * nn;
  K.row_ptr.assign(K.n + 1, 0);
  for (int a = 0; a < nn; ++a) {
    auto& v = adj[a];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    for (int r = 0; r < 3; ++r) K.row_ptr[3 * a + r + 1] = 3 * (int)v.size();
  }
  for (int i = 0; i < K.n; ++i) K.row_ptr[i + 1] += K.row_ptr[i];
  K.col.resize(K.row_ptr[K.n]);
  for (int a = 0; a < nn; ++a)
    for (int r = 0; r < 3; ++r) {
      int k = K.row_ptr[3 * a + r];
      for (int b : adj[a])
        for (int c = 0; c < 3; ++c) K.col[k++] = 3 * b + c;
    }
  K.val.assign(K.col.size(), 0.0);
  return K;
}

static void assemble_stiffness(const Mesh& m, const State& s, const Material& p, Csr& K) {  // fem.cpp:151-169
  const int nt = m.nt();
  std::vector<Block12> blocks(nt);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < nt; ++e) element_stiffness(m, s, p, e, blocks[e]);
  std::fill(K.val.begin(), K.val.end(), 0.0);
  for (int e = 0; e < nt; ++e) {
    const auto& t = m.tets[e];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) K.add(3 * t[i] + a, 3 * t[j] + b, blocks[e][(3 * i + a) * 12 + 3 * j + b]);
  }
}

static std::vector<double> lumped_mass(const Mesh& m, const Material& p) {  // fem.cpp:171-179
  std::vector<double> mass(3 * (size_t)m.nn(), 0.0);
  for (int e = 0; e < m.nt(); ++e) {
    const double q = p.density * m.vol[e] / 4.0;
    for (int i = 0; i < 4; ++i)
      for (int a = 0; a < 3; ++a) mass[3 * (size_t)m.tets[e][i] + a] += q;
  }
  return mass;
}

static double total_strain_energy(const Mesh& m, const State& s, const Material& p) {  // fem.cpp:190-199
  double total = 0.0;
  for (int e = 0; e < m.nt(); ++e) {
    const double scale = s.chi[e] * m.vol[e];
    if (scale == 0.0) continue;
    total += scale * energy_density(deformation_gradient(m, s.u, e), p);
  }
  return total;
}

struct CgResult {
  int iterations = 0;
  double relative_residual = 0.0;
  bool converged = false, negative_curvature = false;
};
static double dot(const std::vector<double>& a, const std::vector<double>& b) {  // sparse.cpp:139-143
  double acc = 0.0;
  for (size_t i = 0; i < a.size(); ++i) acc += a[i] * b[i];
  return acc;
}
static CgResult cg_solve(const Csr& A, const std::vector<double>& b, std::vector<double>& x, double tol, int max_iters) {  // sparse.cpp:129-188
  CgResult res;
  const int n = A.n;
  const std::vector<double> diag = A.diagonal();
  std::vector<double> pre(n);
  for (int i = 0; i < n; ++i) pre[i] = (std::abs(diag[i]) > 1e-300) ? 1.0 / diag[i] : 1.0;
  const double bnorm = std::sqrt(dot(b, b));
  if (bnorm == 0.0) {
    std::fill(x.begin(), x.end(), 0.0);
    res.converged = true;
    return res;
  }
  const std::vector<double> ax = A.multiply(x);
  std::vector<double> r(n), z(n);
  for (int i = 0; i < n; ++i) r[i] = b[i] - ax[i];
  for (int i = 0; i < n; ++i) z[i] = pre[i] * r[i];
  std::vector<double> p = z;
  double rz = dot(r, z);
  for (int it = 0; it < max_iters; ++it) {
    const std::vector<double> Ap = A.multiply(p);
    const double pAp = dot(p, Ap);
    if (pAp <= 0.0) {
      res.negative_curvature = pAp < 0.0;
      res.iterations = it;
      res.relative_residual = std::sqrt(dot(r, r)) / bnorm;
      res.converged = res.relative_residual <= tol;
      return res;
    }
    const double alpha = rz / pAp;
    for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (int i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
    res.iterations = it + 1;
    const double rnorm = std::sqrt(dot(r, r));
    if (rnorm / bnorm <= tol) {
      res.relative_residual = rnorm / bnorm;
      res.converged = true;
      return res;
    }
    for (int i = 0; i < n; ++i) z[i] = pre[i] * r[i];
    const double rz_new = dot(r, z);
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  res.relative_residual = std::sqrt(dot(r, r)) / bnorm;
  res.converged = res.relative_residual <= tol;
  return res;
}

// ---------------------------------------------------------------- fracture (fracture.cpp)
static inline V6 transform_row(const V3& d) {  // fracture.cpp:9-14
  return {d[0] * d[0], d[1] * d[1], d[2] * d[2], d[0] * d[1], d[0] * d[2], d[1] * d[2]};
}
using M6 = std::array<V6, 6>;  // rows
static bool build_T(const Mesh& m, const std::vector<V3>& u, int tet, M6& T) {  // fracture.cpp:16-28
  const auto& t = m.tets[tet];
  for (int k = 0; k < 6; ++k) {
    const int a = t[kLocalEdges[k][0]], b = t[kLocalEdges[k][1]];
    const V3 pb = add3(m.X[b], u[b]), pa = add3(m.X[a], u[a]);
    const V3 d = sub3(pb, pa);
    const double len = norm3(d);
    if (len < 1e-14 * std::max(1.0, m.rest_len[m.tet_edges[tet][k]])) return false;
    const V3 dn = {d[0] / len, d[1] / len, d[2] / len};
    T[k] = transform_row(dn);
  }
  return true;
}
static inline V6 matvec6(const M6& T, const V6& s) {  // R3 sequential
  V6 r;
  for (int k = 0; k < 6; ++k) {
    double acc = T[k][0] * s[0];
    for (int j = 1; j < 6; ++j) acc = acc + T[k][j] * s[j];
    r[k] = acc;
  }
  return r;
}

struct Table {  // NonlocalTable (fracture.hpp:27-30) in CSR form
  std::vector<int> ptr, ids;
  std::vector<double> w;
};

// build_nonlocal_table (fracture.cpp:32-54). brute force is the literal O(T^2) loop; the
// default grid-binned build visits a superset of all tets within r_d, sorts candidates
// ascending and then applies the identical reject tests and the identical ascending wsum
// accumulation, so the table is identical entry-for-entry and bit-for-bit.
static Table build_nonlocal_table(const Mesh& m, double r_d, bool brute) {
  Table tb;
  const int nt = m.nt();
  tb.ptr.assign(nt + 1, 0);
  if (r_d <= 0.0) {
    tb.ids.resize(nt);
    tb.w.assign(nt, 1.0);
    for (int e = 0; e < nt; ++e) { tb.ptr[e + 1] = e + 1; tb.ids[e] = e; }
    return tb;
  }
  std::vector<std::vector<std::pair<int, double>>> lists(nt);
  auto fill = [&](int e, const std::vector<int>& cand) {
    auto& list = lists[e];
    double wsum = 0.0;
    for (int o : cand) {
      const double r = norm3(sub3(m.centroid[o], m.centroid[e]));
      if (r > r_d) continue;
      const double w = 1.0 - r / r_d;
      if (w <= 0.0) continue;
      list.emplace_back(o, w);
      wsum += w;
    }
    for (auto& ow : list) ow.second /= wsum;
  };
  if (brute) {
    std::vector<int> all(nt);
    std::iota(all.begin(), all.end(), 0);
#pragma omp parallel for schedule(dynamic, 64)
    for (int e = 0; e < nt; ++e) fill(e, all);
  } else {
    V3 lo = m.centroid[0], hi = m.centroid[0];
    for (const auto& c : m.centroid)
      for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], c[a]); hi[a] = std::max(hi[a], c[a]); }
    // bins at least r_d wide: every tet within r_d lies in the 27 surrounding bins
    double cell = r_d * (1.0 + 1e-9);
    int dims[3];
    for (;;) {
      double nb_est = 1.0;
      for (int a = 0; a < 3; ++a) nb_est *= std::floor((hi[a] - lo[a]) / cell) + 1.0;
      if (nb_est <= 4.0 * nt + 1024.0) break;
      cell *= 2.0;
    }
    for (int a = 0; a < 3; ++a) dims[a] = std::max(1, (int)std::floor((hi[a] - lo[a]) / cell) + 1);
    auto bin_of = [&](const V3& c, int a) {
      int b = (int)std::floor((c[a] - lo[a]) / cell);
      return std::min(std::max(b, 0), dims[a] - 1);
    };
    const size_t nb = (size_t)dims[0] * dims[1] * dims[2];
    std::vector<int> bstart(nb + 1, 0), bitems(nt);
    std::vector<size_t> tb_bin(nt);
    for (int e = 0; e < nt; ++e) {
      const auto& c = m.centroid[e];
      tb_bin[e] = ((size_t)bin_of(c, 0) * dims[1] + bin_of(c, 1)) * dims[2] + bin_of(c, 2);
      bstart[tb_bin[e] + 1]++;
    }
    for (size_t b = 0; b < nb; ++b) bstart[b + 1] += bstart[b];
    {
      std::vector<int> cur(bstart.begin(), bstart.end() - 1);
      for (int e = 0; e < nt; ++e) bitems[cur[tb_bin[e]]++] = e;
    }
#pragma omp parallel
    {
      std::vector<int> cand;
#pragma omp for schedule(dynamic, 256)
      for (int e = 0; e < nt; ++e) {
        cand.clear();
        const auto& c = m.centroid[e];
        const int bx = bin_of(c, 0), by = bin_of(c, 1), bz = bin_of(c, 2);
        for (int ix = std::max(bx - 1, 0); ix <= std::min(bx + 1, dims[0] - 1); ++ix)
          for (int iy = std::max(by - 1, 0); iy <= std::min(by + 1, dims[1] - 1); ++iy)
            for (int iz = std::max(bz - 1, 0); iz <= std::min(bz + 1, dims[2] - 1); ++iz) {
              const size_t b = ((size_t)ix * dims[1] + iy) * dims[2] + iz;
              for (int q = bstart[b]; q < bstart[b + 1]; ++q) cand.push_back(bitems[q]);
            }
        std::sort(cand.begin(), cand.end());
        fill(e, cand);
      }
    }
  }
  for (int e = 0; e < nt; ++e) tb.ptr[e + 1] = tb.ptr[e] + (int)lists[e].size();
  tb.ids.resize(tb.ptr[nt]);
  tb.w.resize(tb.ptr[nt]);
  for (int e = 0; e < nt; ++e)
    for (size_t q = 0; q < lists[e].size(); ++q) {
      tb.ids[tb.ptr[e] + q] = lists[e][q].first;
      tb.w[tb.ptr[e] + q] = lists[e][q].second;
    }
  return tb;
}

struct Report {  // EdgeStressReport (fracture.hpp:33-38)
  std::vector<V6> sigma_f;
  std::vector<double> screening;
  std::vector<char> degenerate;
};

static std::vector<V6> per_tet_cauchy(const Mesh& m, const std::vector<V3>& u, const Material& p) {  // solver.cpp:79-88
  const int nt = m.nt();
  std::vector<V6> sigma(nt);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < nt; ++e) sigma[e] = cauchy(deformation_gradient(m, u, e), p, nullptr);
  return sigma;
}

static Report nonlocal_screen(const Mesh& m, const std::vector<V3>& u, const std::vector<V6>& sigma_c,
                              const Table& tb) {  // fracture.cpp:56-91
  const int nt = m.nt();
  Report rep;
  rep.sigma_f.assign(nt, V6{0, 0, 0, 0, 0, 0});
  rep.degenerate.assign(nt, 0);
  std::vector<V6> screened(nt, V6{0, 0, 0, 0, 0, 0});
#pragma omp parallel for schedule(static)
  for (int e = 0; e < nt; ++e) {
    M6 T;
    if (!build_T(m, u, e, T)) {
      rep.degenerate[e] = 1;
      continue;
    }
    rep.sigma_f[e] = matvec6(T, sigma_c[e]);
    V6 avg = {0, 0, 0, 0, 0, 0};
    for (int q = tb.ptr[e]; q < tb.ptr[e + 1]; ++q) {
      const double w = tb.w[q];
      const V6& so = sigma_c[tb.ids[q]];
      for (int k = 0; k < 6; ++k) avg[k] = avg[k] + w * so[k];
    }
    screened[e] = matvec6(T, avg);
  }
  const double ninf = -std::numeric_limits<double>::infinity();
  rep.screening.assign(m.ne(), ninf);
  for (int e = 0; e < nt; ++e) {
    if (rep.degenerate[e]) continue;
    for (int k = 0; k < 6; ++k) {
      const int ed = m.tet_edges[e][k];
      rep.screening[ed] = std::max(rep.screening[ed], screened[e][k]);
    }
  }
  for (auto& s : rep.screening)
    if (s == ninf) s = 0.0;
  return rep;
}

static std::vector<int> update_damage(std::vector<uint8_t>& zeta, const std::vector<double>& screening,
                                      double thres) {  // fracture.cpp:93-104
  std::vector<int> newly;
  for (size_t e = 0; e < zeta.size(); ++e) {
    if (zeta[e]) continue;
    if (screening[e] >= thres) {
      zeta[e] = 1;
      newly.push_back((int)e);
    }
  }
  return newly;
}

static std::pair<std::array<int, 4>, int> fragment_components(const Mesh& m, const std::vector<uint8_t>& zeta,
                                                              int tet) {  // fracture.cpp:106-125
  std::array<int, 4> label = {0, 1, 2, 3};
  auto root = [&label](int i) {
    while (label[i] != i) i = label[i];
    return i;
  };
  for (int k = 0; k < 6; ++k) {
    if (zeta[m.tet_edges[tet][k]]) continue;
    const int a = root(kLocalEdges[k][0]), b = root(kLocalEdges[k][1]);
    if (a != b) label[std::max(a, b)] = std::min(a, b);
  }
  int count = 0;
  for (int i = 0; i < 4; ++i) {
    label[i] = root(i);
    if (label[i] == i) ++count;
  }
  return {label, count};
}

static std::vector<double> compute_chi(const Mesh& m, const std::vector<uint8_t>& zeta,
                                       const std::vector<V6>& sigma_f, double thres) {  // fracture.cpp:127-157
  const int nt = m.nt();
  std::vector<double> chi(nt, 1.0);
  const double eps = 1e-12 * thres;
  for (int e = 0; e < nt; ++e) {
    int intact = 0;
    for (int k = 0; k < 6; ++k) intact += zeta[m.tet_edges[e][k]] ? 0 : 1;
    if (intact == 6) { chi[e] = 1.0; continue; }
    if (intact == 0) { chi[e] = 0.0; continue; }
    if (fragment_components(m, zeta, e).second >= 2) { chi[e] = 0.0; continue; }
    double surviving = 0.0, total = 0.0;
    for (int k = 0; k < 6; ++k) {
      const double s = std::abs(sigma_f[e][k]);
      total += s;
      if (!zeta[m.tet_edges[e][k]]) surviving += s;
    }
    chi[e] = (total < eps) ? (double)intact / 6.0 : surviving / total;
  }
  return chi;
}

// ---------------------------------------------------------------- collision (collision.cpp)
struct Sched {
  std::vector<double> times;
  std::vector<V3> values;
  V3 eval(double t) const {  // collision.cpp:8-18
    if (times.empty()) return {0, 0, 0};
    if (t <= times.front()) return values.front();
    if (t >= times.back()) return values.back();
    const size_t hi = (size_t)(std::upper_bound(times.begin(), times.end(), t) - times.begin());
    const size_t lo = hi - 1;
    const double span = times[hi] - times[lo];
    const double w = span > 0.0 ? (t - times[lo]) / span : 0.0;
    V3 r;
    for (int a = 0; a < 3; ++a) r[a] = (1.0 - w) * values[lo][a] + w * values[hi][a];
    return r;
  }
  V3 rate(double t) const {  // collision.cpp:20-30
    if (times.size() < 2) return {0, 0, 0};
    if (t < times.front() || t > times.back()) return {0, 0, 0};
    size_t hi = (size_t)(std::upper_bound(times.begin(), times.end(), t) - times.begin());
    if (hi == 0) hi = 1;
    if (hi >= times.size()) hi = times.size() - 1;
    const size_t lo = hi - 1;
    const double span = times[hi] - times[lo];
    if (!(span > 0.0)) return {0, 0, 0};
    V3 r;
    for (int a = 0; a < 3; ++a) r[a] = (values[hi][a] - values[lo][a]) / span;
    return r;
  }
};
static Sched sched_from(int32_t n, const double* t, const double* v) {
  Sched s;
  for (int i = 0; i < n; ++i) {
    s.times.push_back(t[i]);
    s.values.push_back({v[3 * i], v[3 * i + 1], v[3 * i + 2]});
  }
  return s;
}

struct Collider {
  int kind = 0;  // 0 sphere, 1 halfspace
  Sched center;
  double radius = 0.0;
  V3 point{0, 0, 0}, normal{0, 0, 1};
  double stiffness = 1e6, restitution = 0.0, friction = 0.0;
  void validate() const {  // collision.cpp:32-40
    if (kind == 0 && !(radius > 0.0)) throw FormatError("sphere radius must be positive");
    if (kind == 1 && std::abs(norm3(normal) - 1.0) > 1e-9) throw FormatError("halfspace normal must be unit length");
    if (!(stiffness > 0.0)) throw FormatError("collider stiffness must be positive");
    if (restitution < 0.0 || restitution > 1.0) throw FormatError("restitution must be in [0, 1]");
    if (friction < 0.0) throw FormatError("friction must be non-negative");
  }
};

struct CollisionResult {
  std::vector<double> force;
  std::vector<double> per_collider;
  int contact_count = 0, deep_penetrations = 0;  // collision.hpp:37-41
  double max_depth = 0.0;
};
static CollisionResult detect_and_respond(const Mesh& m, const std::vector<V3>& u, const std::vector<V3>& v,
                                          const std::vector<double>& mass, const std::vector<Collider>& cols,
                                          double t, double dt) {  // collision.cpp:49-111
  CollisionResult out;
  const int n = m.nn();
  out.force.assign(3 * (size_t)n, 0.0);
  out.per_collider.assign(cols.size(), 0.0);
  for (size_t c = 0; c < cols.size(); ++c) {
    const Collider& col = cols[c];
    V3 cc{0, 0, 0}, cv{0, 0, 0};
    if (col.kind == 0) { cc = col.center.eval(t); cv = col.center.rate(t); }
    V3 sum{0, 0, 0};
    for (int i = 0; i < n; ++i) {
      const V3 x = add3(m.X[i], u[i]);
      double depth;
      V3 normal;
      if (col.kind == 0) {
        const V3 rel = sub3(x, cc);
        const double dist = norm3(rel);
        depth = col.radius - dist;
        if (depth <= 0.0) continue;
        normal = dist > 1e-12 ? V3{rel[0] / dist, rel[1] / dist, rel[2] / dist} : V3{0, 0, 1};
        if (depth > 0.5 * col.radius) out.deep_penetrations++;
      } else {
        const V3 rel = sub3(x, col.point);
        depth = -((rel[0] * col.normal[0] + rel[1] * col.normal[1]) + rel[2] * col.normal[2]);
        if (depth <= 0.0) continue;
        normal = col.normal;
      }
      out.contact_count++;
      out.max_depth = std::max(out.max_depth, depth);
      const double kd = col.stiffness * depth;
      V3 f = {kd * normal[0], kd * normal[1], kd * normal[2]};
      const V3 vrel = sub3(v[i], cv);
      const double vn = (vrel[0] * normal[0] + vrel[1] * normal[1]) + vrel[2] * normal[2];
      double impulse = 0.0;
      const double mi = mass[3 * (size_t)i];
      if (vn < 0.0) {
        impulse = -(1.0 + col.restitution) * vn * mi / dt;
        for (int a = 0; a < 3; ++a) f[a] += impulse * normal[a];
      }
      if (col.friction > 0.0) {
        const V3 vt = {vrel[0] - vn * normal[0], vrel[1] - vn * normal[1], vrel[2] - vn * normal[2]};
        const double vtn = norm3(vt);
        if (vtn > 1e-12) {
          const double cap = col.friction * (kd + impulse);
          const double want = mi * vtn / dt;
          const double mag = std::min(cap, want);
          for (int a = 0; a < 3; ++a) f[a] -= mag * (vt[a] / vtn);
        }
      }
      for (int a = 0; a < 3; ++a) {
        out.force[3 * (size_t)i + a] += f[a];
        sum[a] += f[a];
      }
    }
    out.per_collider[c] = norm3(sum);
  }
  return out;
}

// ---------------------------------------------------------------- simulation (solver.cpp)
struct SolverConfig {
  double dt = 1e-3, newton_tol = 0.0, cg_tol = 1e-8;
  int newton_max_iters = 40, cg_max_iters = 4000;
  double ls_backtrack = 0.5, ls_sufficient_decrease = 1e-4;
  int ls_max_halvings = 40;
  V3 gravity{0, 0, 0};
  bool full_newton = false;
  int collision_substeps = 1;
  void validate() const {  // solver.cpp:10-20
    if (!(dt > 0.0)) throw FormatError("dt must be positive");
    if (!(cg_tol > 0.0)) throw FormatError("cg_tol must be positive");
    if (newton_max_iters <= 0 || cg_max_iters <= 0) throw FormatError("iteration limits must be positive");
    if (!(ls_backtrack > 0.0 && ls_backtrack < 1.0)) throw FormatError("line-search backtrack factor must be in (0, 1)");
    if (!(ls_sufficient_decrease > 0.0 && ls_sufficient_decrease < 1.0))
      throw FormatError("line-search sufficient-decrease constant must be in (0, 1)");
    if (collision_substeps < 1) throw FormatError("collision_substeps must be >= 1");
  }
};

// AngleAxisd::toRotationMatrix
static M3 angle_axis(double angle, const V3& axis) {
  const double s = std::sin(angle), c = std::cos(angle);
  const V3 sa = {s * axis[0], s * axis[1], s * axis[2]};
  const V3 ca = {(1.0 - c) * axis[0], (1.0 - c) * axis[1], (1.0 - c) * axis[2]};
  M3 r;
  double tmp = ca[0] * axis[1];
  r.a[0][1] = tmp - sa[2];
  r.a[1][0] = tmp + sa[2];
  tmp = ca[0] * axis[2];
  r.a[0][2] = tmp + sa[1];
  r.a[2][0] = tmp - sa[1];
  tmp = ca[1] * axis[2];
  r.a[1][2] = tmp - sa[0];
  r.a[2][1] = tmp + sa[0];
  for (int a = 0; a < 3; ++a) r.a[a][a] = ca[a] * axis[a] + c;
  return r;
}

struct BC {
  int kind = 0;
  std::string name;
  std::vector<int> nodes;
  Sched translation, angle;
  V3 axis_point{0, 0, 0}, axis_dir{1, 0, 0};
  V3 displacement_at(const Mesh& m, int node, double t) const {  // solver.cpp:22-29
    if (kind == 0) return translation.eval(t);
    const double theta = angle.eval(t)[0];
    const double nn = (axis_dir[0] * axis_dir[0] + axis_dir[1] * axis_dir[1]) + axis_dir[2] * axis_dir[2];
    V3 ax = axis_dir;
    if (nn > 0.0) {
      const double l = std::sqrt(nn);
      ax = {axis_dir[0] / l, axis_dir[1] / l, axis_dir[2] / l};
    }
    const M3 R = angle_axis(theta, ax);
    const V3 rel = sub3(m.X[node], axis_point);
    V3 out;
    for (int a = 0; a < 3; ++a) {
      const double rr = (R.a[a][0] * rel[0] + R.a[a][1] * rel[1]) + R.a[a][2] * rel[2];
      out[a] = (rr + axis_point[a]) - m.X[node][a];
    }
    return out;
  }
};

struct Sim {
  Mesh mesh;
  Material mat;
  SolverConfig cfg;
  std::vector<BC> bcs;
  std::vector<Collider> cols;
  State st;
  Csr K;
  std::vector<double> mass;
  Table table;
  std::vector<double> f_user;  // nodal external load hook; not in the reference
  double newton_tol = 0.0, last_load = 0.0;
  std::vector<double> last_rhs;
  double phase[4] = {0, 0, 0, 0};

  std::vector<int> fixed_dofs() const {  // solver.cpp:62-72
    std::vector<int> d;
    for (const auto& bc : bcs)
      for (int n : bc.nodes) { d.push_back(3 * n); d.push_back(3 * n + 1); d.push_back(3 * n + 2); }
    std::sort(d.begin(), d.end());
    return d;
  }

  std::vector<int> damage_pass() {  // solver.cpp:90-103 (viz split is render-only: out of scope)
    const auto sigma_c = per_tet_cauchy(mesh, st.u, mat);
    const Report rep = nonlocal_screen(mesh, st.u, sigma_c, table);
    const auto newly = update_damage(st.zeta, rep.screening, mat.sigma_thres);
    const auto chi = compute_chi(mesh, st.zeta, rep.sigma_f, mat.sigma_thres);
    for (int e = 0; e < mesh.nt(); ++e) {
      const double value = rep.degenerate[e] ? 0.0 : chi[e];
      st.chi[e] = std::min(st.chi[e], value);
    }
    return newly;
  }

  double solve_linear(std::vector<double>& dx, std::vector<double>& rhs, const std::vector<int>& fixed,
                      const std::vector<double>& fv, int* iters) {  // solver.cpp:105-136
    K.project_dirichlet(fixed, fv, rhs);
    last_rhs = rhs;
    for (int d : fixed) dx[d] = fv[d];
    CgResult cg = cg_solve(K, rhs, dx, cfg.cg_tol, cfg.cg_max_iters);
    if (iters) *iters += cg.iterations;
    if (cg.converged) return cg.relative_residual;
    cg = cg_solve(K, rhs, dx, cfg.cg_tol, 4 * cfg.cg_max_iters);
    if (iters) *iters += cg.iterations;
    if (cg.converged) return cg.relative_residual;
    std::vector<double> fd = K.diagonal();
    for (auto& x : fd) x = std::abs(x);
    for (int d : fixed) fd[d] = 0.0;
    double shift = 1e-8;
    for (int attempt = 0; attempt < 8; ++attempt) {
      K.shift_diagonal(fd, shift);
      std::fill(dx.begin(), dx.end(), 0.0);
      for (int d : fixed) dx[d] = fv[d];
      cg = cg_solve(K, rhs, dx, cfg.cg_tol, cfg.cg_max_iters);
      if (iters) *iters += cg.iterations;
      if (cg.converged) return cg.relative_residual;
      shift *= 10.0;
    }
    std::ostringstream msg;
    msg << "linear solve failed: relative residual " << cg.relative_residual << " after " << cg.iterations
        << " iterations" << (cg.negative_curvature ? " (negative curvature)" : "");
    throw SolveError(msg.str());
  }

  void apply_boundary_displacements(double t) {  // solver.cpp:74-77
    for (const auto& bc : bcs)
      for (int n : bc.nodes) st.u[n] = bc.displacement_at(mesh, n, t);
  }

  // quasi_static_step (solver.cpp:138-217): Newton on the zero-inertia equilibrium with a backtracking line
  // search on the degraded strain energy, load halving on failure, then a damage pass.
  double quasi_time = 0.0;
  or_step_stats quasi_static_step(double t_load) {
    or_step_stats stats{};
    const auto fixed = fixed_dofs();
    const int ndof = 3 * mesh.nn();
    const std::vector<double> zero_fixed(ndof, 0.0);
    auto newton_solve = [&]() -> bool {
      for (int it = 0; it <= cfg.newton_max_iters; ++it) {
        const auto f_int = assemble_forces(mesh, st, mat);
        std::vector<double> residual = f_int;
        for (int d : fixed) residual[d] = 0.0;
        double rn = 0.0;
        for (double x : residual) rn += x * x;
        stats.residual = std::sqrt(rn);
        stats.newton_iterations = it;
        if (stats.residual <= newton_tol) return true;
        if (it == cfg.newton_max_iters) return false;
        assemble_stiffness(mesh, st, mat, K);
        std::vector<double> rhs = residual;
        std::vector<double> dx(ndof, 0.0);
        solve_linear(dx, rhs, fixed, zero_fixed, &stats.cg_iterations);
        const double e0 = total_strain_energy(mesh, st, mat);
        double slope = -dot(residual, dx);
        if (slope >= 0.0) {
          dx = residual;
          slope = -dot(residual, residual);
        }
        const std::vector<V3> saved = st.u;
        double step = 1.0;
        bool accepted = false;
        for (int h = 0; h <= cfg.ls_max_halvings; ++h) {
          for (int n = 0; n < mesh.nn(); ++n)
            for (int a = 0; a < 3; ++a) st.u[n][a] = saved[n][a] + step * dx[3 * (size_t)n + a];
          const double e1 = total_strain_energy(mesh, st, mat);
          if (e1 <= e0 + cfg.ls_sufficient_decrease * step * slope) {
            accepted = true;
            break;
          }
          step *= cfg.ls_backtrack;
        }
        if (!accepted) st.u = saved;
      }
      return false;
    };
    double current = quasi_time;
    double increment = t_load - current;
    if (increment <= 0.0) {
      apply_boundary_displacements(t_load);
      if (!newton_solve()) throw SolveError("equilibrium solve failed at fixed load");
    } else {
      int halvings = 0;
      State backup = st;
      while (current < t_load - 1e-15) {
        const double target = std::min(t_load, current + increment);
        apply_boundary_displacements(target);
        if (newton_solve()) {
          current = target;
          backup = st;
        } else {
          st = backup;
          ++halvings;
          if (halvings > 10) {
            std::ostringstream msg;
            msg << "quasi-static step failed: Newton did not reach " << newton_tol << " (residual " << stats.residual
                << ") after 10 load halvings at load time " << target;
            throw SolveError(msg.str());
          }
          increment *= 0.5;
        }
      }
    }
    quasi_time = t_load;
    st.time = t_load;
    const auto newly = damage_pass();
    stats.newly_broken = (int)newly.size();
    return stats;
  }

  or_step_stats dynamic_step() {  // solver.cpp:219-333 (semi-implicit step, or full Newton: solver.cpp:266-313)
    using clk = std::chrono::steady_clock;
    or_step_stats stats{};
    const double t = st.time, dt = cfg.dt;
    const int nn = mesh.nn(), ndof = 3 * nn;
    auto t0 = clk::now();
    const auto newly = damage_pass();
    stats.newly_broken = (int)newly.size();
    auto t1 = clk::now();

    std::vector<double> f_ext(ndof, 0.0);
    for (int n = 0; n < nn; ++n)
      for (int a = 0; a < 3; ++a) f_ext[3 * (size_t)n + a] = mass[3 * (size_t)n] * cfg.gravity[a];
    if (!f_user.empty())
      for (int i = 0; i < ndof; ++i) f_ext[i] += f_user[i];
    last_load = 0.0;
    if (!cols.empty()) {
      const int sub = cfg.collision_substeps;
      std::vector<V3> probe = st.u;
      std::vector<double> coll(ndof, 0.0);
      for (int s = 0; s < sub; ++s) {
        const double tau = dt * (double)s / (double)sub;
        if (s > 0)
          for (int n = 0; n < nn; ++n)
            for (int a = 0; a < 3; ++a) probe[n][a] = st.u[n][a] + tau * st.v[n][a];
        const auto hit = detect_and_respond(mesh, probe, st.v, mass, cols, t + tau, dt);
        for (int i = 0; i < ndof; ++i) coll[i] += hit.force[i] / (double)sub;
        double load = 0.0;
        for (double f : hit.per_collider) load += f;
        last_load = std::max(last_load, load);
      }
      for (int i = 0; i < ndof; ++i) f_ext[i] += coll[i];
    }
    stats.load = last_load;

    std::vector<double> v(ndof);
    for (int n = 0; n < nn; ++n)
      for (int a = 0; a < 3; ++a) v[3 * (size_t)n + a] = st.v[n][a];
    const auto fixed = fixed_dofs();
    std::vector<double> fixed_dv(ndof, 0.0);
    for (const auto& bc : bcs)
      for (int n : bc.nodes) {
        const V3 d1 = bc.displacement_at(mesh, n, t + dt), d0 = bc.displacement_at(mesh, n, t);
        for (int a = 0; a < 3; ++a) fixed_dv[3 * (size_t)n + a] = (d1[a] - d0[a]) / dt - st.v[n][a];
      }
    const double alpha = mat.damp_mass, beta = mat.damp_stiff;

    // solver.cpp:264-313: one Newton iteration on the backward-Euler residual M dv - dt (f_ext + f(u + dt v+) - B v+)
    // from v+ = v (semi-implicit), or up to newton_max_iters of them (dynamic_full_newton)
    const int max_outer = cfg.full_newton ? cfg.newton_max_iters : 1;
    const std::vector<V3> u_start = st.u;
    std::vector<double> dv_total(ndof, 0.0);
    auto t2 = clk::now(), t3 = t2;
    double msum = 0.0;
    for (double m : mass) msum += m;
    for (int outer = 0; outer < max_outer; ++outer) {
      const auto f_int = assemble_forces(mesh, st, mat);
      assemble_stiffness(mesh, st, mat, K);
      const auto kv = K.multiply(v);
      std::vector<double> rhs(ndof);
      for (int i = 0; i < ndof; ++i) rhs[i] = dt * (f_ext[i] + f_int[i]);
      if (alpha != 0.0)
        for (int i = 0; i < ndof; ++i) rhs[i] -= dt * alpha * (mass[i] * v[i]);
      const double c = dt * beta + (outer == 0 ? dt * dt : 0.0);
      for (int i = 0; i < ndof; ++i) rhs[i] -= c * kv[i];
      if (outer > 0)
        for (int i = 0; i < ndof; ++i) rhs[i] -= mass[i] * dv_total[i];
      const double kscale = dt * beta + dt * dt;
      for (auto& x : K.val) x *= kscale;
      std::vector<double> mdiag(ndof);
      for (int i = 0; i < ndof; ++i) mdiag[i] = (1.0 + dt * alpha) * mass[i];
      K.shift_diagonal(mdiag, 1.0);
      t2 = clk::now();

      std::vector<double> fixed_rhs(ndof, 0.0);
      for (int d : fixed) fixed_rhs[d] = outer == 0 ? fixed_dv[d] : 0.0;
      std::vector<double> dv(ndof, 0.0);
      std::vector<double> rhs_work = rhs;
      solve_linear(dv, rhs_work, fixed, fixed_rhs, &stats.cg_iterations);
      t3 = clk::now();
      for (int i = 0; i < ndof; ++i) {
        dv_total[i] += dv[i];
        v[i] += dv[i];
      }
      if (!cfg.full_newton) break;
      // the true residual at the trial state (solver.cpp:298-312)
      for (int n = 0; n < nn; ++n)
        for (int a = 0; a < 3; ++a) {
          st.v[n][a] = v[3 * (size_t)n + a];
          st.u[n][a] = u_start[n][a] + dt * st.v[n][a];
        }
      const auto f_new = assemble_forces(mesh, st, mat);
      assemble_stiffness(mesh, st, mat, K);
      std::vector<double> res(ndof);
      for (int i = 0; i < ndof; ++i) res[i] = mass[i] * dv_total[i] - dt * (f_ext[i] + f_new[i]);
      if (alpha != 0.0)
        for (int i = 0; i < ndof; ++i) res[i] += dt * alpha * (mass[i] * v[i]);
      if (beta != 0.0) {
        const auto kvn = K.multiply(v);
        for (int i = 0; i < ndof; ++i) res[i] += dt * beta * kvn[i];
      }
      for (int d : fixed) res[d] = 0.0;
      stats.newton_iterations = outer + 1;
      double rn = 0.0;
      for (double x : res) rn += x * x;
      if (std::sqrt(rn) <= std::max(newton_tol, 1e-12 * msum)) break;
    }
    if (!cfg.full_newton)
      for (int n = 0; n < nn; ++n)
        for (int a = 0; a < 3; ++a) {
          st.v[n][a] = v[3 * (size_t)n + a];
          st.u[n][a] += dt * st.v[n][a];
        }
    for (const auto& bc : bcs)
      for (int n : bc.nodes) {
        const V3 d1 = bc.displacement_at(mesh, n, t + dt), d0 = bc.displacement_at(mesh, n, t);
        st.u[n] = d1;
        for (int a = 0; a < 3; ++a) st.v[n][a] = (d1[a] - d0[a]) / dt;
      }
    st.time = t + dt;
    stats.residual = 0.0;
    auto t4 = clk::now();
    auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    phase[0] += sec(t0, t1);
    phase[1] += sec(t1, t2);
    phase[2] += sec(t2, t3);
    phase[3] += sec(t3, t4);
    return stats;
  }
};

}  // namespace orc

// ==================================================================== C ABI
using namespace orc;
struct or_mesh { Mesh m; };
struct or_sim { Sim s; };

static thread_local std::string g_err;
template <class F>
static int guard(F&& f) {
  try {
    f();
    return OR_OK;
  } catch (const FormatError& e) { g_err = e.what(); return OR_FORMAT_ERROR; }
  catch (const GeometryError& e) { g_err = e.what(); return OR_GEOMETRY_ERROR; }
  catch (const SolveError& e) { g_err = e.what(); return OR_SOLVE_ERROR; }
  catch (const std::exception& e) { g_err = e.what(); return OR_INTERNAL_ERROR; }
}
static M3 m3_from(const double* a) {
  M3 m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m.a[r][c] = a[3 * r + c];
  return m;
}
static void m3_to(const M3& m, double* a) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[3 * r + c] = m.a[r][c];
}
static std::vector<V3> v3_from(const double* p, int n) {
  std::vector<V3> v(n);
  for (int i = 0; i < n; ++i) v[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  return v;
}
static State state_from(const Mesh& m, const double* u, const double* chi) {
  State s = rest_state(m);
  if (u) s.u = v3_from(u, m.nn());
  if (chi) s.chi.assign(chi, chi + m.nt());
  return s;
}

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }
int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void or_set_num_threads(int n) {  // CPU-baseline timing at a chosen thread count (bench.py)
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_mesh_create(const double* nodes, int32_t n_nodes, const int32_t* tets, int32_t n_tets, or_mesh** out) {
  return guard([&] {
    std::vector<std::array<int, 4>> t(n_tets);
    for (int i = 0; i < n_tets; ++i) t[i] = {tets[4 * i], tets[4 * i + 1], tets[4 * i + 2], tets[4 * i + 3]};
    *out = new or_mesh{make_mesh(v3_from(nodes, n_nodes), std::move(t))};
  });
}
int or_mesh_make_box(const double size[3], const int32_t cells[3], const double origin[3], double jitter,
                     uint64_t seed, or_mesh** out) {
  return guard([&] {
    *out = new or_mesh{make_box({size[0], size[1], size[2]}, {cells[0], cells[1], cells[2]},
                                {origin[0], origin[1], origin[2]}, jitter, seed)};
  });
}
int or_mesh_load_tetgen(const char* node_text, const char* ele_text, or_mesh** out) {
  return guard([&] { *out = new or_mesh{load_tetgen(node_text, ele_text)}; });
}
void or_mesh_destroy(or_mesh* m) { delete m; }
void or_mesh_counts(const or_mesh* m, int32_t* nodes, int32_t* tets, int32_t* edges) {
  *nodes = m->m.nn(); *tets = m->m.nt(); *edges = m->m.ne();
}
void or_mesh_get(const or_mesh* mh, double* rest_xyz, int32_t* tets, int32_t* edges, int32_t* tet_edges,
                 double* volumes, double* binv9, double* centroids, double* rest_lengths) {
  const Mesh& m = mh->m;
  for (int i = 0; i < m.nn(); ++i)
    for (int a = 0; a < 3; ++a) if (rest_xyz) rest_xyz[3 * i + a] = m.X[i][a];
  for (int e = 0; e < m.nt(); ++e) {
    for (int a = 0; a < 4; ++a) if (tets) tets[4 * e + a] = m.tets[e][a];
    for (int k = 0; k < 6; ++k) if (tet_edges) tet_edges[6 * e + k] = m.tet_edges[e][k];
    if (volumes) volumes[e] = m.vol[e];
    if (binv9) m3_to(m.binv[e], binv9 + 9 * (size_t)e);
    for (int a = 0; a < 3; ++a) if (centroids) centroids[3 * e + a] = m.centroid[e][a];
  }
  for (int i = 0; i < m.ne(); ++i) {
    if (edges) { edges[2 * i] = m.edges[i][0]; edges[2 * i + 1] = m.edges[i][1]; }
    if (rest_lengths) rest_lengths[i] = m.rest_len[i];
  }
}
int64_t or_mesh_edge_tets(const or_mesh* mh, int32_t* ptr, int32_t* ids) {
  const Mesh& m = mh->m;
  int64_t k = 0;
  for (int i = 0; i < m.ne(); ++i) {
    if (ptr) ptr[i] = (int32_t)k;
    for (int t : m.edge_tets[i]) { if (ids) ids[k] = t; ++k; }
  }
  if (ptr) ptr[m.ne()] = (int32_t)k;
  return k;
}
double or_mesh_mean_face_area(const or_mesh* m) { return mean_face_area(m->m); }

int or_material_from_youngs(double E, double nu, double rho, double sigma_thres, double r_d, int32_t model,
                            or_material* out) {
  return guard([&] {
    Material p;
    p.youngs = E; p.poisson = nu; p.density = rho; p.sigma_thres = sigma_thres; p.r_d = r_d; p.model = model;
    p.mu = E / (2.0 * (1.0 + nu));                            // material.cpp:32-35
    p.lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    validate(p);
    std::memset(out, 0, sizeof *out);
    out->youngs = p.youngs; out->poisson = p.poisson; out->density = p.density; out->mu = p.mu;
    out->lambda = p.lambda; out->sigma_thres = p.sigma_thres; out->r_d = p.r_d; out->energy_model = p.model;
  });
}
double or_energy_density(const double F[9], const or_material* p) { return energy_density(m3_from(F), mat_from(p)); }
void or_pk1(const double F[9], const or_material* p, double P[9]) { m3_to(pk1(m3_from(F), mat_from(p)), P); }
void or_pk1_differential(const double F[9], const double dF[9], const or_material* p, double out[9]) {
  m3_to(pk1_differential(m3_from(F), m3_from(dF), mat_from(p)), out);
}
int or_cauchy_sixvector(const double F[9], const or_material* p, double out[6]) {
  bool fb = false;
  const V6 c = cauchy(m3_from(F), mat_from(p), &fb);
  for (int k = 0; k < 6; ++k) out[k] = c[k];
  return fb ? 1 : 0;
}

void or_deformation_gradient(const or_mesh* m, const double* u, int32_t tet, double F[9]) {
  m3_to(deformation_gradient(m->m, v3_from(u, m->m.nn()), tet), F);
}
void or_element_internal_force(const or_mesh* m, const double* u, const double* chi, const or_material* p,
                               int32_t tet, double f[12]) {
  const State s = state_from(m->m, u, chi);
  const auto nf = element_internal_force(m->m, s, mat_from(p), tet);
  for (int i = 0; i < 4; ++i)
    for (int a = 0; a < 3; ++a) f[3 * i + a] = nf[i][a];
}
int or_edge_decomposed_forces(const or_mesh* m, const double* u, const or_material* p, int32_t tet, double coeff[6],
                              double* residual) {
  const State s = state_from(m->m, u, nullptr);
  const EdgeDecomposition d = edge_decomposed_forces(m->m, s, mat_from(p), tet);
  for (int k = 0; k < 6; ++k) coeff[k] = d.coeff[k];
  if (residual) *residual = d.residual;
  return d.ok ? 1 : 0;
}
void or_element_stiffness(const or_mesh* m, const double* u, const double* chi, const or_material* p,
                          int32_t tet, double k[144]) {
  const State s = state_from(m->m, u, chi);
  Block12 b;
  element_stiffness(m->m, s, mat_from(p), tet, b);
  std::memcpy(k, b.data(), sizeof(double) * 144);
}
void or_assemble_forces(const or_mesh* m, const double* u, const double* chi, const or_material* p, double* f) {
  const State s = state_from(m->m, u, chi);
  const auto v = assemble_forces(m->m, s, mat_from(p));
  std::memcpy(f, v.data(), sizeof(double) * v.size());
}
int64_t or_pattern_nnz(const or_mesh* m) { return (int64_t)make_system_pattern(m->m).col.size(); }
uint64_t or_pattern(const or_mesh* m, int32_t* row_ptr, int32_t* cols) {
  const Csr K = make_system_pattern(m->m);
  if (row_ptr) std::memcpy(row_ptr, K.row_ptr.data(), sizeof(int) * K.row_ptr.size());
  if (cols) std::memcpy(cols, K.col.data(), sizeof(int) * K.col.size());
  return K.structure_hash();
}
void or_assemble_stiffness(const or_mesh* m, const double* u, const double* chi, const or_material* p,
                           double* vals) {
  const State s = state_from(m->m, u, chi);
  Csr K = make_system_pattern(m->m);
  assemble_stiffness(m->m, s, mat_from(p), K);
  std::memcpy(vals, K.val.data(), sizeof(double) * K.val.size());
}
void or_lumped_mass(const or_mesh* m, const or_material* p, double* mass3n) {
  const auto v = lumped_mass(m->m, mat_from(p));
  std::memcpy(mass3n, v.data(), sizeof(double) * v.size());
}
double or_total_strain_energy(const or_mesh* m, const double* u, const double* chi, const or_material* p) {
  return total_strain_energy(m->m, state_from(m->m, u, chi), mat_from(p));
}

int or_build_T(const or_mesh* m, const double* u, int32_t tet, double T[36]) {
  M6 t;
  const bool ok = build_T(m->m, v3_from(u, m->m.nn()), tet, t);
  if (ok)
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) T[6 * r + c] = t[r][c];
  return ok ? 1 : 0;
}
int64_t or_nonlocal_table(const or_mesh* m, double r_d, int32_t brute, int32_t* ptr, int32_t* ids, double* w) {
  const Table tb = build_nonlocal_table(m->m, r_d, brute != 0);
  if (ptr) std::memcpy(ptr, tb.ptr.data(), sizeof(int) * tb.ptr.size());
  if (ids) std::memcpy(ids, tb.ids.data(), sizeof(int) * tb.ids.size());
  if (w) std::memcpy(w, tb.w.data(), sizeof(double) * tb.w.size());
  return (int64_t)tb.ids.size();
}
void or_per_tet_cauchy(const or_mesh* m, const double* u, const or_material* p, double* sigma6) {
  const auto s = per_tet_cauchy(m->m, v3_from(u, m->m.nn()), mat_from(p));
  for (size_t e = 0; e < s.size(); ++e)
    for (int k = 0; k < 6; ++k) sigma6[6 * e + k] = s[e][k];
}
void or_nonlocal_screen(const or_mesh* m, const double* u, const double* sigma6, double r_d, double* screening,
                        double* sigma_f6, uint8_t* degenerate) {
  const Mesh& mm = m->m;
  std::vector<V6> sc(mm.nt());
  for (int e = 0; e < mm.nt(); ++e)
    for (int k = 0; k < 6; ++k) sc[e][k] = sigma6[6 * (size_t)e + k];
  const Table tb = build_nonlocal_table(mm, r_d, false);
  const Report rep = nonlocal_screen(mm, v3_from(u, mm.nn()), sc, tb);
  if (screening) std::memcpy(screening, rep.screening.data(), sizeof(double) * rep.screening.size());
  for (int e = 0; e < mm.nt(); ++e) {
    for (int k = 0; k < 6; ++k) if (sigma_f6) sigma_f6[6 * (size_t)e + k] = rep.sigma_f[e][k];
    if (degenerate) degenerate[e] = (uint8_t)rep.degenerate[e];
  }
}
int32_t or_update_damage(uint8_t* zeta, int32_t n_edges, const double* screening, double thres, int32_t* newly) {
  std::vector<uint8_t> z(zeta, zeta + n_edges);
  const auto nb = update_damage(z, std::vector<double>(screening, screening + n_edges), thres);
  std::memcpy(zeta, z.data(), n_edges);
  for (size_t i = 0; i < nb.size(); ++i) newly[i] = nb[i];
  return (int32_t)nb.size();
}
void or_compute_chi(const or_mesh* m, const uint8_t* zeta, const double* sigma_f6, const or_material* p, double* chi) {
  const Mesh& mm = m->m;
  std::vector<V6> sf(mm.nt());
  for (int e = 0; e < mm.nt(); ++e)
    for (int k = 0; k < 6; ++k) sf[e][k] = sigma_f6[6 * (size_t)e + k];
  const auto c = compute_chi(mm, std::vector<uint8_t>(zeta, zeta + mm.ne()), sf, p->sigma_thres);
  std::memcpy(chi, c.data(), sizeof(double) * c.size());
}
int32_t or_fragment_components(const or_mesh* m, const uint8_t* zeta, int32_t tet, int32_t labels[4]) {
  const auto r = fragment_components(m->m, std::vector<uint8_t>(zeta, zeta + m->m.ne()), tet);
  for (int i = 0; i < 4; ++i) labels[i] = r.first[i];
  return r.second;
}

static Csr csr_from(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals) {
  Csr A;
  A.n = n;
  A.row_ptr.assign(row_ptr, row_ptr + n + 1);
  A.col.assign(cols, cols + row_ptr[n]);
  A.val.assign(vals, vals + row_ptr[n]);
  return A;
}
void or_spmv_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* x,
                 double* y) {  // FixedPatternSparse::multiply (sparse.cpp:49-60) on caller-owned arrays, no copies
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) acc += vals[k] * x[cols[k]];
    y[i] = acc;
  }
}
void or_cg_solve_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, const double* vals, const double* b,
                     double* x, double tol, int32_t max_iters, or_cg_result* res) {
  const Csr A = csr_from(n, row_ptr, cols, vals);
  std::vector<double> xv(x, x + n);
  const CgResult r = cg_solve(A, std::vector<double>(b, b + n), xv, tol, max_iters);
  std::memcpy(x, xv.data(), sizeof(double) * n);
  res->iterations = r.iterations;
  res->converged = r.converged;
  res->negative_curvature = r.negative_curvature;
  res->relative_residual = r.relative_residual;
}
void or_project_dirichlet_csr(int32_t n, const int32_t* row_ptr, const int32_t* cols, double* vals,
                              const int32_t* dofs, int32_t n_dofs, const double* values, double* rhs) {
  Csr A = csr_from(n, row_ptr, cols, vals);
  std::vector<double> r(rhs, rhs + n);
  A.project_dirichlet(std::vector<int>(dofs, dofs + n_dofs), std::vector<double>(values, values + n), r);
  std::memcpy(vals, A.val.data(), sizeof(double) * A.val.size());
  std::memcpy(rhs, r.data(), sizeof(double) * n);
}

void or_solver_config_default(or_solver_config* c) {
  std::memset(c, 0, sizeof *c);
  const SolverConfig d;
  c->dt = d.dt; c->newton_tol = d.newton_tol; c->newton_max_iters = d.newton_max_iters;
  c->cg_max_iters = d.cg_max_iters; c->cg_tol = d.cg_tol; c->ls_backtrack = d.ls_backtrack;
  c->ls_sufficient_decrease = d.ls_sufficient_decrease; c->ls_max_halvings = d.ls_max_halvings;
  c->dynamic_full_newton = 0; c->collision_substeps = d.collision_substeps;
}

static Collider collider_from(const or_collider& c) {
  Collider cl;
  cl.kind = c.kind;
  cl.center = sched_from(c.n_keys, c.key_times, c.key_values);
  cl.radius = c.radius;
  cl.point = {c.point[0], c.point[1], c.point[2]};
  cl.normal = {c.normal[0], c.normal[1], c.normal[2]};
  cl.stiffness = c.stiffness; cl.restitution = c.restitution; cl.friction = c.friction;
  return cl;
}

void or_schedule_eval(int32_t n_keys, const double* times, const double* values, double t, double val[3],
                      double rate[3]) {
  const Sched s = sched_from(n_keys, times, values);
  const V3 a = s.eval(t), b = s.rate(t);
  for (int k = 0; k < 3; ++k) { val[k] = a[k]; rate[k] = b[k]; }
}

int or_collider_validate(const or_collider* c) {
  return guard([&] { collider_from(*c).validate(); });
}

int or_detect_and_respond(const or_mesh* mesh, const double* u, const double* v, const double* mass3n,
                          const or_collider* cols, int32_t n_cols, double t, double dt, double* force3n,
                          double* per_collider, int32_t counts[2], double* max_depth) {
  return guard([&] {
    const Mesh& m = mesh->m;
    const int n = m.nn();
    std::vector<V3> uu(n), vv(n);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) { uu[i][a] = u[3 * i + a]; vv[i][a] = v[3 * i + a]; }
    std::vector<double> mass(mass3n, mass3n + 3 * (size_t)n);
    std::vector<Collider> cs;
    for (int i = 0; i < n_cols; ++i) cs.push_back(collider_from(cols[i]));
    const CollisionResult r = detect_and_respond(m, uu, vv, mass, cs, t, dt);
    std::copy(r.force.begin(), r.force.end(), force3n);
    std::copy(r.per_collider.begin(), r.per_collider.end(), per_collider);
    counts[0] = r.contact_count;
    counts[1] = r.deep_penetrations;
    *max_depth = r.max_depth;
  });
}

int or_sim_create(const or_mesh* mesh, const or_material* mat, const or_solver_config* cfg,
                  const or_boundary_condition* bcs, int32_t n_bcs, const or_collider* cols, int32_t n_cols,
                  or_sim** out) {
  return guard([&] {
    auto h = std::make_unique<or_sim>();
    Sim& s = h->s;
    s.mesh = mesh->m;
    s.mat = mat_from(mat);
    SolverConfig c;
    c.dt = cfg->dt; c.newton_tol = cfg->newton_tol; c.newton_max_iters = cfg->newton_max_iters;
    c.cg_max_iters = cfg->cg_max_iters; c.cg_tol = cfg->cg_tol; c.ls_backtrack = cfg->ls_backtrack;
    c.ls_sufficient_decrease = cfg->ls_sufficient_decrease; c.ls_max_halvings = cfg->ls_max_halvings;
    c.full_newton = cfg->dynamic_full_newton != 0;
    c.gravity = {cfg->gravity[0], cfg->gravity[1], cfg->gravity[2]};
    c.collision_substeps = cfg->collision_substeps;
    s.cfg = c;
    for (int i = 0; i < n_bcs; ++i) {
      BC b;
      b.kind = bcs[i].kind;
      b.name = "bc" + std::to_string(i);
      b.nodes.assign(bcs[i].nodes, bcs[i].nodes + bcs[i].n_nodes);
      const Sched sc = sched_from(bcs[i].n_keys, bcs[i].key_times, bcs[i].key_values);
      if (b.kind == 0) b.translation = sc; else b.angle = sc;
      b.axis_point = {bcs[i].axis_point[0], bcs[i].axis_point[1], bcs[i].axis_point[2]};
      b.axis_dir = {bcs[i].axis_dir[0], bcs[i].axis_dir[1], bcs[i].axis_dir[2]};
      s.bcs.push_back(std::move(b));
    }
    for (int i = 0; i < n_cols; ++i) s.cols.push_back(collider_from(cols[i]));
    // member-initialiser order of Simulation::Simulation (solver.cpp:31-60)
    s.st = rest_state(s.mesh);
    s.K = make_system_pattern(s.mesh);
    s.mass = lumped_mass(s.mesh, s.mat);
    s.table = build_nonlocal_table(s.mesh, s.mat.r_d, false);
    validate(s.mat);
    s.cfg.validate();
    for (const auto& cl : s.cols) cl.validate();
    std::vector<char> seen(s.mesh.nn(), 0);
    for (const auto& b : s.bcs) {
      if (b.nodes.empty()) throw FormatError("boundary condition '" + b.name + "' selects no nodes");
      for (int n : b.nodes) {
        if (n < 0 || n >= s.mesh.nn()) throw FormatError("boundary condition '" + b.name + "' references node out of range");
        if (seen[n]) throw FormatError("node " + std::to_string(n) + " appears in two boundary conditions");
        seen[n] = 1;
      }
    }
    s.newton_tol = s.cfg.newton_tol > 0.0 ? s.cfg.newton_tol : 1e-6 * s.mat.sigma_thres * mean_face_area(s.mesh);
    *out = h.release();
  });
}
void or_sim_destroy(or_sim* s) { delete s; }
int or_sim_dynamic_step(or_sim* s, or_step_stats* stats) {
  return guard([&] {
    const or_step_stats r = s->s.dynamic_step();
    if (stats) *stats = r;
  });
}
int or_sim_damage_pass(or_sim* s, int32_t* ids, int64_t cap, int64_t* n) {
  return guard([&] {
    const auto nb = s->s.damage_pass();
    *n = (int64_t)nb.size();
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n); ++i) ids[i] = nb[i];
  });
}
void or_sim_get_state(const or_sim* sh, double* u, double* v, uint8_t* zeta, double* chi, double* time) {
  const Sim& s = sh->s;
  for (int i = 0; i < s.mesh.nn(); ++i)
    for (int a = 0; a < 3; ++a) {
      if (u) u[3 * i + a] = s.st.u[i][a];
      if (v) v[3 * i + a] = s.st.v[i][a];
    }
  if (zeta) std::memcpy(zeta, s.st.zeta.data(), s.st.zeta.size());
  if (chi) std::memcpy(chi, s.st.chi.data(), sizeof(double) * s.st.chi.size());
  if (time) *time = s.st.time;
}
void or_sim_set_state(or_sim* sh, const double* u, const double* v, const uint8_t* zeta, const double* chi,
                      const double* time) {
  Sim& s = sh->s;
  if (u) s.st.u = v3_from(u, s.mesh.nn());
  if (v) s.st.v = v3_from(v, s.mesh.nn());
  if (zeta) s.st.zeta.assign(zeta, zeta + s.mesh.ne());
  if (chi) s.st.chi.assign(chi, chi + s.mesh.nt());
  if (time) s.st.time = *time;
}
void or_sim_set_external_forces(or_sim* s, const double* f3n) {
  if (f3n) s->s.f_user.assign(f3n, f3n + 3 * (size_t)s->s.mesh.nn());
  else s->s.f_user.clear();
}
uint64_t or_sim_pattern_hash(const or_sim* s) { return s->s.K.structure_hash(); }
double or_sim_last_collider_load(const or_sim* s) { return s->s.last_load; }
void or_sim_mass(const or_sim* s, double* m3n) { std::memcpy(m3n, s->s.mass.data(), sizeof(double) * s->s.mass.size()); }
void or_sim_last_system(const or_sim* s, double* vals, double* rhs) {
  if (vals) std::memcpy(vals, s->s.K.val.data(), sizeof(double) * s->s.K.val.size());
  if (rhs && !s->s.last_rhs.empty()) std::memcpy(rhs, s->s.last_rhs.data(), sizeof(double) * s->s.last_rhs.size());
}
int or_sim_quasi_static_step(or_sim* s, double t_load, or_step_stats* stats) {
  return guard([&] {
    const or_step_stats r = s->s.quasi_static_step(t_load);
    if (stats) *stats = r;
  });
}
double or_sim_newton_tolerance(const or_sim* s) { return s->s.newton_tol; }
void or_sim_phase_times(const or_sim* s, double t[4]) {
  for (int i = 0; i < 4; ++i) t[i] = s->s.phase[i];
}

}  // extern "C"
