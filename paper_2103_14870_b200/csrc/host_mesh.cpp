// host_mesh.cpp — see host_mesh.hpp. Setup only; compiled with -ffp-contract=off.
#include "host_mesh.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace gfb {
namespace {

// Eigen 3x3 determinant (bruteforce_det3_helper): (h0 - h1) + h2, first-row expansion; m row-major
inline double det3(const double* m) {
  const double h0 = m[0] * (m[4] * m[8] - m[5] * m[7]);
  const double h1 = m[1] * (m[3] * m[8] - m[5] * m[6]);
  const double h2 = m[2] * (m[3] * m[7] - m[4] * m[6]);
  return (h0 - h1) + h2;
}
inline double norm3(double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); }

// Eigen compute_inverse<3>: cofactor column 0, det = (c00 m00 + c10 m10) + c20 m20, invdet = 1/det,
// out(r,c) = cofactor(c,r) * invdet.
void inverse3(const double* m, double* out) {
  auto cof = [m](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return m[3 * i1 + j1] * m[3 * i2 + j2] - m[3 * i1 + j2] * m[3 * i2 + j1];
  };
  const double c00 = cof(0, 0), c10 = cof(1, 0), c20 = cof(2, 0);
  const double invdet = 1.0 / ((c00 * m[0] + c10 * m[3]) + c20 * m[6]);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out[3 * r + c] = cof(c, r) * invdet;
}

// Counter-based splitmix64 interior-node jitter (identical to the oracle's generator).
inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline double unit_jitter(uint64_t seed, uint64_t node, int comp) {
  const uint64_t r = mix64(mix64(seed) + 3ull * node + (uint64_t)comp);
  return 2.0 * ((double)(r >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

void validate_and_graph(HostMesh& m) {  // induce_edge_graph (mesh.cpp:34-70)
  if (m.nt == 0) throw GeometryError("mesh has no tetrahedra");
  for (int32_t e = 0; e < m.nt; ++e) {
    const int32_t* t = &m.tets[4 * (size_t)e];
    for (int i = 0; i < 4; ++i) {
      if (t[i] < 0 || t[i] >= m.nn)
        throw GeometryError("tet " + std::to_string(e) + " references node " + std::to_string(t[i]) + " out of range");
      for (int j = i + 1; j < 4; ++j)
        if (t[i] == t[j]) throw GeometryError("tet " + std::to_string(e) + " repeats node " + std::to_string(t[i]));
    }
  }
  // bucket the 6T (min,max) pairs by min node; sorted unique per bucket == lexicographic edge order
  std::vector<int32_t> cnt(m.nn + 1, 0);
  for (int32_t e = 0; e < m.nt; ++e)
    for (const auto& le : kLocalEdge) {
      const int32_t a = m.tets[4 * (size_t)e + le[0]], b = m.tets[4 * (size_t)e + le[1]];
      cnt[std::min(a, b) + 1]++;
    }
  for (int32_t i = 0; i < m.nn; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> buf(cnt[m.nn]);
  {
    std::vector<int32_t> cur(cnt.begin(), cnt.end() - 1);
    for (int32_t e = 0; e < m.nt; ++e)
      for (const auto& le : kLocalEdge) {
        const int32_t a = m.tets[4 * (size_t)e + le[0]], b = m.tets[4 * (size_t)e + le[1]];
        buf[cur[std::min(a, b)]++] = std::max(a, b);
      }
  }
  std::vector<int32_t> first(m.nn + 1, 0);  // first edge id of each min-node bucket
  std::vector<int32_t> uniq_len(m.nn, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int32_t i = 0; i < m.nn; ++i) {
    auto b = buf.begin() + cnt[i], e = buf.begin() + cnt[i + 1];
    std::sort(b, e);
    uniq_len[i] = (int32_t)(std::unique(b, e) - b);
  }
  for (int32_t i = 0; i < m.nn; ++i) first[i + 1] = first[i] + uniq_len[i];
  m.ne = first[m.nn];
  m.edges.resize(2 * (size_t)m.ne);
  for (int32_t i = 0; i < m.nn; ++i)
    for (int32_t q = 0; q < uniq_len[i]; ++q) {
      m.edges[2 * (size_t)(first[i] + q)] = i;
      m.edges[2 * (size_t)(first[i] + q) + 1] = buf[cnt[i] + q];
    }
  m.tet_edges.resize(6 * (size_t)m.nt);
#pragma omp parallel for schedule(static)
  for (int32_t e = 0; e < m.nt; ++e)
    for (int k = 0; k < 6; ++k) {
      const int32_t a = m.tets[4 * (size_t)e + kLocalEdge[k][0]], b = m.tets[4 * (size_t)e + kLocalEdge[k][1]];
      const int32_t lo = std::min(a, b), hi = std::max(a, b);
      const auto bb = buf.begin() + cnt[lo], ee = bb + uniq_len[lo];
      m.tet_edges[6 * (size_t)e + k] = first[lo] + (int32_t)(std::lower_bound(bb, ee, hi) - bb);
    }
  m.et_ptr.assign(m.ne + 1, 0);
  for (size_t q = 0; q < m.tet_edges.size(); ++q) m.et_ptr[m.tet_edges[q] + 1]++;
  for (int32_t i = 0; i < m.ne; ++i) m.et_ptr[i + 1] += m.et_ptr[i];
  m.et_ids.resize(m.et_ptr[m.ne]);
  std::vector<int32_t> cur(m.et_ptr.begin(), m.et_ptr.end() - 1);
  for (int32_t e = 0; e < m.nt; ++e)
    for (int k = 0; k < 6; ++k) m.et_ids[cur[m.tet_edges[6 * (size_t)e + k]]++] = e;
}

void rest_quantities(HostMesh& m) {  // mesh.cpp:72-100
  m.vol.resize(m.nt);
  m.binv.resize(9 * (size_t)m.nt);
  m.centroid.resize(3 * (size_t)m.nt);
  std::vector<int32_t> bad;
#pragma omp parallel for schedule(static)
  for (int32_t e = 0; e < m.nt; ++e) {
    const int32_t* t = &m.tets[4 * (size_t)e];
    const double* p0 = &m.X[3 * (size_t)t[0]];
    double dm[9];  // columns = X[t_c] - X[t_0]
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) dm[3 * r + c] = m.X[3 * (size_t)t[c + 1] + r] - p0[r];
    const double det = det3(dm);
    if (!(det > 0.0)) {
#pragma omp critical
      bad.push_back(e);
      continue;
    }
    m.vol[e] = det / 6.0;
    inverse3(dm, &m.binv[9 * (size_t)e]);
    for (int r = 0; r < 3; ++r) {
      const double s = ((p0[r] + m.X[3 * (size_t)t[1] + r]) + m.X[3 * (size_t)t[2] + r]) + m.X[3 * (size_t)t[3] + r];
      m.centroid[3 * (size_t)e + r] = 0.25 * s;
    }
  }
  if (!bad.empty()) {
    const int32_t e = *std::min_element(bad.begin(), bad.end());
    const int32_t* t = &m.tets[4 * (size_t)e];
    double dm[9];
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) dm[3 * r + c] = m.X[3 * (size_t)t[c + 1] + r] - m.X[3 * (size_t)t[0] + r];
    throw GeometryError("tet " + std::to_string(e) + " is degenerate or inverted (det = " + std::to_string(det3(dm)) + ")");
  }
  m.rest_len.resize(m.ne);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < m.ne; ++i) {
    const double* a = &m.X[3 * (size_t)m.edges[2 * (size_t)i]];
    const double* b = &m.X[3 * (size_t)m.edges[2 * (size_t)i + 1]];
    m.rest_len[i] = norm3(b[0] - a[0], b[1] - a[1], b[2] - a[2]);
  }
}

std::vector<std::pair<int, std::vector<std::string>>> tokenize(const std::string& text) {
  std::vector<std::pair<int, std::vector<std::string>>> out;
  std::istringstream in(text);
  std::string line;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    const auto h = line.find('#');
    if (h != std::string::npos) line.erase(h);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    for (std::string t; ls >> t;) tok.push_back(t);
    if (!tok.empty()) out.emplace_back(no, std::move(tok));
  }
  return out;
}
long to_long(const std::string& s, int line) {
  try {
    size_t pos = 0;
    const long v = std::stol(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw FormatError("line " + std::to_string(line) + ": expected integer, got '" + s + "'");
  }
}
double to_double(const std::string& s, int line) {
  try {
    size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw FormatError("line " + std::to_string(line) + ": expected number, got '" + s + "'");
  }
}

}  // namespace

double HostMesh::mean_face_area() const {  // mesh.cpp:18-32
  static constexpr int fl[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
  double sum = 0.0;
  long count = 0;
  for (int32_t e = 0; e < nt; ++e)
    for (const auto& f : fl) {
      const double* a = &X[3 * (size_t)tets[4 * (size_t)e + f[0]]];
      const double* b = &X[3 * (size_t)tets[4 * (size_t)e + f[1]]];
      const double* c = &X[3 * (size_t)tets[4 * (size_t)e + f[2]]];
      const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
      sum += 0.5 * norm3(u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]);
      ++count;
    }
  return count ? sum / (double)count : 0.0;
}

HostMesh mesh_from_arrays(std::vector<double> X, std::vector<int32_t> tets) {  // make_mesh (mesh.cpp:102-109)
  HostMesh m;
  m.nn = (int32_t)(X.size() / 3);
  m.nt = (int32_t)(tets.size() / 4);
  m.X = std::move(X);
  m.tets = std::move(tets);
  validate_and_graph(m);
  rest_quantities(m);
  return m;
}

HostMesh mesh_box(const double size[3], const int32_t cells[3], const double origin[3], double jitter,
                  uint64_t seed) {  // structured_mesh + make_box_mesh (primitives.cpp:13-79)
  static constexpr int kCube[6][4] = {{0, 1, 3, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 6, 4, 7}, {0, 4, 5, 7}, {0, 5, 1, 7}};
  const int32_t nx = cells[0], ny = cells[1], nz = cells[2];
  if (nx < 1 || ny < 1 || nz < 1) throw GeometryError("cell counts must be positive");
  const double h[3] = {size[0] / nx, size[1] / ny, size[2] / nz};
  const int64_t nnodes = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  const int64_t ntets = 6ll * nx * ny * nz;
  if (ntets > INT32_MAX / 6 || nnodes > INT32_MAX / 3) throw GeometryError("box mesh too large for 32-bit ids");
  auto nid = [&](int64_t i, int64_t j, int64_t k) { return (int32_t)((i * (ny + 1) + j) * (nz + 1) + k); };
  std::vector<double> X(3 * (size_t)nnodes);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i <= nx; ++i)
    for (int32_t j = 0; j <= ny; ++j)
      for (int32_t k = 0; k <= nz; ++k) {
        const int32_t id = nid(i, j, k);
        double p[3] = {origin[0] + i * h[0], origin[1] + j * h[1], origin[2] + k * h[2]};
        if (jitter != 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz)
          for (int c = 0; c < 3; ++c) p[c] = p[c] + (jitter * h[c]) * unit_jitter(seed, (uint64_t)id, c);
        for (int c = 0; c < 3; ++c) X[3 * (size_t)id + c] = p[c];
      }
  std::vector<int32_t> tets(4 * (size_t)ntets);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < nx; ++i)
    for (int32_t j = 0; j < ny; ++j)
      for (int32_t k = 0; k < nz; ++k) {
        int32_t corner[8];
        for (int b = 0; b < 8; ++b) corner[b] = nid(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1));
        const size_t base = 6 * (((size_t)i * ny + j) * nz + k);
        for (int q = 0; q < 6; ++q) {
          int32_t* t = &tets[4 * (base + q)];
          for (int v = 0; v < 4; ++v) t[v] = corner[kCube[q][v]];
          double dm[9];  // orientation fix (primitives.cpp:56-62)
          for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) dm[3 * r + c] = X[3 * (size_t)t[c + 1] + r] - X[3 * (size_t)t[0] + r];
          if (det3(dm) < 0.0) std::swap(t[2], t[3]);
        }
      }
  return mesh_from_arrays(std::move(X), std::move(tets));
}

HostMesh mesh_tetgen(const std::string& node_text, const std::string& ele_text) {  // load_tetgen (mesh.cpp:157-221)
  const auto nl = tokenize(node_text);
  if (nl.empty()) throw FormatError(".node: file is empty");
  const int hl = nl[0].first;
  const auto& ht = nl[0].second;
  if (ht.size() < 2) throw FormatError("line " + std::to_string(hl) + ": .node header needs '<count> <dim> [attrs] [markers]'");
  const long np = to_long(ht[0], hl), dim = to_long(ht[1], hl);
  if (dim != 3) throw FormatError("line " + std::to_string(hl) + ": only 3-dimensional .node files are supported");
  if (np <= 0) throw FormatError("line " + std::to_string(hl) + ": point count must be positive");
  if ((long)nl.size() - 1 < np)
    throw FormatError(".node: expected " + std::to_string(np) + " point lines, found " + std::to_string(nl.size() - 1));
  long base = -1;
  std::vector<double> X(3 * (size_t)np);
  for (long i = 0; i < np; ++i) {
    const int line = nl[i + 1].first;
    const auto& t = nl[i + 1].second;
    if (t.size() < 4) throw FormatError("line " + std::to_string(line) + ": point record needs '<index> x y z'");
    const long idx = to_long(t[0], line);
    if (base < 0) base = idx == 0 ? 0 : 1;
    const long at = idx - base;
    if (at < 0 || at >= np) throw FormatError("line " + std::to_string(line) + ": point index " + std::to_string(idx) + " out of range");
    for (int c = 0; c < 3; ++c) X[3 * at + c] = to_double(t[1 + c], line);
  }
  const auto el = tokenize(ele_text);
  if (el.empty()) throw FormatError(".ele: file is empty");
  const int ehl = el[0].first;
  const auto& eht = el[0].second;
  if (eht.size() < 2) throw FormatError("line " + std::to_string(ehl) + ": .ele header needs '<count> <nodes-per-tet> [attrs]'");
  const long ntet = to_long(eht[0], ehl), per = to_long(eht[1], ehl);
  if (per != 4) throw FormatError("line " + std::to_string(ehl) + ": only 4-node tetrahedra are supported");
  if (ntet <= 0) throw FormatError("line " + std::to_string(ehl) + ": element count must be positive");
  if ((long)el.size() - 1 < ntet)
    throw FormatError(".ele: expected " + std::to_string(ntet) + " element lines, found " + std::to_string(el.size() - 1));
  long ebase = -1;
  std::vector<int32_t> tets(4 * (size_t)ntet);
  for (long i = 0; i < ntet; ++i) {
    const int line = el[i + 1].first;
    const auto& t = el[i + 1].second;
    if (t.size() < 5) throw FormatError("line " + std::to_string(line) + ": element record needs '<index> n1 n2 n3 n4'");
    const long idx = to_long(t[0], line);
    if (ebase < 0) ebase = idx == 0 ? 0 : 1;
    const long at = idx - ebase;
    if (at < 0 || at >= ntet) throw FormatError("line " + std::to_string(line) + ": element index " + std::to_string(idx) + " out of range");
    for (int k = 0; k < 4; ++k) {
      const long node = to_long(t[1 + k], line) - base;
      if (node < 0 || node >= np)
        throw FormatError("line " + std::to_string(line) + ": node index " + std::to_string(node + base) +
                          " out of range (have " + std::to_string(np) + " points)");
      tets[4 * at + k] = (int32_t)node;
    }
  }
  return mesh_from_arrays(std::move(X), std::move(tets));
}

NodePattern make_node_pattern(const HostMesh& m) {
  // every node pair that shares a tet is an edge, so row i = {i} U edge-neighbours(i)
  NodePattern p;
  p.row_ptr.assign(m.nn + 1, 0);
  for (int32_t i = 0; i < m.nn; ++i) p.row_ptr[i + 1] = 1;
  for (int32_t e = 0; e < m.ne; ++e) {
    p.row_ptr[m.edges[2 * (size_t)e] + 1]++;
    p.row_ptr[m.edges[2 * (size_t)e + 1] + 1]++;
  }
  for (int32_t i = 0; i < m.nn; ++i) p.row_ptr[i + 1] += p.row_ptr[i];
  p.cols.resize(p.row_ptr[m.nn]);
  std::vector<int32_t> cur(p.row_ptr.begin(), p.row_ptr.end() - 1);
  for (int32_t i = 0; i < m.nn; ++i) p.cols[cur[i]++] = i;
  for (int32_t e = 0; e < m.ne; ++e) {
    const int32_t a = m.edges[2 * (size_t)e], b = m.edges[2 * (size_t)e + 1];
    p.cols[cur[a]++] = b;
    p.cols[cur[b]++] = a;
  }
  p.diag.resize(m.nn);
  int32_t maxdeg = 0;
#pragma omp parallel for schedule(static) reduction(max : maxdeg)
  for (int32_t i = 0; i < m.nn; ++i) {
    std::sort(p.cols.begin() + p.row_ptr[i], p.cols.begin() + p.row_ptr[i + 1]);
    p.diag[i] = (int32_t)(std::lower_bound(p.cols.begin() + p.row_ptr[i], p.cols.begin() + p.row_ptr[i + 1], i) - p.cols.begin());
    maxdeg = std::max(maxdeg, p.row_ptr[i + 1] - p.row_ptr[i]);
  }
  p.max_degree = maxdeg;
  if ((int64_t)p.cols.size() * 9 > INT32_MAX) throw GeometryError("system pattern exceeds 32-bit scalar CSR offsets");
  return p;
}

uint64_t NodePattern::structure_hash(int32_t nn) const {  // FNV-1a over (n, row_ptr, col) of the scalar CSR
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  mix((uint64_t)(3 * (int64_t)nn));
  for (int32_t i = 0; i < nn; ++i) {
    const int32_t deg = row_ptr[i + 1] - row_ptr[i];
    for (int a = 0; a < 3; ++a) mix((uint64_t)(9 * row_ptr[i] + 3 * a * deg));
  }
  mix((uint64_t)(9 * row_ptr[nn]));
  for (int32_t i = 0; i < nn; ++i)
    for (int a = 0; a < 3; ++a)
      for (int32_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q)
        for (int b = 0; b < 3; ++b) mix((uint64_t)(3 * cols[q] + b));
  return h;
}

void NodePattern::scalar_csr(int32_t nn, int32_t* rp, int32_t* co) const {
  for (int32_t i = 0; i < nn; ++i) {
    const int32_t deg = row_ptr[i + 1] - row_ptr[i];
    for (int a = 0; a < 3; ++a) {
      const int32_t start = 9 * row_ptr[i] + 3 * a * deg;
      if (rp) rp[3 * i + a] = start;
      if (co)
        for (int32_t q = 0; q < deg; ++q)
          for (int b = 0; b < 3; ++b) co[start + 3 * q + b] = 3 * cols[row_ptr[i] + q] + b;
    }
  }
  if (rp) rp[3 * nn] = 9 * row_ptr[nn];
}

NodeTets make_node_tets(const HostMesh& m, const NodePattern& p) {
  NodeTets nt;
  nt.ptr.assign(m.nn + 1, 0);
  for (size_t q = 0; q < m.tets.size(); ++q) nt.ptr[m.tets[q] + 1]++;
  for (int32_t i = 0; i < m.nn; ++i) nt.ptr[i + 1] += nt.ptr[i];
  nt.tet.resize(nt.ptr[m.nn]);
  nt.slot.resize(nt.ptr[m.nn]);
  std::vector<int32_t> cur(nt.ptr.begin(), nt.ptr.end() - 1);
  for (int32_t e = 0; e < m.nt; ++e)
    for (int k = 0; k < 4; ++k) nt.tet[cur[m.tets[4 * (size_t)e + k]]++] = e;
  int32_t maxval = 0;
#pragma omp parallel for schedule(static) reduction(max : maxval)
  for (int32_t i = 0; i < m.nn; ++i) {
    maxval = std::max(maxval, nt.ptr[i + 1] - nt.ptr[i]);
    const auto rb = p.cols.begin() + p.row_ptr[i], re = p.cols.begin() + p.row_ptr[i + 1];
    for (int32_t q = nt.ptr[i]; q < nt.ptr[i + 1]; ++q) {
      uint32_t s = 0;
      for (int k = 0; k < 4; ++k) {
        const uint32_t pos = (uint32_t)(std::lower_bound(rb, re, m.tets[4 * (size_t)nt.tet[q] + k]) - rb);
        s |= (pos & 0xffu) << (8 * k);
      }
      nt.slot[q] = s;
    }
  }
  nt.max_valence = maxval;
  return nt;
}

// build_nonlocal_table (fracture.cpp:32-54). Candidates come from a uniform grid of >= r_d bins
// (a superset of every tet within r_d), sorted ascending; the reject tests, weights and the
// ascending wsum accumulation are the reference's, so entries are bit-identical to the O(T^2) loop.
NonlocalTable make_nonlocal_table(const HostMesh& m, double r_d) {
  NonlocalTable tb;
  const int32_t nt = m.nt;
  tb.ptr.assign(nt + 1, 0);
  if (r_d <= 0.0) {
    tb.ids.resize(nt);
    tb.w.assign(nt, 1.0);
    for (int32_t e = 0; e < nt; ++e) {
      tb.ptr[e + 1] = e + 1;
      tb.ids[e] = e;
    }
    return tb;
  }
  const double* c = m.centroid.data();
  double lo[3] = {c[0], c[1], c[2]}, hi[3] = {c[0], c[1], c[2]};
  for (int32_t e = 0; e < nt; ++e)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], c[3 * (size_t)e + a]);
      hi[a] = std::max(hi[a], c[3 * (size_t)e + a]);
    }
  double cell = r_d * (1.0 + 1e-9);
  for (;;) {
    double est = 1.0;
    for (int a = 0; a < 3; ++a) est *= std::floor((hi[a] - lo[a]) / cell) + 1.0;
    if (est <= 4.0 * nt + 1024.0) break;
    cell *= 2.0;
  }
  int64_t dims[3];
  for (int a = 0; a < 3; ++a) dims[a] = std::max<int64_t>(1, (int64_t)std::floor((hi[a] - lo[a]) / cell) + 1);
  auto bin = [&](int32_t e, int a) {
    const int64_t b = (int64_t)std::floor((c[3 * (size_t)e + a] - lo[a]) / cell);
    return std::min(std::max<int64_t>(b, 0), dims[a] - 1);
  };
  const int64_t nb = dims[0] * dims[1] * dims[2];
  std::vector<int64_t> bstart(nb + 1, 0);
  std::vector<int64_t> tbin(nt);
  for (int32_t e = 0; e < nt; ++e) {
    tbin[e] = (bin(e, 0) * dims[1] + bin(e, 1)) * dims[2] + bin(e, 2);
    bstart[tbin[e] + 1]++;
  }
  for (int64_t b = 0; b < nb; ++b) bstart[b + 1] += bstart[b];
  std::vector<int32_t> items(nt);
  {
    std::vector<int64_t> cur(bstart.begin(), bstart.end() - 1);
    for (int32_t e = 0; e < nt; ++e) items[cur[tbin[e]]++] = e;
  }
  std::vector<std::vector<int32_t>> lid(nt);
  std::vector<std::vector<double>> lw(nt);
#pragma omp parallel
  {
    std::vector<int32_t> cand;
#pragma omp for schedule(dynamic, 256)
    for (int32_t e = 0; e < nt; ++e) {
      cand.clear();
      const int64_t bx = bin(e, 0), by = bin(e, 1), bz = bin(e, 2);
      for (int64_t ix = std::max<int64_t>(bx - 1, 0); ix <= std::min(bx + 1, dims[0] - 1); ++ix)
        for (int64_t iy = std::max<int64_t>(by - 1, 0); iy <= std::min(by + 1, dims[1] - 1); ++iy)
          for (int64_t iz = std::max<int64_t>(bz - 1, 0); iz <= std::min(bz + 1, dims[2] - 1); ++iz) {
            const int64_t b = (ix * dims[1] + iy) * dims[2] + iz;
            cand.insert(cand.end(), items.begin() + bstart[b], items.begin() + bstart[b + 1]);
          }
      std::sort(cand.begin(), cand.end());
      double wsum = 0.0;
      auto& ids = lid[e];
      auto& ws = lw[e];
      const double* ce = c + 3 * (size_t)e;
      for (const int32_t o : cand) {
        const double* co = c + 3 * (size_t)o;
        const double r = norm3(co[0] - ce[0], co[1] - ce[1], co[2] - ce[2]);
        if (r > r_d) continue;
        const double w = 1.0 - r / r_d;
        if (w <= 0.0) continue;
        ids.push_back(o);
        ws.push_back(w);
        wsum += w;
      }
      for (double& w : ws) w /= wsum;
    }
  }
  for (int32_t e = 0; e < nt; ++e) tb.ptr[e + 1] = tb.ptr[e] + (int64_t)lid[e].size();
  tb.ids.resize(tb.ptr[nt]);
  tb.w.resize(tb.ptr[nt]);
#pragma omp parallel for schedule(static)
  for (int32_t e = 0; e < nt; ++e) {
    std::copy(lid[e].begin(), lid[e].end(), tb.ids.begin() + tb.ptr[e]);
    std::copy(lw[e].begin(), lw[e].end(), tb.w.begin() + tb.ptr[e]);
  }
  return tb;
}

}  // namespace gfb
