// host_viz.cpp — RenderMesh (host_viz.hpp): the render-side consumer of the newly-broken edge lists
// (grafem::VizMesh, viz.cpp:20-412). See the header for the rules the output follows.
#include "host_viz.hpp"

#include <algorithm>
#include <cstdio>
#include <numeric>

namespace gfb {

namespace {

using V3 = std::array<double, 3>;

V3 sub(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
double dot(const V3& a, const V3& b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
// signed volume of the tet (origin, a, b, c)
double tri_vol(const V3& a, const V3& b, const V3& c) { return dot(a, cross(b, c)) / 6.0; }

constexpr int kFaceLocal[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};  // face k: opposite local node k

}  // namespace

RenderMesh::RenderMesh(HostMesh mesh) : m_(std::move(mesh)) {
  const int32_t nt = m_.nt;
  // unique faces, ids in order of first appearance over (tet, local face)
  struct Rec {
    std::array<int32_t, 3> key;
    int32_t pos;  // 4 tet + local face
  };
  std::vector<Rec> recs(4 * (size_t)nt);
  for (int32_t t = 0; t < nt; ++t)
    for (int fi = 0; fi < 4; ++fi) {
      std::array<int32_t, 3> k = {m_.tets[4 * (size_t)t + kFaceLocal[fi][0]], m_.tets[4 * (size_t)t + kFaceLocal[fi][1]],
                                  m_.tets[4 * (size_t)t + kFaceLocal[fi][2]]};
      std::sort(k.begin(), k.end());
      recs[4 * (size_t)t + fi] = {k, 4 * t + fi};
    }
  std::sort(recs.begin(), recs.end(), [](const Rec& a, const Rec& b) { return a.key != b.key ? a.key < b.key : a.pos < b.pos; });
  struct Group {
    int32_t first, begin, end;  // first appearance; [begin, end) in recs
  };
  std::vector<Group> groups;
  for (int32_t i = 0; i < (int32_t)recs.size();) {
    int32_t j = i;
    while (j < (int32_t)recs.size() && recs[j].key == recs[i].key) ++j;
    groups.push_back({recs[i].pos, i, j});
    i = j;
  }
  std::sort(groups.begin(), groups.end(), [](const Group& a, const Group& b) { return a.first < b.first; });
  auto edge_id = [this](int32_t a, int32_t b) {
    const int32_t lo = std::min(a, b), hi = std::max(a, b);
    int32_t l = 0, r = m_.ne;
    while (l < r) {  // edges are (min, max) pairs in lexicographic order (mesh.cpp:50-57)
      const int32_t mid = (l + r) / 2;
      const int32_t e0 = m_.edges[2 * (size_t)mid], e1 = m_.edges[2 * (size_t)mid + 1];
      if (e0 < lo || (e0 == lo && e1 < hi)) l = mid + 1;
      else r = mid;
    }
    if (l >= m_.ne || m_.edges[2 * (size_t)l] != lo || m_.edges[2 * (size_t)l + 1] != hi)
      throw GeometryError("face edge lookup failed");
    return l;
  };
  auto X = [this](int32_t n) { return V3{m_.X[3 * (size_t)n], m_.X[3 * (size_t)n + 1], m_.X[3 * (size_t)n + 2]}; };
  face_nodes_.resize(groups.size());
  face_edges_.resize(groups.size());
  tet_faces_.resize(nt);
  for (int32_t f = 0; f < (int32_t)groups.size(); ++f) {
    const Group& g = groups[f];
    const auto& k = recs[g.begin].key;
    face_nodes_[f] = k;
    face_edges_[f] = {edge_id(k[0], k[1]), edge_id(k[0], k[2]), edge_id(k[1], k[2])};
    for (int32_t i = g.begin; i < g.end; ++i) tet_faces_[recs[i].pos / 4][recs[i].pos % 4] = f;
    if (g.end - g.begin == 1) {  // boundary face: orient outward, away from the opposite vertex (viz.cpp:48-55)
      const int32_t t = recs[g.begin].pos / 4, fi = recs[g.begin].pos % 4;
      const int32_t* tv = &m_.tets[4 * (size_t)t];
      std::array<int32_t, 3> tri = {tv[kFaceLocal[fi][0]], tv[kFaceLocal[fi][1]], tv[kFaceLocal[fi][2]]};
      const V3 a = X(tri[0]);
      if (dot(cross(sub(X(tri[1]), a), sub(X(tri[2]), a)), sub(X(tv[fi]), a)) > 0.0) std::swap(tri[1], tri[2]);
      boundary_.push_back(tri);
      boundary_face_.push_back(f);
    }
  }
  // edge -> faces, ascending face id
  ef_ptr_.assign(m_.ne + 1, 0);
  for (const auto& fe : face_edges_)
    for (int32_t e : fe) ++ef_ptr_[e + 1];
  std::partial_sum(ef_ptr_.begin(), ef_ptr_.end(), ef_ptr_.begin());
  ef_ids_.resize(ef_ptr_.back());
  std::vector<int32_t> fill(ef_ptr_.begin(), ef_ptr_.end() - 1);
  for (int32_t f = 0; f < (int32_t)face_edges_.size(); ++f)
    for (int32_t e : face_edges_[f]) ef_ids_[fill[e]++] = f;
}

int RenderMesh::nodes_of(Kind k, int32_t entity, int32_t out[4]) const {
  switch (k) {
    case kEdge:
      out[0] = m_.edges[2 * (size_t)entity];
      out[1] = m_.edges[2 * (size_t)entity + 1];
      return 2;
    case kFace:
      for (int i = 0; i < 3; ++i) out[i] = face_nodes_[entity][i];
      return 3;
    default:
      for (int i = 0; i < 4; ++i) out[i] = m_.tets[4 * (size_t)entity + i];
      return 4;
  }
}

int RenderMesh::group(Kind k, int32_t entity, int32_t node, const uint8_t* zeta, int32_t out[4]) const {
  int32_t nodes[4];
  const int n = nodes_of(k, entity, nodes);
  // the entity's edges as (local a, local b, edge id), in the reference's order (viz.cpp:79-107)
  int32_t le[6][3];
  int ne = 0;
  auto add = [&](int a, int b, int32_t id) {
    le[ne][0] = a;
    le[ne][1] = b;
    le[ne][2] = id;
    ++ne;
  };
  if (k == kEdge) {
    add(0, 1, entity);
  } else if (k == kFace) {
    const auto& fe = face_edges_[entity];
    add(0, 1, fe[0]);
    add(0, 2, fe[1]);
    add(1, 2, fe[2]);
  } else {
    for (int q = 0; q < 6; ++q) add(kLocalEdge[q][0], kLocalEdge[q][1], m_.tet_edges[6 * (size_t)entity + q]);
  }
  int label[4] = {0, 1, 2, 3};
  auto root = [&label](int i) {
    while (label[i] != i) i = label[i];
    return i;
  };
  for (int q = 0; q < ne; ++q) {  // union-find over the intact edges, smaller root wins
    if (zeta[le[q][2]]) continue;
    const int a = root(le[q][0]), b = root(le[q][1]);
    if (a != b) label[std::max(a, b)] = std::min(a, b);
  }
  int self = 0;
  while (nodes[self] != node) ++self;
  const int target = root(self);
  int cnt = 0;
  for (int i = 0; i < n; ++i)
    if (root(i) == target) out[cnt++] = nodes[i];
  return cnt;
}

int32_t RenderMesh::group_rep(Kind k, int32_t entity, int32_t node, const uint8_t* zeta) const {
  int32_t g[4];
  const int n = group(k, entity, node, zeta, g);
  return *std::min_element(g, g + n);
}

std::array<double, 3> RenderMesh::rest_point(Kind k, int32_t entity) const {
  int32_t nodes[4];
  const int n = nodes_of(k, entity, nodes);
  V3 p{0.0, 0.0, 0.0};
  if (k == kTet) {
    for (int a = 0; a < 3; ++a) p[a] = m_.centroid[3 * (size_t)entity + a];  // rest centroid (mesh.cpp:90)
  } else if (n == 2) {
    for (int a = 0; a < 3; ++a) p[a] = 0.5 * (m_.X[3 * (size_t)nodes[0] + a] + m_.X[3 * (size_t)nodes[1] + a]);
  } else {
    for (int a = 0; a < 3; ++a)
      p[a] = ((m_.X[3 * (size_t)nodes[0] + a] + m_.X[3 * (size_t)nodes[1] + a]) + m_.X[3 * (size_t)nodes[2] + a]) / 3.0;
  }
  return p;
}

// rest point + the mean displacement of a node group (viz.cpp:197-211)
static V3 follow(const V3& rest, const int32_t* g, int n, const double* u) {
  V3 mean{0.0, 0.0, 0.0};
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) mean[a] += u[3 * (size_t)g[i] + a];
  V3 p;
  for (int a = 0; a < 3; ++a) p[a] = rest[a] + mean[a] / (double)n;
  return p;
}

std::array<double, 3> RenderMesh::moved_point(Kind k, int32_t entity, int32_t side_node, const double* u,
                                               const uint8_t* zeta) const {
  int32_t g[4];
  const int n = group(k, entity, side_node, zeta, g);
  return follow(rest_point(k, entity), g, n, u);
}

std::array<double, 3> RenderMesh::child_position(int64_t c, const double* u, const uint8_t* zeta) const {
  if (c < 0 || c >= (int64_t)children_.size()) throw FormatError("child index out of range");
  const Child& ch = children_[c];
  int32_t g[4];
  const int n = group(ch.kind, ch.entity, ch.rep, zeta, g);
  return follow(ch.rest, g, n, u);
}

void RenderMesh::ensure_children(Kind k, int32_t entity, const uint8_t* zeta) {
  int32_t nodes[4], reps[4];
  const int n = nodes_of(k, entity, nodes);
  for (int i = 0; i < n; ++i) reps[i] = group_rep(k, entity, nodes[i], zeta);
  std::sort(reps, reps + n);
  const int nr = (int)(std::unique(reps, reps + n) - reps);
  for (int i = 0; i < nr; ++i) {  // ascending representative (viz.cpp:178-180)
    const uint64_t kk = key(k, entity, reps[i]);
    if (child_of_.count(kk)) continue;
    Child ch{k, entity, reps[i], rest_point(k, entity), {}};
    int32_t g[4];
    ch.parents.assign(g, g + group(k, entity, reps[i], zeta, g));
    child_of_.emplace(kk, (int32_t)children_.size());
    children_.push_back(std::move(ch));
  }
}

void RenderMesh::apply_splits(const int32_t* newly_broken, int64_t n, const uint8_t* zeta) {
  for (int64_t q = 0; q < n; ++q) {
    const int32_t e = newly_broken[q];
    if (e < 0 || e >= m_.ne) throw GeometryError("unknown edge id in split request");
    ensure_children(kEdge, e, zeta);
    for (int32_t p = ef_ptr_[e]; p < ef_ptr_[e + 1]; ++p) {
      const int32_t f = ef_ids_[p];
      ensure_children(kFace, f, zeta);
      for (int32_t fe : face_edges_[f]) ensure_children(kEdge, fe, zeta);  // midpoints of the split face's quads
    }
    for (int32_t p = m_.et_ptr[e]; p < m_.et_ptr[e + 1]; ++p) ensure_children(kTet, m_.et_ids[p], zeta);
  }
}

int64_t RenderMesh::handle(Kind k, int32_t entity, int32_t side_node, const uint8_t* zeta) const {
  const auto it = child_of_.find(key(k, entity, group_rep(k, entity, side_node, zeta)));
  if (it == child_of_.end()) throw GeometryError("missing split vertex; splits not applied");
  return (int64_t)m_.nn + it->second;
}

int32_t RenderMesh::face_edge(int32_t f, int32_t a, int32_t b) const {
  const int32_t lo = std::min(a, b), hi = std::max(a, b);
  for (int32_t e : face_edges_[f])
    if (m_.edges[2 * (size_t)e] == lo && m_.edges[2 * (size_t)e + 1] == hi) return e;
  throw GeometryError("face edge lookup failed");
}

void RenderMesh::edge_faces_in_tet(int32_t t, int32_t a, int32_t b, int32_t out[2]) const {
  int found = 0;
  for (int fi = 0; fi < 4 && found < 2; ++fi) {
    const auto& fn = face_nodes_[tet_faces_[t][fi]];
    const bool ha = fn[0] == a || fn[1] == a || fn[2] == a, hb = fn[0] == b || fn[1] == b || fn[2] == b;
    if (ha && hb) out[found++] = tet_faces_[t][fi];
  }
  if (out[0] > out[1]) std::swap(out[0], out[1]);
}

RenderMesh::Surface RenderMesh::build_surface(const double* u, const uint8_t* zeta) const {
  std::vector<std::array<int64_t, 3>> tris;
  // exterior: the boundary triangle while intact, else three corner quads (viz.cpp:226-257)
  for (size_t bi = 0; bi < boundary_.size(); ++bi) {
    const auto& tri = boundary_[bi];
    const int32_t f = boundary_face_[bi];
    const auto& fe = face_edges_[f];
    if (!(zeta[fe[0]] || zeta[fe[1]] || zeta[fe[2]])) {
      tris.push_back({tri[0], tri[1], tri[2]});
      continue;
    }
    for (int k = 0; k < 3; ++k) {
      const int32_t a = tri[k], b = tri[(k + 1) % 3], c = tri[(k + 2) % 3];
      const int64_t hab = handle(kEdge, face_edge(f, a, b), a, zeta), hf = handle(kFace, f, a, zeta);
      const int64_t hca = handle(kEdge, face_edge(f, c, a), a, zeta);
      tris.push_back({a, hab, hf});
      tris.push_back({a, hf, hca});
    }
  }
  // fracture surfaces: both sides' dual quads of every broken edge in every incident tet (viz.cpp:259-296)
  for (int32_t e = 0; e < m_.ne; ++e) {
    if (!zeta[e]) continue;
    const int32_t na = m_.edges[2 * (size_t)e], nb = m_.edges[2 * (size_t)e + 1];
    for (int32_t p = m_.et_ptr[e]; p < m_.et_ptr[e + 1]; ++p) {
      const int32_t t = m_.et_ids[p];
      int32_t fp[2] = {-1, -1};
      edge_faces_in_tet(t, na, nb, fp);
      const V3 pm = rest_point(kEdge, e), p1 = rest_point(kFace, fp[0]), pt = rest_point(kTet, t);
      for (int side = 0; side < 2; ++side) {
        const int32_t s = side == 0 ? na : nb, o = side == 0 ? nb : na;
        const int64_t hm = handle(kEdge, e, s, zeta), hf1 = handle(kFace, fp[0], s, zeta);
        const int64_t ht = handle(kTet, t, s, zeta), hf2 = handle(kFace, fp[1], s, zeta);
        const V3 outward = sub(V3{m_.X[3 * (size_t)o], m_.X[3 * (size_t)o + 1], m_.X[3 * (size_t)o + 2]},
                               V3{m_.X[3 * (size_t)s], m_.X[3 * (size_t)s + 1], m_.X[3 * (size_t)s + 2]});
        if (!(dot(cross(sub(p1, pm), sub(pt, pm)), outward) < 0.0)) {  // quad normal away from the owning side
          tris.push_back({hm, hf1, ht});
          tris.push_back({hm, ht, hf2});
        } else {
          tris.push_back({hm, ht, hf1});
          tris.push_back({hm, hf2, ht});
        }
      }
    }
  }
  // compact to the referenced vertices: original nodes ascending, then children (viz.cpp:298-316)
  std::vector<int64_t> used;
  used.reserve(3 * tris.size());
  for (const auto& t : tris) used.insert(used.end(), t.begin(), t.end());
  std::sort(used.begin(), used.end());
  used.erase(std::unique(used.begin(), used.end()), used.end());
  Surface s;
  s.xyz.reserve(3 * used.size());
  for (int64_t h : used) {
    V3 p;
    if (h < m_.nn) {
      for (int a = 0; a < 3; ++a) p[a] = m_.X[3 * (size_t)h + a] + u[3 * (size_t)h + a];
      ++s.n_original;
    } else {
      p = child_position(h - m_.nn, u, zeta);
    }
    s.xyz.insert(s.xyz.end(), p.begin(), p.end());
  }
  s.tris.reserve(tris.size());
  auto idx = [&used](int64_t h) { return (int32_t)(std::lower_bound(used.begin(), used.end(), h) - used.begin()); };
  for (const auto& t : tris) s.tris.push_back({idx(t[0]), idx(t[1]), idx(t[2])});
  return s;
}

void RenderMesh::export_frame(const std::string& path, const double* u, const uint8_t* zeta) const {
  const Surface s = build_surface(u, zeta);
  FILE* fp = std::fopen(path.c_str(), "w");
  if (!fp) throw FormatError("cannot write '" + path + "'");
  bool ok = true;
  for (size_t v = 0; v < s.xyz.size() / 3; ++v)
    ok &= std::fprintf(fp, "v %.17g %.17g %.17g\n", s.xyz[3 * v], s.xyz[3 * v + 1], s.xyz[3 * v + 2]) > 0;
  for (const auto& t : s.tris) ok &= std::fprintf(fp, "f %d %d %d\n", t[0] + 1, t[1] + 1, t[2] + 1) > 0;
  ok &= std::fclose(fp) == 0;
  if (!ok) throw FormatError("short write to '" + path + "'");
}

std::array<double, 4> RenderMesh::fragment_volumes(int32_t tet, const double* u, const uint8_t* zeta) const {
  if (tet < 0 || tet >= m_.nt) throw FormatError("tet index out of range");
  const int32_t* tv = &m_.tets[4 * (size_t)tet];
  auto X = [this](int32_t n) { return V3{m_.X[3 * (size_t)n], m_.X[3 * (size_t)n + 1], m_.X[3 * (size_t)n + 2]}; };
  std::array<double, 4> vol{0.0, 0.0, 0.0, 0.0};
  for (int corner = 0; corner < 4; ++corner) {
    const int32_t g = tv[corner];
    V3 pg = X(g);
    for (int a = 0; a < 3; ++a) pg[a] += u[3 * (size_t)g + a];
    double v = 0.0;
    // the corner's pieces of its three faces (viz.cpp:347-372)
    for (int fi = 0; fi < 4; ++fi) {
      if (fi == corner) continue;
      std::array<int32_t, 3> tri = {tv[kFaceLocal[fi][0]], tv[kFaceLocal[fi][1]], tv[kFaceLocal[fi][2]]};
      const V3 a = X(tri[0]);
      if (dot(cross(sub(X(tri[1]), a), sub(X(tri[2]), a)), sub(X(tv[fi]), a)) > 0.0) std::swap(tri[1], tri[2]);
      while (tri[0] != g) std::rotate(tri.begin(), tri.begin() + 1, tri.end());
      const int32_t f = tet_faces_[tet][fi];
      const V3 mab = moved_point(kEdge, face_edge(f, tri[0], tri[1]), g, u, zeta);
      const V3 cf = moved_point(kFace, f, g, u, zeta);
      const V3 mca = moved_point(kEdge, face_edge(f, tri[2], tri[0]), g, u, zeta);
      v += tri_vol(pg, mab, cf);
      v += tri_vol(pg, cf, mca);
    }
    // the corner's dual quads of its three edges (viz.cpp:374-408)
    for (int k = 0; k < 6; ++k) {
      const int32_t la = tv[kLocalEdge[k][0]], lb = tv[kLocalEdge[k][1]];
      if (la != g && lb != g) continue;
      const int32_t other = la == g ? lb : la;
      const int32_t e = m_.tet_edges[6 * (size_t)tet + k];
      int32_t fp[2] = {-1, -1};
      edge_faces_in_tet(tet, g, other, fp);
      const V3 pm = moved_point(kEdge, e, g, u, zeta), p1 = moved_point(kFace, fp[0], g, u, zeta);
      const V3 pt = moved_point(kTet, tet, g, u, zeta), p2 = moved_point(kFace, fp[1], g, u, zeta);
      const V3 rm = rest_point(kEdge, e), r1 = rest_point(kFace, fp[0]), rt = rest_point(kTet, tet);
      if (!(dot(cross(sub(r1, rm), sub(rt, rm)), sub(X(other), X(g))) < 0.0)) {
        v += tri_vol(pm, p1, pt);
        v += tri_vol(pm, pt, p2);
      } else {
        v += tri_vol(pm, pt, p1);
        v += tri_vol(pm, p2, pt);
      }
    }
    vol[corner] = v;
  }
  return vol;
}

}  // namespace gfb
