// Mesh validation and element geometry (fp64, host).
// PAPER.md §5: flat triangles, collocation at centroids.
// Kernel normal n = -(v1-v0)×(v2-v0)/‖·‖ for CCW-from-outside triangles
// (reading C1: Eq. (2)/(4) hold with n pointing into the scatterer).
#include <algorithm>
#include <cmath>
#include <unordered_map>

#include "fda_internal.h"

namespace fda {

double Vec3::norm() const { return std::sqrt(x * x + y * y + z * z); }

fda_status build_geometry(const double* V, int64_t nv, const int32_t* F, int64_t nt, Geometry& g,
                          std::string& err) {
  if (nt < 1 || nv < 3) {
    err = "mesh needs at least one triangle and three vertices";
    return FDA_E_INVALID_ARG;
  }
  Vec3 lo(1e300, 1e300, 1e300), hi(-1e300, -1e300, -1e300);
  for (int64_t i = 0; i < nv; ++i) {
    Vec3 p(V[3 * i], V[3 * i + 1], V[3 * i + 2]);
    if (!std::isfinite(p.x) || !std::isfinite(p.y) || !std::isfinite(p.z)) {
      err = "non-finite vertex coordinate";
      return FDA_E_MESH;
    }
    lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
    hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
  }
  const double diag2 = (hi - lo).dot(hi - lo);
  g.n = nt;
  g.v0.resize(nt); g.v1.resize(nt); g.v2.resize(nt);
  g.centroid.resize(nt); g.normal.resize(nt); g.area.resize(nt); g.hmax.resize(nt);
  g.perm.resize(nt);
  std::unordered_map<uint64_t, int32_t> edges;
  edges.reserve(static_cast<size_t>(3 * nt));
  double signed_vol = 0.0;
  for (int64_t t = 0; t < nt; ++t) {
    int32_t ia = F[3 * t], ib = F[3 * t + 1], ic = F[3 * t + 2];
    if (ia < 0 || ib < 0 || ic < 0 || ia >= nv || ib >= nv || ic >= nv) {
      err = "triangle " + std::to_string(t) + " has a vertex index out of range";
      return FDA_E_INVALID_ARG;
    }
    if (ia == ib || ib == ic || ia == ic) {
      err = "triangle " + std::to_string(t) + " repeats a vertex";
      return FDA_E_MESH;
    }
    Vec3 a(V[3 * ia], V[3 * ia + 1], V[3 * ia + 2]);
    Vec3 b(V[3 * ib], V[3 * ib + 1], V[3 * ib + 2]);
    Vec3 c(V[3 * ic], V[3 * ic + 1], V[3 * ic + 2]);
    Vec3 cr = (b - a).cross(c - a);
    double nrm = cr.norm();
    if (!(0.5 * nrm > 1e-14 * diag2)) {
      err = "triangle " + std::to_string(t) + " is degenerate (area <= 1e-14 diag^2)";
      return FDA_E_MESH;
    }
    g.v0[t] = a; g.v1[t] = b; g.v2[t] = c;
    g.area[t] = 0.5 * nrm;
    g.normal[t] = cr * (-1.0 / nrm);
    g.centroid[t] = (a + b + c) * (1.0 / 3.0);
    g.hmax[t] = std::max({(b - a).norm(), (c - b).norm(), (a - c).norm()});
    g.perm[t] = t;
    signed_vol += a.dot(b.cross(c)) / 6.0;
    const int32_t e[3][2] = {{ia, ib}, {ib, ic}, {ic, ia}};
    for (auto& ed : e) {
      uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(ed[0])) << 32) | static_cast<uint32_t>(ed[1]);
      if (++edges[key] > 1) {
        err = "directed edge used twice: mesh is non-manifold or inconsistently oriented";
        return FDA_E_MESH;
      }
    }
  }
  for (auto& kv : edges) {
    uint64_t rev = (kv.first << 32) | (kv.first >> 32);
    if (edges.find(rev) == edges.end()) {
      err = "mesh is open (an edge has no opposite half-edge); the exterior solver needs a closed surface";
      return FDA_E_MESH;
    }
  }
  if (signed_vol <= 0.0) {
    err = "mesh is oriented inward (negative signed volume); triangles must be CCW seen from outside";
    return FDA_E_MESH;
  }
  return FDA_OK;
}

}  // namespace fda
