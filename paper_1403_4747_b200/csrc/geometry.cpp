// Mesh validation and element geometry (fp64, host).
// PAPER.md §5: flat triangles, collocation at centroids.
// Kernel normal n = -(v1-v0)×(v2-v0)/‖·‖ for CCW-from-outside triangles
// (reading C1: Eq. (2)/(4) hold with n pointing into the scatterer).
#include <algorithm>
#include <cmath>
#include <parallel/algorithm>
#include <vector>

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
  // per triangle (parallel): geometry and the first failing check; the lowest failing index is reported
  std::vector<int8_t> bad(nt, 0);   // 1 index out of range, 2 repeated vertex, 3 degenerate
  double signed_vol = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : signed_vol)
  for (int64_t t = 0; t < nt; ++t) {
    const int32_t ia = F[3 * t], ib = F[3 * t + 1], ic = F[3 * t + 2];
    if (ia < 0 || ib < 0 || ic < 0 || ia >= nv || ib >= nv || ic >= nv) { bad[t] = 1; continue; }
    if (ia == ib || ib == ic || ia == ic) { bad[t] = 2; continue; }
    Vec3 a(V[3 * ia], V[3 * ia + 1], V[3 * ia + 2]);
    Vec3 b(V[3 * ib], V[3 * ib + 1], V[3 * ib + 2]);
    Vec3 c(V[3 * ic], V[3 * ic + 1], V[3 * ic + 2]);
    Vec3 cr = (b - a).cross(c - a);
    double nrm = cr.norm();
    if (!(0.5 * nrm > 1e-14 * diag2)) { bad[t] = 3; continue; }
    g.v0[t] = a; g.v1[t] = b; g.v2[t] = c;
    g.area[t] = 0.5 * nrm;
    g.normal[t] = cr * (-1.0 / nrm);
    g.centroid[t] = (a + b + c) * (1.0 / 3.0);
    g.hmax[t] = std::max({(b - a).norm(), (c - b).norm(), (a - c).norm()});
    g.perm[t] = t;
    signed_vol += a.dot(b.cross(c)) / 6.0;
  }
  for (int64_t t = 0; t < nt; ++t) {
    if (!bad[t]) continue;
    const std::string tri = "triangle " + std::to_string(t);
    if (bad[t] == 1) { err = tri + " has a vertex index out of range"; return FDA_E_INVALID_ARG; }
    if (bad[t] == 2) { err = tri + " repeats a vertex"; return FDA_E_MESH; }
    err = tri + " is degenerate (area <= 1e-14 diag^2)";
    return FDA_E_MESH;
  }
  // closed, consistently oriented 2-manifold: every directed edge once, and its reverse present
  std::vector<uint64_t> edges((size_t)3 * nt);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < nt; ++t) {
    const uint32_t v[3] = {(uint32_t)F[3 * t], (uint32_t)F[3 * t + 1], (uint32_t)F[3 * t + 2]};
    for (int k = 0; k < 3; ++k) edges[3 * t + k] = ((uint64_t)v[k] << 32) | v[(k + 1) % 3];
  }
  __gnu_parallel::sort(edges.begin(), edges.end());
  bool dup = false, open = false;
#pragma omp parallel for schedule(static) reduction(|| : dup, open)
  for (int64_t e = 0; e < (int64_t)edges.size(); ++e) {
    if (e > 0 && edges[e] == edges[e - 1]) dup = true;
    const uint64_t rev = (edges[e] << 32) | (edges[e] >> 32);
    if (!std::binary_search(edges.begin(), edges.end(), rev)) open = true;
  }
  if (dup) {
    err = "directed edge used twice: mesh is non-manifold or inconsistently oriented";
    return FDA_E_MESH;
  }
  if (open) {
    err = "mesh is open (an edge has no opposite half-edge); the exterior solver needs a closed surface";
    return FDA_E_MESH;
  }
  if (signed_vol <= 0.0) {
    err = "mesh is oriented inward (negative signed volume); triangles must be CCW seen from outside";
    return FDA_E_MESH;
  }
  return FDA_OK;
}

}  // namespace fda
