// C ABI of the FDA library (include/fda.h): argument checking, build
// orchestration (PAPER.md Algorithm Step 1, and §4 tables) and
// host-table export for host-logic tests.
#include <chrono>
#include <cuda_runtime.h>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <new>
#include <stdexcept>
#include <omp.h>
#include <nvtx3/nvToolsExt.h>

#include "fda_internal.h"

namespace {
// NVTX ranges around the public calls and the build phases (header-only NVTX v3: no-ops
// unless a profiler such as Nsight Systems is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace fda;

template <class T, class A>
static fda_status put(const std::vector<T, A>& v, void* dst, int64_t* count, int32_t* eb) {
  *count = (int64_t)v.size();
  *eb = (int32_t)sizeof(T);
  if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(T));
  return FDA_OK;
}


extern "C" {

fda_status fda_options_default(fda_options* opt) {
  if (!opt) return FDA_E_INVALID_ARG;
  std::memset(opt, 0, sizeof(*opt));
  opt->max_leaf = 64;
  opt->p_eq = 8;
  opt->p_chk_lf = 8;
  opt->p_chk_hf = 12;
  opt->eq_scale = 1.05;
  opt->chk_scale_lf = 2.95;
  opt->tier1_rho = 1.5;
  opt->tier2_rho = 3.0;
  opt->direct_all = 0;
  opt->device = 0;
  opt->build_threads = 0;
  opt->use_graph = 1;
  opt->verbose = 0;
  opt->m2l_lowrank = 1;
  opt->rhs_operator = 0;
  opt->rank = 0;
  opt->nranks = 1;
  opt->tensor_cores = 2;
  opt->hf_leaves = 0;
  opt->lr_tensor_cores = 2;
  opt->build_on_device = 1;
  opt->m2l_bf16 = 1;
  return FDA_OK;
}

const char* fda_status_string(fda_status s) {
  switch (s) {
    case FDA_OK: return "FDA_OK";
    case FDA_E_INVALID_ARG: return "FDA_E_INVALID_ARG";
    case FDA_E_MESH: return "FDA_E_MESH";
    case FDA_E_NOMEM: return "FDA_E_NOMEM";
    case FDA_E_CUDA: return "FDA_E_CUDA";
    case FDA_E_NCCL: return "FDA_E_NCCL";
    case FDA_E_NOT_CONVERGED: return "FDA_E_NOT_CONVERGED";
    case FDA_E_STATE: return "FDA_E_STATE";
    case FDA_E_INTERNAL: return "FDA_E_INTERNAL";
  }
  return "unknown";
}

static thread_local std::string g_build_error;

const char* fda_last_error(const fda_ctx* ctx) {
  if (!ctx) return g_build_error.c_str();
  return ctx->err.c_str();
}

fda_status fda_build(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt, double k,
                     fda_cplx alpha, double eps, const fda_options* opt, fda_ctx** out) {
  NvtxRange nvtx_range("fda_build");
  g_build_error.clear();
  if (!out || !vertices || !triangles) { g_build_error = "null pointer argument"; return FDA_E_INVALID_ARG; }
  *out = nullptr;
  if (!(k > 0) || !std::isfinite(k)) { g_build_error = "k must be > 0"; return FDA_E_INVALID_ARG; }
  if (!(eps > 0 && eps <= 0.1)) { g_build_error = "eps must lie in (0, 0.1]"; return FDA_E_INVALID_ARG; }
  if (alpha.im == 0.0 || !std::isfinite(alpha.re) || !std::isfinite(alpha.im)) {
    g_build_error = "alpha must have a non-zero imaginary part (Burton-Miller coupling, i/k recommended)";
    return FDA_E_INVALID_ARG;
  }
  if (nt < 1) { g_build_error = "nt must be >= 1"; return FDA_E_INVALID_ARG; }
  auto t0 = std::chrono::steady_clock::now();
  fda_ctx* ctx = new (std::nothrow) fda_ctx();
  if (!ctx) return FDA_E_NOMEM;
  ctx->p.k = k;
  ctx->p.alpha = cd(alpha.re, alpha.im);
  ctx->p.eps = eps;
  if (opt) ctx->p.opt = *opt; else fda_options_default(&ctx->p.opt);
  fda_options& o = ctx->p.opt;
  if (o.nranks < 1) o.nranks = 1;
  if (o.rank < 0 || o.rank >= o.nranks) {
    g_build_error = "opt.rank must lie in [0, opt.nranks)";
    delete ctx;
    return FDA_E_INVALID_ARG;
  }
  if (o.max_leaf < 1 || o.max_leaf > 128 || o.p_eq < 2 || o.p_chk_lf < 2 || o.p_chk_hf < 2 || !(o.eq_scale > 0) ||
      !(o.chk_scale_lf > o.eq_scale) || !(o.tier1_rho >= 0) || !(o.tier2_rho >= o.tier1_rho) ||
      o.tensor_cores < 0 || o.tensor_cores > 5 || o.hf_leaves < 0 || o.hf_leaves > 1 ||
      o.lr_tensor_cores < 0 || o.lr_tensor_cores > 2) {
    g_build_error = "invalid fda_options";
    delete ctx;
    return FDA_E_INVALID_ARG;
  }
  int saved_threads = omp_get_max_threads();
  if (o.build_threads > 0) omp_set_num_threads(o.build_threads);
  fda_status st = FDA_OK;
  try {
    auto tp = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
      auto now = std::chrono::steady_clock::now();
      if (o.verbose) fprintf(stderr, "[fda_build] %-12s %8.3f s\n", name, std::chrono::duration<double>(now - tp).count());
      nvtxMarkA(name);   // end of a build phase on the profiler timeline
      tp = now;
    };
    st = build_geometry(vertices, nv, triangles, nt, ctx->g, ctx->err);
    if (st == FDA_OK) {
      phase("geometry");
      build_tree(ctx->g, ctx->p, ctx->t);
      phase("tree");
      build_lists(ctx->g, ctx->p, ctx->t, ctx->plan);
      phase("lists");
      Plan& pl = ctx->plan;
      const int nlev = (int)ctx->t.levels.size();
      std::vector<bool> need(nlev, false);
      for (int l = 0; l < nlev; ++l)
        need[l] = pl.out_level_begin[l + 1] > pl.out_level_begin[l] || pl.in_level_begin[l + 1] > pl.in_level_begin[l];
      build_clouds_and_svd(ctx->p, ctx->t, need);
      phase("svd");
      // state offsets (complex entries)
      pl.out_offset.resize(pl.out_states.size());
      pl.in_offset.resize(pl.in_states.size());
      int64_t off = 0;
      for (size_t s = 0; s < pl.out_states.size(); ++s) {
        pl.out_offset[s] = off;
        off += (ctx->t.levels[ctx->t.boxes[pl.out_states[s].box].level].rank + 3) & ~3;   // 32-B aligned states
      }
      pl.out_size = off;
      off = 0;
      for (size_t s = 0; s < pl.in_states.size(); ++s) {
        pl.in_offset[s] = off;
        off += (ctx->t.levels[ctx->t.boxes[pl.in_states[s].box].level].rank + 3) & ~3;
      }
      pl.in_size = off;
      // operator tables: the device build (fp64 on opt.device) where possible, the host for
      // the rest (HF-leaf S2M / L2T) and for host-only contexts
      // sharding (opt.nranks > 1): own leaves, exchange plan, pruned ops and the matrices this
      // rank needs, decided before any table is built (partition.cpp)
      std::vector<char> needed;
      apply_partition(ctx->p, ctx->t, pl, needed);
      const bool on_dev = o.build_on_device != 0 && o.device >= 0;
      operator_layout(ctx->t, pl, needed);
      std::vector<char> done;
      LowRank lr;
      if (on_dev) {
        st = build_operators_device(ctx, done, lr);
        if (st != FDA_OK) throw std::runtime_error(ctx->err);
        phase("operators (device)");
      }
      const size_t pool_dev_size = pl.pool.size();
      build_operators(ctx->g, ctx->p, ctx->t, pl, done, lr);
      if (ctx->pool_dev) {   // the host-side part into the device pool: the §4.2 factors appended at the
                             // end, and any matrix the device build left to the host (HF-leaf S2M / L2T)
        if ((int64_t)pl.pool.size() > ctx->pool_dev_cap) throw std::runtime_error("device pool capacity exceeded");
        float2* dp = static_cast<float2*>(ctx->pool_dev);
        auto up = [&](size_t off, size_t cnt) {
          if (cnt && cudaMemcpy(dp + off, pl.pool.data() + off, cnt * sizeof(float2), cudaMemcpyHostToDevice) !=
                         cudaSuccess)
            throw std::runtime_error("upload of host-built matrices failed");
        };
        up(pool_dev_size, pl.pool.size() - pool_dev_size);
        for (size_t id = 0; id < done.size(); ++id)
          if (!done[id] && pl.mats[id].rows > 0) up((size_t)pl.mats[id].offset, (size_t)pl.mats[id].rows * pl.mats[id].cols);
      }
      phase("operators");
      // §4.2: route the M2L ops whose K̃ was factored (r < T/2) to the two-stage path
      pl.n_m2l_total = 0;
      pl.m2l_lr.clear();
      pl.tmp_size = 0;
      for (size_t l = 0; l < pl.m2l.size(); ++l) {
        std::vector<Op> dense;
        // levels where a factored K̃ is shared by fewer than 16 ops on average (the
        // coarse HF levels: ~10 at config 2 L2) keep the dense K̃ — the grouped dense
        // translation kernel tiles 16 ops per CTA, the fused factored one 64
        // (the share is counted on the GLOBAL op list before any sharding, so every rank of a
        // sharded build routes a level the same way)
        const bool use_lr = !pl.lr_V.empty() && l < pl.m2l_share.size() && pl.m2l_share[l] >= 16.0;
        for (const Op& op : pl.m2l[l]) {
          ++pl.n_m2l_total;
          if (use_lr && pl.lr_V[op.mat] >= 0) {
            LrOp lo{op.src, op.dst, pl.lr_V[op.mat], pl.lr_U[op.mat], pl.tmp_size, (int)l};
            pl.tmp_size += pl.mats[pl.lr_V[op.mat]].rows;
            pl.m2l_lr.push_back(lo);
          } else {
            dense.push_back(op);
          }
        }
        pl.m2l[l].swap(dense);
      }
      for (int kind = 0; kind <= (o.rhs_operator ? 1 : 0); ++kind) {
        if (on_dev) {
          st = build_corrections_device(ctx, kind);
          if (st != FDA_OK) throw std::runtime_error(ctx->err);
        } else {
          build_corrections(ctx->g, ctx->p, pl, kind);
        }
      }
      phase("corrections");
    }
  } catch (const std::bad_alloc&) {
    ctx->err = "host allocation failed during build";
    st = FDA_E_NOMEM;
  } catch (const std::exception& e) {
    ctx->err = std::string("build failed: ") + e.what();
    st = FDA_E_INTERNAL;
  }
  if (o.build_threads > 0) omp_set_num_threads(saved_threads);
  if (st == FDA_OK && o.device >= 0) st = engine_create(ctx);
  if (st != FDA_OK) {
    g_build_error = ctx->err;
    engine_destroy(ctx);
    if (ctx->pool_dev) cudaFree(ctx->pool_dev);   // not adopted by an engine
    for (void* c : ctx->corr_dev)
      if (c) cudaFree(c);
    delete ctx;
    return st;
  }
  // statistics
  fda_build_info& I = ctx->info;
  const Plan& pl = ctx->plan;
  const Tree& t = ctx->t;
  I.n_elements = nt;
  I.n_levels = (int32_t)t.levels.size();
  I.n_hf_levels = 0;
  for (int l = 0; l < I.n_levels && l < 32; ++l) {
    I.rank[l] = t.levels[l].rank;
    I.dirs[l] = t.levels[l].ndir;
    I.width[l] = t.levels[l].width;
    if (t.levels[l].hf) ++I.n_hf_levels;
  }
  I.n_boxes = (int64_t)t.boxes.size();
  I.n_leaves = (int64_t)t.leaves.size();
  I.n_out_states = (int64_t)pl.out_states.size();
  I.n_in_states = (int64_t)pl.in_states.size();
  I.n_m2l_pairs = pl.n_m2l_total;
  for (auto& v : pl.m2m) I.n_m2m_ops += (int64_t)v.size();
  for (auto& v : pl.l2l) I.n_l2l_ops += (int64_t)v.size();
  I.n_direct_leaf_pairs = (int64_t)pl.near_idx.size();
  for (size_t i = 0; i + 1 < pl.near_ptr.size(); ++i) {
    const Box& B = t.boxes[t.leaves[i]];
    for (int64_t e = pl.near_ptr[i]; e < pl.near_ptr[i + 1]; ++e) {
      const Box& C = t.boxes[t.leaves[pl.near_idx[e]]];
      I.n_direct_element_pairs += (B.end - B.begin) * (C.end - C.begin);
    }
  }
  I.n_corrections = (int64_t)pl.corr_col.size();
  I.n_matrices = (int64_t)pl.mats.size();
  I.table_bytes = (int64_t)pl.pool.size() * 8 + (int64_t)pl.corr_col.size() * 12 + (int64_t)pl.corr_col_rhs.size() * 12;
  I.t_build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = ctx;
  return FDA_OK;
}

fda_status fda_matvec(fda_ctx* ctx, const void* x, void* y, int32_t flags, void* stream) {
  if (!ctx) return FDA_E_INVALID_ARG;
  if (!x || !y || x == y) { ctx->err = "x and y must be non-null and must not alias"; return FDA_E_INVALID_ARG; }
  if (!ctx->dev) { ctx->err = "context was built host-only (opt.device = -1): no device matvec"; return FDA_E_STATE; }
  NvtxRange nvtx_range("fda_matvec");
  return engine_apply(ctx, x, y, flags, stream, 0);
}

fda_status fda_rhs_plane_wave(fda_ctx* ctx, const double dir[3], void* b, int32_t flags) {
  if (!ctx || !dir || !b) return FDA_E_INVALID_ARG;
  double nrm = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
  if (!(nrm > 0)) { ctx->err = "plane-wave direction must be non-zero"; return FDA_E_INVALID_ARG; }
  if (!ctx->dev) { ctx->err = "context was built host-only"; return FDA_E_STATE; }
  return engine_rhs_plane_wave(ctx, dir, b, flags);
}

fda_status fda_exchange_local(fda_ctx** ctxs, int32_t n) {
  if (!ctxs || n < 2) return FDA_E_INVALID_ARG;
  std::vector<fda::Context*> cs(n);
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || !ctxs[i]->dev || ctxs[i]->p.opt.nranks != n || ctxs[i]->p.opt.rank != i) {
      if (ctxs[i]) ctxs[i]->err = "fda_exchange_local: ctxs[i] must be rank i of an n-rank device build";
      return FDA_E_INVALID_ARG;
    }
    cs[i] = ctxs[i];
  }
  return fda::engine_exchange_local(cs.data(), n);
}

fda_status fda_rhs_point_source(fda_ctx* ctx, const double src[3], void* b, int32_t flags) {
  if (!ctx || !src || !b) return FDA_E_INVALID_ARG;
  if (!std::isfinite(src[0]) || !std::isfinite(src[1]) || !std::isfinite(src[2])) {
    ctx->err = "point-source position must be finite";
    return FDA_E_INVALID_ARG;
  }
  const fda::Vec3 xs(src[0], src[1], src[2]);
  for (const fda::Vec3& c : ctx->g.centroid)
    if ((c - xs).norm() == 0.0) { ctx->err = "point source coincides with a collocation point"; return FDA_E_INVALID_ARG; }
  if (!ctx->dev) { ctx->err = "context was built host-only"; return FDA_E_STATE; }
  return engine_rhs_point_source(ctx, src, b, flags);
}

fda_status fda_rhs_apply(fda_ctx* ctx, const void* v, void* b, int32_t flags, void* stream) {
  if (!ctx) return FDA_E_INVALID_ARG;
  if (!v || !b || v == b) { ctx->err = "v and b must be non-null and must not alias"; return FDA_E_INVALID_ARG; }
  if (!ctx->dev) { ctx->err = "context was built host-only (opt.device = -1)"; return FDA_E_STATE; }
  if (!ctx->p.opt.rhs_operator) { ctx->err = "context was built without opt.rhs_operator"; return FDA_E_STATE; }
  NvtxRange nvtx_range("fda_rhs_apply");
  return engine_apply(ctx, v, b, flags, stream, 1);
}

fda_status bm_solve(fda_ctx* ctx, const void* rhs, void* u, double tol, int32_t max_iter, int32_t restart,
                    fda_solve_info* info, int32_t flags) {
  if (!ctx) return FDA_E_INVALID_ARG;
  if (!rhs || !u || rhs == u) { ctx->err = "rhs and u must be non-null and must not alias"; return FDA_E_INVALID_ARG; }
  if (!(tol > 0) || max_iter < 1 || restart < 0) { ctx->err = "tol > 0, max_iter >= 1, restart >= 0"; return FDA_E_INVALID_ARG; }
  if (flags & FDA_HOST_C64) { ctx->err = "bm_solve takes complex128 host vectors (FDA_HOST_C64 is for fda_matvec)"; return FDA_E_INVALID_ARG; }
  if (!ctx->dev) { ctx->err = "context was built host-only"; return FDA_E_STATE; }
  NvtxRange nvtx_range("bm_solve");
  return engine_solve(ctx, rhs, u, tol, max_iter, restart, info, flags);
}

fda_status fda_nccl_unique_id(void* id128) {
  if (!id128) return FDA_E_INVALID_ARG;
  return nccl_unique_id(id128, g_build_error);
}

fda_status fda_comm_init(fda_ctx* ctx, const void* id128) {
  if (!ctx || !id128) return FDA_E_INVALID_ARG;
  if (ctx->p.opt.nranks <= 1) { ctx->err = "fda_comm_init needs a context built with opt.nranks > 1"; return FDA_E_STATE; }
  if (!ctx->dev) { ctx->err = "context was built host-only"; return FDA_E_STATE; }
  return engine_comm_init(ctx, id128);
}

fda_status fda_stats(const fda_ctx* ctx, fda_build_info* info) {
  if (!ctx || !info) return FDA_E_INVALID_ARG;
  *info = ctx->info;
  return FDA_OK;
}

fda_status fda_set_profiling(fda_ctx* ctx, int32_t on) {
  if (!ctx) return FDA_E_INVALID_ARG;
  ctx->profiling = on != 0;
  return FDA_OK;
}

fda_status fda_near_time(fda_ctx* ctx, double* ms) {
  if (!ctx || !ms) return FDA_E_INVALID_ARG;
  if (!ctx->dev) { ctx->err = "context was built host-only"; return FDA_E_STATE; }
  return engine_near_time(ctx, ms);
}

fda_status fda_stage_times(fda_ctx* ctx, double* ms, int32_t* n) {
  if (!ctx || !ms || !n) return FDA_E_INVALID_ARG;
  if (!ctx->dev) return FDA_E_STATE;
  return engine_stage_times(ctx, ms, n);
}

fda_status fda_kernel_times(fda_ctx* ctx, double* ms, int32_t* n) {
  if (!ctx || !ms || !n) return FDA_E_INVALID_ARG;
  if (!ctx->dev) return FDA_E_STATE;
  return engine_kernel_times(ctx, ms, n);
}

fda_status fda_debug_table(const fda_ctx* ctx, const char* name, void* dst, int64_t* count, int32_t* eb) {
  if (!ctx || !name || !count || !eb) return FDA_E_INVALID_ARG;
  const Plan& p = ctx->plan;
  const Tree& t = ctx->t;
  const Geometry& g = ctx->g;
  std::string nm(name);
  auto ops = [&](const std::vector<std::vector<Op>>& v) {
    std::vector<int64_t> o;
    for (size_t l = 0; l < v.size(); ++l)
      for (auto& op : v[l]) { o.push_back((int64_t)l); o.push_back(op.src); o.push_back(op.dst); o.push_back(op.mat); }
    return o;
  };
  if (nm == "perm") return put(g.perm, dst, count, eb);
  if (nm == "verts") {
    std::vector<double> v;
    for (int64_t i = 0; i < g.n; ++i)
      for (const Vec3* q : {&g.v0[i], &g.v1[i], &g.v2[i]}) { v.push_back(q->x); v.push_back(q->y); v.push_back(q->z); }
    return put(v, dst, count, eb);
  }
  if (nm == "leaf_range") {
    std::vector<int64_t> v;
    for (int64_t b : t.leaves) { v.push_back(t.boxes[b].begin); v.push_back(t.boxes[b].end); }
    return put(v, dst, count, eb);
  }
  if (nm == "leaf_S") return put(p.leaf_S, dst, count, eb);
  if (nm == "leaf_T") return put(p.leaf_T, dst, count, eb);
  if (nm == "leaf_out") return put(p.leaf_out, dst, count, eb);
  if (nm == "leaf_in") return put(p.leaf_in, dst, count, eb);
  if (nm == "out_offset") return put(p.out_offset, dst, count, eb);
  if (nm == "in_offset") return put(p.in_offset, dst, count, eb);
  if (nm == "sizes") return put(std::vector<int64_t>{p.out_size, p.in_size}, dst, count, eb);
  if (nm == "hf_s2m" || nm == "hf_s2m_rhs" || nm == "hf_l2t") {   // (leaf, state, matrix) triples
    const auto& L = nm == "hf_s2m" ? p.hf_s2m : (nm == "hf_s2m_rhs" ? p.hf_s2m_rhs : p.hf_l2t);
    std::vector<int64_t> v;
    for (const auto& o : L) { v.push_back(o.leaf); v.push_back(o.state); v.push_back(o.mat); }
    return put(v, dst, count, eb);
  }
  if (nm == "xsend" || nm == "xrecv") {   // per peer: count, sorted out-state ids
    const auto& L = nm == "xsend" ? p.xsend : p.xrecv;
    std::vector<int64_t> v;
    for (const auto& q : L) {
      v.push_back((int64_t)q.size());
      v.insert(v.end(), q.begin(), q.end());
    }
    return put(v, dst, count, eb);
  }
  if (nm == "m2m") return put(ops(p.m2m), dst, count, eb);
  if (nm == "m2l") return put(ops(p.m2l), dst, count, eb);
  if (nm == "l2l") return put(ops(p.l2l), dst, count, eb);
  if (nm == "m2l_lr") {  // level, src, dst, matV, matU, tmp
    std::vector<int64_t> v;
    for (auto& o : p.m2l_lr)
      for (int64_t x : {(int64_t)o.level, o.src, o.dst, o.matV, o.matU, o.tmp}) v.push_back(x);
    return put(v, dst, count, eb);
  }
  if (nm == "mats") {
    std::vector<int64_t> v;
    for (auto& m : p.mats) { v.push_back(m.offset); v.push_back(m.rows); v.push_back(m.cols); }
    return put(v, dst, count, eb);
  }
  if (nm == "specs") {
    std::vector<int64_t> v;
    for (auto& s : p.specs) {
      for (int64_t x : {(int64_t)s.kind, (int64_t)s.level, (int64_t)s.octant, (int64_t)s.dir, s.leaf, s.dx, s.dy, s.dz}) v.push_back(x);
    }
    return put(v, dst, count, eb);
  }
  if (nm == "pool" || nm == "corr_val" || nm == "corr_val_rhs") {
    // device build: the device-built values were never downloaded; read them from the engine
    const int which = nm == "pool" ? 0 : (nm == "corr_val" ? 1 : 2);
    const bool on_dev = which == 0 ? ctx->pool_partial : (which == 1 ? p.corr_val.empty() && !p.corr_col.empty()
                                                                      : p.corr_val_rhs.empty() && !p.corr_col_rhs.empty());
    if (on_dev && ctx->dev) {
      const int64_t n = which == 0 ? (int64_t)p.pool.size() : (int64_t)(which == 1 ? p.corr_col : p.corr_col_rhs).size();
      if (count) *count = n;
      if (eb) *eb = (int32_t)sizeof(cf);
      if (!dst) return FDA_OK;
      return engine_read_table(const_cast<fda_ctx*>(ctx), which, dst, n);
    }
  }
  if (nm == "pool") return put(p.pool, dst, count, eb);
  if (nm == "near_ptr") return put(p.near_ptr, dst, count, eb);
  if (nm == "near_idx") return put(p.near_idx, dst, count, eb);
  if (nm == "corr_ptr") return put(p.corr_ptr, dst, count, eb);
  if (nm == "corr_col") return put(p.corr_col, dst, count, eb);
  if (nm == "corr_val") return put(p.corr_val, dst, count, eb);
  if (nm == "corr_ptr_rhs") return put(p.corr_ptr_rhs, dst, count, eb);
  if (nm == "corr_col_rhs") return put(p.corr_col_rhs, dst, count, eb);
  if (nm == "corr_val_rhs") return put(p.corr_val_rhs, dst, count, eb);
  if (nm == "leaf_S_rhs") return put(p.leaf_S_rhs, dst, count, eb);
  if (nm == "out_states" || nm == "in_states") {
    const auto& S = nm == "out_states" ? p.out_states : p.in_states;
    std::vector<int64_t> v;
    for (auto& s : S) { v.push_back(s.box); v.push_back(s.dir); }
    return put(v, dst, count, eb);
  }
  if (nm == "boxes") {  // level, ix, iy, iz, parent, begin, end, leaf
    std::vector<int64_t> v;
    for (auto& b : t.boxes)
      for (int64_t x : {(int64_t)b.level, b.ix, b.iy, b.iz, b.parent, b.begin, b.end, (int64_t)b.leaf}) v.push_back(x);
    return put(v, dst, count, eb);
  }
  if (nm == "box_center") {
    std::vector<double> v;
    for (auto& b : t.boxes) { v.push_back(b.center.x); v.push_back(b.center.y); v.push_back(b.center.z); }
    return put(v, dst, count, eb);
  }
  if (nm == "levels") {  // width, hf, nf, rank
    std::vector<double> v;
    for (auto& L : t.levels) { v.push_back(L.width); v.push_back(L.hf); v.push_back(L.nf); v.push_back(L.rank); }
    return put(v, dst, count, eb);
  }
  if (nm == "owned")
    return put(std::vector<int64_t>{p.own_leaf0, p.own_leaf1, p.own_e0, p.own_e1}, dst, count, eb);
  if (nm == "launches") return put(std::vector<int64_t>{ctx->launches_per_matvec}, dst, count, eb);
  if (nm == "kernel_tasks")
    return put(std::vector<int64_t>(ctx->kernel_tasks, ctx->kernel_tasks + 18), dst, count, eb);
  if (nm == "kernel_flops")
    return put(std::vector<double>(ctx->kernel_flops, ctx->kernel_flops + 18), dst, count, eb);
  if (nm == "root") {
    return put(std::vector<double>{t.root_center.x, t.root_center.y, t.root_center.z, t.root_width, t.lambda},
               dst, count, eb);
  }
  const_cast<fda_ctx*>(ctx)->err = "unknown table name: " + nm;
  return FDA_E_INVALID_ARG;
}

void fda_free(fda_ctx* ctx) {
  if (!ctx) return;
  engine_destroy(ctx);
  delete ctx;
}

}  // extern "C"
