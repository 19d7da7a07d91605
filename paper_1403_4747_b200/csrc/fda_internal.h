// Internal data structures of the FDA library (host side, fp64 build).
// See DESIGN.md §4 for the layout in HBM and §2 for the citations.
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>
#include <unordered_map>

#include "../../include/fda.h"

namespace fda {

struct Context;
using cd = std::complex<double>;
using cf = std::complex<float>;

// allocator that leaves new elements uninitialised (the 20+ GB matrix pool is fully overwritten by
// the operator build; zero-filling it cost seconds at config 5)
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind { using other = NoInitAlloc<U>; };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) {}
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    if constexpr (sizeof...(Args) > 0) ::new ((void*)p) U(std::forward<Args>(args)...);
  }
};
using PoolVec = std::vector<cf, NoInitAlloc<cf>>;

struct Vec3 {
  double x, y, z;
  Vec3() : x(0), y(0), z(0) {}
  Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  Vec3 operator-() const { return {-x, -y, -z}; }
  double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
  Vec3 cross(const Vec3& o) const { return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x}; }
  double norm() const;
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

struct Mat3 {  // row-major rotation
  double m[3][3];
  Vec3 apply(const Vec3& v) const {
    return {m[0][0] * v.x + m[0][1] * v.y + m[0][2] * v.z, m[1][0] * v.x + m[1][1] * v.y + m[1][2] * v.z,
            m[2][0] * v.x + m[2][1] * v.y + m[2][2] * v.z};
  }
  Vec3 apply_t(const Vec3& v) const {
    return {m[0][0] * v.x + m[1][0] * v.y + m[2][0] * v.z, m[0][1] * v.x + m[1][1] * v.y + m[2][1] * v.z,
            m[0][2] * v.x + m[1][2] * v.y + m[2][2] * v.z};
  }
};

// ---------------------------------------------------------------- geometry
struct Geometry {
  int64_t n = 0;                 // elements
  std::vector<Vec3> v0, v1, v2;  // triangle vertices (tree order)
  std::vector<Vec3> centroid;    // collocation points x_i
  std::vector<Vec3> normal;      // kernel normal, into the body (C1)
  std::vector<double> area, hmax;
  std::vector<int64_t> perm;     // tree position -> caller index
};

// ---------------------------------------------------------------- octree
struct Box {
  int level;
  int64_t ix, iy, iz;            // integer coordinates at this level
  Vec3 center;
  int64_t parent;
  int64_t child[8];
  int64_t begin, end;            // element range (tree order)
  bool leaf;
  int octant;                    // index in parent
};

struct Level {
  double width;
  bool hf;                       // w >= λ (reading C8)
  int nf;                        // face subdivisions per cube face (HF), 0 for LF
  int ndir;                      // 6 nf²  (0 for LF)
  int64_t box_begin, box_end;    // boxes of this level are contiguous
  int rank = 0;                  // retained SVD rank T_l
  // reference-frame clouds (relative to the box centre)
  std::vector<Vec3> eq;          // OUT_EQUIV = cube grid p_eq, side eq_scale*w
  std::vector<Vec3> chk;         // OUT_CHECK: LF cube (chk_scale*w) or HF frustum (+z)
  // truncated SVD of G_up = G(chk, eq) = U Σ V^H
  std::vector<cd> U;             // m × T (column-major: U[c*m + i])
  std::vector<cd> V;             // n × T
  std::vector<double> S;         // T
};

// state = (box, direction); direction -1 = non-directional (LF)
struct State {
  int64_t box;
  int dir;
};

// one translation op: dst += M[mat] * src
struct Op {
  int64_t src, dst;  // global state indices
  int64_t mat;       // matrix id
};

// factored M2L op (§4.2): tmp = V̂ src ; dst += Û tmp
struct LrOp {
  int64_t src, dst;  // global out / in state indices
  int64_t matV, matU;
  int64_t tmp;       // complex offset of this op's r-vector in the tmp buffer
  int level;
};

// leaf-level op of an HF leaf (opt.hf_leaves): one directional state of the leaf
struct LeafOp {
  int64_t leaf;      // leaf index
  int64_t state;     // out-state (S2M) or in-state (L2T) id
  int64_t mat;       // S̃_{B,u} (T × n_B) or T̃_{B,w} (n_B × T)
};

struct MatInfo {
  int64_t offset;    // complex64 elements into the matrix pool
  int32_t rows, cols;
};

enum MatKind { MK_S2M = 0, MK_L2T = 1, MK_M2M = 2, MK_L2L = 3, MK_M2L = 4, MK_S2M_RHS = 5 };

// what a matrix is (geometry it is built from); see operators.cpp
struct MatSpec {
  int kind;
  int level;      // M2M/L2L: parent level; M2L: level; S2M/L2T: leaf level
  int octant;     // M2M/L2L: child octant
  int dir;        // M2M: parent out dir; L2L: parent in dir; M2L: source out dir (-1 LF)
  int64_t leaf;   // S2M/L2T: leaf box id
  int64_t dx, dy, dz;  // M2L: integer offset c_D - c_C (units of w)
};

struct Tree {
  double lambda = 0;
  Vec3 root_center;
  double root_width;
  std::vector<Box> boxes;
  std::vector<Level> levels;
  std::vector<int64_t> leaves;   // box ids of leaves (tree order of elements)
};

struct Plan {
  // states (global numbering, grouped by level)
  std::vector<State> out_states, in_states;
  std::vector<int64_t> out_level_begin, in_level_begin;   // size nlev+1
  std::vector<int64_t> out_offset, in_offset;              // complex offset of each state vector
  int64_t out_size = 0, in_size = 0;                       // total complex entries
  std::vector<int64_t> box_out_lf, box_in_lf;              // LF state of a box or -1
  // per leaf
  std::vector<int64_t> leaf_box;
  std::vector<int64_t> leaf_S, leaf_T;                     // matrix ids (-1 = none)
  std::vector<int64_t> leaf_out, leaf_in;                  // state ids (-1 = none)
  // ops per level (index = level of the destination for m2m/m2l, of source for l2l)
  std::vector<std::vector<Op>> m2m, m2l, l2l;
  // §4.2 factored M2L ops (plan.m2l keeps the dense ones)
  std::vector<LrOp> m2l_lr;
  std::vector<double> m2l_share;     // per level: global M2L ops per distinct K̃ (before sharding)
  int64_t tmp_size = 0;
  std::vector<int64_t> lr_V, lr_U;   // per matrix id: factor ids (-1 = dense)
  int64_t n_m2l_total = 0;
  // sharding (nranks > 1): owned leaves [own_leaf0, own_leaf1), elements [own_e0, own_e1)
  int64_t own_leaf0 = 0, own_leaf1 = 0, own_e0 = 0, own_e1 = 0;
  std::vector<int64_t> rank_e0, rank_e1;   // every rank's element range (tree order)
  // exchange of partial outgoing states between the passes (partition.cpp):
  // per peer rank, the sorted out-state ids this rank sends / receives
  std::vector<std::vector<int64_t>> xsend, xrecv;
  // direct (near) lists: CSR over leaves -> source leaves
  std::vector<int64_t> near_ptr, near_idx;
  // corrections: CSR over elements (tree order); index 1 = RHS operator
  std::vector<int64_t> corr_ptr, corr_col;
  std::vector<cf> corr_val;
  std::vector<int64_t> corr_ptr_rhs, corr_col_rhs;
  std::vector<cf> corr_val_rhs;
  std::vector<int64_t> leaf_S_rhs;   // per leaf: S̃ with G sources (RHS pass), -1 = none
  // HF leaves (opt.hf_leaves): directional S2M / L2T, one op per used wedge
  std::vector<LeafOp> hf_s2m, hf_s2m_rhs, hf_l2t;
  // matrices
  std::vector<MatInfo> mats;
  std::vector<MatSpec> specs;    // parallel to mats
  PoolVec pool;                  // complex64 matrix pool (column-major per matrix), uninitialised until built
};

struct Params {
  double k;
  cd alpha;
  double eps;
  fda_options opt;
  double lambda() const;
};

// geometry.cpp
fda_status build_geometry(const double* V, int64_t nv, const int32_t* F, int64_t nt, Geometry& g,
                          std::string& err);
// octree.cpp
void build_tree(Geometry& g, const Params& p, Tree& t);
void build_lists(const Geometry& g, const Params& p, Tree& t, Plan& plan);
int wedge_of(int64_t dx, int64_t dy, int64_t dz, int nf);
int anti_dir(int dir, int nf);
int child_dir(int dir, int nf);
Vec3 dir_center(int dir, int nf);
Mat3 rotation_to_z(const Vec3& u);
// operators.cpp
struct LowRank {                       // §4.2 factors K̃ ≈ Û V̂ per M2L matrix id (R = -1: dense)
  std::vector<int> R;
  std::vector<std::vector<cd>> U, V;
};
void build_clouds_and_svd(const Params& p, Tree& t, const std::vector<bool>& need);
// plan.mats (offset, rows, cols) + zeroed pool; matrices with needed[id] = 0 get no storage
void operator_layout(const Tree& t, Plan& plan, const std::vector<char>& needed);
Mat3 out_frame(const Level& L, int dir);
Mat3 in_frame(const Level& L, int dir);
Vec3 octant_offset(int o, double wc);
void lowrank_one(const Params& p, int64_t id, int T, const cd* M, LowRank& lr);
// every spec with done[id] == 0 (done empty: all) on the host, then the §4.2 factors appended
void build_operators(const Geometry& g, const Params& p, Tree& t, Plan& plan, const std::vector<char>& done,
                     LowRank& lr);
// build_dev.cu: the same tables computed on the device in fp64 (opt.device >= 0, opt.build_on_device)
fda_status build_operators_device(Context* ctx, std::vector<char>& done, LowRank& lr);
fda_status build_corrections_device(Context* ctx, int kind);
// corrections.cpp: pair search (CSR, tier 0 self / 1 / 2 per entry) and the host evaluation
// rows outside [row0, row1) (other ranks' elements) are left empty
void correction_pairs(const Geometry& g, const Params& p, std::vector<int64_t>& ptr, std::vector<int64_t>& col,
                      std::vector<int8_t>& tier, int64_t row0, int64_t row1);
void build_corrections(const Geometry& g, const Params& p, Plan& plan, int kind = 0);
// partition.cpp
// before the operator tables: own leaves / elements, exchange plan, pruned ops, needed[matrix id]
void apply_partition(const Params& p, const Tree& t, Plan& plan, std::vector<char>& needed);
// quad.cpp (fp64 kernels and rules)
cd lhs_kernel(const Vec3& x, const Vec3& nx, const Vec3& y, const Vec3& ny, double k, cd alpha);
cd rhs_kernel(const Vec3& x, const Vec3& nx, const Vec3& y, double k, cd alpha);
// kind 0: LHS integrand (Eq. 5); kind 1: RHS integrand G + α ∂G/∂n_x (Eq. 4 right side)
cd entry_rule(int tier, const Vec3& x, const Vec3& nx, const Vec3& a, const Vec3& b, const Vec3& c,
              const Vec3& ny, double area, double k, cd alpha, int kind = 0);
cd self_lhs(const Vec3& a, const Vec3& b, const Vec3& c, double k, cd alpha);
cd self_rhs(const Vec3& a, const Vec3& b, const Vec3& c, double k, cd alpha);
cd G(const Vec3& x, const Vec3& y, double k);
cd dGdnx(const Vec3& x, const Vec3& nx, const Vec3& y, double k);
cd dGdny(const Vec3& x, const Vec3& y, const Vec3& ny, double k);
extern const double Q3_BARY[3][3];
// rule tables for the device build: T1 448 × (b0, b1, b2, w), Q6 6 × (b0, b1, b2, w), GL20 20 × (x, w)
void quad_tables(std::vector<double>& t1, std::vector<double>& q6, std::vector<double>& gl);
// linalg.cpp
void svd_jacobi(int m, int n, std::vector<cd>& A /*col-major m×n, overwritten*/, std::vector<double>& S,
                std::vector<cd>& V /*n×n col-major*/);
void zgemm_cm(int m, int n, int kk, const cd* A, int lda, const cd* B, int ldb, cd* C, int ldc,
              bool conjA_T = false);
int lowrank_factor(int m, int n, const cd* A, double eps, std::vector<cd>& Uh, std::vector<cd>& Vh);
int svd_range(int m, int n, const std::vector<cd>& A, double eps, std::vector<double>& S, std::vector<cd>& U,
              std::vector<cd>& V);

// engine.cu (device side)
struct Context;
fda_status engine_create(Context* ctx);
// kind 0: the LHS operator A (fda_matvec); kind 1: the RHS operator B (fda_rhs_apply)
fda_status engine_apply(Context* ctx, const void* x, void* y, int32_t flags, void* stream, int kind);
fda_status engine_rhs_plane_wave(Context* ctx, const double dir[3], void* b, int32_t flags);
fda_status engine_rhs_point_source(Context* ctx, const double src[3], void* b, int32_t flags);
fda_status engine_solve(Context* ctx, const void* rhs, void* u, double tol, int32_t max_iter, int32_t restart,
                        fda_solve_info* info, int32_t flags);
fda_status engine_stage_times(Context* ctx, double* ms, int32_t* n);
fda_status engine_kernel_times(Context* ctx, double* ms, int32_t* n);
fda_status engine_near_time(Context* ctx, double* ms);
fda_status engine_comm_init(Context* ctx, const void* id128);
fda_status engine_read_table(Context* ctx, int which, void* dst, int64_t count);   // 0 pool, 1 / 2 corr_val (LHS / RHS)
fda_status engine_exchange_local(Context** ctxs, int n);
fda_status nccl_unique_id(void* id128, std::string& err);
void engine_destroy(Context* ctx);

struct Context {
  Params p;
  Geometry g;
  Tree t;
  Plan plan;
  std::string err;
  fda_build_info info{};
  void* dev = nullptr;   // engine-owned device state
  int64_t launches_per_matvec = 0;
  void* pool_dev = nullptr;        // device build: the matrix pool already on the device (engine adopts it)
  int64_t pool_dev_cap = 0;        // its capacity (complex entries)
  bool pool_partial = false;       // device build: the host plan.pool lacks the device-built matrices
                                   // (never downloaded; fda_debug_table reads them from the device)
  void* corr_dev[2] = {nullptr, nullptr};   // device build: correction values (LHS, RHS) left on the
  int64_t corr_dev_n[2] = {0, 0};           // device for the engine (plan.corr_val[_rhs] stays empty)
  int64_t kernel_tasks[18] = {};   // CTA tasks per translation kernel family × (M2M, M2L, L2L)
  double kernel_flops[18] = {};    // their algorithmic flops (complex-equivalent, 8·rows·cols per op)
  bool profiling = false;
};

}  // namespace fda

struct fda_ctx : public fda::Context {};
