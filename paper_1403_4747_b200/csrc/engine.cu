// Device engine: uploads the build tables to HBM and runs the FDA matvec
// (PAPER.md Algorithm Steps 2-4) and the GMRES solve (§5,
// P:907-910) on one B200.
//
// Per matvec:
//   main stream : gather → [memset states] → S2M → M2M (leaf level … top)
//                 → M2L (every level) → L2L (top … leaf level) → L2T ─┐
//   near stream :          near field (Q3 direct pairs + corrections) ─┴→ scatter
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <parallel/algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "fda_internal.h"
#include "kernels.cuh"

namespace fda {

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ctx->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call; \
      return FDA_E_CUDA;                                                           \
    }                                                                              \
  } while (0)

// one translation op in offsets: dst[dof : +rows] (+)= M[mat] · src[so : +cols]
struct XOp {
  int64_t so, dof, mat;
};

// ------------------------------------------------------------------ NCCL (loaded on first use)
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};
NcclApi& nccl(std::string& err) {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return api;
    }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
    api.send = (decltype(api.send))dlsym(h, "ncclSend");
    api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.bcast = (decltype(api.bcast))dlsym(h, "ncclBroadcast");
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.errStr && api.send &&
             api.recv && api.groupStart && api.groupEnd && api.bcast;
    if (!api.ok) err = "libnccl.so.2 lacks a required symbol";
  }
  return api;
}
}  // namespace

fda_status nccl_unique_id(void* id128, std::string& err) {
  NcclApi& a = nccl(err);
  if (!a.ok) return FDA_E_NCCL;
  ncclUniqueId id;
  ncclResult_t r = a.getUniqueId(&id);
  if (r != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + a.errStr(r);
    return FDA_E_NCCL;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  std::memcpy(id128, &id, 128);
  return FDA_OK;
}

struct XStage {
  bool atomic = true;
  TcTask* tc[TC_NV] = {};          // tensor-core tasks per kernel variant (opt.tensor_cores)
  int n_tc[TC_NV] = {};
  TcTask* tcw[2] = {};             // warp-specialised persistent kernel, 1 / 2 row tiles (opt.tensor_cores = 4)
  int n_tcw[2] = {}, grid_tcw[2] = {};
  XTask* tasks[XV] = {};
  int ntask[XV] = {};
  int64_t* src = nullptr;
  int64_t* dst = nullptr;
  double fl[3] = {0, 0, 0};        // algorithmic flops (8·rows·cols per op) on k_xlate / k_xlate_tc / k_xlate_tcw
  XbfTask* bf = nullptr;           // BF16x3 persistent kernel (k_xlate_bf): tasks, CTAs, ring plan
  int n_bf = 0, grid_bf = 0;
  LrTcPlan bf_plan;
  double fl_bf = 0;
};

// GMRES workspace (engine_solve; cached per context)
struct Gm {
  float2 *V = nullptr, *w = nullptr, *b = nullptr, *x = nullptr;
  float2* full = nullptr;                         // sharded: one full-length tree-order vector
  double2 *partial = nullptr, *hbuf = nullptr;   // hbuf: [h1 (m+1) | h2 (m+1) | y (m+1)]
  double *np = nullptr, *nrm = nullptr;
  int m = 0;
};

struct Dev {
  int device = 0;
  Gm gm;
  int gm_cap = 0;                   // Krylov vectors the cached workspace holds
  std::vector<void*> gm_allocs;
  int n = 0, nleaf = 0;
  cudaStream_t s_near = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_n0 = nullptr, ev_n1 = nullptr;
  cudaEvent_t ev_l0 = nullptr, ev_l1 = nullptr;   // near kernel of the last matvec, recorded on its stream
  bool live = false;                                // ev_l0/ev_l1 hold a completed-or-pending matvec
  int32_t* perm = nullptr;
  float4 *tgt_pos = nullptr, *tgt_nrm = nullptr;
  SrcElem* src = nullptr;
  float* src_w = nullptr;
  NearTask* near_tasks = nullptr;  // one per owned leaf, by descending near-field work (LPT block order)
  int2* near_slots = nullptr;      // per task: (source element, index into near_off) of every direct source
  bool alpha_pure_imag = false;
  int n_near = 0;                  // near-field CTAs (owned leaves)
  bool near_wide = true;           // near CTA shape: 256 threads / 512 staged sources (else 128 / 256)
  int e0 = 0, e1 = 0;              // owned element range (tree order)
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  // sharded: exchange of partial outgoing states (partition.cpp); per peer the
  // entries (complex) sent / received, packed in state-id order
  float2 *sendb = nullptr, *recvb = nullptr;
  int64_t *xs_idx = nullptr, *xr_idx = nullptr;       // outb position of every packed entry
  int64_t n_send = 0, n_recv = 0;
  std::vector<int64_t> soff, scnt, roff, rcnt;         // per peer, in complex entries
  float4* near_off = nullptr;
  int32_t *corr_ptr = nullptr, *corr_col = nullptr;
  float2* corr_val = nullptr;
  int32_t *corr_ptr_rhs = nullptr, *corr_col_rhs = nullptr;   // RHS operator (kind 1)
  float2* corr_val_rhs = nullptr;
  LeafTask* s2m_rhs = nullptr;
  int n_s2m_rhs = 0;
  float2* pool = nullptr;
  float2 *outb = nullptr, *inb = nullptr;
  int64_t out_size = 0, in_size = 0;
  LeafTask *s2m = nullptr, *l2t = nullptr, *l2t_add = nullptr;
  int n_s2m = 0, n_l2t = 0, n_l2t_add = 0, max_T = 0;
  std::vector<XStage> m2m, l2l;
  // M2L per level (levels are independent of each other; level l needs only
  // the outgoing states of level l): dense ops, §4.2 factored ops with r ≤ 32
  // (fused kernel) and with r > 32 (two stages through tmp)
  struct M2LLevel {
    XStage dense, a, b;
    LrTask* lr_tasks[LR_NCLS] = {};  // fused §4.2 tasks per phase-1 row class (m2l_lr_class)
    int n_lr[LR_NCLS] = {};
    int64_t* lr_src = nullptr;
    int64_t* lr_dst = nullptr;
    LrTcTask* lrtc = nullptr;        // fused §4.2 tasks on the tensor cores (k_m2l_tcw, persistent)
    int n_lrtc = 0;
    int lrtc_grid = 0;
    LrTcPlan lrtc_plan;
    bool lrtc_bf16 = false;          // k_m2l_bf (BF16x3) instead of k_m2l_tcw (3xTF32)
    int64_t split0 = 0, split1 = 0;  // float range of this level's out-states (bf16 split)
    double fl_lr = 0, fl_lrtc = 0;   // algorithmic flops (16·r·T per factored op) on k_m2l_lr / k_m2l_tcw
    bool any() const {
      int n = n_lrtc + dense.n_bf + a.n_bf + b.n_bf;
      for (int c = 0; c < LR_NCLS; ++c) n += n_lr[c];
      for (int v = 0; v < TC_NV; ++v) n += dense.n_tc[v] + a.n_tc[v] + b.n_tc[v];
      for (int q = 0; q < 2; ++q) n += dense.n_tcw[q] + a.n_tcw[q] + b.n_tcw[q];
      for (int v = 0; v < XV; ++v) n += dense.ntask[v] + a.ntask[v] + b.ntask[v];
      return n > 0;
    }
  };
  std::vector<M2LLevel> m2lv;
  static const int kM2LStreams = 6;
  cudaStream_t s_m2l[kM2LStreams] = {};
  std::vector<cudaEvent_t> ev_up;
  std::vector<std::vector<cudaEvent_t>> ev_m2l;   // per level: one event per M2L graph branch
  float2* tmpb = nullptr;
  int64_t tmp_size = 0;
  cudaStream_t s_cap = nullptr;
  cudaGraphExec_t graph_exec[6] = {};   // [kind]: unsharded matvec; [2 + kind] / [4 + kind]: sharded UP / DOWN
  bool use_graph = false;
  float2 *x_tree = nullptr, *y_near = nullptr, *y_far = nullptr;
  double2 *xh = nullptr, *yh = nullptr;
  double *cen = nullptr, *nrm = nullptr;
  KernelParams kp{};
  bool timed = false;
  std::vector<void*> allocs;
  // tensor-core operand pool: per matrix, per 128-row tile, per TC_KC-float K chunk: [hi | lo] A tiles
  bool use_tc = false;
  int64_t tc_size = 0;                           // floats of the tensor-core operand pool
  std::vector<TcLayoutJob> tc_jobs;              // its contents, laid out on the device (k_tc_layout)
  std::unordered_map<int64_t, int64_t> tc_off;   // matrix id → float offset
  std::unordered_map<int64_t, int64_t> tc_boff;  // matrix id → float offset of its k_m2l_tcw B operand
  std::unordered_map<int64_t, int64_t> tc_bfoff; // … of its k_m2l_bf (bf16) B operand
  std::unordered_map<int64_t, int64_t> tc_xbfoff; // … of its k_xlate_bf (bf16) B operand
  float* tcpool = nullptr;
  __nv_bfloat16 *outb_hi = nullptr, *outb_lo = nullptr;   // bf16 hi / lo planes of outb (k_m2l_bf, k_xlate_bf)
  __nv_bfloat16 *inb_hi = nullptr, *inb_lo = nullptr;     // bf16 hi / lo planes of inb (k_xlate_bf L2L)
  bool use_xbf = false;            // dense translations on k_xlate_bf (BF16x3)
  std::vector<char> split_out, split_in;   // per level: split its out- / in-states into bf16 planes on the main stream
  // per-kernel-family device times of a profiled (serialised) matvec: event marks
  // recorded around every launch on the one stream (fda_kernel_times)
  bool kt_on = false;
  std::vector<cudaEvent_t> kt_ev;
  std::vector<int> kt_fam;        // family of the launch that ends at mark i (-1: a start mark)
  int kt_n = 0;
};

// kernel families of fda_kernel_times (include/fda.h)
enum KFam { KF_GATHER = 0, KF_NEAR, KF_S2M, KF_XLATE, KF_XLATE_TC, KF_XLATE_TCW, KF_M2L_LR, KF_M2L_TCW, KF_L2T,
            KF_SCATTER, KF_MEMSET, KF_XLATE_BF, KF_COUNT };

static void kt_mark(Dev* d, cudaStream_t s, int fam) {
  if (!d->kt_on) return;
  if (d->kt_n >= (int)d->kt_ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) { d->kt_on = false; return; }
    d->kt_ev.push_back(e);
    d->kt_fam.push_back(-1);
  }
  d->kt_fam[d->kt_n] = fam;
  cudaEventRecord(d->kt_ev[d->kt_n++], s);
}
#define KT(fam, s, ...)       \
  do {                        \
    kt_mark(d, s, -1);        \
    __VA_ARGS__;              \
    kt_mark(d, s, fam);       \
  } while (0)

template <class T>
static fda_status upload(Context* ctx, Dev* d, T** dst, const T* src, size_t count) {
  *dst = nullptr;
  if (count == 0) count = 1;  // keep valid pointers for empty tables
  CK(cudaMalloc((void**)dst, count * sizeof(T)));
  d->allocs.push_back(*dst);
  if (src) CK(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
  return FDA_OK;
}
template <class T>
static fda_status alloc(Context* ctx, Dev* d, T** dst, size_t count) {
  return upload<T>(ctx, d, dst, nullptr, count);
}

#define UP(...)                                 \
  do {                                          \
    fda_status s_ = upload(ctx, d, __VA_ARGS__); \
    if (s_ != FDA_OK) return s_;                \
  } while (0)
#define AL(...)                                \
  do {                                         \
    fda_status s_ = alloc(ctx, d, __VA_ARGS__); \
    if (s_ != FDA_OK) return s_;               \
  } while (0)

// ---- tensor-core operand layout (kernels_tc.cu): the real 2R × 2C matrix with
// interleaved rows / columns (A[2i][2j] = Re M, A[2i][2j+1] = −Im M, A[2i+1][2j] = Im M,
// A[2i+1][2j+1] = Re M), TF32 hi/lo, per 128-row tile and TC_KC-float K chunk, canonical
// K-major core matrices: element (r, k) of a 128 × TC_KC tile at ((k/4 · 16 + r/8) · 8 + r%8) · 4 + k%4

static int tc_tiles(int rows) { return (2 * rows + 127) / 128; }

// A operand of the tensor-core translation kernels: the real interleaved 2R × 2C form of
// matrix m, TF32 hi / lo, per 128-row tile and TC_KC-float K chunk (layout in
// kernels_tc.cu: k_tc_layout, built on the device from the complex64 pool)
static int64_t tc_matrix(Context* ctx, Dev* d, int64_t m) {
  auto it = d->tc_off.find(m);
  if (it != d->tc_off.end()) return it->second;
  const MatInfo& mi = ctx->plan.mats[m];
  const int ntile = tc_tiles(mi.rows), nkc = (2 * mi.cols + TC_KC - 1) / TC_KC;
  const int64_t off = d->tc_size;
  d->tc_size += (int64_t)ntile * nkc * 2 * 128 * TC_KC;
  d->tc_jobs.push_back(TcLayoutJob{off, mi.offset, mi.rows, mi.cols, ntile, nkc, 0, 0});
  d->tc_off.emplace(m, off);
  return off;
}

// B operand of k_m2l_tcw: the real 2R × 2C form of matrix m as nrp ≥ 2R rows × K = 2C
// (zero-padded to nkc 16-float chunks), per chunk [hi: nrp × 16 | lo: nrp × 16] in the
// canonical K-major no-swizzle layout (core matrices of 8 rows × 16 B)
static int64_t tc_bop(Context* ctx, Dev* d, int64_t m, int nrp, int nkc) {
  auto it = d->tc_boff.find(m);
  if (it != d->tc_boff.end()) return it->second;
  const MatInfo& mi = ctx->plan.mats[m];
  const int64_t off = d->tc_size;
  d->tc_size += (int64_t)nkc * 2 * nrp * TC_KC;
  d->tc_jobs.push_back(TcLayoutJob{off, mi.offset, mi.rows, mi.cols, nrp, nkc, 1, 0});
  d->tc_boff.emplace(m, off);
  return off;
}

// bf16 B operand of k_m2l_bf: as tc_bop with 32-element K chunks of bf16 hi / lo
// (row blocks of rb rows per chunk, rb = 0: one block; k_m2l_bf streams B2 in two N-halves)
static int64_t tc_bop_bf(Context* ctx, Dev* d, int64_t m, int nrp, int nkc32, int rb = 0) {
  auto it = d->tc_bfoff.find(m);
  if (it != d->tc_bfoff.end()) return it->second;
  const MatInfo& mi = ctx->plan.mats[m];
  const int64_t off = d->tc_size;
  d->tc_size += (int64_t)nkc32 * nrp * 32;   // 2 planes × nrp × 32 bf16 = nrp × 32 floats per chunk
  d->tc_jobs.push_back(TcLayoutJob{off, mi.offset, mi.rows, mi.cols, nrp, nkc32, 2, rb});
  d->tc_bfoff.emplace(m, off);
  return off;
}

// bf16 B operand of k_xlate_bf: the real 2R × 2C form of a translation matrix, nrp = 2R padded to 16
static int64_t tc_xbf(Context* ctx, Dev* d, int64_t m, int nrp, int nkc32) {
  auto it = d->tc_xbfoff.find(m);
  if (it != d->tc_xbfoff.end()) return it->second;
  const MatInfo& mi = ctx->plan.mats[m];
  const int64_t off = d->tc_size;
  d->tc_size += (int64_t)nkc32 * nrp * 32;
  d->tc_jobs.push_back(TcLayoutJob{off, mi.offset, mi.rows, mi.cols, nrp, nkc32, 2, 0});
  d->tc_xbfoff.emplace(m, off);
  return off;
}

// Group the ops of one stage (one level, or all M2L levels at once) by matrix
// and cut each group into tiles of the kernel variant (rows × ops per CTA)
// that pads the group least.  Stages with fewer CTAs than ~4 waves are split
// along K (cols) so that small, latency-bound stages still fill the GPU.
static fda_status build_xstage(Context* ctx, Dev* d, const std::vector<XOp>& ops, bool atomic, XStage& st,
                               bool tc_ok = true, bool force_tc = false, bool bf_ok = false) {

  const Plan& p = ctx->plan;
  st.atomic = atomic;
  if (ops.empty()) return FDA_OK;
  // BF16x3 persistent kernel (k_xlate_bf, d->use_xbf): ≤ 128 ops per task, every matrix R ≤ 128
  // (N = 2R ≤ 256); stages with taller matrices keep the 3xTF32 / CUDA-core kernels
  bool use_bf = false;
  if (bf_ok && d->use_xbf && atomic) {
    // every eligible stage (A/B at config 4: routing only stages with ≥ 64 / 256 / 1000 ops per
    // matrix to k_xlate_bf, the rest to k_xlate / k_xlate_tc, is slower: 4.985-5.010 vs 4.920 ms)
    bool fits = true;
    for (const XOp& o : ops) fits &= p.mats[o.mat].rows <= 128;
    use_bf = fits;
  }
  std::vector<size_t> ord(ops.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
  // Locality order for k_xlate_bf on large stages whose matrices are each shared by many ops:
  // ops sorted by (block of destination offsets, matrix, destination) instead of (matrix,
  // destination), so that the tasks running at any time touch one block of destination states
  // and the sources they read instead of streaming the level's states once per matrix (config 5
  // M2M L7 in matrix order: 7.0 GB of DRAM traffic per launch, ncu).  A block holds ≈ 2·128 ops
  // per matrix on average (A/B, config 5: k_xlate_bf 23.6 → 22.5 ms; 1·128: 24.9 ms; the
  // non-persistent k_xlate_tc is slower in this order, 24.7 → 28.2 ms, and keeps matrix order).
  bool blocked = false;
  {
    const double mult = 2.0;
    if (use_bf && ops.size() >= 200000) {
      std::vector<int64_t> mv;
      mv.reserve(ops.size());
      int64_t dmin = ops[0].dof, dmax = ops[0].dof;
      for (const XOp& o : ops) {
        mv.push_back(o.mat);
        dmin = std::min(dmin, o.dof);
        dmax = std::max(dmax, o.dof);
      }
      __gnu_parallel::sort(mv.begin(), mv.end());
      const double nm = (double)(std::unique(mv.begin(), mv.end()) - mv.begin());
      if ((double)ops.size() / nm >= 256) {
        blocked = true;
        const int64_t bspan =
            std::max<int64_t>(1, (int64_t)(mult * 128.0 * (double)(dmax - dmin + 1) * nm / (double)ops.size()));
        __gnu_parallel::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
          const int64_t ba = (ops[a].dof - dmin) / bspan, bb = (ops[b].dof - dmin) / bspan;
          if (ba != bb) return ba < bb;
          return ops[a].mat != ops[b].mat ? ops[a].mat < ops[b].mat : ops[a].dof < ops[b].dof;
        });
      }
    }
  }
  if (!blocked)
    __gnu_parallel::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
      return ops[a].mat != ops[b].mat ? ops[a].mat < ops[b].mat : ops[a].dof < ops[b].dof;
    });
  std::vector<int64_t> so, dof;
  if (use_bf) {
    {
      std::vector<XbfTask> bt;
      int nmax = 16;
      for (size_t i = 0; i < ord.size();) {
        const int64_t m = ops[ord[i]].mat;
        size_t j = i;
        while (j < ord.size() && ops[ord[j]].mat == m) ++j;
        const int R = p.mats[m].rows, C = p.mats[m].cols;
        const int n = ((2 * R + 15) / 16) * 16, nk = (2 * C + 31) / 32;
        nmax = std::max(nmax, n);
        const int64_t off = tc_xbf(ctx, d, m, n, nk);
        const int32_t base = (int32_t)so.size();
        for (size_t q = i; q < j; ++q) {
          so.push_back(ops[ord[q]].so);
          dof.push_back(ops[ord[q]].dof);
        }
        const int64_t nops = (int64_t)(j - i);
        for (int64_t c0 = 0; c0 < nops; c0 += 128) {
          XbfTask t;
          t.b_off = off;
          t.R = R;
          t.C = C;
          t.n = n;
          t.nk = nk;
          t.op_begin = base + (int32_t)c0;
          t.op_count = (int32_t)std::min<int64_t>(128, nops - c0);
          bt.push_back(t);
          st.fl_bf += 8.0 * R * C * t.op_count;
        }
        i = j;
      }
      // longest tasks first (the persistent CTAs stride over them), unless in locality order
      if (!blocked)
        std::stable_sort(bt.begin(), bt.end(), [](const XbfTask& x, const XbfTask& y) {
        return (int64_t)x.nk * x.n * x.op_count > (int64_t)y.nk * y.n * y.op_count;
      });
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      st.n_bf = (int)bt.size();
      st.grid_bf = std::min(st.n_bf, nsm);
      st.bf_plan = xlate_bf_plan(nmax);
      UP(&st.bf, bt.data(), bt.size());
      UP(&st.src, so.data(), so.size());
      UP(&st.dst, dof.data(), dof.size());
      return FDA_OK;
    }
  }
  std::vector<XTask> tasks[XV];
  bool tc = d->use_tc && atomic && tc_ok;
  if (tc && ctx->p.opt.tensor_cores == 2 && !force_tc) {   // auto: large, well-shared stages only
    double flops = 0;
    std::unordered_map<int64_t, int> nm;
    for (const XOp& o : ops) {
      flops += 8.0 * p.mats[o.mat].rows * p.mats[o.mat].cols;
      nm[o.mat] = 1;
    }
    // ≥ 0.1 GFLOP per stage (round 1: 1 GFLOP): the LF levels' M2M / L2L (8 octant matrices shared
    // by 10⁴ ops) then run on tcgen05 — A/B config 4 5.134 → 5.020 ms, config 3 1.562 → 1.535,
    // config 2 0.424 → 0.428 (profiles/r02_ab_tc_threshold.jsonl)
    tc = flops >= 0.1e9 && (double)ops.size() >= 64.0 * (double)nm.size();
  }
  if (tc) {
    std::vector<TcTask> tct[TC_NV];
    for (size_t i = 0; i < ord.size();) {
      const int64_t m = ops[ord[i]].mat;
      size_t j = i;
      while (j < ord.size() && ops[ord[j]].mat == m) ++j;
      const int R = p.mats[m].rows, C = p.mats[m].cols, ntile = tc_tiles(R);
      if (ntile > 3) { ctx->err = "matrix too tall for the tensor-core path (rows > 192)"; return FDA_E_INTERNAL; }
      const int64_t nops = (int64_t)(j - i);
      // 2-stage variants with several CTAs per SM (default; measured faster on configs 3-5 than the
      // 3-stage one-CTA-per-SM variants, which opt.tensor_cores = 3 selects for A/B runs)
      const bool multi = ctx->p.opt.tensor_cores != 3;
      const int v = tc_variant(!multi && nops >= 160 && ntile <= 2 ? 256 : 128, ntile, multi), nmax = tc_variant_ops(v);
      const int64_t off = tc_matrix(ctx, d, m);
      const int32_t base = (int32_t)so.size();
      for (size_t q = i; q < j; ++q) {
        so.push_back(ops[ord[q]].so);
        dof.push_back(ops[ord[q]].dof);
      }
      for (int64_t c0 = 0; c0 < nops; c0 += nmax) {
        TcTask t;
        t.a_off = off;
        t.R = R;
        t.C = C;
        t.nkc = (2 * C + TC_KC - 1) / TC_KC;
        t.ntile = ntile;
        t.op_begin = base + (int32_t)c0;
        t.op_count = (int32_t)std::min<int64_t>(nmax, nops - c0);
        t.kc0 = 0;
        t.kc1 = t.nkc;
        tct[v].push_back(t);
      }
      i = j;
    }
    // split-K for stages with fewer tasks than ~2 waves (one CTA per SM): ≥ 3 chunks per part
    int64_t total = 0;
    for (int v = 0; v < TC_NV; ++v) total += (int64_t)tct[v].size();
    const int64_t target = 2 * 148;
    if (total > 0 && total < target)
      for (int v = 0; v < TC_NV; ++v) {
        std::vector<TcTask> out;
        for (const TcTask& t : tct[v]) {
          const int parts = (int)std::max<int64_t>(1, std::min<int64_t>((target + total - 1) / total, t.nkc / 3));
          const int per = (t.nkc + parts - 1) / parts;
          for (int c = 0; c < t.nkc; c += per) {
            TcTask u = t;
            u.kc0 = c;
            u.kc1 = std::min(t.nkc, c + per);
            out.push_back(u);
          }
        }
        tct[v].swap(out);
      }
    auto tfl = [](const TcTask& t) { return 8.0 * t.R * t.C * t.op_count * (double)(t.kc1 - t.kc0) / t.nkc; };
    if (ctx->p.opt.tensor_cores == 4) {   // N = 128, ≤ 2 tiles → the warp-specialised persistent kernel
      std::vector<TcTask> w[2];
      for (int v = 0; v < TC_NV; ++v) {
        if (tc_variant_ops(v) != 128) continue;
        std::vector<TcTask> keep;
        for (const TcTask& t : tct[v]) (t.ntile <= 2 ? w[t.ntile - 1] : keep).push_back(t);
        tct[v].swap(keep);
      }
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      for (int q = 0; q < 2; ++q) {
        std::stable_sort(w[q].begin(), w[q].end(),
                         [](const TcTask& x, const TcTask& y) { return x.kc1 - x.kc0 > y.kc1 - y.kc0; });
        st.n_tcw[q] = (int)w[q].size();
        st.grid_tcw[q] = std::min<int>(st.n_tcw[q], nsm);
        for (const TcTask& t : w[q]) st.fl[2] += tfl(t);
        if (st.n_tcw[q]) UP(&st.tcw[q], w[q].data(), w[q].size());
      }
    }
    for (int v = 0; v < TC_NV; ++v) {
      st.n_tc[v] = (int)tct[v].size();
      for (const TcTask& t : tct[v]) st.fl[1] += tfl(t);
      if (st.n_tc[v]) UP(&st.tc[v], tct[v].data(), tct[v].size());
    }
    UP(&st.src, so.data(), so.size());
    UP(&st.dst, dof.data(), dof.size());
    return FDA_OK;
  }
  size_t i = 0;
  while (i < ord.size()) {
    const int64_t m = ops[ord[i]].mat;
    size_t j = i;
    while (j < ord.size() && ops[ord[j]].mat == m) ++j;
    const int rows = p.mats[m].rows, cols = p.mats[m].cols;
    const int64_t nops = (int64_t)(j - i);
    int best = 1;
    int64_t best_cost = -1;
    for (int v = 0; v < XV; ++v) {
      const int64_t R = xvar_rows(v), O = xvar_ops(v);
      const int64_t cost = ((rows + R - 1) / R) * R * ((nops + O - 1) / O) * O;
      if (best_cost < 0 || cost < best_cost) { best = v; best_cost = cost; }
    }
    const int R = xvar_rows(best), O = xvar_ops(best);
    const int32_t base = (int32_t)so.size();
    for (size_t q = i; q < j; ++q) {
      so.push_back(ops[ord[q]].so);
      dof.push_back(ops[ord[q]].dof);
    }
    for (int64_t c0 = 0; c0 < nops; c0 += O)
      for (int r0 = 0; r0 < rows; r0 += R) {
        XTask t;
        t.mat_off = p.mats[m].offset;
        t.rows = rows;
        t.cols = cols;
        t.row0 = r0;
        t.op_begin = base + (int32_t)c0;
        t.op_count = (int32_t)std::min<int64_t>(O, nops - c0);
        t.k_begin = 0;
        t.k_end = cols;
        t.pad = 0;
        tasks[best].push_back(t);
      }
    i = j;
  }
  int64_t total = 0;
  for (int v = 0; v < XV; ++v) total += (int64_t)tasks[v].size();
  const int64_t target = 4 * 148 * 4;  // ≈ 4 waves of 4 resident CTAs per SM
  if (atomic && total < target) {
    const int64_t split = (target + total - 1) / total;
    for (int v = 0; v < XV; ++v) {
      std::vector<XTask> out;
      for (const XTask& t : tasks[v]) {
        const int nk = (t.cols + XK - 1) / XK;
        const int sp = (int)std::min<int64_t>(split, nk);
        const int per = (nk + sp - 1) / sp;
        for (int c = 0; c < nk; c += per) {
          XTask u = t;
          u.k_begin = c * XK;
          u.k_end = std::min(t.cols, (c + per) * XK);
          out.push_back(u);
        }
      }
      tasks[v].swap(out);
    }
  }
  for (int v = 0; v < XV; ++v) {
    st.ntask[v] = (int)tasks[v].size();
    for (const XTask& t : tasks[v]) st.fl[0] += 8.0 * std::min(xvar_rows(v), t.rows - t.row0) * (t.k_end - t.k_begin) * t.op_count;
    if (st.ntask[v]) UP(&st.tasks[v], tasks[v].data(), tasks[v].size());
  }
  UP(&st.src, so.data(), so.size());
  UP(&st.dst, dof.data(), dof.size());
  return FDA_OK;
}

// one translation stage: its tensor-core tasks read the context's own operand pool (d->tcpool)
static void launch_stage(Dev* d, const XStage& st, const float2* src, float2* dst, cudaStream_t s,
                         const __nv_bfloat16* shi = nullptr, const __nv_bfloat16* slo = nullptr) {
  const float2* pool = d->pool;
  const float* tcpool = d->tcpool;
  if (st.n_bf)
    KT(KF_XLATE_BF, s, launch_xlate_bf(st.n_bf, st.bf, st.src, st.dst, tcpool, shi, slo, dst, st.bf_plan, st.grid_bf, s));
  for (int q = 0; q < 2; ++q)
    if (st.n_tcw[q])
      KT(KF_XLATE_TCW, s, launch_xlate_tcw(q + 1, st.n_tcw[q], st.tcw[q], st.src, st.dst, tcpool, src, dst, st.grid_tcw[q], s));
  for (int v = 0; v < TC_NV; ++v)
    if (st.n_tc[v]) KT(KF_XLATE_TC, s, launch_xlate_tc(v, st.n_tc[v], st.tc[v], st.src, st.dst, tcpool, src, dst, s));
  for (int v = 0; v < XV; ++v)
    if (st.ntask[v])
      KT(KF_XLATE, s, launch_xlate(v, st.atomic, st.ntask[v], st.tasks[v], st.src, st.dst, pool, src, dst, s));
}

fda_status engine_create(Context* ctx) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    ctx->err = "no CUDA device available (the FDA matvec runs only on the GPU; use opt.device = -1 for a host-only build)";
    return FDA_E_CUDA;
  }
  if (ctx->p.opt.device >= ndev) { ctx->err = "opt.device out of range"; return FDA_E_INVALID_ARG; }
  Dev* d = new Dev();
  ctx->dev = d;
  d->device = ctx->p.opt.device;
  CK(cudaSetDevice(d->device));
  auto tp = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    auto now = std::chrono::steady_clock::now();
    if (ctx->p.opt.verbose)
      fprintf(stderr, "[engine_create] %-14s %8.3f s\n", name, std::chrono::duration<double>(now - tp).count());
    tp = now;
  };
  const Geometry& g = ctx->g;
  const Tree& t = ctx->t;
  const Plan& p = ctx->plan;
  const int n = (int)g.n;
  const int nleaf = (int)t.leaves.size();
  d->n = n;
  d->nleaf = nleaf;
  d->kp.k = (float)ctx->p.k;
  d->kp.alpha_re = (float)ctx->p.alpha.real();
  d->kp.alpha_im = (float)ctx->p.alpha.imag();
  d->kp.ak_re = (float)(ctx->p.k * ctx->p.alpha.real());
  d->kp.ak_im = (float)(ctx->p.k * ctx->p.alpha.imag());
  d->kp.inv_k = (float)(1.0 / ctx->p.k);
  d->kp.skip_corr = getenv("FDA_NEAR_NOCORR") && atoi(getenv("FDA_NEAR_NOCORR")) != 0;
  d->use_tc = ctx->p.opt.tensor_cores != 0;
  // opt.tensor_cores = 5: dense translations on the BF16x3 persistent kernel (unsharded contexts)
  // k_xlate_bf for the dense translations: opt.tensor_cores = 5 always; auto mode (2) on problems
  // with ≥ 10 GFLOP of dense translations per matvec (A/B, one B200: config 4 (17 GFLOP) 4.99 →
  // 4.92 ms, config 5 (2.2 TFLOP) 60.0 → 57 ms; configs 2 (1.1) and 3 (6.4) are faster on the
  // CUDA-core / 3xTF32 kernels, whose smaller CTAs fill the short levels better)
  {
    double xf = 0;
    for (const auto* lv : {&ctx->plan.m2m, &ctx->plan.l2l, &ctx->plan.m2l})
      for (const auto& ops : *lv)
        for (const Op& o : ops) xf += 8.0 * ctx->plan.mats[o.mat].rows * ctx->plan.mats[o.mat].cols;
    d->use_xbf = ctx->p.opt.nranks <= 1 &&
                 (ctx->p.opt.tensor_cores == 5 || (ctx->p.opt.tensor_cores == 2 && ctx->p.opt.m2l_bf16 != 0 && xf >= 10e9));
  }
  if (d->use_xbf) CK(xlate_bf_prepare());
  if (d->use_tc) CK(tc_prepare());

  if (d->use_tc) CK(xlate_tcw_prepare());
  if (d->use_tc) CK(m2l_tcw_prepare());
  if (d->use_tc) CK(m2l_bf_prepare());
  CK(m2l_lr_prepare());

  // leaf-local element data in wave units (fp32 k·(offset from the owning leaf
  // centre), computed in fp64); the near kernel's weight carries k² (kernels.cu)
  const double kw = ctx->p.k;
  std::vector<float4> tpos(n), tnrm(n);
  std::vector<SrcElem> src(n);
  std::vector<float> w(n);
  std::vector<int32_t> perm(n);
  std::vector<double> cen(3 * (size_t)n), nrm(3 * (size_t)n);
  const double inv12pi = 1.0 / (12.0 * M_PI);  // Q3 weight 1/3 and 1/(4π)
  for (int i = 0; i < nleaf; ++i) {
    const Box& B = t.boxes[t.leaves[i]];
    if (B.end - B.begin > 128) { ctx->err = "leaf with more than 128 elements (depth cap hit)"; return FDA_E_INTERNAL; }
    for (int64_t e = B.begin; e < B.end; ++e) {
      Vec3 x = (g.centroid[e] - B.center) * kw;
      tpos[e] = make_float4((float)x.x, (float)x.y, (float)x.z, 0.f);
      tnrm[e] = make_float4((float)g.normal[e].x, (float)g.normal[e].y, (float)g.normal[e].z, 0.f);
      Vec3 q[3];
      for (int k = 0; k < 3; ++k)
        q[k] = (g.v0[e] * Q3_BARY[k][0] + g.v1[e] * Q3_BARY[k][1] + g.v2[e] * Q3_BARY[k][2] - B.center) * kw;
      src[e].a = make_float4((float)q[0].x, (float)q[0].y, (float)q[0].z, (float)g.normal[e].x);
      src[e].b = make_float4((float)q[1].x, (float)q[1].y, (float)q[1].z, (float)g.normal[e].y);
      src[e].c = make_float4((float)q[2].x, (float)q[2].y, (float)q[2].z, (float)g.normal[e].z);
      w[e] = (float)(g.area[e] * inv12pi * kw * kw);
    }
  }
  for (int i = 0; i < n; ++i) {
    perm[i] = (int32_t)g.perm[i];
    cen[3 * i] = g.centroid[i].x; cen[3 * i + 1] = g.centroid[i].y; cen[3 * i + 2] = g.centroid[i].z;
    nrm[3 * i] = g.normal[i].x; nrm[3 * i + 1] = g.normal[i].y; nrm[3 * i + 2] = g.normal[i].z;
  }
  std::vector<float4> noff(p.near_idx.size());
  for (int i = 0; i < nleaf; ++i) {
    const Box& B = t.boxes[t.leaves[i]];
    for (int64_t e = p.near_ptr[i]; e < p.near_ptr[i + 1]; ++e) {
      const Box& C = t.boxes[t.leaves[p.near_idx[e]]];
      Vec3 o = (B.center - C.center) * kw;
      noff[e] = make_float4((float)o.x, (float)o.y, (float)o.z, 0.f);
    }
  }
  if (p.corr_col.size() >= (size_t)INT32_MAX || p.near_idx.size() >= (size_t)INT32_MAX) {
    ctx->err = "table too large for 32-bit indices";
    return FDA_E_INTERNAL;
  }
  std::vector<int32_t> cptr(p.corr_ptr.size()), ccol(p.corr_col.size());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)cptr.size(); ++i) cptr[i] = (int32_t)p.corr_ptr[i];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)ccol.size(); ++i) ccol[i] = (int32_t)p.corr_col[i];
  // LPT order of the near-field CTAs: estimated work = targets × (3·sources + corrections)
  std::vector<int64_t> work(nleaf, 0), nsrc(nleaf, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nleaf; ++i) {
    const Box& B = t.boxes[t.leaves[i]];
    for (int64_t e = p.near_ptr[i]; e < p.near_ptr[i + 1]; ++e) {
      const Box& C = t.boxes[t.leaves[p.near_idx[e]]];
      nsrc[i] += C.end - C.begin;
    }
    work[i] = (B.end - B.begin) * 3 * nsrc[i] + (p.corr_ptr[B.end] - p.corr_ptr[B.begin]);
  }
  std::vector<int32_t> order;
  for (int i = 0; i < nleaf; ++i)   // sharded: this rank evaluates the near field of its own leaves only
    if (i >= p.own_leaf0 && i < p.own_leaf1) order.push_back(i);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
  // slot table: per task (LPT order) the source elements of all its direct leaves (prefix sums,
  // then filled in parallel)
  std::vector<NearTask> ntask(order.size());
  std::vector<int64_t> sbeg(order.size() + 1, 0);
  for (size_t q = 0; q < order.size(); ++q) sbeg[q + 1] = sbeg[q] + nsrc[order[q]];
  if (sbeg.back() >= (int64_t)INT32_MAX) { ctx->err = "near-field slot table too large"; return FDA_E_INTERNAL; }
  std::vector<int2> slots((size_t)sbeg.back());
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < (int64_t)order.size(); ++q) {
    const int32_t i = order[q];
    const Box& B = t.boxes[t.leaves[i]];
    int64_t o = sbeg[q];
    for (int64_t e = p.near_ptr[i]; e < p.near_ptr[i + 1]; ++e) {
      const Box& C = t.boxes[t.leaves[p.near_idx[e]]];
      for (int64_t el = C.begin; el < C.end; ++el) slots[o++] = make_int2((int)el, (int)e);
    }
    ntask[q] = NearTask{(int32_t)B.begin, (int32_t)(B.end - B.begin), (int32_t)sbeg[q], (int32_t)sbeg[q + 1]};
  }
  d->n_near = (int)order.size();
  // 256-thread near CTAs pay when a target leaf sees many direct sources (kernels.cu)
  d->near_wide = d->n_near > 0 && (double)slots.size() >= 400.0 * (double)d->n_near;
  d->e0 = (int)p.own_e0;
  d->e1 = (int)p.own_e1;
  d->nranks = ctx->p.opt.nranks;
  d->alpha_pure_imag = ctx->p.alpha.real() == 0.0;

  UP(&d->perm, perm.data(), perm.size());
  UP(&d->tgt_pos, tpos.data(), tpos.size());
  UP(&d->tgt_nrm, tnrm.data(), tnrm.size());
  UP(&d->src, src.data(), src.size());
  UP(&d->src_w, w.data(), w.size());
  UP(&d->near_tasks, ntask.data(), ntask.size());
  UP(&d->near_slots, slots.data(), slots.size());
  UP(&d->near_off, noff.data(), noff.size());
  UP(&d->corr_ptr, cptr.data(), cptr.size());
  UP(&d->corr_col, ccol.data(), ccol.size());
  if (ctx->corr_dev[0]) {   // device build: adopt the correction values it left on the device
    d->corr_val = static_cast<float2*>(ctx->corr_dev[0]);
    d->allocs.push_back(d->corr_val);
    ctx->corr_dev[0] = nullptr;
  } else {
    UP(&d->corr_val, reinterpret_cast<const float2*>(p.corr_val.data()), p.corr_val.size());
  }
  if (ctx->p.opt.rhs_operator) {
    if (p.corr_col_rhs.size() >= (size_t)INT32_MAX) { ctx->err = "RHS table too large"; return FDA_E_INTERNAL; }
    std::vector<int32_t> rp(p.corr_ptr_rhs.begin(), p.corr_ptr_rhs.end()),
        rc(p.corr_col_rhs.begin(), p.corr_col_rhs.end());
    UP(&d->corr_ptr_rhs, rp.data(), rp.size());
    UP(&d->corr_col_rhs, rc.data(), rc.size());
    if (ctx->corr_dev[1]) {
      d->corr_val_rhs = static_cast<float2*>(ctx->corr_dev[1]);
      d->allocs.push_back(d->corr_val_rhs);
      ctx->corr_dev[1] = nullptr;
    } else {
      UP(&d->corr_val_rhs, reinterpret_cast<const float2*>(p.corr_val_rhs.data()), p.corr_val_rhs.size());
    }
  }
  if (ctx->pool_dev) {   // device build: adopt the pool it left on the device
    d->pool = static_cast<float2*>(ctx->pool_dev);
    d->allocs.push_back(d->pool);
    ctx->pool_dev = nullptr;
  } else {
    UP(&d->pool, reinterpret_cast<const float2*>(p.pool.data()), p.pool.size());
  }
  UP(&d->cen, cen.data(), cen.size());
  UP(&d->nrm, nrm.data(), nrm.size());
  d->out_size = p.out_size;
  d->in_size = p.in_size;
  AL(&d->outb, (size_t)p.out_size);
  AL(&d->inb, (size_t)p.in_size);
  AL(&d->x_tree, (size_t)n);
  AL(&d->y_near, (size_t)n);
  AL(&d->y_far, (size_t)n);
  AL(&d->xh, (size_t)n);
  AL(&d->yh, (size_t)n);

  // leaf tasks
  std::vector<LeafTask> s2m, l2t, s2m_rhs;
  for (int i = 0; i < nleaf; ++i) {
    const Box& B = t.boxes[t.leaves[i]];
    const int T = t.levels[B.level].rank;
    if (p.leaf_S[i] >= 0) {
      LeafTask lt{p.mats[p.leaf_S[i]].offset, p.out_offset[p.leaf_out[i]], (int32_t)B.begin,
                  (int32_t)(B.end - B.begin), T, 0};
      s2m.push_back(lt);
      d->max_T = std::max(d->max_T, T);
      if (T > 320) { ctx->err = "rank above 320"; return FDA_E_INTERNAL; }
      if (ctx->p.opt.rhs_operator && p.leaf_S_rhs[i] >= 0) {
        LeafTask lr = lt;
        lr.mat_off = p.mats[p.leaf_S_rhs[i]].offset;
        s2m_rhs.push_back(lr);
      }
    }
    LeafTask lt{-1, 0, (int32_t)B.begin, (int32_t)(B.end - B.begin), 0, 0};
    if (p.leaf_T[i] >= 0) {
      lt.mat_off = p.mats[p.leaf_T[i]].offset;
      lt.state_off = p.in_offset[p.leaf_in[i]];
      lt.T = T;
      if (T > 320) { ctx->err = "rank above 320"; return FDA_E_INTERNAL; }
    }
    l2t.push_back(lt);
  }
  // HF leaves (opt.hf_leaves): one task per directional state; their L2T tasks accumulate
  std::vector<LeafTask> l2t_add;
  auto leaf_task = [&](const LeafOp& o, bool in) {
    const Box& B = t.boxes[t.leaves[o.leaf]];
    const int T = t.levels[B.level].rank;
    return LeafTask{p.mats[o.mat].offset, in ? p.in_offset[o.state] : p.out_offset[o.state], (int32_t)B.begin,
                    (int32_t)(B.end - B.begin), T, 0};
  };
  for (const LeafOp& o : p.hf_s2m) {
    s2m.push_back(leaf_task(o, false));
    d->max_T = std::max(d->max_T, s2m.back().T);
  }
  for (const LeafOp& o : p.hf_s2m_rhs) s2m_rhs.push_back(leaf_task(o, false));
  for (const LeafOp& o : p.hf_l2t) l2t_add.push_back(leaf_task(o, true));
  for (const LeafTask& lt : s2m)
    if (lt.T > 320) { ctx->err = "rank above 320"; return FDA_E_INTERNAL; }
  d->n_l2t_add = (int)l2t_add.size();
  if (d->n_l2t_add) UP(&d->l2t_add, l2t_add.data(), l2t_add.size());
  d->n_s2m = (int)s2m.size();
  d->n_l2t = (int)l2t.size();
  UP(&d->s2m, s2m.data(), s2m.size());
  d->n_s2m_rhs = (int)s2m_rhs.size();
  UP(&d->s2m_rhs, s2m_rhs.data(), s2m_rhs.size());
  UP(&d->l2t, l2t.data(), l2t.size());

  phase("leaf tables");
  const int nlev = (int)t.levels.size();
  d->m2m.resize(nlev); d->l2l.resize(nlev);
  auto xops = [&](const std::vector<Op>& ops, const std::vector<int64_t>& so, const std::vector<int64_t>& dof,
                  bool src_in) {
    std::vector<XOp> v;
    v.reserve(ops.size());
    for (const Op& o : ops) {
      (void)src_in;
      v.push_back(XOp{so[o.src], dof[o.dst], o.mat});
    }
    return v;
  };
  d->m2lv.resize(nlev);
  for (int l = 0; l < nlev; ++l) {
    fda_status s;
    if ((s = build_xstage(ctx, d, xops(p.m2m[l], p.out_offset, p.out_offset, false), true, d->m2m[l], true, false,
                          true)) != FDA_OK)
      return s;
    if ((s = build_xstage(ctx, d, xops(p.l2l[l], p.in_offset, p.in_offset, true), true, d->l2l[l], true, false,
                          true)) != FDA_OK)
      return s;
    if ((s = build_xstage(ctx, d, xops(p.m2l[l], p.out_offset, p.in_offset, false), true, d->m2lv[l].dense, true,
                          false, true)) != FDA_OK)
      return s;
  }
  {
    // §4.2 factored ops: r ≤ 64 → fused kernel; r > 64 → tmp = V̂ src (atomic into a zeroed tmp
    // region, so small stages can be split along K) then in += Û tmp
    // With opt.tensor_cores = 1 the factored ops go to the two stages instead, on the
    // tensor cores (V̂ then Û); the auto mode keeps the fused CUDA-core kernel, which is
    // faster for these thin factors (config 5: 37 ms vs 49 ms).
    std::vector<std::vector<XOp>> a(nlev), b(nlev);
    std::vector<std::vector<LrOp>> fused(nlev);
    std::vector<char> lr_tc(nlev, 0);
    if (d->use_tc) {
      std::vector<double> fl(nlev, 0.0);
      std::vector<int64_t> nops(nlev, 0);
      std::vector<std::unordered_map<int64_t, int>> nm(nlev);
      for (const LrOp& o : p.m2l_lr) {
        fl[o.level] += 16.0 * p.mats[o.matV].rows * p.mats[o.matV].cols;
        ++nops[o.level];
        nm[o.level][o.matV] = 1;
      }
      for (int l = 0; l < nlev; ++l)
        lr_tc[l] = nops[l] > 0 && ctx->p.opt.tensor_cores == 1;   // auto: the fused CUDA-core kernel
                                                                   // measured faster (config 3/5)
    }
    // fused tensor-core kernel (opt.lr_tensor_cores): per level, the ops with r ≤ 32, T ≤ LRTC_MAX_T.
    // Auto (2): levels with ≥ 64 ops per factored K̃ and ≥ 3 GFLOP of factored work — the
    // persistent kernel owns every SM while it runs, which pays on large levels (config 5:
    // M2L 32.0 vs 35.0 ms; config 3: matvec 1.735 vs 1.767 ms) but not on small ones that
    // share the GPU with the near field inside the graph (config 2, largest level 1.6 GFLOP:
    // matvec 0.473 vs 0.471 ms at a 1.5 GFLOP threshold)
    std::vector<char> lr_f(nlev, 0);
    const int lrtc_max_r = ctx->p.opt.m2l_bf16 != 0 ? LRBF_MAX_R : LRTC_MAX_R;
    if (d->use_tc && ctx->p.opt.lr_tensor_cores != 0) {
      std::vector<int64_t> nops(nlev, 0);
      std::vector<double> fl(nlev, 0.0);
      std::vector<std::unordered_map<int64_t, int>> nm(nlev);
      for (const LrOp& o : p.m2l_lr) {
        if (p.mats[o.matV].rows > lrtc_max_r || p.mats[o.matV].cols > LRTC_MAX_T) continue;
        ++nops[o.level];
        fl[o.level] += 16.0 * p.mats[o.matV].rows * p.mats[o.matV].cols;
        nm[o.level][o.matV] = 1;
      }
      // auto (2): BF16x3 (default) on every eligible level — measured faster than the fused
      // CUDA-core kernel on configs 2 / 3 / 4 (matvec 0.475 → 0.427, 1.634 → 1.549,
      // 5.116 → 5.047 ms, profiles/r02_ab_routing.jsonl); 3xTF32 only on levels with ≥ 64 ops
      // per factored K̃ and ≥ 3 GFLOP (round 1)
      const bool bf = ctx->p.opt.m2l_bf16 != 0;
      for (int l = 0; l < nlev; ++l)
        lr_f[l] = nops[l] > 0 && !lr_tc[l] &&
                  (ctx->p.opt.lr_tensor_cores == 1 || bf ||
                   ((double)nops[l] >= 64.0 * (double)nm[l].size() && fl[l] >= 3e9));
    }
    std::vector<std::vector<LrOp>> ftc(nlev);
    int64_t tmp_off = 0;
    for (const LrOp& o : p.m2l_lr) {
      if (lr_f[o.level] && p.mats[o.matV].rows <= lrtc_max_r && p.mats[o.matV].cols <= LRTC_MAX_T) {
        ftc[o.level].push_back(o);
        continue;
      }
      if (p.mats[o.matV].rows <= LR_MAX_R && !lr_tc[o.level]) {
        fused[o.level].push_back(o);
        continue;
      }
      a[o.level].push_back(XOp{p.out_offset[o.src], tmp_off, o.matV});
      b[o.level].push_back({tmp_off, p.in_offset[o.dst], o.matU});
      tmp_off += (p.mats[o.matV].rows + 1) & ~1;   // even offsets (16-B aligned tensor-core operands)
    }
    d->tmp_size = tmp_off;
    AL(&d->tmpb, (size_t)std::max<int64_t>(1, tmp_off));
    for (int l = 0; l < nlev; ++l) {
      fda_status s;
      auto& F = fused[l];
      __gnu_parallel::stable_sort(F.begin(), F.end(), [](const LrOp& x, const LrOp& y) {
        return x.matV != y.matV ? x.matV < y.matV : x.dst < y.dst;
      });
      std::vector<LrTask> lt[LR_NCLS];
      std::vector<int64_t> ls, ld;
      for (size_t i = 0; i < F.size();) {
        size_t j = i;
        const size_t cap = (size_t)m2l_lr_ops(m2l_lr_class(p.mats[F[i].matV].rows));
        while (j < F.size() && F[j].matV == F[i].matV && j - i < cap) ++j;
        LrTask tk;
        tk.v_off = p.mats[F[i].matV].offset;
        tk.u_off = p.mats[F[i].matU].offset;
        tk.T = p.mats[F[i].matV].cols;
        tk.r = p.mats[F[i].matV].rows;
        tk.op_begin = (int32_t)ls.size();
        tk.op_count = (int32_t)(j - i);
        for (size_t q = i; q < j; ++q) {
          ls.push_back(p.out_offset[F[q].src]);
          ld.push_back(p.in_offset[F[q].dst]);
        }
        // the R1 = 24 class only pays on large levels (fewer, fuller launches otherwise)
        int cls = m2l_lr_class(tk.r);
        if (cls == 1 && F.size() < 200000) cls = 2;
        lt[cls].push_back(tk);
        i = j;
      }
      // longest CTAs first (phase-1 rows 16 / 32 / 64, phase-2 row tiles of 32)
      auto cost = [](const LrTask& t) {
        const int r1 = m2l_lr_rows(m2l_lr_class(t.r));   // (the LPT key; class 1 → 2 merges change little)
        return (int64_t)(r1 * t.T + ((t.T + 31) / 32) * 32 * t.r) * t.op_count;
      };
      Dev::M2LLevel& L = d->m2lv[l];
      {   // tensor-core tasks: ≤ 128 ops per factored K̃, op offsets appended to ls / ld
        auto& Ft = ftc[l];
        // Locality order on levels whose states exceed the L2 (config 5: 0.2-0.6 GB per level):
        // ops sorted by (block of destination states, K̃, destination), so that the tasks running
        // at any time touch one block of destination states and their sources instead of half
        // the level (one K̃'s ops span every box of the level).  A block holds ≈ 4·128 ops per K̃
        // on average; tasks keep this order (no longest-first sort).  A/B, config 5: k_m2l_bf
        // 26.7 → 25.1 ms; on L2-resident levels (config 4) the LPT order is faster (1.18 vs 1.33).
        bool blocked = false;
        int64_t dmin = 0, bspan = 1;
        if (!Ft.empty()) {
          int64_t dmax = Ft[0].dst;
          dmin = Ft[0].dst;
          for (const LrOp& o : Ft) {
            dmin = std::min(dmin, o.dst);
            dmax = std::max(dmax, o.dst);
          }
          const int64_t lev_bytes = 8 * (p.in_offset[dmax] - p.in_offset[dmin] + p.mats[Ft[0].matV].cols);
          if (lev_bytes > ((int64_t)64 << 20)) {
            std::vector<int64_t> mv(Ft.size());
            for (size_t q = 0; q < Ft.size(); ++q) mv[q] = Ft[q].matV;
            __gnu_parallel::sort(mv.begin(), mv.end());
            const double nm = (double)(std::unique(mv.begin(), mv.end()) - mv.begin());
            if ((double)Ft.size() / nm >= 512) {
              blocked = true;
              bspan = std::max<int64_t>(1, (int64_t)(4.0 * 128.0 * (double)(dmax - dmin + 1) * nm / (double)Ft.size()));
            }
          }
        }
        if (blocked)
          __gnu_parallel::stable_sort(Ft.begin(), Ft.end(), [dmin, bspan](const LrOp& x, const LrOp& y) {
            const int64_t bx = (x.dst - dmin) / bspan, by = (y.dst - dmin) / bspan;
            if (bx != by) return bx < by;
            return x.matV != y.matV ? x.matV < y.matV : x.dst < y.dst;
          });
        else
          __gnu_parallel::stable_sort(Ft.begin(), Ft.end(), [](const LrOp& x, const LrOp& y) {
            return x.matV != y.matV ? x.matV < y.matV : x.dst < y.dst;
          });
        std::vector<LrTcTask> tt;
        for (size_t i = 0; i < Ft.size();) {
          size_t j = i;
          while (j < Ft.size() && Ft[j].matV == Ft[i].matV && j - i < 128 &&
                 (!blocked || (Ft[j].dst - dmin) / bspan == (Ft[i].dst - dmin) / bspan))
            ++j;
          const int r = p.mats[Ft[i].matV].rows, T = p.mats[Ft[i].matV].cols;
          LrTcTask tk;
          tk.T = T;
          tk.r = r;
          tk.n1 = 2 * ((r + 7) / 8) * 8;
          tk.n2 = 2 * ((T + 7) / 8) * 8;
          if (ctx->p.opt.m2l_bf16) {   // BF16x3: 32-element K chunks of bf16 hi / lo
            tk.nk1 = (2 * T + 31) / 32;
            tk.b1_off = tc_bop_bf(ctx, d, Ft[i].matV, tk.n1, tk.nk1);
            tk.b2_off = tc_bop_bf(ctx, d, Ft[i].matU, tk.n2, (tk.n1 + 31) / 32);
          } else {
            tk.nk1 = (2 * T + TC_KC - 1) / TC_KC;
            tk.b1_off = tc_bop(ctx, d, Ft[i].matV, tk.n1, tk.nk1);
            tk.b2_off = tc_bop(ctx, d, Ft[i].matU, tk.n2, tk.n1 / TC_KC);
          }
          tk.op_begin = (int32_t)ls.size();
          tk.op_count = (int32_t)(j - i);
          for (size_t q = i; q < j; ++q) {
            ls.push_back(p.out_offset[Ft[q].src]);
            ld.push_back(p.in_offset[Ft[q].dst]);
          }
          tt.push_back(tk);
          i = j;
        }
        // one ring layout per launch; tasks longest first (the persistent CTAs stride over them)
        int n1m = 16;
        for (const LrTcTask& tk : tt) n1m = std::max(n1m, tk.n1);
        if (!blocked)
          std::stable_sort(tt.begin(), tt.end(), [](const LrTcTask& x, const LrTcTask& y) {
            return (int64_t)(x.nk1 + x.n1 / TC_KC) * x.n2 > (int64_t)(y.nk1 + y.n1 / TC_KC) * y.n2;
          });
        if (!tt.empty()) {
          int n2m = 16;
          for (const LrTcTask& tk : tt) n2m = std::max(n2m, tk.n2);
          L.lrtc_bf16 = ctx->p.opt.m2l_bf16 != 0;
          L.lrtc_plan = L.lrtc_bf16 ? m2l_bf_plan(n1m, n2m) : m2l_tcw_plan(n1m, n2m);
          // this level's out-states (contiguous offsets) are split into bf16 planes after its M2M
          const int64_t s0 = p.out_level_begin[l], s1 = p.out_level_begin[l + 1];
          if (s1 > s0) {
            L.split0 = 2 * p.out_offset[s0];
            L.split1 = 2 * (s1 < (int64_t)p.out_offset.size() ? p.out_offset[s1] : p.out_size);
          }
        }
        {
          int dev = 0, nsm = 148;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
          L.lrtc_grid = std::min<int>((int)tt.size(), nsm);
        }
        L.n_lrtc = (int)tt.size();
        for (const LrTcTask& tk : tt) L.fl_lrtc += 16.0 * tk.r * tk.T * tk.op_count;
        if (L.n_lrtc) UP(&L.lrtc, tt.data(), tt.size());
      }
      for (int c = 0; c < LR_NCLS; ++c) {
        std::stable_sort(lt[c].begin(), lt[c].end(),
                         [&](const LrTask& x, const LrTask& y) { return cost(x) > cost(y); });
        L.n_lr[c] = (int)lt[c].size();
        for (const LrTask& tk : lt[c]) L.fl_lr += 16.0 * tk.r * tk.T * tk.op_count;
        if (L.n_lr[c]) UP(&L.lr_tasks[c], lt[c].data(), lt[c].size());
      }
      if (!ls.empty()) {
        UP(&L.lr_src, ls.data(), ls.size());
        UP(&L.lr_dst, ld.data(), ld.size());
      }
      if ((s = build_xstage(ctx, d, a[l], true, L.a, true, lr_tc[l] != 0)) != FDA_OK) return s;
      if ((s = build_xstage(ctx, d, b[l], true, L.b, true, lr_tc[l] != 0)) != FDA_OK) return s;
    }
  }
  phase("translations");
  if (d->use_tc) {
    AL(&d->tcpool, (size_t)std::max<int64_t>(1, d->tc_size));
    CK(cudaMemset(d->tcpool, 0, sizeof(float) * std::max<int64_t>(1, d->tc_size)));
    if (!d->tc_jobs.empty()) {
      TcLayoutJob* dj = nullptr;
      CK(cudaMalloc((void**)&dj, sizeof(TcLayoutJob) * d->tc_jobs.size()));
      CK(cudaMemcpy(dj, d->tc_jobs.data(), sizeof(TcLayoutJob) * d->tc_jobs.size(), cudaMemcpyHostToDevice));
      launch_tc_layout((int)d->tc_jobs.size(), dj, d->pool, d->tcpool, 0);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaFree(dj);
    }
    std::vector<TcLayoutJob>().swap(d->tc_jobs);
    bool any_bf = false;
    for (auto& L : d->m2lv) any_bf |= L.n_lrtc > 0 && L.lrtc_bf16;
    // k_xlate_bf sources: which levels' out- / in-states the main stream splits into bf16 planes
    // (k_m2l_bf's branch then skips its own split of that level; other levels keep the split in
    // the branch, off the M2M chain)
    d->split_out.assign(nlev, 0);
    d->split_in.assign(nlev, 0);
    bool any_in = false;
    if (d->use_xbf)
      for (int l = 0; l < nlev; ++l) {
        if (l + 1 < nlev && d->m2m[l].n_bf) d->split_out[l + 1] = 1;
        if (d->m2lv[l].dense.n_bf) d->split_out[l] = 1;
        if (d->l2l[l].n_bf) d->split_in[l] = 1, any_in = true;
        any_bf |= d->split_out[l] != 0;
      }
    if (any_in) {
      AL(&d->inb_hi, (size_t)2 * std::max<int64_t>(1, p.in_size));
      AL(&d->inb_lo, (size_t)2 * std::max<int64_t>(1, p.in_size));
    }
    if (any_bf) {
      AL(&d->outb_hi, (size_t)2 * std::max<int64_t>(1, p.out_size));
      AL(&d->outb_lo, (size_t)2 * std::max<int64_t>(1, p.out_size));
    }
  }
  // sharded: packed exchange lists (partition.cpp xsend / xrecv)
  d->rank = ctx->p.opt.rank;
  if (d->nranks > 1) {
    const int R = d->nranks;
    auto Tof = [&](int64_t st) { return (int64_t)t.levels[t.boxes[p.out_states[st].box].level].rank; };
    std::vector<int64_t> xs, xr;
    d->soff.assign(R, 0); d->scnt.assign(R, 0); d->roff.assign(R, 0); d->rcnt.assign(R, 0);
    for (int q = 0; q < R; ++q) {
      d->soff[q] = (int64_t)xs.size();
      for (int64_t st : p.xsend[q])
        for (int64_t e = 0; e < Tof(st); ++e) xs.push_back(p.out_offset[st] + e);
      d->scnt[q] = (int64_t)xs.size() - d->soff[q];
      d->roff[q] = (int64_t)xr.size();
      for (int64_t st : p.xrecv[q])
        for (int64_t e = 0; e < Tof(st); ++e) xr.push_back(p.out_offset[st] + e);
      d->rcnt[q] = (int64_t)xr.size() - d->roff[q];
    }
    d->n_send = (int64_t)xs.size();
    d->n_recv = (int64_t)xr.size();
    UP(&d->xs_idx, xs.data(), xs.size());
    UP(&d->xr_idx, xr.data(), xr.size());
    AL(&d->sendb, (size_t)std::max<int64_t>(1, d->n_send));
    AL(&d->recvb, (size_t)std::max<int64_t>(1, d->n_recv));
    CK(cudaMemset(d->recvb, 0, sizeof(float2) * std::max<int64_t>(1, d->n_recv)));
  }
  // kernels per matvec: gather, near, s2m, every non-empty translation launch, l2t, scatter
  int64_t nl = 4 + (d->n_s2m > 0) + (d->n_l2t_add > 0);  // gather, near, l2t, scatter (+ s2m, HF-leaf L2T)
  auto cnt = [&](const XStage& st) {
    nl += st.n_bf > 0;
    for (int q = 0; q < 2; ++q) nl += st.n_tcw[q] > 0;
    for (int v = 0; v < TC_NV; ++v) nl += st.n_tc[v] > 0;
    for (int v = 0; v < XV; ++v) nl += st.ntask[v] > 0;
  };
  for (auto& st : d->m2m) cnt(st);
  for (auto& st : d->l2l) cnt(st);
  for (auto& L : d->m2lv) {
    cnt(L.dense); cnt(L.a); cnt(L.b);
    for (int c = 0; c < LR_NCLS; ++c) nl += L.n_lr[c] > 0;
    nl += L.n_lrtc > 0;
    nl += L.n_lrtc > 0 && L.lrtc_bf16;   // k_split_bf16 before k_m2l_bf
  }
  for (size_t l = 0; l < d->split_out.size(); ++l) nl += d->split_out[l] + d->split_in[l];   // k_split_bf16
  if (d->nranks > 1) nl += 2;            // k_pack, k_unpack_add
  ctx->launches_per_matvec = nl;
  // CTA tasks per translation kernel family (fda_debug_table "kernel_tasks"; lets the tests
  // assert where the translations were routed): [k_xlate, k_xlate_tc, k_xlate_tcw, k_m2l_lr,
  // k_m2l_tcw], each split into M2M | M2L | L2L
  {
    int64_t* kt = ctx->kernel_tasks;
    for (int i = 0; i < 18; ++i) kt[i] = 0;
    double* kf = ctx->kernel_flops;
    for (int i = 0; i < 18; ++i) kf[i] = 0;
    auto add = [&](const XStage& st, int which) {
      kt[5 * 3 + which] += st.n_bf;
      kf[5 * 3 + which] += st.fl_bf;
      for (int v = 0; v < XV; ++v) kt[0 * 3 + which] += st.ntask[v];
      for (int v = 0; v < TC_NV; ++v) kt[1 * 3 + which] += st.n_tc[v];
      for (int q = 0; q < 2; ++q) kt[2 * 3 + which] += st.n_tcw[q];
      for (int f = 0; f < 3; ++f) kf[f * 3 + which] += st.fl[f];
    };
    for (auto& st : d->m2m) add(st, 0);
    for (auto& st : d->l2l) add(st, 2);
    for (auto& L : d->m2lv) {
      add(L.dense, 1); add(L.a, 1); add(L.b, 1);
      for (int c = 0; c < LR_NCLS; ++c) kt[3 * 3 + 1] += L.n_lr[c];
      kt[4 * 3 + 1] += L.n_lrtc;
      kf[3 * 3 + 1] += L.fl_lr;
      kf[4 * 3 + 1] += L.fl_lrtc;
    }
  }
  // priorities: the far-field chain (S2M → M2M → M2L → L2L → L2T, captured
  // from s_cap and the M2L branch streams) is the critical path of the graph;
  // the near field (no dependencies until the final join) runs at the lowest
  // priority and fills the SMs the chain leaves idle
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CK(cudaStreamCreateWithPriority(&d->s_near, cudaStreamNonBlocking, prio_lo));
  CK(cudaStreamCreateWithPriority(&d->s_cap, cudaStreamNonBlocking, prio_hi));
  for (auto& sm : d->s_m2l) CK(cudaStreamCreateWithPriority(&sm, cudaStreamNonBlocking, prio_hi));
  d->ev_up.resize(nlev);
  d->ev_m2l.resize(nlev);
  for (auto& v : d->ev_m2l) {
    v.resize(LR_NCLS + 2);
    for (auto& e : v) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  for (auto& e : d->ev_up) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  d->use_graph = ctx->p.opt.use_graph != 0 && d->nranks <= 1;
  CK(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming));
  phase("upload/exchange");
  for (auto& e : d->ev) CK(cudaEventCreate(&e));
  CK(cudaEventCreate(&d->ev_n0));
  CK(cudaEventCreate(&d->ev_l0));
  CK(cudaEventCreate(&d->ev_l1));
  CK(cudaEventCreate(&d->ev_n1));
  CK(cudaDeviceSynchronize());
  return FDA_OK;
}

// device → host copy of the adopted matrix pool or correction values (fda_debug_table)
fda_status engine_read_table(Context* ctx, int which, void* dst, int64_t count) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  if (!d) return FDA_E_STATE;
  CK(cudaSetDevice(d->device));
  const void* src = which == 0 ? (const void*)d->pool : (which == 1 ? (const void*)d->corr_val : (const void*)d->corr_val_rhs);
  if (!src) return FDA_E_STATE;
  CK(cudaMemcpy(dst, src, (size_t)count * sizeof(float2), cudaMemcpyDeviceToHost));
  return FDA_OK;
}

fda_status engine_comm_init(Context* ctx, const void* id128) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  CK(cudaSetDevice(d->device));
  NcclApi& a = nccl(ctx->err);
  if (!a.ok) return FDA_E_NCCL;
  if (d->comm) { a.commDestroy(d->comm); d->comm = nullptr; }
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ncclResult_t r = a.commInitRank(&d->comm, ctx->p.opt.nranks, id, ctx->p.opt.rank);
  if (r != ncclSuccess) {
    ctx->err = std::string("ncclCommInitRank: ") + a.errStr(r);
    d->comm = nullptr;
    return FDA_E_NCCL;
  }
  return FDA_OK;
}

// sum the ranks' rows (each rank holds its own rows, zeros elsewhere)
static fda_status reduce_y(Context* ctx, Dev* d, void* y, bool f64, cudaStream_t s) {
  if (d->nranks <= 1) return FDA_OK;
  if (!d->comm) { ctx->err = "sharded context: call fda_comm_init before fda_matvec (or pass FDA_LOCAL)"; return FDA_E_STATE; }
  NcclApi& a = nccl(ctx->err);
  ncclResult_t r = a.allReduce(y, y, (size_t)2 * d->n, f64 ? ncclDouble : ncclFloat, ncclSum, d->comm, s);
  if (r != ncclSuccess) {
    ctx->err = std::string("ncclAllReduce: ") + a.errStr(r);
    return FDA_E_NCCL;
  }
  return FDA_OK;
}

void engine_destroy(Context* ctx) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  if (!d) return;
  cudaSetDevice(d->device);
  cudaDeviceSynchronize();
  if (d->comm) {
    std::string e;
    NcclApi& a = nccl(e);
    if (a.ok) a.commDestroy(d->comm);
  }
  for (void* a : d->allocs) cudaFree(a);
  for (void* a : d->gm_allocs) cudaFree(a);
  for (auto& ge : d->graph_exec)
    if (ge) cudaGraphExecDestroy(ge);
  if (d->s_near) cudaStreamDestroy(d->s_near);
  if (d->s_cap) cudaStreamDestroy(d->s_cap);
  for (auto& sm : d->s_m2l)
    if (sm) cudaStreamDestroy(sm);
  for (auto& e : d->ev_up) cudaEventDestroy(e);
  for (auto& v : d->ev_m2l)
    for (auto& e : v) cudaEventDestroy(e);
  if (d->ev_fork) cudaEventDestroy(d->ev_fork);
  if (d->ev_join) cudaEventDestroy(d->ev_join);
  for (auto& e : d->ev) if (e) cudaEventDestroy(e);
  if (d->ev_n0) cudaEventDestroy(d->ev_n0);
  if (d->ev_l0) cudaEventDestroy(d->ev_l0);
  if (d->ev_l1) cudaEventDestroy(d->ev_l1);
  if (d->ev_n1) cudaEventDestroy(d->ev_n1);
  for (auto& e : d->kt_ev) cudaEventDestroy(e);
  delete d;
  ctx->dev = nullptr;
}

// bf16 hi / lo planes of level l's out-states (in = false) or in-states (in = true), on stream s
static void split_level(Context* ctx, Dev* d, int l, bool in, cudaStream_t s) {
  const Plan& p = ctx->plan;
  const auto& lb = in ? p.in_level_begin : p.out_level_begin;
  const auto& off = in ? p.in_offset : p.out_offset;
  const int64_t s0 = lb[l], s1 = lb[l + 1];
  if (s1 <= s0) return;
  const int64_t f0 = 2 * off[s0], f1 = 2 * (s1 < (int64_t)off.size() ? off[s1] : (in ? p.in_size : p.out_size));
  const float* x = reinterpret_cast<const float*>(in ? d->inb : d->outb);
  __nv_bfloat16* hi = in ? d->inb_hi : d->outb_hi;
  __nv_bfloat16* lo = in ? d->inb_lo : d->outb_lo;
  KT(KF_XLATE_BF, s, launch_split_bf16(x + f0, f1 - f0, hi + f0, lo + f0, s));
}

// the tensor-core factored M2L of one level: k_m2l_bf (after splitting the level's out-states
// into bf16 hi / lo planes, unless the main stream did: d->split_out) or k_m2l_tcw
static void launch_lrtc(Dev* d, const Dev::M2LLevel& L, cudaStream_t st, bool split = true) {
  if (!L.n_lrtc) return;
  if (L.lrtc_bf16) {
    KT(KF_M2L_TCW, st, {
      if (split)
        launch_split_bf16(reinterpret_cast<const float*>(d->outb) + L.split0, L.split1 - L.split0,
                          d->outb_hi + L.split0, d->outb_lo + L.split0, st);
      launch_m2l_bf(L.n_lrtc, L.lrtc, L.lr_src, L.lr_dst, d->tcpool, d->outb_hi, d->outb_lo, d->inb, L.lrtc_plan,
                    L.lrtc_grid, st);
    });
  } else {
    KT(KF_M2L_TCW, st,
       launch_m2l_tcw(L.n_lrtc, L.lrtc, L.lr_src, L.lr_dst, d->tcpool, d->outb, d->inb, L.lrtc_plan, L.lrtc_grid, st));
  }
}

// the device part of one matvec: x_tree → y_near, y_far (tree order)
static fda_status run_core(Context* ctx, Dev* d, cudaStream_t s, int kind) {
  // profiling mode serialises the near field on the main stream so that every
  // stage time is the isolated duration of its kernels
  const bool prof = ctx->profiling;
  cudaStream_t sn = prof ? s : d->s_near;
  CK(cudaEventRecord(d->ev_fork, s));
  CK(cudaStreamWaitEvent(sn, d->ev_fork, 0));
  if (prof) CK(cudaEventRecord(d->ev_n0, sn));
  // near-kernel timing events: external event nodes when captured (so every graph replay
  // re-timestamps them), plain records in eager runs (the flag is only valid under capture)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(sn, &cap));
  const unsigned evf = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  CK(cudaEventRecordWithFlags(d->ev_l0, sn, evf));
  KT(KF_NEAR, sn,
     launch_near(d->n_near, d->near_tasks, d->near_slots, d->near_off, d->tgt_pos, d->tgt_nrm, d->src, d->src_w,
                 kind ? d->corr_ptr_rhs : d->corr_ptr, kind ? d->corr_col_rhs : d->corr_col,
                 kind ? d->corr_val_rhs : d->corr_val, d->x_tree, d->y_near, d->kp, d->alpha_pure_imag, kind,
                 d->near_wide, sn));
  CK(cudaEventRecordWithFlags(d->ev_l1, sn, evf));
  d->live = true;
  if (prof) CK(cudaEventRecord(d->ev_n1, sn));
  CK(cudaEventRecord(d->ev_join, sn));

  if (prof) CK(cudaEventRecord(d->ev[1], s));
  kt_mark(d, s, -1);
  if (d->out_size) CK(cudaMemsetAsync(d->outb, 0, sizeof(float2) * d->out_size, s));
  if (d->in_size) CK(cudaMemsetAsync(d->inb, 0, sizeof(float2) * d->in_size, s));
  if (d->tmp_size) CK(cudaMemsetAsync(d->tmpb, 0, sizeof(float2) * d->tmp_size, s));
  kt_mark(d, s, KF_MEMSET);
  if (kind) KT(KF_S2M, s, launch_s2m(d->n_s2m_rhs, d->s2m_rhs, d->pool, d->x_tree, d->outb, d->max_T, s));
  else KT(KF_S2M, s, launch_s2m(d->n_s2m, d->s2m, d->pool, d->x_tree, d->outb, d->max_T, s));
  if (prof) CK(cudaEventRecord(d->ev[2], s));
  const int nlev = (int)d->m2m.size();
  const bool xbf = !d->split_out.empty();
  auto split_out = [&](int l) { if (xbf && d->split_out[l]) split_level(ctx, d, l, false, s); };
  auto split_in = [&](int l) { if (xbf && d->split_in[l]) split_level(ctx, d, l, true, s); };
  auto m2l_level = [&](int l, cudaStream_t st) {
    const Dev::M2LLevel& L = d->m2lv[l];
    launch_lrtc(d, L, st, !(xbf && d->split_out[l]));
    for (int c = LR_NCLS - 1; c >= 0; --c)
      if (L.n_lr[c])
        KT(KF_M2L_LR, st, launch_m2l_lr(c, L.n_lr[c], L.lr_tasks[c], L.lr_src, L.lr_dst, d->pool, d->outb, d->inb, st));
    launch_stage(d, L.dense, d->outb, d->inb, st, d->outb_hi, d->outb_lo);
    launch_stage(d, L.a, d->outb, d->tmpb, st);
    launch_stage(d, L.b, d->tmpb, d->inb, st);
  };
  if (prof) {
    // serialised: every stage time is the isolated duration of its kernels
    for (int l = nlev - 1; l >= 0; --l) {
      launch_stage(d, d->m2m[l], d->outb, d->outb, s, d->outb_hi, d->outb_lo);
      split_out(l);
    }
    CK(cudaEventRecord(d->ev[3], s));
    for (int l = 0; l < nlev; ++l) m2l_level(l, s);
    CK(cudaEventRecord(d->ev[4], s));
    for (int l = 0; l < nlev; ++l) {
      split_in(l);
      launch_stage(d, d->l2l[l], d->inb, d->inb, s, d->inb_hi, d->inb_lo);
    }
    CK(cudaEventRecord(d->ev[5], s));
  } else {
    // dependency DAG: the M2L branches of level l (fused classes and the
    // dense / two-stage ops, each on its own stream) start as soon as the
    // outgoing states of level l exist, overlapping the M2M chain above it;
    // L2L out of level l waits for every M2L branch into level l.
    int k = 0;
    std::vector<int> nbr(nlev, 0);
    for (int l = nlev - 1; l >= 0; --l) {
      launch_stage(d, d->m2m[l], d->outb, d->outb, s, d->outb_hi, d->outb_lo);   // writes level-l out-states
      split_out(l);
      if (!d->m2lv[l].any()) continue;
      const Dev::M2LLevel& L = d->m2lv[l];
      CK(cudaEventRecord(d->ev_up[l], s));
      auto branch = [&](auto&& launch) -> fda_status {
        cudaStream_t sm = d->s_m2l[k++ % Dev::kM2LStreams];
        CK(cudaStreamWaitEvent(sm, d->ev_up[l], 0));
        launch(sm);
        CK(cudaEventRecord(d->ev_m2l[l][nbr[l]++], sm));
        return FDA_OK;
      };
      fda_status bs;
      if (L.n_lrtc &&
          (bs = branch([&](cudaStream_t sm) {
             launch_lrtc(d, L, sm, !(xbf && d->split_out[l]));
           })) != FDA_OK)
        return bs;
      for (int c = LR_NCLS - 1; c >= 0; --c)
        if (L.n_lr[c] &&
            (bs = branch([&](cudaStream_t sm) {
               launch_m2l_lr(c, L.n_lr[c], L.lr_tasks[c], L.lr_src, L.lr_dst, d->pool, d->outb, d->inb, sm);
             })) != FDA_OK)
          return bs;
      if ((bs = branch([&](cudaStream_t sm) {
             launch_stage(d, L.dense, d->outb, d->inb, sm, d->outb_hi, d->outb_lo);
             launch_stage(d, L.a, d->outb, d->tmpb, sm);
             launch_stage(d, L.b, d->tmpb, d->inb, sm);
           })) != FDA_OK)
        return bs;
    }
    for (int l = 0; l < nlev; ++l) {
      for (int b = 0; b < nbr[l]; ++b) CK(cudaStreamWaitEvent(s, d->ev_m2l[l][b], 0));
      split_in(l);
      launch_stage(d, d->l2l[l], d->inb, d->inb, s, d->inb_hi, d->inb_lo);
    }
  }
  KT(KF_L2T, s, launch_l2t(d->n_l2t, d->l2t, d->pool, d->inb, d->y_far, s));
  if (d->n_l2t_add) KT(KF_L2T, s, launch_l2t(d->n_l2t_add, d->l2t_add, d->pool, d->inb, d->y_far, s, /*accumulate=*/true));
  if (prof) CK(cudaEventRecord(d->ev[6], s));
  CK(cudaStreamWaitEvent(s, d->ev_join, 0));
  CK(cudaGetLastError());
  return FDA_OK;
}

// ---- sharded matvec (nranks > 1): partial upward pass →
// exchange of partial outgoing states → downward pass for the owned targets.
// Eager launches; the near field runs on its own stream across the exchange.
// the near field of the owned leaves, forked onto its own stream (joined by the caller
// through ev_join): eager, so that it overlaps the exchange between the two graph halves
static fda_status launch_sharded_near(Context* ctx, Dev* d, cudaStream_t s, int kind) {
  // profiling mode serialises the near field on the main stream (stage times as in run_core)
  const bool prof = ctx->profiling;
  cudaStream_t sn = prof ? s : d->s_near;
  CK(cudaEventRecord(d->ev_fork, s));
  CK(cudaStreamWaitEvent(sn, d->ev_fork, 0));
  if (prof) CK(cudaEventRecord(d->ev_n0, sn));
  CK(cudaEventRecord(d->ev_l0, sn));
  launch_near(d->n_near, d->near_tasks, d->near_slots, d->near_off, d->tgt_pos, d->tgt_nrm, d->src, d->src_w,
              kind ? d->corr_ptr_rhs : d->corr_ptr, kind ? d->corr_col_rhs : d->corr_col,
              kind ? d->corr_val_rhs : d->corr_val, d->x_tree, d->y_near, d->kp, d->alpha_pure_imag, kind, d->near_wide, sn);
  CK(cudaEventRecord(d->ev_l1, sn));
  d->live = true;
  if (prof) CK(cudaEventRecord(d->ev_n1, sn));
  CK(cudaEventRecord(d->ev_join, sn));
  CK(cudaGetLastError());
  return FDA_OK;
}

// the partial upward pass (S2M of own leaves, M2M into boxes holding own elements) and the
// packing of the partials other ranks need: one stream, captured as a graph
static fda_status run_sharded_up(Context* ctx, Dev* d, cudaStream_t s, int kind) {
  const bool prof = ctx->profiling;
  if (prof) CK(cudaEventRecord(d->ev[1], s));
  if (d->out_size) CK(cudaMemsetAsync(d->outb, 0, sizeof(float2) * d->out_size, s));
  if (d->in_size) CK(cudaMemsetAsync(d->inb, 0, sizeof(float2) * d->in_size, s));
  if (d->tmp_size) CK(cudaMemsetAsync(d->tmpb, 0, sizeof(float2) * d->tmp_size, s));
  if (kind) launch_s2m(d->n_s2m_rhs, d->s2m_rhs, d->pool, d->x_tree, d->outb, d->max_T, s);
  else launch_s2m(d->n_s2m, d->s2m, d->pool, d->x_tree, d->outb, d->max_T, s);
  if (prof) CK(cudaEventRecord(d->ev[2], s));
  const int nlev = (int)d->m2m.size();
  for (int l = nlev - 1; l >= 0; --l) launch_stage(d, d->m2m[l], d->outb, d->outb, s);   // partials
  launch_pack(d->outb, d->xs_idx, d->sendb, d->n_send, s);
  if (prof) CK(cudaEventRecord(d->ev[3], s));
  CK(cudaGetLastError());
  return FDA_OK;
}

static fda_status exchange_nccl(Context* ctx, Dev* d, cudaStream_t s) {
  if (!d->comm) { ctx->err = "sharded context: call fda_comm_init before fda_matvec"; return FDA_E_STATE; }
  NcclApi& a = nccl(ctx->err);
  if (!a.ok) return FDA_E_NCCL;
  ncclResult_t r = a.groupStart();
  for (int q = 0; q < d->nranks && r == ncclSuccess; ++q) {
    if (q == d->rank) continue;
    if (d->scnt[q] > 0) r = a.send(d->sendb + d->soff[q], (size_t)(2 * d->scnt[q]), ncclFloat, q, d->comm, s);
    if (r == ncclSuccess && d->rcnt[q] > 0)
      r = a.recv(d->recvb + d->roff[q], (size_t)(2 * d->rcnt[q]), ncclFloat, q, d->comm, s);
  }
  ncclResult_t r2 = a.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    ctx->err = std::string("NCCL exchange of outgoing states: ") + a.errStr(r);
    return FDA_E_NCCL;
  }
  return FDA_OK;
}

static fda_status run_sharded_down(Context* ctx, Dev* d, cudaStream_t s) {
  launch_unpack_add(d->recvb, d->xr_idx, d->outb, d->n_recv, s);
  const int nlev = (int)d->m2m.size();
  CK(cudaEventRecord(d->ev_up[0], s));
  int k = 0;
  std::vector<int> nbr(nlev, 0);
  for (int l = nlev - 1; l >= 0; --l) {   // M2L branches of every level, concurrent
    const Dev::M2LLevel& L = d->m2lv[l];
    if (!L.any()) continue;
    if (L.n_lrtc) {
      cudaStream_t sm = d->s_m2l[k++ % Dev::kM2LStreams];
      CK(cudaStreamWaitEvent(sm, d->ev_up[0], 0));
      launch_lrtc(d, L, sm);
      CK(cudaEventRecord(d->ev_m2l[l][nbr[l]++], sm));
    }
    for (int c = LR_NCLS - 1; c >= -1; --c) {
      if (c >= 0 && !L.n_lr[c]) continue;
      cudaStream_t sm = d->s_m2l[k++ % Dev::kM2LStreams];
      CK(cudaStreamWaitEvent(sm, d->ev_up[0], 0));
      if (c >= 0) {
        launch_m2l_lr(c, L.n_lr[c], L.lr_tasks[c], L.lr_src, L.lr_dst, d->pool, d->outb, d->inb, sm);
      } else {
        launch_stage(d, L.dense, d->outb, d->inb, sm);
        launch_stage(d, L.a, d->outb, d->tmpb, sm);
        launch_stage(d, L.b, d->tmpb, d->inb, sm);
      }
      CK(cudaEventRecord(d->ev_m2l[l][nbr[l]++], sm));
    }
  }
  const bool prof = ctx->profiling;
  if (prof) {   // M2L stage = exchange unpack + every M2L branch
    for (int l = 0; l < nlev; ++l)
      for (int b = 0; b < nbr[l]; ++b) CK(cudaStreamWaitEvent(s, d->ev_m2l[l][b], 0));
    CK(cudaEventRecord(d->ev[4], s));
  }
  for (int l = 0; l < nlev; ++l) {
    for (int b = 0; b < nbr[l]; ++b) CK(cudaStreamWaitEvent(s, d->ev_m2l[l][b], 0));
    launch_stage(d, d->l2l[l], d->inb, d->inb, s);
  }
  if (prof) CK(cudaEventRecord(d->ev[5], s));
  launch_l2t(d->n_l2t, d->l2t, d->pool, d->inb, d->y_far, s);
  launch_l2t(d->n_l2t_add, d->l2t_add, d->pool, d->inb, d->y_far, s, /*accumulate=*/true);
  if (prof) CK(cudaEventRecord(d->ev[6], s));
  CK(cudaGetLastError());
  return FDA_OK;
}

// capture fn(stream) once into d->graph_exec[slot] (all buffers are internal, so the graph
// serves every call) and launch it on s
template <class Fn>
static fda_status launch_captured(Context* ctx, Dev* d, cudaStream_t s, int slot, Fn&& fn) {
  cudaGraphExec_t& ge = d->graph_exec[slot];
  if (!ge) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(d->s_cap, cudaStreamCaptureModeThreadLocal));
    fda_status st = fn(d->s_cap);
    cudaError_t e = cudaStreamEndCapture(d->s_cap, &g);
    if (st != FDA_OK) return st;
    if (e != cudaSuccess) {
      ctx->err = std::string("graph capture failed: ") + cudaGetErrorString(e);
      return FDA_E_CUDA;
    }
    e = cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      ge = nullptr;
      ctx->err = std::string("graph instantiate failed: ") + cudaGetErrorString(e);
      return FDA_E_CUDA;
    }
  }
  CK(cudaGraphLaunch(ge, s));
  return FDA_OK;
}

// run_core through a CUDA graph (captured once: all its buffers are internal,
// so the same graph serves every call); profiled calls run it eagerly.
// phase (sharded contexts only): 0 = whole matvec with the NCCL exchange,
// FDA_PHASE_UP / FDA_PHASE_DOWN = the halves around an external exchange
// (fda_exchange_local, the one-GPU test transport)
static fda_status core(Context* ctx, Dev* d, cudaStream_t s, int kind, int phase = 0) {
  if (d->nranks > 1) {
    // sharded: near field (eager, own stream) ∥ [UP graph → NCCL exchange →
    // DOWN graph]; the halves are CUDA graphs (graph_exec[2 + kind] / [4 + kind]) unless profiling
    fda_status st = FDA_OK;
    const bool graphs = !ctx->profiling && ctx->p.opt.use_graph != 0;
    if (phase != FDA_PHASE_DOWN) {
      if ((st = launch_sharded_near(ctx, d, s, kind)) != FDA_OK) return st;
      st = graphs ? launch_captured(ctx, d, s, 2 + kind, [&](cudaStream_t cs) { return run_sharded_up(ctx, d, cs, kind); })
                  : run_sharded_up(ctx, d, s, kind);
      if (st != FDA_OK) return st;
    }
    if (phase == 0 && (st = exchange_nccl(ctx, d, s)) != FDA_OK) return st;
    if (phase != FDA_PHASE_UP) {
      st = graphs ? launch_captured(ctx, d, s, 4 + kind, [&](cudaStream_t cs) { return run_sharded_down(ctx, d, cs); })
                  : run_sharded_down(ctx, d, s);
      if (st != FDA_OK) return st;
      CK(cudaStreamWaitEvent(s, d->ev_join, 0));   // the near field of this matvec
    }
    return st;
  }
  if (ctx->profiling || !d->use_graph) return run_core(ctx, d, s, kind);
  return launch_captured(ctx, d, s, kind, [&](cudaStream_t cs) { return run_core(ctx, d, cs, kind); });
}

// device-pointer matvec in caller order (float2 in, float2 out)
static fda_status matvec_dev(Context* ctx, Dev* d, const float2* x, float2* y, cudaStream_t s, int kind = 0,
                             bool local = false, int phase = 0) {
  const bool prof = ctx->profiling && (d->nranks <= 1 || phase == 0);
  d->kt_on = prof && d->nranks <= 1;
  d->kt_n = 0;
  if (prof) CK(cudaEventRecord(d->ev[0], s));
  if (phase != FDA_PHASE_DOWN) KT(KF_GATHER, s, launch_gather_f32(x, d->perm, d->x_tree, d->n, s));
  if (prof) CK(cudaEventRecord(d->ev[1], s));
  fda_status st = core(ctx, d, s, kind, phase);
  if (st != FDA_OK) return st;
  if (phase == FDA_PHASE_UP) return FDA_OK;
  KT(KF_SCATTER, s, launch_scatter_f32(d->y_near, d->y_far, d->perm, y, d->n, d->e0, d->e1, s));
  d->kt_on = false;
  if (prof) CK(cudaEventRecord(d->ev[7], s));
  d->timed = prof;
  CK(cudaGetLastError());
  if (!local) {
    fda_status r = reduce_y(ctx, d, y, false, s);
    if (r != FDA_OK) return r;
  }
  return FDA_OK;
}

fda_status engine_apply(Context* ctx, const void* x, void* y, int32_t flags, void* stream, int kind) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  CK(cudaSetDevice(d->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool local = (flags & FDA_LOCAL) != 0;
  const int phase = flags & (FDA_PHASE_UP | FDA_PHASE_DOWN);
  if (phase) {
    if (d->nranks <= 1 || !(flags & FDA_DEVICE) || !local || phase == (FDA_PHASE_UP | FDA_PHASE_DOWN)) {
      ctx->err = "FDA_PHASE_UP / FDA_PHASE_DOWN need a sharded context, FDA_DEVICE and FDA_LOCAL";
      return FDA_E_INVALID_ARG;
    }
  }
  if (flags & FDA_DEVICE)
    return matvec_dev(ctx, d, static_cast<const float2*>(x), static_cast<float2*>(y), s, kind, local, phase);
  // host complex128 (or, with FDA_HOST_C64, complex64) in/out; the device buffers xh / yh hold
  // n complex128, which also fit n complex64
  const bool c64 = (flags & FDA_HOST_C64) != 0;
  const bool prof = ctx->profiling && (d->nranks <= 1 || phase == 0);
  CK(cudaMemcpyAsync(d->xh, x, (c64 ? sizeof(float2) : sizeof(double2)) * d->n, cudaMemcpyHostToDevice, s));
  if (prof) CK(cudaEventRecord(d->ev[0], s));
  if (c64) launch_gather_f32(reinterpret_cast<const float2*>(d->xh), d->perm, d->x_tree, d->n, s);
  else launch_gather_f64(d->xh, d->perm, d->x_tree, d->n, s);
  if (prof) CK(cudaEventRecord(d->ev[1], s));
  fda_status st = core(ctx, d, s, kind);
  if (st != FDA_OK) return st;
  if (c64) launch_scatter_f32(d->y_near, d->y_far, d->perm, reinterpret_cast<float2*>(d->yh), d->n, d->e0, d->e1, s);
  else launch_scatter_f64(d->y_near, d->y_far, d->perm, d->yh, d->n, d->e0, d->e1, s);
  if (prof) CK(cudaEventRecord(d->ev[7], s));
  d->timed = prof;
  if (!local) {
    fda_status r = reduce_y(ctx, d, d->yh, !c64, s);
    if (r != FDA_OK) return r;
  }
  CK(cudaMemcpyAsync(y, d->yh, (c64 ? sizeof(float2) : sizeof(double2)) * d->n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return FDA_OK;
}

// one-GPU test transport of the sharded exchange: copies every rank's packed
// partials for every peer into that peer's receive buffer (what the grouped
// ncclSend / ncclRecv of exchange_nccl does across GPUs)
fda_status engine_exchange_local(Context** ctxs, int n) {
  for (int r = 0; r < n; ++r) {
    Dev* dr = static_cast<Dev*>(ctxs[r]->dev);
    for (int q = 0; q < n; ++q) {
      if (q == r) continue;
      Dev* dq = static_cast<Dev*>(ctxs[q]->dev);
      if (dr->rcnt[q] != dq->scnt[r]) {
        ctxs[r]->err = "exchange plan mismatch between ranks";
        return FDA_E_INTERNAL;
      }
      if (dr->rcnt[q] > 0) {
        Context* ctx = ctxs[r];
        CK(cudaMemcpy(dr->recvb + dr->roff[q], dq->sendb + dq->soff[r], sizeof(float2) * dr->rcnt[q],
                      cudaMemcpyDeviceToDevice));
      }
    }
  }
  return FDA_OK;
}

// device time of the near-field kernel in the last matvec (events on its own
// stream, recorded inside the captured graph: the kernel as it runs
// concurrently with the far field)
fda_status engine_near_time(Context* ctx, double* ms) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  if (!d->live) { ctx->err = "no matvec yet"; return FDA_E_STATE; }
  CK(cudaEventSynchronize(d->ev_l1));
  float v = 0.f;
  CK(cudaEventElapsedTime(&v, d->ev_l0, d->ev_l1));
  *ms = v;
  return FDA_OK;
}

fda_status engine_kernel_times(Context* ctx, double* ms, int32_t* n) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  if (!d->timed || d->kt_n == 0) {
    ctx->err = "no profiled device-pointer matvec yet (fda_set_profiling(ctx, 1), then fda_matvec with FDA_DEVICE)";
    return FDA_E_STATE;
  }
  CK(cudaEventSynchronize(d->kt_ev[d->kt_n - 1]));
  double acc[KF_COUNT] = {0};
  for (int i = 1; i < d->kt_n; ++i) {
    if (d->kt_fam[i] < 0 || d->kt_fam[i - 1] >= 0) continue;
    float v = 0.f;
    CK(cudaEventElapsedTime(&v, d->kt_ev[i - 1], d->kt_ev[i]));
    acc[d->kt_fam[i]] += v;
  }
  const int m = std::min<int>(*n, KF_COUNT);
  for (int i = 0; i < m; ++i) ms[i] = acc[i];
  *n = m;
  return FDA_OK;
}

fda_status engine_stage_times(Context* ctx, double* ms, int32_t* n) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  if (!d->timed) { ctx->err = "no profiled matvec yet (call fda_set_profiling(ctx, 1) first)"; return FDA_E_STATE; }
  CK(cudaEventSynchronize(d->ev[7]));
  float v[8] = {0};
  CK(cudaEventElapsedTime(&v[0], d->ev[0], d->ev_n0));
  CK(cudaEventElapsedTime(&v[1], d->ev_n0, d->ev_n1));
  CK(cudaEventElapsedTime(&v[2], d->ev[1], d->ev[2]));
  CK(cudaEventElapsedTime(&v[3], d->ev[2], d->ev[3]));
  CK(cudaEventElapsedTime(&v[4], d->ev[3], d->ev[4]));
  CK(cudaEventElapsedTime(&v[5], d->ev[4], d->ev[5]));
  CK(cudaEventElapsedTime(&v[6], d->ev[5], d->ev[6]));
  CK(cudaEventElapsedTime(&v[7], d->ev[6], d->ev[7]));
  int m = std::min(*n, 8);
  for (int i = 0; i < m; ++i) ms[i] = v[i];
  *n = m;
  return FDA_OK;
}

fda_status engine_rhs_plane_wave(Context* ctx, const double dir[3], void* b, int32_t flags) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  CK(cudaSetDevice(d->device));
  double nn = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
  if (flags & FDA_DEVICE) {
    launch_plane_wave(d->cen, d->nrm, d->perm, d->n, ctx->p.k, ctx->p.alpha.real(), ctx->p.alpha.imag(),
                      dir[0] / nn, dir[1] / nn, dir[2] / nn, static_cast<float2*>(b), nullptr, 0);
    CK(cudaGetLastError());
    return FDA_OK;
  }
  launch_plane_wave(d->cen, d->nrm, d->perm, d->n, ctx->p.k, ctx->p.alpha.real(), ctx->p.alpha.imag(), dir[0] / nn,
                    dir[1] / nn, dir[2] / nn, nullptr, d->yh, 0);
  CK(cudaGetLastError());
  CK(cudaMemcpy(b, d->yh, sizeof(double2) * d->n, cudaMemcpyDeviceToHost));
  return FDA_OK;
}

fda_status engine_rhs_point_source(Context* ctx, const double src[3], void* b, int32_t flags) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  CK(cudaSetDevice(d->device));
  const double are = ctx->p.alpha.real(), aim = ctx->p.alpha.imag();
  if (flags & FDA_DEVICE) {
    launch_point_source(d->cen, d->nrm, d->perm, d->n, ctx->p.k, are, aim, src[0], src[1], src[2],
                        static_cast<float2*>(b), nullptr, 0);
    CK(cudaGetLastError());
    return FDA_OK;
  }
  launch_point_source(d->cen, d->nrm, d->perm, d->n, ctx->p.k, are, aim, src[0], src[1], src[2], nullptr, d->yh, 0);
  CK(cudaGetLastError());
  CK(cudaMemcpy(b, d->yh, sizeof(double2) * d->n, cudaMemcpyDeviceToHost));
  return FDA_OK;
}

// ------------------------------------------------------------------ GMRES
// bm_solve: GMRES (§5; reading C20) on device vectors in
// caller order.  Arnoldi with classical Gram-Schmidt applied twice (CGS2),
// fp64 accumulation of every inner product, coefficients kept on the device;
// one small device→host copy per iteration feeds the Givens rotations.

static const int kChunks = 128;

// ---- sharded GMRES (nranks > 1): every Krylov vector holds only this rank's rows
// (tree order, the contiguous element range [e0, e1)); inner products are local partial sums
// all-reduced over the ranks (one ncclAllReduce of j + 1 complex values per CGS pass), the
// matvec input is all-gathered (one ncclBroadcast per rank's slice, grouped) and the matvec
// returns the LOCAL rows (no all-reduce of y)
static fda_status allgather_tree(Context* ctx, Dev* d, float2* full, cudaStream_t s) {
  NcclApi& a = nccl(ctx->err);
  if (!a.ok) return FDA_E_NCCL;
  const Plan& p = ctx->plan;
  ncclResult_t r = a.groupStart();
  for (int q = 0; q < d->nranks && r == ncclSuccess; ++q) {
    const int64_t n0 = p.rank_e0[q], nq = p.rank_e1[q] - p.rank_e0[q];
    if (nq > 0) r = a.bcast(full + n0, full + n0, (size_t)(2 * nq), ncclFloat, q, d->comm, s);
  }
  ncclResult_t r2 = a.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    ctx->err = std::string("NCCL all-gather of the Krylov vector: ") + a.errStr(r);
    return FDA_E_NCCL;
  }
  return FDA_OK;
}
static fda_status allreduce_d(Context* ctx, Dev* d, double* v, size_t count, cudaStream_t s) {
  NcclApi& a = nccl(ctx->err);
  if (!a.ok) return FDA_E_NCCL;
  const ncclResult_t r = a.allReduce(v, v, count, ncclDouble, ncclSum, d->comm, s);
  if (r != ncclSuccess) {
    ctx->err = std::string("NCCL all-reduce of GMRES dot products: ") + a.errStr(r);
    return FDA_E_NCCL;
  }
  return FDA_OK;
}
static fda_status matvec_own(Context* ctx, Dev* d, const float2* x_own, float2* y_own, cudaStream_t s) {
  const int64_t e0 = d->e0, nl = d->e1 - d->e0;
  if (nl > 0) CK(cudaMemcpyAsync(d->x_tree + e0, x_own, sizeof(float2) * nl, cudaMemcpyDeviceToDevice, s));
  fda_status st = allgather_tree(ctx, d, d->x_tree, s);
  if (st != FDA_OK) return st;
  if ((st = core(ctx, d, s, 0, 0)) != FDA_OK) return st;
  launch_add_slice(d->y_near, d->y_far, e0, nl, y_own, s);
  CK(cudaGetLastError());
  return FDA_OK;
}

// h[0..nv) = V[0..nv)^H w  → device
static void dots_dev(Gm& gm, int nv, const float2* w, int64_t n, double2* h) {
  launch_dots(gm.V, n, nv, w, n, gm.partial, kChunks, 0);
  launch_reduce_partials(gm.partial, nv, kChunks, h, 0);
}

// ‖w‖ into gm.nrm (device) — over the ranks' slices when sharded
static fda_status norm_dev(Context* ctx, Dev* d, Gm& gm, const float2* w, int64_t n) {
  launch_norm2(w, n, gm.np, kChunks, 0);
  if (d->nranks > 1) {
    launch_reduce_sum(gm.np, kChunks, gm.nrm, 0);
    fda_status st = allreduce_d(ctx, d, gm.nrm, 1, 0);
    if (st != FDA_OK) return st;
    launch_sqrt1(gm.nrm, 0);
  } else {
    launch_reduce_norm(gm.np, kChunks, gm.nrm, 0);
  }
  return FDA_OK;
}
static fda_status norm_host(Context* ctx, Dev* d, Gm& gm, const float2* w, int64_t n, double& out) {
  fda_status st = norm_dev(ctx, d, gm, w, n);
  if (st != FDA_OK) return st;
  CK(cudaMemcpy(&out, gm.nrm, sizeof(double), cudaMemcpyDeviceToHost));
  return FDA_OK;
}

fda_status engine_solve(Context* ctx, const void* rhs, void* u, double tol, int32_t max_iter, int32_t restart,
                        fda_solve_info* info, int32_t flags) {
  Dev* d = static_cast<Dev*>(ctx->dev);
  CK(cudaSetDevice(d->device));
  CK(cudaDeviceSynchronize());
  auto t0 = std::chrono::steady_clock::now();
  // sharded (nranks > 1): the Krylov vectors hold this rank's rows only (tree order)
  const bool sh = d->nranks > 1;
  if (sh && !d->comm) { ctx->err = "sharded context: call fda_comm_init before bm_solve"; return FDA_E_STATE; }
  const int64_t n = sh ? (int64_t)(d->e1 - d->e0) : d->n;
  const int m = restart > 0 ? std::min(restart, max_iter) : max_iter;
  auto mv = [&](const float2* xv, float2* yv) -> fda_status {
    return sh ? matvec_own(ctx, d, xv, yv, 0) : matvec_dev(ctx, d, xv, yv, 0);
  };
  // h[0..nv) = V^H w over all ranks
  auto dots = [&](Gm& g, int nv, const float2* w, double2* h) -> fda_status {
    dots_dev(g, nv, w, n, h);
    return sh ? allreduce_d(ctx, d, reinterpret_cast<double*>(h), (size_t)2 * nv, 0) : FDA_OK;
  };
  // workspace cached in the context (allocated on the first solve, grown on demand)
  if (d->gm_cap < m + 1) {
    for (void* q : d->gm_allocs) cudaFree(q);
    d->gm_allocs.clear();
    d->gm_cap = 0;
    auto A = [&](void** q, size_t bytes) -> bool {
      if (cudaMalloc(q, bytes) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      d->gm_allocs.push_back(*q);
      return true;
    };
    Gm& w = d->gm;
    if (!A((void**)&w.V, sizeof(float2) * std::max<int64_t>(1, n) * (m + 1)) || !A((void**)&w.w, sizeof(float2) * std::max<int64_t>(1, n)) ||
        !A((void**)&w.full, sizeof(float2) * d->n) ||
        !A((void**)&w.b, sizeof(float2) * std::max<int64_t>(1, n)) || !A((void**)&w.x, sizeof(float2) * std::max<int64_t>(1, n)) ||
        !A((void**)&w.partial, sizeof(double2) * kChunks * (m + 1)) ||
        !A((void**)&w.hbuf, sizeof(double2) * 3 * (m + 1)) || !A((void**)&w.np, sizeof(double) * kChunks) ||
        !A((void**)&w.nrm, sizeof(double))) {
      for (void* q : d->gm_allocs) cudaFree(q);
      d->gm_allocs.clear();
      ctx->err = "device allocation for the GMRES workspace failed";
      return FDA_E_NOMEM;
    }
    d->gm_cap = m + 1;
  }
  Gm gm = d->gm;
  gm.m = m;
  auto cleanup = []() {};
  fda_status st = FDA_OK;
#define GCK(expr)       \
  do {                  \
    st = (expr);        \
    if (st != FDA_OK) { \
      cleanup();        \
      return st;        \
    }                   \
  } while (0)
#define GCU(call)                                                                  \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ctx->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call; \
      cleanup();                                                                   \
      return FDA_E_CUDA;                                                           \
    }                                                                              \
  } while (0)
  double2* h1 = gm.hbuf;
  double2* h2 = gm.hbuf + (m + 1);
  double2* yd = gm.hbuf + 2 * (m + 1);
  if (sh) {   // caller order → tree order (full), then this rank's slice
    if (flags & FDA_DEVICE) {
      launch_gather_f32(static_cast<const float2*>(rhs), d->perm, gm.full, d->n, 0);
    } else {
      GCU(cudaMemcpy(d->xh, rhs, sizeof(double2) * d->n, cudaMemcpyHostToDevice));
      launch_gather_f64(d->xh, d->perm, gm.full, d->n, 0);
    }
    if (n > 0) GCU(cudaMemcpy(gm.b, gm.full + d->e0, sizeof(float2) * n, cudaMemcpyDeviceToDevice));
  } else if (flags & FDA_DEVICE) {
    GCU(cudaMemcpy(gm.b, rhs, sizeof(float2) * n, cudaMemcpyDeviceToDevice));
  } else {
    GCU(cudaMemcpy(d->xh, rhs, sizeof(double2) * n, cudaMemcpyHostToDevice));
    launch_f64_to_f32(d->xh, gm.b, n, 0);
  }
  if (n > 0) GCU(cudaMemset(gm.x, 0, sizeof(float2) * n));
  double bnorm = 0;
  GCK(norm_host(ctx, d, gm, gm.b, n, bnorm));
  int it = 0;
  double res = 1.0;
  bool conv = bnorm == 0.0;
  std::vector<cd> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1);
  std::vector<double2> hh(2 * (m + 1) + 1);
  while (!conv && it < max_iter) {
    float2* v0 = gm.V;
    double beta;
    if (it == 0) {
      if (n > 0) GCU(cudaMemcpy(v0, gm.b, sizeof(float2) * n, cudaMemcpyDeviceToDevice));
      beta = bnorm;
    } else {  // restart: r = b - A x
      GCK(mv(gm.x, gm.w));
      if (n > 0) GCU(cudaMemcpy(v0, gm.b, sizeof(float2) * n, cudaMemcpyDeviceToDevice));
      launch_axpby(v0, gm.w, -1.0, 1.0, n, 0);
      GCK(norm_host(ctx, d, gm, v0, n, beta));
    }
    launch_scale(v0, v0, 1.0 / beta, 0.0, n, 0);
    std::fill(H.begin(), H.end(), cd(0));
    std::fill(g.begin(), g.end(), cd(0));
    g[0] = beta;
    int jd = 0;
    for (int j = 0; j < m && it < max_iter; ++j) {
      float2* vj = gm.V + (int64_t)j * n;
      GCK(mv(vj, gm.w));
      GCK(dots(gm, j + 1, gm.w, h1));
      launch_update(gm.w, gm.V, n, j + 1, h1, n, -1.0, 0);
      GCK(dots(gm, j + 1, gm.w, h2));
      launch_update(gm.w, gm.V, n, j + 1, h2, n, -1.0, 0);
      GCK(norm_dev(ctx, d, gm, gm.w, n));
      launch_scale_by_inv(gm.V + (int64_t)(j + 1) * n, gm.w, gm.nrm, n, 0);
      // one copy: h1, h2 and the norm
      GCU(cudaMemcpy(hh.data(), h1, sizeof(double2) * (m + 1 + j + 1), cudaMemcpyDeviceToHost));   // h1 | h2
      double hn;
      GCU(cudaMemcpy(&hn, gm.nrm, sizeof(double), cudaMemcpyDeviceToHost));
      for (int i = 0; i <= j; ++i)
        H[(size_t)j * (m + 1) + i] = cd(hh[i].x + hh[m + 1 + i].x, hh[i].y + hh[m + 1 + i].y);
      H[(size_t)j * (m + 1) + j + 1] = hn;
      // Givens rotations (complex): [c̄ s̄; -s c]
      for (int i = 0; i < j; ++i) {
        cd a = H[(size_t)j * (m + 1) + i], bb = H[(size_t)j * (m + 1) + i + 1];
        H[(size_t)j * (m + 1) + i] = std::conj(cs[i]) * a + std::conj(sn[i]) * bb;
        H[(size_t)j * (m + 1) + i + 1] = -sn[i] * a + cs[i] * bb;
      }
      cd a = H[(size_t)j * (m + 1) + j], bb = H[(size_t)j * (m + 1) + j + 1];
      double den = std::sqrt(std::norm(a) + std::norm(bb));
      cs[j] = a / den;
      sn[j] = bb / den;
      H[(size_t)j * (m + 1) + j] = den;
      H[(size_t)j * (m + 1) + j + 1] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = std::conj(cs[j]) * g[j];
      ++it;
      jd = j + 1;
      res = std::abs(g[j + 1]) / bnorm;
      if (res <= tol || hn == 0.0) { conv = res <= tol; break; }
    }
    // y = R⁻¹ g ; x += V y
    std::vector<double2> y(jd);
    std::vector<cd> yc(jd);
    for (int i = jd - 1; i >= 0; --i) {
      cd s = g[i];
      for (int k = i + 1; k < jd; ++k) s -= H[(size_t)k * (m + 1) + i] * yc[k];
      yc[i] = s / H[(size_t)i * (m + 1) + i];
      y[i] = make_double2(yc[i].real(), yc[i].imag());
    }
    if (jd > 0) {
      GCU(cudaMemcpy(yd, y.data(), sizeof(double2) * jd, cudaMemcpyHostToDevice));
      launch_update(gm.x, gm.V, n, jd, yd, n, +1.0, 0);
    }
    if (restart <= 0) break;
  }
  // true residual ‖b - A x‖ / ‖b‖ (one extra matvec)
  double true_res = 0;
  if (bnorm > 0) {
    GCK(mv(gm.x, gm.w));
    launch_axpby(gm.w, gm.b, 1.0, -1.0, n, 0);  // w = b - A x
    double rn;
    GCK(norm_host(ctx, d, gm, gm.w, n, rn));
    true_res = rn / bnorm;
  }
  if (sh) {   // this rank's slice → full tree-order u on every rank → caller order
    if (n > 0) GCU(cudaMemcpy(gm.full + d->e0, gm.x, sizeof(float2) * n, cudaMemcpyDeviceToDevice));
    GCK(allgather_tree(ctx, d, gm.full, 0));
    GCU(cudaMemset(d->y_far, 0, sizeof(float2) * d->n));
    if (flags & FDA_DEVICE) {
      launch_scatter_f32(gm.full, d->y_far, d->perm, static_cast<float2*>(u), d->n, 0, d->n, 0);
    } else {
      launch_scatter_f64(gm.full, d->y_far, d->perm, d->yh, d->n, 0, d->n, 0);
      GCU(cudaMemcpy(u, d->yh, sizeof(double2) * d->n, cudaMemcpyDeviceToHost));
    }
  } else if (flags & FDA_DEVICE) {
    GCU(cudaMemcpy(u, gm.x, sizeof(float2) * n, cudaMemcpyDeviceToDevice));
  } else {
    launch_f32_to_f64(gm.x, d->yh, n, 0);
    GCU(cudaMemcpy(u, d->yh, sizeof(double2) * n, cudaMemcpyDeviceToHost));
  }
  GCU(cudaDeviceSynchronize());
  cleanup();
  if (info) {
    info->iterations = it;
    info->converged = conv ? 1 : 0;
    info->rel_residual = res;
    info->true_residual = true_res;
    info->t_solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return conv ? FDA_OK : FDA_E_NOT_CONVERGED;
}

}  // namespace fda
