// C ABI (include/dd_aux.h): host driver of the B200 auxiliary-matrix solver.
//
// dd_aux_analyze builds, on the host, everything integer about the factorization
// ("very fast symbolic factorization step"): the block elimination order,
// the clique-completion fill, the elimination tree and its levels, the HBM layout of
// the factor and every per-level descriptor table the kernels consume.  dd_aux_factor
// and dd_aux_solve only upload tables and enqueue kernels level by level (SURVEY.md
// §8(a) a5: "Per level, in order: K1 -> K2 -> K3, stream order as the only barrier").
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <numeric>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dd_aux.h"
#include "analyze.hpp"
#include "launch.hpp"

using namespace ddaux;
using namespace ddk;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(DD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define LAUNCH_CHECK(what)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess) return fail(DD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Blob {  // host image of the device table region
  std::vector<uint8_t> data;
  template <class T>
  size_t put(const std::vector<T>& v) {
    size_t off = align256(data.size());
    data.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(data.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
};

struct LevelRanges {
  int n0, n1;     // level nodes
  int s0, s1;     // K2 strips (L = W D^{-1})
  int k0, k1;     // K2 GEMM tiles
  int r0, r1;     // rowperm entries
  int t0, t1;     // K3 targets: [t0, ta) update the next level's panels, [ta, t1) the rest
  int ta, ta1;               // [t0, ta1): diagonal blocks of the next level's nodes (K3a1), [ta1, ta): the
                             // rest of their panels (K3a2)
  int64_t tiles_a, tiles_b;  // implicit tile counts of the two parts
  int64_t tiles_a1;          // tiles of K3a1
  int f0, f1;     // forward-solve tiles
  int b0, b1;     // backward-solve tiles
  int d0, d1;     // diagonal-solve tiles (node, 64-row tile)
  int i0, i1;     // inverse work items (node, TB column tile)
  double fl_k1, fl_k2, fl_k3;      // algorithmic flops of the level's factor kernels
  int max_s;                       // largest diagonal block of the level
  int max_rp;                      // largest padded struct-row count of the level's nodes
  double fl_diag, fl_upd;          // solve flops per rhs: one diagonal sweep / one update sweep
};

}  // namespace

struct GraphCache {           // one instantiated CUDA graph + the pointer key it was captured for
  cudaGraphExec_t exec = nullptr;
  std::vector<uintptr_t> key;
  int64_t dl[16] = {0};       // launches / flops the captured sequence accounts for per replay
  double df[16] = {0};
};

struct dd_aux_handle_s {
  int dtype = DD_REAL64;
  bool cplx = false;
  dd_aux_options opt{};
  Graph g;
  Symbolic S;
  std::vector<int64_t> blk_size, colptr, odof_blk;
  std::vector<int32_t> rowidx;
  int64_t n = 0, n_pad = 0, nnzb_in = 0;
  int order_used = 0;
  // layout
  std::vector<NodeDev> nodes;
  int64_t nA = 0;            // arena elements per plane
  int64_t d_off = 0, e_off = 0;
  int64_t nW = 0, nK1 = 0;   // level workspace elements per plane
  int max_s = 0;
  // tables
  Blob blob;
  size_t off_nodes = 0, off_stpos = 0, off_strow = 0, off_lvlnodes = 0, off_strips = 0, off_rowperm = 0,
         off_targets = 0, off_contribs = 0, off_tiles = 0, off_ftargets = 0, off_fcontribs = 0, off_btiles = 0,
         off_sprows = 0, off_blksize = 0, off_odof = 0, off_dtiles = 0, off_litems = 0, off_k2items = 0;
  int64_t nT = 0;             // rows of the solve's level buffer T
  size_t off_spsegs = 0;       // SpSeg table (filled at factor time)
  std::vector<SpSeg> spsegs;   // voff holds the CSC position until factor
  int n_sprows = 0;
  std::vector<LevelRanges> lv;
  // factor buffer offsets (bytes)
  size_t tables_bytes = 0, off_arena = 0, off_ipiv = 0, off_perm = 0, off_gperm = 0, off_ginv = 0, off_stats = 0,
         off_totals = 0, off_norm = 0, factor_bytes = 0;
  // work buffer offsets (bytes)
  size_t w_off_W = 0, w_off_K1 = 0, w_off_load = 0, work_bytes = 0;
  // info
  double flops_factor = 0, flops_solve = 0, value_bytes = 0;
  int64_t max_front = 0, max_width = 0;
  bool factored = false, singular = false;
  const void* factored_ptr = nullptr;
  double nnz_full = 0;  // entries of the full symmetric A (K6 flops)
  // lookahead: high-priority side stream + per-level events
  cudaStream_t side = nullptr;
  cudaStream_t side2 = nullptr;   // k_rowperm: concurrent with k_linv / K2 of the same level
  cudaEvent_t evR = nullptr;      // joins side2 back into the caller's stream
  bool norm_valid = false;  // ||A||_inf of the current factorization's d_vals computed on device
  bool m3 = false;         // complex products in the 3M form (options.complex_3m)
  int k3cfg = 1;           // K3 tile configuration (env DD_AUX_K3CFG, read at analyze)
  bool lookahead = true;   // env DD_AUX_LOOKAHEAD=0 disables the side-stream overlap
  std::vector<cudaEvent_t> evA, evA2, evB, evK;  // evK[l]: K1 of level l done (perm ready)
  cudaEvent_t evLoad = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr;  // factor timing (finfo.ms_load / ms_factor)
  // f3/f2 Schur mode (dd_aux_analyze_partial): the last n_schur block ids are kept (not eliminated)
  int64_t n_schur = 0;
  int n_elim = 0;                  // eliminated positions [0, n_elim); kept positions [n_elim, N)
  int64_t r0 = 0;                  // first padded solve row of the kept blocks
  int64_t n_aux = 0, n_aux_dof = 0;
  std::vector<int64_t> aux_odof;   // [n_aux] first auxiliary DoF of each auxiliary block
  std::vector<int32_t> schur_target, schur_group;  // per kept block (0-based among the kept)
  std::vector<int64_t> grp_ptr;    // groups (distinct schur_group, ascending): members in clq_blk order
  std::vector<int32_t> grp_kept;   // kept indices sorted by (group, target)
  std::vector<int64_t> grp_m;      // m_g
  std::vector<int32_t> kept_gperm, kept_ginv, kept_perm;  // identity maps of the kept rows (uploaded per factor)
  size_t off_sx_items = 0, off_sx_tiles = 0, off_sg_items = 0, off_sg_contrib = 0, off_ss_items = 0,
         off_soff = 0;
  int n_sx_tiles = 0, n_sg_items = 0, n_ss_items = 0;
  std::vector<int64_t> soff_host;  // S_offset of the last export (kept alive for the async upload)
  // f1 assembly tables (host images kept alive for the async upload)
  std::vector<AsmItem> asm_items;
  std::vector<AsmContrib> asm_cons;
  double asm_bytes = 0;
  // CUDA graphs (options.use_graphs): factor level loop and whole solve, captured on `cap`
  GraphCache gfactor, gsolve;
  cudaStream_t cap = nullptr;
  // tracing
  bool trace = false;
  std::vector<cudaEvent_t> pool;
  struct Rec { int ph, e0, e1, level; };
  int cur_level = -1;                          // level being enqueued (per-level trace)
  std::vector<double> lvl_ms, lvl_fl;          // [nlevels * 16]
  std::vector<Rec> recs;
  int64_t launches[16] = {0};
  double flops[16] = {0};
  double ms_acc[16] = {0};
  int ev() {
    int id = (int)recs.size() * 2;
    while ((int)pool.size() < id + 2) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return id;
  }
  ~dd_aux_handle_s() {
    for (auto e : pool) cudaEventDestroy(e);
    for (auto e : evA) cudaEventDestroy(e);
    for (auto e : evB) cudaEventDestroy(e);
    for (auto e : evA2) cudaEventDestroy(e);
    for (auto e : evK) cudaEventDestroy(e);
    if (evLoad) cudaEventDestroy(evLoad);
    for (auto e : {t0, t1, t2})
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (evR) cudaEventDestroy(evR);
    if (gfactor.exec) cudaGraphExecDestroy(gfactor.exec);
    if (gsolve.exec) cudaGraphExecDestroy(gsolve.exec);
    if (cap) cudaStreamDestroy(cap);
  }
};

namespace {
// bracket one kernel launch: counts + flops always, CUDA events when tracing
struct TraceScope {
  dd_aux_handle_s* h;
  int ph, id = -1;
  cudaStream_t st;
  double fl;
  TraceScope(dd_aux_handle_s* h_, int ph_, double fl_, cudaStream_t st_) : h(h_), ph(ph_), st(st_), fl(fl_) {
    h->launches[ph] += 1;
    h->flops[ph] += fl;
    if (h->trace) {
      id = h->ev();
      cudaEventRecord(h->pool[id], st);
    }
  }
  ~TraceScope() {
    if (id >= 0) {
      cudaEventRecord(h->pool[id + 1], st);
      h->recs.push_back({ph, id, id + 1, h->cur_level});
      if (h->cur_level >= 0) {
        if (h->lvl_fl.size() < (size_t)(h->cur_level + 1) * 16) {
          h->lvl_fl.resize((size_t)(h->cur_level + 1) * 16, 0.0);
          h->lvl_ms.resize((size_t)(h->cur_level + 1) * 16, 0.0);
        }
        h->lvl_fl[(size_t)h->cur_level * 16 + ph] += fl;
      }
    }
  }
};

// Enqueue fn(stream) directly, or (options.use_graphs, tracing off) replay a CUDA graph of it
// captured once per pointer key on the handle's capture stream.  Launch
// and flop counters advance by the captured sequence's counts on every replay.
template <class Fn>
int run_graph(dd_aux_handle_s* h, GraphCache& gc, const std::vector<uintptr_t>& key, Fn&& fn, cudaStream_t st) {
  if (!h->opt.use_graphs || h->trace) return fn(st);
  if (!gc.exec || gc.key != key) {
    if (gc.exec) {
      cudaGraphExecDestroy(gc.exec);
      gc.exec = nullptr;
    }
    if (!h->cap) CUDA_TRY(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    int64_t l0[16];
    double f0[16];
    for (int q = 0; q < 16; ++q) {
      l0[q] = h->launches[q];
      f0[q] = h->flops[q];
    }
    CUDA_TRY(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    const int rc = fn(h->cap);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(h->cap, &g);
    for (int q = 0; q < 16; ++q) {
      gc.dl[q] = h->launches[q] - l0[q];
      gc.df[q] = h->flops[q] - f0[q];
      h->launches[q] = l0[q];
      h->flops[q] = f0[q];
    }
    if (rc) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return rc;
    }
    if (e != cudaSuccess) return fail(DD_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
    const cudaError_t ei = cudaGraphInstantiate(&gc.exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) {
      gc.exec = nullptr;
      return fail(DD_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
    }
    gc.key = key;
  }
  CUDA_TRY(cudaGraphLaunch(gc.exec, st));
  for (int q = 0; q < 16; ++q) {
    h->launches[q] += gc.dl[q];
    h->flops[q] += gc.df[q];
  }
  return DD_OK;
}
}  // namespace

extern "C" {

void dd_aux_default_options(dd_aux_options* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->order = DD_ORDER_AUTO;
  opt->refine_steps = 1;
  opt->complex_3m = 1;
}

const char* dd_aux_last_error(void) { return g_err.c_str(); }
const char* dd_aux_version(void) { return "dd_aux 0.1 (sm_100a, FP64 DMMA)"; }

}  // extern "C"

static int build_schur_tables(dd_aux_handle_t h);
struct SchurIn {  // dd_aux_analyze_partial's kept-block description
  const int32_t* target;
  const int32_t* group;
  int64_t n_aux;
  const int64_t* aux_size;
};

// dd_aux_analyze and dd_aux_analyze_partial: with n_schur > 0 the last n_schur block ids are kept
// (their Schur complement is formed, they are not eliminated); the order option then applies to
// the eliminated blocks and the kept ones follow in ascending id.
static int analyze_impl(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx,
                        int32_t dtype, const dd_aux_options* opt_in, int64_t n_schur, const SchurIn* sin,
                        dd_aux_handle_t* out) {
  if (nblk <= 0) return fail(-1, "nblk must be > 0");
  if (!blk_size) return fail(-2, "blk_size is NULL");
  if (!colptr) return fail(-3, "colptr is NULL");
  if (!rowidx) return fail(-4, "rowidx is NULL");
  if (dtype != DD_REAL64 && dtype != DD_COMPLEX128) return fail(-5, "dtype must be DD_REAL64 or DD_COMPLEX128");
  if (!out) return fail(-7, "out is NULL");
  std::string msg = validate_pattern(nblk, blk_size, colptr, rowidx);
  if (!msg.empty()) return fail(DD_ERR_PATTERN, msg);
  for (int64_t j = 0; j < nblk; ++j)
    if (blk_size[j] > (dtype == DD_COMPLEX128 ? K1_MAX_BLOCK_CPLX : K1_MAX_BLOCK_REAL))
      return fail(DD_ERR_PATTERN, "interface size " + std::to_string(blk_size[j]) + " exceeds the supported maximum " +
                                      std::to_string(dtype == DD_COMPLEX128 ? K1_MAX_BLOCK_CPLX : K1_MAX_BLOCK_REAL) +
                                      (dtype == DD_COMPLEX128 ? " (complex)" : " (real)"));
  dd_aux_options opt;
  dd_aux_default_options(&opt);
  if (opt_in) opt = *opt_in;
  if (opt.order < DD_ORDER_AUTO || opt.order > DD_ORDER_USER) return fail(-6, "invalid order option");
  if (opt.refine_steps < 0) return fail(-6, "refine_steps must be >= 0");
  if (!(opt.refine_tol >= 0)) return fail(-6, "refine_tol must be >= 0");
  if (opt.perturb && !(opt.perturb_tau > 0 && opt.perturb_tau < 1)) return fail(-6, "perturb needs 0 < perturb_tau < 1");

  dd_aux_handle_s* h = new (std::nothrow) dd_aux_handle_s();
  if (!h) return fail(DD_ERR_INTERNAL, "out of host memory");
  h->dtype = dtype;
  h->cplx = dtype == DD_COMPLEX128;
  h->opt = opt;
  h->opt.user_order = nullptr;
  h->blk_size.assign(blk_size, blk_size + nblk);
  h->colptr.assign(colptr, colptr + nblk + 1);
  h->rowidx.assign(rowidx, rowidx + colptr[nblk]);
  h->nnzb_in = colptr[nblk];
  h->g = graph_from_pattern(nblk, blk_size, colptr, rowidx);
  const int N = (int)nblk;
  h->odof_blk.assign(N + 1, 0);
  for (int i = 0; i < N; ++i) h->odof_blk[i + 1] = h->odof_blk[i] + blk_size[i];
  h->n = h->odof_blk[N];

  const bool verbose = getenv("DD_AUX_VERBOSE") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    auto now = std::chrono::steady_clock::now();
    if (verbose) fprintf(stderr, "[dd_aux_analyze] %-14s %8.3f s\n", what, std::chrono::duration<double>(now - tprev).count());
    tprev = now;
  };
  // ---------------------------------------------------------------- ordering (reading L8)
  const int NE = (int)(nblk - n_schur);  // eliminated blocks: ids [0, NE)
  h->n_schur = n_schur;
  h->n_elim = NE;
  Graph ge;                               // the block graph of the eliminated blocks
  if (n_schur > 0) {
    ge.n = NE;
    ge.adj.assign(NE, {});
    ge.w.assign(h->g.w.begin(), h->g.w.begin() + NE);
    for (int v = 0; v < NE; ++v)
      for (int u : h->g.adj[v])
        if (u < NE) ge.adj[v].push_back(u);
  }
  const Graph& go = n_schur > 0 ? ge : h->g;
  std::vector<int> order;
  if (opt.order == DD_ORDER_USER) {
    if (!opt.user_order) {
      delete h;
      return fail(-6, "DD_ORDER_USER needs user_order");
    }
    order.assign(opt.user_order, opt.user_order + NE);
    std::vector<char> seen(NE, 0);
    for (int v : order) {
      if (v < 0 || v >= NE || seen[v]) {
        delete h;
        return fail(-6, n_schur ? "user_order is not a permutation of the eliminated blocks [0, nblk - n_schur)"
                                : "user_order is not a permutation");
      }
      seen[v] = 1;
    }
    h->order_used = DD_ORDER_USER;
  } else if (opt.order == DD_ORDER_NATURAL) {
    order.resize(NE);
    for (int i = 0; i < NE; ++i) order[i] = i;
    h->order_used = DD_ORDER_NATURAL;
  } else if (opt.order == DD_ORDER_MINDEG) {
    order = order_mindeg(go);
    h->order_used = DD_ORDER_MINDEG;
  } else if (opt.order == DD_ORDER_ND) {
    order = order_nd(go);
    h->order_used = DD_ORDER_ND;
  } else {
    auto md = order_mindeg(go);
    auto nd = order_nd(go);
    if (order_flops(go, nd) < order_flops(go, md)) {
      order = nd;
      h->order_used = DD_ORDER_ND;
    } else {
      order = md;
      h->order_used = DD_ORDER_MINDEG;
    }
  }
  for (int k = NE; k < N; ++k) order.push_back(k);  // kept blocks last, ascending id
  mark("ordering");
  h->S = symbolic_from_order(h->g, order);
  if (n_schur > 0) {  // only eliminated positions are scheduled: drop the kept ones from the levels
    Symbolic& Sm = h->S;
    int nl = 0;
    for (int t = 0; t < NE; ++t) nl = std::max(nl, Sm.level[t] + 1);
    Sm.level_nodes.assign(nl, {});
    for (int t = 0; t < NE; ++t) Sm.level_nodes[Sm.level[t]].push_back(t);
    Sm.nlevels = nl;
  }
  const Symbolic& S = h->S;

  mark("symbolic");
  // ---------------------------------------------------------------- layout
  const int64_t mu = h->cplx ? 4 : 1;
  {  // algorithmic flops of the eliminated positions (all of them unless Schur mode)
    double ff = 0, fs = 0;
    for (int t = 0; t < NE; ++t) {
      const double sv = (double)blk_size[S.order[t]];
      double rv = 0;
      for (int u : S.st[t]) rv += (double)blk_size[S.order[u]];
      ff += sv * sv * sv / 3.0 + rv * sv * sv + rv * rv * sv;
      fs += 2.0 * (sv * sv + 2.0 * rv * sv);
    }
    h->flops_factor = mu * ff;
    h->flops_solve = mu * fs;
  }
  h->nodes.resize(N);
  std::vector<int32_t> st_pos, st_row;
  int64_t ydof = 0, panel_off = 0;
  for (int t = 0; t < N; ++t) {
    NodeDev& nd = h->nodes[t];
    const int blk = S.order[t];
    nd.blk = blk;
    nd.s = (int32_t)blk_size[blk];
    nd.sp = (int32_t)pad2(nd.s);
    nd.st0 = (int32_t)st_pos.size();
    nd.nst = (int32_t)S.st[t].size();
    int64_t ro = nd.sp, r = 0;
    for (int u : S.st[t]) {
      st_pos.push_back(u);
      st_row.push_back((int32_t)ro);
      int64_t su = blk_size[S.order[u]];
      ro += pad2(su);
      r += su;
    }
    nd.rp = (int32_t)(ro - nd.sp);
    nd.ld = (int32_t)pad8(ro);
    nd.ldw = (int32_t)pad8(std::max<int64_t>(nd.rp, 2));
    nd.panel = panel_off;
    panel_off += (int64_t)nd.ld * nd.s;
    nd.ydof = ydof;
    ydof += nd.sp;
    nd.odof = h->odof_blk[blk];
    if (t < NE) {
      h->max_front = std::max<int64_t>(h->max_front, nd.s + r);
      h->max_s = std::max(h->max_s, nd.s);
      h->value_bytes += (double)(nd.s * (int64_t)nd.s + r * nd.s) * (h->cplx ? 16.0 : 8.0);
    }
  }
  h->n_pad = ydof;
  h->r0 = NE < N ? h->nodes[NE].ydof : ydof;
  int64_t off = panel_off;
  for (int t = 0; t < N; ++t) {
    NodeDev& nd = h->nodes[t];
    nd.linv = off;
    off += (int64_t)((nd.s + TB - 1) / TB) * TB * TB;
  }
  for (int t = 0; t < N; ++t) {  // full inverses L_tt^{-1} (lower, unit diagonal)
    NodeDev& nd = h->nodes[t];
    nd.ldi = (int32_t)pad8(nd.s);
    nd.inv = off;
    off += (int64_t)nd.ldi * nd.s;
  }
  h->d_off = off;
  off += pad8(h->n_pad);
  h->e_off = off;
  off += pad8(h->n_pad);
  h->nA = (off + 31) & ~int64_t(31);
  // level workspace (W panels and K1 scratch) -- reused by every level
  for (int l = 0; l < S.nlevels; ++l) {
    int64_t w = 0, k1 = 0;
    for (int t : S.level_nodes[l]) {
      NodeDev& nd = h->nodes[t];
      nd.w = w;
      w += (int64_t)nd.ldw * nd.s;
      nd.k1w = k1;
      k1 += (int64_t)nd.sp * K1NB_MAX;
    }
    h->nW = std::max(h->nW, w);
    h->nK1 = std::max(h->nK1, k1);
    h->max_width = std::max<int64_t>(h->max_width, (int64_t)S.level_nodes[l].size());
  }
  h->nW = (h->nW + 31) & ~int64_t(31);
  h->nK1 = (h->nK1 + 31) & ~int64_t(31);

  mark("layout");
  // ---------------------------------------------------------------- per-level tables
  auto row_in_panel = [&](int j, int i) -> int {  // row offset of block at position i inside panel j
    if (i == j) return 0;
    const NodeDev& nj = h->nodes[j];
    auto b = st_pos.begin() + nj.st0, e = b + nj.nst;
    auto it = std::lower_bound(b, e, i);
    return st_row[it - st_pos.begin()];
  };
  // reverse index: for node t, the earlier panels k with t in struct(k)
  std::vector<std::vector<std::pair<int, int>>> appears(N);
  for (int k = 0; k < N; ++k)
    for (int q = 0; q < h->nodes[k].nst; ++q) appears[st_pos[h->nodes[k].st0 + q]].push_back({k, st_row[h->nodes[k].st0 + q]});

  std::vector<int32_t> lvl_nodes;
  std::vector<Strip> strips;
  std::vector<Tile> k2items;
  std::vector<RowPerm> rowperm;
  std::vector<UpdTarget> targets;
  std::vector<UpdContrib> contribs;
  std::vector<int64_t> tprefix;  // per target: tiles before it within its level
  std::vector<SolveTarget> ftargets;
  std::vector<SolveContrib> fcontribs;
  std::vector<int2> btiles;
  std::vector<DTile> dtiles, litems;
  {
    const char* ev = getenv("DD_AUX_K3CFG");
    // default tile config per scalar type (measured on B200): real 64x64 at
    // 4 CTAs/SM with per-warp masking; complex 64x32, 2 stages, 4 CTAs/SM: 3M (Gauss) by default,
    // 4M with per-warp masking when complex_3m = 0; all with 16-byte fragment loads (VEC)
    h->k3cfg = ev ? atoi(ev) : (h->cplx ? (opt.complex_3m ? 9 : 10) : 13);
#ifndef DD_AUX_AB
    if (h->k3cfg != 9 && h->k3cfg != 10 && h->k3cfg != 13) h->k3cfg = h->cplx ? (opt.complex_3m ? 9 : 10) : 13;
#endif
    h->m3 = h->cplx && opt.complex_3m;
    const char* la = getenv("DD_AUX_LOOKAHEAD");
    h->lookahead = la ? atoi(la) != 0 : true;
  }
  const int BM3 = k3_bm(h->cplx, h->k3cfg), BN3 = k3_bn(h->cplx, h->k3cfg), SBM = solve_bm(h->cplx);
  const int K2BM = 64;
  for (int l = 0; l < S.nlevels; ++l) {
    LevelRanges R{};
    const auto& L = S.level_nodes[l];
    R.n0 = (int)lvl_nodes.size();
    for (int t : L) lvl_nodes.push_back(t);
    R.n1 = (int)lvl_nodes.size();
    R.s0 = (int)strips.size();
    for (int t : L) {
      const NodeDev& nd = h->nodes[t];
      for (int r0 = 0; r0 < nd.rp; r0 += K2BM) strips.push_back(Strip{t, r0, std::min(K2BM, nd.rp - r0), 0});
    }
    R.s1 = (int)strips.size();
    R.k0 = (int)k2items.size();
    for (int t : L) {
      const NodeDev& nd = h->nodes[t];
      for (int tm = 0; tm * BM3 < nd.rp; ++tm)
        for (int tn = 0; tn * BN3 < nd.s; ++tn) k2items.push_back(Tile{t, tm, tn, 0});
    }
    R.k1 = (int)k2items.size();
    R.r0 = (int)rowperm.size();
    for (int t : L)
      for (auto& kr : appears[t]) rowperm.push_back(RowPerm{t, kr.first, kr.second, 0});
    R.r1 = (int)rowperm.size();
    // K3 targets: (i, j) in struct(k)^2, i at/after j, contributors in ascending position
    std::unordered_map<int64_t, int> tmap;
    std::vector<std::vector<UpdContrib>> tcon;
    std::vector<std::pair<int, int>> tij;
    for (int k : L) {
      const NodeDev& nk = h->nodes[k];
      for (int a = 0; a < nk.nst; ++a)
        for (int b = 0; b <= a; ++b) {
          int i = st_pos[nk.st0 + a], j = st_pos[nk.st0 + b];
          int64_t key = (int64_t)i * N + j;
          auto it = tmap.find(key);
          int id;
          if (it == tmap.end()) {
            id = (int)tij.size();
            tmap.emplace(key, id);
            tij.push_back({i, j});
            tcon.push_back({});
          } else {
            id = it->second;
          }
          tcon[id].push_back(UpdContrib{k, st_row[nk.st0 + a] - nk.sp, st_row[nk.st0 + b], 0});
        }
    }
    // K3 targets in launch order: (a) targets in panels of the NEXT level's nodes first (the
    // lookahead), then (b) the rest; each part sorted by K cost (sum of contributor sizes),
    // descending.  Tiles are implicit: tprefix[t] = tiles before target t (per level).
    std::vector<char> next(N, 0);
    if (l + 1 < S.nlevels)
      for (int t : S.level_nodes[l + 1]) next[t] = 1;
    // (K1 of level l+1 waits for K3a1 only: every update of a diagonal block is a (t, t) target)
    std::vector<std::pair<int64_t, int>> cost_a1, cost_a, cost_b;
    for (size_t id = 0; id < tij.size(); ++id) {
      int64_t kcost = 0;
      for (auto& c : tcon[id]) kcost += h->nodes[c.k].s;
      if (next[tij[id].second] && tij[id].first == tij[id].second) cost_a1.push_back({kcost, (int)id});
      else (next[tij[id].second] ? cost_a : cost_b).push_back({kcost, (int)id});
    }
    auto bycost = [](const std::pair<int64_t, int>& x, const std::pair<int64_t, int>& y) {
      return x.first != y.first ? x.first > y.first : x.second < y.second;
    };
    std::sort(cost_a1.begin(), cost_a1.end(), bycost);
    std::sort(cost_a.begin(), cost_a.end(), bycost);
    std::sort(cost_b.begin(), cost_b.end(), bycost);
    R.t0 = (int)targets.size();
    int64_t tiles_lvl = 0;
    auto emit = [&](const std::pair<int64_t, int>& cp) {
      const int id = cp.second;
      const int i = tij[id].first, j = tij[id].second;
      UpdTarget tg{};
      tg.j = j;
      tg.ro = row_in_panel(j, i);
      tg.M = h->nodes[i].s;
      tg.N = h->nodes[j].s;
      tg.c0 = (int)contribs.size();
      for (auto& c : tcon[id]) contribs.push_back(c);
      tg.c1 = (int)contribs.size();
      tg.diag = (i == j);
      int64_t nt = 0;
      const int ntm = (tg.M + BM3 - 1) / BM3, ntn = (tg.N + BN3 - 1) / BN3;
      for (int tm = 0; tm < ntm; ++tm) nt += tg.diag ? std::min(ntn, (tm * BM3 + BM3 - 1) / BN3 + 1) : ntn;
      tprefix.push_back(tiles_lvl);
      tiles_lvl += nt;
      targets.push_back(tg);
    };
    for (auto& cp : cost_a1) emit(cp);
    R.ta1 = (int)targets.size();
    R.tiles_a1 = tiles_lvl;
    for (auto& cp : cost_a) emit(cp);
    R.ta = (int)targets.size();
    R.tiles_a = tiles_lvl;
    for (auto& cp : cost_b) emit(cp);
    R.t1 = (int)targets.size();
    R.tiles_b = tiles_lvl - R.tiles_a;
    // forward-solve targets: y_i -= L_ik z_k over the level's contributors
    std::unordered_map<int, std::vector<SolveContrib>> fmap;
    std::vector<int> fo;
    for (int k : L) {
      const NodeDev& nk = h->nodes[k];
      for (int a = 0; a < nk.nst; ++a) {
        int i = st_pos[nk.st0 + a];
        if (!fmap.count(i)) fo.push_back(i);
        fmap[i].push_back(SolveContrib{k, st_row[nk.st0 + a]});
      }
    }
    R.f0 = (int)ftargets.size();
    for (int i : fo) {
      int c0 = (int)fcontribs.size();
      for (auto& c : fmap[i]) fcontribs.push_back(c);
      int c1 = (int)fcontribs.size();
      for (int tm = 0; tm * SBM < h->nodes[i].s; ++tm) ftargets.push_back(SolveTarget{i, tm, c0, c1});
    }
    R.f1 = (int)ftargets.size();
    R.b0 = (int)btiles.size();
    for (int t : L)
      if (h->nodes[t].nst > 0)
        for (int tm = 0; tm * SBM < h->nodes[t].s; ++tm) btiles.push_back(make_int2(t, tm));
    R.b1 = (int)btiles.size();
    {
      R.d0 = (int)dtiles.size();
      int64_t toff = 0;
      for (int t : L) {
        for (int tm = 0; tm * SBM < h->nodes[t].s; ++tm) dtiles.push_back(DTile{t, tm, toff});
        toff += h->nodes[t].sp;
      }
      h->nT = std::max<int64_t>(h->nT, toff);
      R.d1 = (int)dtiles.size();
      R.i0 = (int)litems.size();
      for (int t : L)
        for (int c = 0; c * TB < h->nodes[t].s; ++c) litems.push_back(DTile{t, c, 0});
      R.i1 = (int)litems.size();
    }
    {
      const double mu = h->cplx ? 4.0 : 1.0;
      R.fl_k1 = R.fl_k2 = R.fl_k3 = R.fl_diag = R.fl_upd = 0;
      R.max_s = 0;
      R.max_rp = 0;
      for (int t : L) {
        R.max_s = std::max(R.max_s, (int)h->nodes[t].s);
        R.max_rp = std::max(R.max_rp, (int)h->nodes[t].rp);
        double sv = h->nodes[t].s, rv = 0;
        for (int q = 0; q < h->nodes[t].nst; ++q) rv += h->nodes[st_pos[h->nodes[t].st0 + q]].s;
        R.fl_k1 += mu * sv * sv * sv / 3.0;
        R.fl_k2 += mu * rv * sv * sv;
        R.fl_k3 += mu * rv * rv * sv;
        R.fl_diag += mu * sv * sv;
        R.fl_upd += mu * 2.0 * rv * sv;
      }
    }
    h->lv.push_back(R);
  }
  mark("level tables");
  // K6 residual rows: block row I of the full symmetric A
  std::vector<std::vector<SpSeg>> rowsegs(N);
  for (int j = 0; j < N; ++j)
    for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p) {
      int i = rowidx[p];
      if (i == j) rowsegs[i].push_back(SpSeg{p, j, 2});
      else {
        rowsegs[i].push_back(SpSeg{p, j, 0});  // stored (i, j)
        rowsegs[j].push_back(SpSeg{p, i, 1});  // (j, i) = stored^T
      }
    }
  for (int j = 0; j < N; ++j)
    for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p)
      h->nnz_full += (double)blk_size[rowidx[p]] * blk_size[j] * (rowidx[p] == j ? 1.0 : 2.0);
  std::vector<SpRow> sprows;
  const int SPM = spmv_bm();
  for (int I = 0; I < N; ++I) {
    std::sort(rowsegs[I].begin(), rowsegs[I].end(), [](const SpSeg& a, const SpSeg& b) { return a.J < b.J; });
    int c0 = (int)h->spsegs.size();
    for (auto& sg : rowsegs[I]) h->spsegs.push_back(sg);
    int c1 = (int)h->spsegs.size();
    for (int tm = 0; tm * SPM < blk_size[I]; ++tm) sprows.push_back(SpRow{I, tm, c0, c1});
  }
  h->n_sprows = (int)sprows.size();

  mark("k6 tables");
  Blob& B = h->blob;
  h->off_nodes = B.put(h->nodes);
  h->off_stpos = B.put(st_pos);
  h->off_strow = B.put(st_row);
  h->off_lvlnodes = B.put(lvl_nodes);
  h->off_strips = B.put(strips);
  h->off_k2items = B.put(k2items);
  h->off_rowperm = B.put(rowperm);
  h->off_targets = B.put(targets);
  h->off_contribs = B.put(contribs);
  h->off_tiles = B.put(tprefix);
  h->off_ftargets = B.put(ftargets);
  h->off_fcontribs = B.put(fcontribs);
  h->off_btiles = B.put(btiles);
  h->off_dtiles = B.put(dtiles);
  h->off_litems = B.put(litems);
  h->off_sprows = B.put(sprows);
  h->off_blksize = B.put(h->blk_size);
  std::vector<int64_t> odof(h->odof_blk.begin(), h->odof_blk.end() - 1);
  h->off_odof = B.put(odof);
  h->off_spsegs = B.put(h->spsegs);
  if (n_schur > 0) {
    h->schur_target.assign(sin->target, sin->target + n_schur);
    h->schur_group.assign(sin->group, sin->group + n_schur);
    h->n_aux = sin->n_aux;
    h->aux_odof.assign(sin->n_aux, 0);
    for (int64_t I = 1; I < sin->n_aux; ++I) h->aux_odof[I] = h->aux_odof[I - 1] + sin->aux_size[I - 1];
    h->n_aux_dof = h->aux_odof[sin->n_aux - 1] + sin->aux_size[sin->n_aux - 1];
    const int rc = build_schur_tables(h);
    if (rc) {
      delete h;
      return rc;
    }
  }
  h->tables_bytes = align256(B.data.size());

  mark("blob");
  // ---------------------------------------------------------------- buffer sizes
  const int planes = h->cplx ? 2 : 1;
  size_t o = h->tables_bytes;
  h->off_arena = o;
  o = align256(o + (size_t)h->nA * planes * sizeof(double));
  h->off_ipiv = o;
  o = align256(o + (size_t)h->n_pad * 4);
  h->off_perm = o;
  o = align256(o + (size_t)h->n_pad * 4);
  h->off_gperm = o;
  o = align256(o + (size_t)h->n_pad * 4);
  h->off_ginv = o;
  o = align256(o + (size_t)h->n * 4);
  h->off_stats = o;
  o = align256(o + (size_t)N * 8 * 8);
  h->off_totals = o;
  o = align256(o + 16 * 8);
  h->off_norm = o;
  o = align256(o + 8);
  h->factor_bytes = o;
  size_t w = 0;
  h->w_off_W = w;  // two W buffers (level parity) for the lookahead
  w = align256(w + (size_t)h->nW * planes * sizeof(double) * 2);
  h->w_off_K1 = w;
  w = align256(w + (size_t)h->nK1 * planes * sizeof(double));
  h->w_off_load = w;
  w = align256(w + (size_t)h->nnzb_in * sizeof(LoadBlock));
  h->work_bytes = w;
  *out = h;
  return DD_OK;
}

extern "C" {

int dd_aux_analyze(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx,
                   int32_t dtype, const dd_aux_options* opt, dd_aux_handle_t* out) {
  return analyze_impl(nblk, blk_size, colptr, rowidx, dtype, opt, 0, nullptr, out);
}

int dd_aux_get_info(dd_aux_handle_t h, dd_aux_info* info) {
  if (!h) return fail(-1, "handle is NULL");
  if (!info) return fail(-2, "info is NULL");
  std::memset(info, 0, sizeof(*info));
  info->n = h->n;
  info->nblk = h->S.nblk;
  info->nnzb_in = h->nnzb_in;
  info->nnzb_filled = h->S.nblk + h->S.nnz_struct;
  info->n_levels = h->S.nlevels;
  info->max_front = h->max_front;
  info->max_level_width = h->max_width;
  info->flops_factor = h->flops_factor;
  info->flops_solve_per_rhs = h->flops_solve;
  info->factor_value_bytes = h->value_bytes;
  info->factor_bytes = h->factor_bytes;
  info->work_bytes = h->work_bytes;
  info->dtype = h->dtype;
  info->order_used = h->order_used;
  info->n_schur = h->n_schur;
  info->n_groups = h->n_schur ? (int64_t)h->grp_ptr.size() - 1 : 0;
  info->n_aux_dof = h->n_aux_dof;
  return DD_OK;
}

int dd_aux_get_order(dd_aux_handle_t h, int32_t* order) {
  if (!h) return fail(-1, "handle is NULL");
  if (!order) return fail(-2, "order is NULL");
  for (int t = 0; t < h->S.nblk; ++t) order[t] = h->S.order[t];
  return DD_OK;
}

int dd_aux_get_etree(dd_aux_handle_t h, int32_t* parent, int32_t* level, int64_t* nnz_struct) {
  if (!h) return fail(-1, "handle is NULL");
  for (int t = 0; t < h->S.nblk; ++t) {
    int blk = h->S.order[t];
    if (parent) parent[blk] = h->S.parent[t] < 0 ? -1 : h->S.order[h->S.parent[t]];
    if (level) level[blk] = h->S.level[t];
  }
  if (nnz_struct) *nnz_struct = h->S.nnz_struct;
  return DD_OK;
}

int dd_aux_get_struct(dd_aux_handle_t h, int64_t* st_ptr, int32_t* st_blk) {
  if (!h) return fail(-1, "handle is NULL");
  const int N = h->S.nblk;
  std::vector<int64_t> cnt(N + 1, 0);
  for (int t = 0; t < N; ++t) cnt[h->S.order[t] + 1] = (int64_t)h->S.st[t].size();
  for (int b = 0; b < N; ++b) cnt[b + 1] += cnt[b];
  if (st_ptr)
    for (int b = 0; b <= N; ++b) st_ptr[b] = cnt[b];
  if (st_blk)
    for (int t = 0; t < N; ++t) {
      int64_t o = cnt[h->S.order[t]];
      for (int u : h->S.st[t]) st_blk[o++] = h->S.order[u];
    }
  return DD_OK;
}

// The solve's column-indexed grids put the right-hand-side tile on gridDim.y (<= 65535): a call
// with more columns runs in chunks of SOLVE_MAX_COLS (columns are independent, and every kernel's
// per-column result is independent of how many columns are solved together, so chunking is
// bitwise neutral).
static constexpr int64_t SOLVE_MAX_COLS = 32768;

int dd_aux_solve_work_bytes(dd_aux_handle_t h, int64_t nrhs, size_t* bytes) {
  if (!h) return fail(-1, "handle is NULL");
  if (nrhs < 0) return fail(-2, "nrhs must be >= 0");
  if (!bytes) return fail(-3, "bytes is NULL");
  nrhs = std::min(nrhs, SOLVE_MAX_COLS);
  const int planes = h->cplx ? 2 : 1;
  const size_t ldy = (size_t)pad8(h->n_pad);
  size_t w = align256(ldy * (size_t)nrhs * planes * sizeof(double));   // y
  w += align256((size_t)h->n * (size_t)nrhs * planes * sizeof(double));  // saved B (refinement)
  w += align256((size_t)nrhs * sizeof(double)) + 256;                    // per-column berr + flag
  w += align256(bupd_part_bytes(h->cplx, (int)nrhs));                    // backward split-K partials
  w += align256((size_t)pad8(std::max<int64_t>(h->nT, 2)) * nrhs * planes * sizeof(double));  // level buffer T
  w += align256(bupd_cnt_bytes(h->cplx, (int)nrhs));                                            // split-K counters
  *bytes = w;
  return DD_OK;
}

int dd_aux_factor(dd_aux_handle_t h, const void* d_vals, const int64_t* val_offset, void* d_factor, void* d_work,
                  void* stream, dd_aux_factor_info* finfo) {
  if (!h) return fail(-1, "handle is NULL");
  if (!d_vals) return fail(-2, "d_vals is NULL");
  if (!val_offset) return fail(-3, "val_offset is NULL");
  if (!d_factor || ((uintptr_t)d_factor & 255)) return fail(-4, "d_factor is NULL or not 256-byte aligned");
  if (!d_work || ((uintptr_t)d_work & 255)) return fail(-5, "d_work is NULL or not 256-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const bool C = h->cplx;
  const int N = h->S.nblk;
  uint8_t* F = (uint8_t*)d_factor;
  uint8_t* Wb = (uint8_t*)d_work;
  h->factored = false;
  h->norm_valid = false;

  // ---- tables: fill the value offsets of the K6 segments, upload everything
  {
    SpSeg* sp = (SpSeg*)(h->blob.data.data() + h->off_spsegs);
    for (size_t q = 0; q < h->spsegs.size(); ++q) sp[q].voff = val_offset[h->spsegs[q].voff];
  }
  CUDA_TRY(cudaMemcpyAsync(F, h->blob.data.data(), h->blob.data.size(), cudaMemcpyHostToDevice, st));
  if (h->n_schur > 0) {  // identity row maps of the kept (never pivoted) blocks
    CUDA_TRY(cudaMemcpyAsync(F + h->off_gperm + (size_t)h->r0 * 4, h->kept_gperm.data(), h->kept_gperm.size() * 4,
                             cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(F + h->off_ginv + (size_t)(h->n - (int64_t)h->kept_ginv.size()) * 4, h->kept_ginv.data(),
                             h->kept_ginv.size() * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(F + h->off_perm + (size_t)h->r0 * 4, h->kept_perm.data(), h->kept_perm.size() * 4,
                             cudaMemcpyHostToDevice, st));
  }
  // ---- K0 load list
  std::vector<LoadBlock> lbs;
  lbs.reserve(h->nnzb_in);
  int64_t max_elems = 0;
  for (int j = 0; j < N; ++j)
    for (int64_t p = h->colptr[j]; p < h->colptr[j + 1]; ++p) {
      int i = h->rowidx[p];
      int pi = h->S.pos[i], pj = h->S.pos[j];
      LoadBlock L{};
      L.voff = val_offset[p];
      L.rows = (int32_t)h->blk_size[i];
      L.cols = (int32_t)h->blk_size[j];
      L.diag = (i == j);
      if (pi >= pj) {  // stored (i,j) in panel pj at the rows of i
        const NodeDev& nj = h->nodes[pj];
        int ro = 0;
        if (i != j) {
          auto b = h->S.st[pj].begin();
          auto it = std::lower_bound(b, h->S.st[pj].end(), pi);
          const int32_t* strow = (const int32_t*)(h->blob.data.data() + h->off_strow);
          ro = strow[nj.st0 + (it - b)];
        }
        L.dst = nj.panel + ro;
        L.ld = nj.ld;
        L.trans = 0;
      } else {  // i eliminated first: block (j, i) = stored^T lives in panel pi at the rows of j
        const NodeDev& ni = h->nodes[pi];
        auto b = h->S.st[pi].begin();
        auto it = std::lower_bound(b, h->S.st[pi].end(), pj);
        const int32_t* strow = (const int32_t*)(h->blob.data.data() + h->off_strow);
        L.dst = ni.panel + strow[ni.st0 + (it - b)];
        L.ld = ni.ld;
        L.trans = 1;
      }
      max_elems = std::max<int64_t>(max_elems, (int64_t)L.rows * L.cols);
      lbs.push_back(L);
    }
  CUDA_TRY(cudaMemcpyAsync(Wb + h->w_off_load, lbs.data(), lbs.size() * sizeof(LoadBlock), cudaMemcpyHostToDevice, st));

  double* arena = (double*)(F + h->off_arena);
  const int64_t aim = C ? h->nA : 0;
  double* work = (double*)Wb;
  const int64_t wim = C ? h->nW : 0;
  double* k1work = (double*)(Wb + h->w_off_K1);
  const int64_t k1im = C ? h->nK1 : 0;
  const NodeDev* dnodes = (const NodeDev*)(F + h->off_nodes);

  // timing events owned by the handle (no leak on an early error return)
  for (auto* e : {&h->t0, &h->t1, &h->t2})
    if (!*e) CUDA_TRY(cudaEventCreate(e));
  cudaEvent_t e0 = h->t0, e1 = h->t1, e2 = h->t2;
  cudaEventRecord(e0, st);
  // ---- a1: zero the arena, load the caller's blocks
  CUDA_TRY(cudaMemsetAsync(arena, 0, (size_t)h->nA * (C ? 2 : 1) * sizeof(double), st));
  {
    TraceScope ts(h, DD_PH_LOAD, 0.0, st);
    launch_load(C, (const double*)d_vals, (const LoadBlock*)(Wb + h->w_off_load), (int)lbs.size(), max_elems, arena,
                aim, st);
  }
  LAUNCH_CHECK("k0_load");
  cudaEventRecord(e1, st);

  K1Args k1{};
  k1.nd = dnodes;
  k1.arena = arena;
  k1.aim = aim;
  k1.work = k1work;
  k1.wim = k1im;
  k1.perm = (int*)(F + h->off_perm);
  k1.ipiv = (int*)(F + h->off_ipiv);
  k1.gperm = (int*)(F + h->off_gperm);
  k1.ginv = (int*)(F + h->off_ginv);
  k1.d_off = h->d_off;
  k1.e_off = h->e_off;
  k1.stats = (int64_t*)(F + h->off_stats);
  k1.nb = getenv("DD_AUX_K1NB") ? atoi(getenv("DD_AUX_K1NB")) : 0;
  k1.fullw = getenv("DD_AUX_K1FULLW") ? atoi(getenv("DD_AUX_K1FULLW")) : 1;
  int64_t* totals_d = (int64_t*)(F + h->off_totals);
  unsigned long long* maxL_d = (unsigned long long*)(totals_d + 8);
  unsigned long long* norm_d = (unsigned long long*)(F + h->off_norm);
  k1.perturb_tau = h->opt.perturb ? h->opt.perturb_tau : 0.0;
  k1.normA = norm_d;
  k1.maxL = maxL_d;
  const int nLv = (int)h->lv.size();
  if (!h->side) {
    int lo, hi;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi));
    CUDA_TRY(cudaEventCreateWithFlags(&h->evLoad, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithPriority(&h->side2, cudaStreamNonBlocking, hi));
    CUDA_TRY(cudaEventCreateWithFlags(&h->evR, cudaEventDisableTiming));
  }
  while ((int)h->evA.size() < nLv) {
    cudaEvent_t a, a2, b, kk;
    CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&a2, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&kk, cudaEventDisableTiming));
    h->evA.push_back(a);
    h->evA2.push_back(a2);
    h->evB.push_back(b);
    h->evK.push_back(kk);
  }
  // a2-a6 as one enqueue function of the stream, so it can be captured once into a CUDA graph
  // (options.use_graphs; SURVEY.md §8(a) a5 "graph-capture the whole level sequence")
  auto levels_body = [&](cudaStream_t st) -> int {
    CUDA_TRY(cudaMemsetAsync(k1.ipiv, 0, (size_t)h->n_pad * 4, st));
    if (h->n_schur > 0)  // kept nodes are never factored: zero stats
      CUDA_TRY(cudaMemsetAsync(F + h->off_stats, 0, (size_t)N * 8 * 8, st));
    CUDA_TRY(cudaMemsetAsync(totals_d, 0, 16 * sizeof(int64_t), st));
    if (k1.perturb_tau > 0) {  // reading L4 (opt-in): ||A||_inf of the caller's blocks before K1
      CUDA_TRY(cudaMemsetAsync(norm_d, 0, sizeof(unsigned long long), st));
      SpmvArgs sa{};
      sa.rows = (const SpRow*)(F + h->off_sprows);
      sa.segs = (const SpSeg*)(F + h->off_spsegs);
      sa.blk_size = (const int64_t*)(F + h->off_blksize);
      sa.odof = (const int64_t*)(F + h->off_odof);
      sa.vals = (const double*)d_vals;
      launch_norm_a(C, sa, h->n_sprows, norm_d, st);
      LAUNCH_CHECK("k_norm_a");
    }
    RowpermArgs rp{(const RowPerm*)(F + h->off_rowperm), dnodes, arena, aim, k1.perm};
    K2Args k2{maxL_d, (const Tile*)(F + h->off_k2items), (const Strip*)(F + h->off_strips), dnodes, arena, aim, work,
              wim, k1.perm, k1.ipiv, h->d_off, h->e_off};
    K3Args k3{(const UpdTarget*)(F + h->off_targets), (const int64_t*)(F + h->off_tiles), 0, 0,
              (const UpdContrib*)(F + h->off_contribs), dnodes, arena, aim, work, wim, 0,
              (unsigned long long*)(totals_d + 9)};
    static const bool k3p = getenv("DD_AUX_K3PERSIST") && atoi(getenv("DD_AUX_K3PERSIST"));  // A/B
    const int* lvlnodes = (const int*)(F + h->off_lvlnodes);
    // ---- a2-a5: level-scheduled factorization with a one-level lookahead.
    // Main stream st: K3a(l) [targets in panels of level l+1] -> K3b(l) [the rest].
    // Side stream (high priority): K1 / rowperm / K2 of level l+1 as soon as K3a(l) is done, so
    // the sequential diagonal factorizations overlap the bulk Schur update of level l.
    // W is double-buffered by level parity (K2(l+1) writes while K3b(l) still reads W(l)).
    const int nL = (int)h->lv.size();
    cudaStream_t sd = h->lookahead ? h->side : st;
    const size_t wpar = (size_t)h->nW * (C ? 2 : 1);  // elements per parity buffer
    auto diag_phase = [&](int l) -> int {              // K1 + rowperm + K2 of level l on the side stream
      const LevelRanges& R = h->lv[l];
      h->cur_level = l;
      k1.nodes = lvlnodes + R.n0;
      {
        TraceScope ts(h, DD_PH_K1, R.fl_k1, sd);
        launch_k1(C, k1, R.n1 - R.n0, R.max_s, sd);
      }
      LAUNCH_CHECK("k1_diag_bk");
      CUDA_TRY(cudaEventRecord(h->evK[l], sd));  // the level's in-block permutations are final
      {
        LinvArgs li{(const DTile*)(F + h->off_litems) + R.i0, dnodes, arena, aim};
        double fl = 0;
        for (int q = R.n0; q < R.n1; ++q) {
          const double sv = h->nodes[((const int*)(h->blob.data.data() + h->off_lvlnodes))[q]].s;
          fl += (C ? 4.0 : 1.0) * sv * sv * sv / 3.0;
        }
        TraceScope ts(h, DD_PH_LINV, fl, sd);
        launch_linv(C, li, R.i1 - R.i0, sd);
      }
      LAUNCH_CHECK("k_linv");
      return DD_OK;
    };
    // rowperm + K2 of level l: need every K3 update of level l-1 into level l's panels (K3a2:
    // it reads the rows of block t in earlier panels, which rowperm permutes)
    // k_rowperm (rows of block t inside EARLIER panels) and K2 (panel t itself) touch disjoint
    // rows: rowperm runs on a third stream, gated by the same event (ready), joined at the end
    static const bool rp3 = !(getenv("DD_AUX_ROWPERM3") && atoi(getenv("DD_AUX_ROWPERM3")) == 0);  // A/B
    cudaStream_t s3 = h->lookahead ? (rp3 ? h->side2 : sd) : st;
    auto panel_phase = [&](int l, cudaEvent_t ready) -> int {
      const LevelRanges& R = h->lv[l];
      h->cur_level = l;
      RowpermArgs r = rp;
      r.list = rp.list + R.r0;
      if (R.r1 > R.r0) {
        if (s3 != st && s3 != sd) {  // needs the level's K1 (perm) and every K3 read of those rows (ready)
          CUDA_TRY(cudaStreamWaitEvent(s3, ready, 0));
          CUDA_TRY(cudaStreamWaitEvent(s3, h->evK[l], 0));
        }
        TraceScope ts(h, DD_PH_ROWPERM, 0.0, s3);
        launch_rowperm(C, r, R.r1 - R.r0, h->max_s, s3);
      }
      LAUNCH_CHECK("k_rowperm");
      K2Args a2 = k2;
      a2.strips = k2.strips + R.s0;
      a2.items = k2.items + R.k0;
      a2.work = work + (l & 1) * wpar;
      if (R.s1 > R.s0) {
        TraceScope ts(h, DD_PH_K2, R.fl_k2, sd);
        launch_k2(C, h->k3cfg, a2, R.k1 - R.k0, R.s1 - R.s0, R.max_s, sd);
      }
      LAUNCH_CHECK("k2_panel");
      CUDA_TRY(cudaEventRecord(h->evB[l], sd));
      return DD_OK;
    };
    CUDA_TRY(cudaEventRecord(h->evLoad, st));
    CUDA_TRY(cudaStreamWaitEvent(sd, h->evLoad, 0));
    if (nL > 0) {
      int rc = diag_phase(0);
      if (!rc) rc = panel_phase(0, h->evLoad);
      if (rc) return rc;
    }
    for (int l = 0; l < nL; ++l) {
      const LevelRanges& R = h->lv[l];
      h->cur_level = l;
      CUDA_TRY(cudaStreamWaitEvent(st, h->evB[l], 0));
      K3Args a3 = k3;
      a3.work = work + (l & 1) * wpar;
      a3.targets = k3.targets + R.t0;
      a3.tprefix = k3.tprefix + R.t0;
      // K3a1: the next level's diagonal blocks first, so its K1 starts while K3a2 / K3b run
      a3.ntargets = R.ta1 - R.t0;
      a3.tile0 = 0;
      const int64_t tiles_a2 = R.tiles_a - R.tiles_a1;
      if (R.tiles_a1 > 0) {
        TraceScope ts(h, DD_PH_K3, (tiles_a2 > 0 || R.tiles_b > 0) ? 0.0 : R.fl_k3, st);
        launch_k3(C, h->k3cfg, a3, (int)R.tiles_a1, st, k3p);
      }
      LAUNCH_CHECK("k3_update");
      CUDA_TRY(cudaEventRecord(h->evA[l], st));
      if (l + 1 < nL) {
        CUDA_TRY(cudaStreamWaitEvent(sd, h->evA[l], 0));
        int rc = diag_phase(l + 1);
        if (rc) return rc;
      }
      // K3a2: the rest of the next level's panels
      a3.targets = k3.targets + R.ta1;
      a3.tprefix = k3.tprefix + R.ta1;
      a3.ntargets = R.ta - R.ta1;
      a3.tile0 = R.tiles_a1;
      h->cur_level = l;
      if (tiles_a2 > 0) {
        TraceScope ts(h, DD_PH_K3, R.tiles_b > 0 ? 0.0 : R.fl_k3, st);
        launch_k3(C, h->k3cfg, a3, (int)tiles_a2, st, k3p);
      }
      LAUNCH_CHECK("k3_update");
      CUDA_TRY(cudaEventRecord(h->evA2[l], st));
      if (l + 1 < nL) {
        CUDA_TRY(cudaStreamWaitEvent(sd, h->evA2[l], 0));
        int rc = panel_phase(l + 1, h->evA2[l]);
        if (rc) return rc;
      }
      a3.targets = k3.targets + R.ta;
      a3.tprefix = k3.tprefix + R.ta;
      a3.ntargets = R.t1 - R.ta;
      a3.tile0 = R.tiles_a;
      h->cur_level = l;
      if (R.tiles_b > 0) {
        TraceScope ts(h, DD_PH_K3, R.fl_k3, st);
        launch_k3(C, h->k3cfg, a3, (int)R.tiles_b, st, k3p);
      }
      LAUNCH_CHECK("k3_update");
    }
    h->cur_level = -1;
    if (s3 != st && s3 != sd) {  // join the rowperm stream (the solve reads the permuted rows)
      CUDA_TRY(cudaEventRecord(h->evR, s3));
      CUDA_TRY(cudaStreamWaitEvent(st, h->evR, 0));
    }
    // ---- a6: statistics
      {
      TraceScope ts(h, DD_PH_STATS, 0.0, st);
      launch_k4((const int64_t*)(F + h->off_stats), N, k1.gperm, totals_d, st);
    }
    LAUNCH_CHECK("k4_stats");
    return DD_OK;
  };
  // on an error part-way through, join the side streams into the caller's stream before returning,
  // so no queued lookahead kernel can outlive the caller's buffers (the caller may free them)
  auto levels = [&](cudaStream_t st) -> int {
    const int rc = levels_body(st);
    if (rc && h->lookahead)
      for (cudaStream_t x : {h->side, h->side2}) {
        cudaEventRecord(h->evR, x);
        cudaStreamWaitEvent(st, h->evR, 0);
      }
    return rc;
  };
  {
    const std::vector<uintptr_t> key = {(uintptr_t)d_factor, (uintptr_t)d_work};
    int rc = run_graph(h, h->gfactor, key, levels, st);
    if (rc) return rc;
  }
  cudaEventRecord(e2, st);
  int64_t totals[16] = {0};
  CUDA_TRY(cudaMemcpyAsync(totals, totals_d, 9 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms_load = 0, ms_fac = 0;
  cudaEventElapsedTime(&ms_load, e0, e1);
  cudaEventElapsedTime(&ms_fac, e1, e2);
  if (finfo) {
    finfo->npos = C ? 0 : totals[0];
    finfo->nneg = C ? 0 : totals[1];
    finfo->nzero = C ? 0 : totals[2];
    finfo->n2x2 = totals[3];
    finfo->nswaps = totals[4];
    finfo->first_zero_pivot = totals[5];
    finfo->ms_load = ms_load;
    finfo->ms_factor = ms_fac;
    finfo->nperturbed = totals[6];
    finfo->nonfinite = totals[7];
    double ml;
    std::memcpy(&ml, &totals[8], sizeof(double));
    finfo->max_abs_L = ml;
  }
  h->factored = true;
  h->factored_ptr = d_factor;
  h->singular = totals[5] != 0;
  if (h->opt.perturb) h->norm_valid = true;  // ||A||_inf of these values is on the device now
  return totals[7] ? DD_NONFINITE : (h->singular ? DD_ZERO_PIVOT : DD_OK);
}

enum { SW_FWD = 1, SW_D = 2, SW_BWD = 4, SW_ALL = 7 };

// phases: SW_FWD forward sweep (levels ascending), SW_D the D^{-1} solve, SW_BWD backward sweep;
// a Schur-mode handle's levels hold only its eliminated positions (kept rows are read / written
// by the update kernels as struct rows, never solved)
static int solve_sweep(dd_aux_handle_t h, const uint8_t* F, double* y, int64_t yim, int64_t ldy, int nrhs,
                       cudaStream_t st, double* part, double* T, const int* flag = nullptr, int phases = SW_ALL,
                       int* cnt = nullptr) {
  // with a device flag the sweep may be skipped: its flops are not counted (conservative trace)
  const double fs = flag ? 0.0 : 1.0;
  const bool C = h->cplx;
  SolveArgs a{};
  a.nd = (const NodeDev*)(F + h->off_nodes);
  a.arena = (const double*)(F + h->off_arena);
  a.aim = C ? h->nA : 0;
  a.y = y;
  a.yim = yim;
  a.ldy = ldy;
  a.nrhs = nrhs;
  a.ftargets = (const SolveTarget*)(F + h->off_ftargets);
  a.fcontribs = (const SolveContrib*)(F + h->off_fcontribs);
  a.btiles = (const int2*)(F + h->off_btiles);
  a.st_pos = (const int*)(F + h->off_stpos);
  a.st_row = (const int*)(F + h->off_strow);
  a.ipiv = (const int*)(F + h->off_ipiv);
  a.d_off = h->d_off;
  a.e_off = h->e_off;
  a.nrows = h->n_pad;
  a.flag = flag;
  a.dtiles = (const DTile*)(F + h->off_dtiles);
  a.T = T;
  a.cnt = cnt;
  a.ldT = pad8(std::max<int64_t>(h->nT, 2));
  a.Tim = C ? a.ldT * nrhs : 0;
  const int* lvlnodes = (const int*)(F + h->off_lvlnodes);
  for (int l = 0; l < (int)h->lv.size() && (phases & SW_FWD); ++l) {
    const LevelRanges& R = h->lv[l];
    h->cur_level = l;
    SolveArgs b = a;
    b.nodes = lvlnodes + R.n0;
    b.dtiles = a.dtiles + R.d0;
    {
      TraceScope ts(h, DD_PH_FDIAG, R.fl_diag * nrhs * fs, st);
      launch_diag_gemm(C, h->m3, false, b, R.d1 - R.d0, st);
    }
    LAUNCH_CHECK("k_diag_g(fwd)");
    b.ftargets = a.ftargets + R.f0;
    if (R.f1 > R.f0) {
      TraceScope ts(h, DD_PH_FUPD, R.fl_upd * nrhs * fs, st);
      launch_fupd(C, h->m3, b, R.f1 - R.f0, st);
    }
    LAUNCH_CHECK("k_fupd");
  }
  if (phases & SW_D) {
    TraceScope ts(h, DD_PH_DSOLVE, 0.0, st);
    h->cur_level = -1;
    launch_dsolve(C, a, st);
  }
  LAUNCH_CHECK("k_dsolve");
  for (int l = (int)h->lv.size() - 1; l >= 0 && (phases & SW_BWD); --l) {
    const LevelRanges& R = h->lv[l];
    h->cur_level = l;
    SolveArgs b = a;
    b.btiles = a.btiles + R.b0;
    if (R.b1 > R.b0) {
      TraceScope ts(h, DD_PH_BUPD, R.fl_upd * nrhs * fs, st);
      launch_bupd(C, h->m3, b, R.b1 - R.b0, R.max_rp, part, st);
    }
    LAUNCH_CHECK("k_bupd");
    b.nodes = lvlnodes + R.n0;
    b.dtiles = a.dtiles + R.d0;
    {
      TraceScope ts(h, DD_PH_BDIAG, R.fl_diag * nrhs * fs, st);
      launch_diag_gemm(C, h->m3, true, b, R.d1 - R.d0, st);
    }
    LAUNCH_CHECK("k_diag_g(bwd)");
  }
  h->cur_level = -1;
  return DD_OK;
}

int dd_aux_solve(dd_aux_handle_t h, const void* d_factor, const void* d_vals, int64_t nrhs, void* d_B, int64_t ldb,
                 void* d_work, void* stream) {
  if (!h) return fail(-1, "handle is NULL");
  if (!d_factor) return fail(-2, "d_factor is NULL");
  if (nrhs < 0) return fail(-4, "nrhs must be >= 0");
  if (nrhs == 0) return DD_OK;
  if (!d_B) return fail(-5, "d_B is NULL");
  if (ldb < h->n) return fail(-6, "ldb < n");
  if (!d_work || ((uintptr_t)d_work & 255)) return fail(-7, "d_work is NULL or not 256-byte aligned");
  if (h->n_schur > 0)
    return fail(-1, "a Schur-mode (partial) factorization has no full solve: use dd_aux_condense / dd_aux_recover");
  if (!h->factored || h->factored_ptr != d_factor) return fail(DD_ERR_NOT_FACTORED, "d_factor holds no factorization of this handle");
  if (h->singular) return fail(DD_ERR_SINGULAR, "the factorization reported a zero pivot");
  const int refine = h->opt.refine_steps;
  if (refine > 0 && !d_vals) return fail(-3, "d_vals is NULL but refine_steps > 0");
  if (nrhs > SOLVE_MAX_COLS) {  // column chunks (direct launches; see SOLVE_MAX_COLS)
    const int g = h->opt.use_graphs;
    h->opt.use_graphs = 0;
    int rc = DD_OK;
    const size_t es = h->cplx ? 16 : 8;
    for (int64_t c0 = 0; c0 < nrhs && rc == DD_OK; c0 += SOLVE_MAX_COLS)
      rc = dd_aux_solve(h, d_factor, d_vals, std::min(SOLVE_MAX_COLS, nrhs - c0), (uint8_t*)d_B + (size_t)c0 * ldb * es,
                        ldb, d_work, stream);
    h->opt.use_graphs = g;
    return rc;
  }
  cudaStream_t st0 = (cudaStream_t)stream;
  const bool in_graph = h->opt.use_graphs && !h->trace;
  auto body = [&](cudaStream_t st) -> int {
    const bool C = h->cplx;
    const int planes = C ? 2 : 1;
    const uint8_t* F = (const uint8_t*)d_factor;
    uint8_t* Wb = (uint8_t*)d_work;
    const int64_t ldy = pad8(h->n_pad);
    double* y = (double*)Wb;
    const int64_t yim = C ? ldy * nrhs : 0;
    double* Bsave = (double*)(Wb + align256((size_t)ldy * nrhs * planes * sizeof(double)));

    PermArgs pa{};
    pa.gperm = (const int*)(F + h->off_gperm);
    pa.nrows = h->n_pad;
    pa.nrhs = (int)nrhs;
    pa.y = y;
    pa.yim = yim;
    pa.ldy = ldy;
    if (refine > 0) {
      TraceScope ts(h, DD_PH_PERM, 0.0, st);
      launch_copy(C, (const double*)d_B, ldb, Bsave, h->n, h->n, (int)nrhs, st);
      LAUNCH_CHECK("k_copy");
    }
    pa.src = (const double*)d_B;
    pa.lds = ldb;
    {
      TraceScope ts(h, DD_PH_PERM, 0.0, st);
      launch_perm_in(C, pa, st);
    }
    LAUNCH_CHECK("k_perm_in");
    double* berr_d = (double*)((uint8_t*)Bsave + align256((size_t)h->n * nrhs * planes * sizeof(double)));
    int* flag_d = (int*)((uint8_t*)berr_d + align256((size_t)nrhs * sizeof(double)));
    double* part = (double*)((uint8_t*)flag_d + 256);
    double* Tbuf = (double*)((uint8_t*)part + align256(bupd_part_bytes(C, (int)nrhs)));
    int* cnt = (int*)((uint8_t*)Tbuf + align256((size_t)pad8(std::max<int64_t>(h->nT, 2)) * nrhs * planes * sizeof(double)));
    static const bool fold = !(getenv("DD_AUX_BUPD_FOLD") && atoi(getenv("DD_AUX_BUPD_FOLD")) == 0);  // A/B
    if (fold) CUDA_TRY(cudaMemsetAsync(cnt, 0, bupd_cnt_bytes(C, (int)nrhs), st));
    else cnt = nullptr;
    int rc = solve_sweep(h, F, y, yim, ldy, (int)nrhs, st, part, Tbuf, nullptr, SW_ALL, cnt);
    if (rc) return rc;
    pa.dst = (double*)d_B;
    pa.ldd = ldb;
    pa.accumulate = 0;
    {
      TraceScope ts(h, DD_PH_PERM, 0.0, st);
      launch_perm_out(C, pa, st);
    }
    LAUNCH_CHECK("k_perm_out");
    const double tol = h->opt.refine_tol;
    unsigned long long* norm_d = (unsigned long long*)(F + h->off_norm);
    for (int r = 0; r < refine; ++r) {
      SpmvArgs sa{};
      sa.rows = (const SpRow*)(F + h->off_sprows);
      sa.segs = (const SpSeg*)(F + h->off_spsegs);
      sa.blk_size = (const int64_t*)(F + h->off_blksize);
      sa.odof = (const int64_t*)(F + h->off_odof);
      sa.vals = (const double*)d_vals;
      sa.X = (const double*)d_B;
      sa.ldx = ldb;
      sa.Bsave = Bsave;
      sa.ldb = h->n;
      sa.ginv = (const int*)(F + h->off_ginv);
      sa.y = y;
      sa.yim = yim;
      sa.ldy = ldy;
      sa.nrhs = (int)nrhs;
      {
        TraceScope ts(h, DD_PH_SPMV, (C ? 8.0 : 2.0) * h->nnz_full * (double)nrhs, st);
        launch_spmv(C, sa, h->n_sprows, st);
      }
      LAUNCH_CHECK("k_spmv");
      const int* flag = nullptr;
      if (tol > 0) {  // adaptive: skip the correction on the device when every column is converged
        if (!h->norm_valid || in_graph) {  // a replayed graph recomputes ||A|| (values may change)
          CUDA_TRY(cudaMemsetAsync(norm_d, 0, sizeof(unsigned long long), st));
          launch_norm_a(C, sa, h->n_sprows, norm_d, st);
          LAUNCH_CHECK("k_norm_a");
          h->norm_valid = !in_graph;
        }
        CUDA_TRY(cudaMemsetAsync(flag_d, 0, sizeof(int), st));
        launch_berr(C, y, yim, ldy, h->n_pad, (const double*)d_B, ldb, h->n, (int)nrhs, norm_d, tol, berr_d, flag_d, st);
        LAUNCH_CHECK("k_berr");
        flag = flag_d;
      }
      rc = solve_sweep(h, F, y, yim, ldy, (int)nrhs, st, part, Tbuf, flag, SW_ALL, cnt);
      if (rc) return rc;
      pa.accumulate = 1;
      pa.flag = flag;
      {
        TraceScope ts(h, DD_PH_PERM, 0.0, st);
        launch_perm_out(C, pa, st);
      }
      LAUNCH_CHECK("k_perm_out");
    }
    return DD_OK;
  };
  double tolv = h->opt.refine_tol;
  uint64_t tolbits;
  std::memcpy(&tolbits, &tolv, 8);
  const std::vector<uintptr_t> key = {(uintptr_t)d_factor, (uintptr_t)d_vals, (uintptr_t)nrhs, (uintptr_t)d_B,
                                      (uintptr_t)ldb, (uintptr_t)d_work, (uintptr_t)refine, (uintptr_t)tolbits};
  return run_graph(h, h->gsolve, key, body, st0);
}

}  // extern "C"

// f1 tables: per output block (CSC order) its 32-column chunks, each with the contributor list
// (cliques containing both interfaces, ascending clique index).  S_offset / val_offset may be
// NULL for the size query (the offsets are then left zero).
static int build_assembly(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                          const int64_t* S_offset, const int64_t* val_offset, std::vector<AsmItem>& items,
                          std::vector<AsmContrib>& cons) {
  const int N = h->S.nblk;
  if (nclq < 0) return fail(-2, "nclq must be >= 0");
  if (nclq > 0 && (!clq_ptr || !clq_blk)) return fail(!clq_ptr ? -3 : -4, "clique arrays are NULL");
  std::vector<std::vector<AsmContrib>> per(h->nnzb_in);
  for (int64_t p = 0; p < nclq; ++p) {
    const int64_t b0 = clq_ptr[p], b1 = clq_ptr[p + 1];
    if (b1 < b0 || b0 < 0) return fail(-3, "clq_ptr is not non-decreasing");
    std::vector<int64_t> off(b1 - b0 + 1, 0);
    for (int64_t a = b0; a < b1; ++a) {
      const int I = clq_blk[a];
      if (I < 0 || I >= N) return fail(DD_ERR_PATTERN, "clique " + std::to_string(p) + ": block id out of range");
      if (a > b0 && I <= clq_blk[a - 1])
        return fail(DD_ERR_PATTERN, "clique " + std::to_string(p) + ": members not strictly ascending");
      off[a - b0 + 1] = off[a - b0] + h->blk_size[I];
    }
    const int64_t m = off.back();
    for (int64_t a = b0; a < b1; ++a)
      for (int64_t b = b0; b <= a; ++b) {
        const int I = clq_blk[a], J = clq_blk[b];  // I >= J
        auto rb = h->rowidx.begin() + h->colptr[J], re = h->rowidx.begin() + h->colptr[J + 1];
        auto itp = std::lower_bound(rb, re, I);
        if (itp == re || *itp != I)
          return fail(DD_ERR_PATTERN, "clique " + std::to_string(p) + ": block (" + std::to_string(I) + "," +
                                          std::to_string(J) + ") is not in the pattern");
        AsmContrib c{};
        c.soff = S_offset ? S_offset[p] : 0;
        c.ld = m;
        c.ra = (int32_t)off[a - b0];
        c.cb = (int32_t)off[b - b0];
        per[itp - h->rowidx.begin()].push_back(c);
      }
  }
  const int CH = asm_chunk();
  items.clear();
  cons.clear();
  for (int j = 0; j < N; ++j)
    for (int64_t q = h->colptr[j]; q < h->colptr[j + 1]; ++q) {
      const int i = h->rowidx[q];
      const int k0 = (int)cons.size();
      for (auto& c : per[q]) cons.push_back(c);
      const int k1 = (int)cons.size();
      for (int c0 = 0; c0 < h->blk_size[j]; c0 += CH) {
        AsmItem it{};
        it.dst = val_offset ? val_offset[q] : 0;
        it.rows = (int32_t)h->blk_size[i];
        it.cols = (int32_t)h->blk_size[j];
        it.c0 = c0;
        it.k0 = k0;
        it.k1 = k1;
        it.pad = (i == j);  // diagonal block (byte accounting only)
        items.push_back(it);
      }
    }
  return DD_OK;
}

extern "C" {

int dd_aux_assemble_work_bytes(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                               size_t* bytes) {
  if (!h) return fail(-1, "handle is NULL");
  if (!bytes) return fail(-5, "bytes is NULL");
  std::vector<AsmItem> items;
  std::vector<AsmContrib> cons;
  int rc = build_assembly(h, nclq, clq_ptr, clq_blk, nullptr, nullptr, items, cons);
  if (rc) return rc;
  *bytes = align256(items.size() * sizeof(AsmItem)) + align256(cons.size() * sizeof(AsmContrib));
  return DD_OK;
}

static int assemble_impl(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                         const void* d_S, const int64_t* S_offset, int32_t symmetrize, const int64_t* val_offset,
                         void* d_vals, void* d_work, void* stream, int accumulate);

int dd_aux_assemble(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                    const void* d_S, const int64_t* S_offset, int32_t symmetrize, const int64_t* val_offset,
                    void* d_vals, void* d_work, void* stream) {
  return assemble_impl(h, nclq, clq_ptr, clq_blk, d_S, S_offset, symmetrize, val_offset, d_vals, d_work, stream, 0);
}

int dd_aux_assemble_acc(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                        const void* d_S, const int64_t* S_offset, int32_t symmetrize, const int64_t* val_offset,
                        void* d_vals, void* d_work, void* stream) {
  if (symmetrize) return fail(-7, "dd_aux_assemble_acc: symmetrize must be 0 (the cliques must be symmetric)");
  return assemble_impl(h, nclq, clq_ptr, clq_blk, d_S, S_offset, 0, val_offset, d_vals, d_work, stream, 1);
}

}  // extern "C"

static int assemble_impl(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                         const void* d_S, const int64_t* S_offset, int32_t symmetrize, const int64_t* val_offset,
                         void* d_vals, void* d_work, void* stream, int accumulate) {
  if (!h) return fail(-1, "handle is NULL");
  if (nclq > 0 && !d_S) return fail(-5, "d_S is NULL");
  if (nclq > 0 && !S_offset) return fail(-6, "S_offset is NULL");
  if (!val_offset) return fail(-8, "val_offset is NULL");
  if (!d_vals) return fail(-9, "d_vals is NULL");
  if (!d_work || ((uintptr_t)d_work & 255)) return fail(-10, "d_work is NULL or not 256-byte aligned");
  std::vector<AsmItem> items;
  std::vector<AsmContrib> cons;
  int rc = build_assembly(h, nclq, clq_ptr, clq_blk, S_offset, val_offset, items, cons);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // the host images live in the handle until the next call, so the async copies never race a free
  h->asm_items.swap(items);
  h->asm_cons.swap(cons);
  uint8_t* W = (uint8_t*)d_work;
  const size_t off_c = align256(h->asm_items.size() * sizeof(AsmItem));
  if (!h->asm_items.empty())
    CUDA_TRY(cudaMemcpyAsync(W, h->asm_items.data(), h->asm_items.size() * sizeof(AsmItem), cudaMemcpyHostToDevice, st));
  if (!h->asm_cons.empty())
    CUDA_TRY(cudaMemcpyAsync(W + off_c, h->asm_cons.data(), h->asm_cons.size() * sizeof(AsmContrib),
                             cudaMemcpyHostToDevice, st));
  AsmArgs a{(const AsmItem*)W, (const AsmContrib*)(W + off_c), (const double*)d_S, (double*)d_vals, accumulate};
  {
    // algorithmic (unique) traffic: output written once + each contribution read once, plus the
    // mirrored block S_p[J, I] for the symmetric part of an off-diagonal block (a diagonal
    // block's transpose is the same memory)
    double bytes = 0;
    const double es = h->cplx ? 16.0 : 8.0;
    for (size_t q = 0; q < h->asm_items.size(); ++q) {
      const AsmItem& it = h->asm_items[q];
      const double cells = (double)it.rows * std::min(asm_chunk(), it.cols - it.c0);
      bytes += cells * es * (1.0 + ((symmetrize && !it.pad) ? 2.0 : 1.0) * (it.k1 - it.k0));
    }
    h->asm_bytes = bytes;
    TraceScope ts(h, DD_PH_ASSEMBLE, 0.0, st);
    launch_assemble(h->cplx, symmetrize != 0, a, (int)h->asm_items.size(), st);
  }
  LAUNCH_CHECK("k_assemble");
  return DD_OK;
}

extern "C" {

double dd_aux_last_assemble_bytes(dd_aux_handle_t h) { return h ? h->asm_bytes : 0.0; }

int dd_aux_set_refine(dd_aux_handle_t h, int32_t refine_steps, double refine_tol) {
  if (!h) return fail(-1, "handle is NULL");
  if (refine_steps < 0) return fail(-2, "refine_steps must be >= 0");
  if (!(refine_tol >= 0)) return fail(-3, "refine_tol must be >= 0");
  h->opt.refine_steps = refine_steps;
  h->opt.refine_tol = refine_tol;
  return DD_OK;
}

int dd_aux_get_pivots(dd_aux_handle_t h, const void* d_factor, int32_t* ipiv, int32_t* perm, void* d, void* e) {
  if (!h) return fail(-1, "handle is NULL");
  if (!d_factor) return fail(-2, "d_factor is NULL");
  if (!h->factored || h->factored_ptr != d_factor) return fail(DD_ERR_NOT_FACTORED, "not factored");
  const uint8_t* F = (const uint8_t*)d_factor;
  const int64_t np = h->n_pad;
  std::vector<int32_t> ip(np), pm(np);
  const bool C = h->cplx;
  std::vector<double> dv(np * (C ? 2 : 1)), ev(np * (C ? 2 : 1));
  CUDA_TRY(cudaMemcpy(ip.data(), F + h->off_ipiv, np * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(pm.data(), F + h->off_perm, np * 4, cudaMemcpyDeviceToHost));
  const double* arena = (const double*)(F + h->off_arena);
  CUDA_TRY(cudaMemcpy(dv.data(), arena + h->d_off, np * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(ev.data(), arena + h->e_off, np * 8, cudaMemcpyDeviceToHost));
  if (C) {
    CUDA_TRY(cudaMemcpy(dv.data() + np, arena + h->nA + h->d_off, np * 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(ev.data() + np, arena + h->nA + h->e_off, np * 8, cudaMemcpyDeviceToHost));
  }
  int64_t q = 0;
  for (int t = 0; t < h->S.nblk; ++t) {
    const NodeDev& nd = h->nodes[t];
    for (int m = 0; m < nd.s; ++m, ++q) {
      int64_t g = nd.ydof + m;
      if (ipiv) ipiv[q] = ip[g];
      if (perm) perm[q] = pm[g];
      if (d) {
        if (C) {
          ((double*)d)[2 * q] = dv[g];
          ((double*)d)[2 * q + 1] = dv[np + g];
        } else {
          ((double*)d)[q] = dv[g];
        }
      }
      if (e) {
        if (C) {
          ((double*)e)[2 * q] = ev[g];
          ((double*)e)[2 * q + 1] = ev[np + g];
        } else {
          ((double*)e)[q] = ev[g];
        }
      }
    }
  }
  return DD_OK;
}

int dd_aux_set_graphs(dd_aux_handle_t h, int32_t enable) {
  if (!h) return fail(-1, "handle is NULL");
  h->opt.use_graphs = enable != 0;
  return DD_OK;
}

int dd_aux_set_trace(dd_aux_handle_t h, int32_t enable) {
  if (!h) return fail(-1, "handle is NULL");
  h->trace = enable != 0;
  return DD_OK;
}

int dd_aux_get_trace(dd_aux_handle_t h, dd_aux_trace* out, int32_t reset) {
  if (!h) return fail(-1, "handle is NULL");
  if (!out) return fail(-2, "out is NULL");
  for (auto& r : h->recs) {
    CUDA_TRY(cudaEventSynchronize(h->pool[r.e1]));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, h->pool[r.e0], h->pool[r.e1]));
    h->ms_acc[r.ph] += ms;
    if (r.level >= 0 && (size_t)r.level * 16 + r.ph < h->lvl_ms.size()) h->lvl_ms[(size_t)r.level * 16 + r.ph] += ms;
  }
  h->recs.clear();
  for (int q = 0; q < 16; ++q) {
    out->ms[q] = h->ms_acc[q];
    out->launches[q] = h->launches[q];
    out->flops[q] = h->flops[q];
  }
  if (reset) {
    std::fill(h->lvl_ms.begin(), h->lvl_ms.end(), 0.0);
    std::fill(h->lvl_fl.begin(), h->lvl_fl.end(), 0.0);
    for (int q = 0; q < 16; ++q) {
      h->ms_acc[q] = 0;
      h->launches[q] = 0;
      h->flops[q] = 0;
    }
  }
  return DD_OK;
}

int dd_aux_get_level_trace(dd_aux_handle_t h, double* ms, double* flops) {
  if (!h) return fail(-1, "handle is NULL");
  const size_t nl = h->S.nlevels;
  for (size_t q = 0; q < nl * 16; ++q) {
    if (ms) ms[q] = q < h->lvl_ms.size() ? h->lvl_ms[q] : 0.0;
    if (flops) flops[q] = q < h->lvl_fl.size() ? h->lvl_fl[q] : 0.0;
  }
  return DD_OK;
}

int dd_aux_destroy(dd_aux_handle_t h) {
  delete h;
  return DD_OK;
}

}  // extern "C"

// ============================================================================ f3 / f2: Schur mode
// Tables of a partial factorization (dd_aux_analyze_partial): export items, condensation gather
// and recovery scatter lists, identity row maps of the kept blocks.
static int build_schur_tables(dd_aux_handle_t h) {
  const int N = h->S.nblk, NE = h->n_elim;
  const int64_t NS = h->n_schur;
  // groups = distinct schur_group values ascending; members by ascending target
  std::vector<int32_t> idx(NS);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) {
    return h->schur_group[a] != h->schur_group[b] ? h->schur_group[a] < h->schur_group[b]
                                                  : h->schur_target[a] < h->schur_target[b];
  });
  h->grp_kept = idx;
  h->grp_ptr.assign(1, 0);
  h->grp_m.clear();
  for (int64_t q = 0; q < NS; ++q) {
    if (q > 0 && h->schur_group[idx[q]] == h->schur_group[idx[q - 1]] &&
        h->schur_target[idx[q]] == h->schur_target[idx[q - 1]])
      return fail(DD_ERR_PATTERN, "two kept blocks of group " + std::to_string(h->schur_group[idx[q]]) +
                                      " have the same schur_target");
    if (q > 0 && h->schur_group[idx[q]] != h->schur_group[idx[q - 1]]) h->grp_ptr.push_back(q);
  }
  h->grp_ptr.push_back(NS);
  const int ng = (int)h->grp_ptr.size() - 1;
  auto row_in = [&](int j, int i) -> int {  // row offset of position i inside panel j, -1 if absent
    const NodeDev& nj = h->nodes[j];
    int64_t ro = nj.sp;
    for (int u : h->S.st[j]) {
      if (u == i) return (int)ro;
      ro += pad2(h->nodes[u].s);
    }
    return -1;
  };
  std::vector<SxItem> items;
  std::vector<SxTile> tiles;
  for (int g = 0; g < ng; ++g) {
    int64_t m = 0;
    std::vector<int64_t> off;
    for (int64_t q = h->grp_ptr[g]; q < h->grp_ptr[g + 1]; ++q) {
      off.push_back(m);
      m += h->blk_size[NE + idx[q]];
    }
    h->grp_m.push_back(m);
    for (int64_t qa = h->grp_ptr[g]; qa < h->grp_ptr[g + 1]; ++qa)
      for (int64_t qb = h->grp_ptr[g]; qb < h->grp_ptr[g + 1]; ++qb) {
        const int ta = h->S.pos[NE + idx[qa]], tb = h->S.pos[NE + idx[qb]];
        SxItem it{};
        it.rows = h->nodes[ta].s;
        it.cols = h->nodes[tb].s;
        it.group = g;
        it.m = (int32_t)m;
        it.dst = off[qa - h->grp_ptr[g]] + off[qb - h->grp_ptr[g]] * m;
        if (ta == tb) {
          it.mode = 2;
          it.src = h->nodes[ta].panel;
          it.ld = h->nodes[ta].ld;
        } else {
          const int lo = std::min(ta, tb), hi = std::max(ta, tb);
          const int ro = row_in(lo, hi);
          if (ro < 0) {
            it.mode = 3;
          } else {
            it.mode = ta > tb ? 0 : 1;
            it.src = h->nodes[lo].panel + ro;
            it.ld = h->nodes[lo].ld;
          }
        }
        const int id = (int)items.size();
        items.push_back(it);
        for (int r0 = 0; r0 < it.rows; r0 += 32)
          for (int c0 = 0; c0 < it.cols; c0 += 32) tiles.push_back(SxTile{id, r0, c0, 0});
      }
  }
  h->n_sx_tiles = (int)tiles.size();
  // condensation gather: per auxiliary block, its kept copies in ascending position
  std::vector<std::vector<int>> copies(h->n_aux);
  for (int64_t k = 0; k < NS; ++k) copies[h->schur_target[k]].push_back(h->S.pos[NE + k]);
  std::vector<SgItem> sg;
  std::vector<int32_t> contrib;
  for (int64_t I = 0; I < h->n_aux; ++I) {
    if (copies[I].empty()) continue;
    std::sort(copies[I].begin(), copies[I].end());
    SgItem it{};
    it.aux_row = h->aux_odof[I];
    it.s = (int32_t)h->blk_size[NE + [&] {  // size of any copy
      for (int64_t k = 0; k < NS; ++k)
        if (h->schur_target[k] == I) return (int)k;
      return 0;
    }()];
    it.c0 = (int32_t)contrib.size();
    for (int t : copies[I]) contrib.push_back(t);
    it.c1 = (int32_t)contrib.size();
    sg.push_back(it);
  }
  h->n_sg_items = (int)sg.size();
  // recovery scatter: per kept position, the auxiliary rows of its target
  std::vector<SgItem> ss;
  for (int64_t k = 0; k < NS; ++k) {
    SgItem it{};
    it.aux_row = h->aux_odof[h->schur_target[k]];
    it.s = (int32_t)h->blk_size[NE + k];
    it.c0 = h->S.pos[NE + k];
    ss.push_back(it);
  }
  h->n_ss_items = (int)ss.size();
  // identity row maps of the kept blocks: rows [r0, n_pad), original DoFs [odof(NE), n)
  h->kept_gperm.clear();
  h->kept_ginv.clear();
  h->kept_perm.clear();
  for (int t = NE; t < N; ++t) {
    const NodeDev& nd = h->nodes[t];
    for (int m = 0; m < nd.sp; ++m) {
      h->kept_gperm.push_back(m < nd.s ? (int32_t)(nd.odof + m) : -1);
      h->kept_perm.push_back(m);
    }
  }
  for (int64_t o = h->odof_blk[NE]; o < h->n; ++o) {
    const int blk = (int)(std::upper_bound(h->odof_blk.begin(), h->odof_blk.end(), o) - h->odof_blk.begin()) - 1;
    const NodeDev& nd = h->nodes[h->S.pos[blk]];
    h->kept_ginv.push_back((int32_t)(nd.ydof + (o - nd.odof)));
  }
  Blob& B = h->blob;
  h->off_sx_items = B.put(items);
  h->off_sx_tiles = B.put(tiles);
  h->off_sg_items = B.put(sg);
  h->off_sg_contrib = B.put(contrib);
  h->off_ss_items = B.put(ss);
  h->off_soff = B.put(std::vector<int64_t>(ng, 0));
  return DD_OK;
}

extern "C" {

int dd_aux_analyze_partial(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx,
                           int32_t dtype, const dd_aux_options* opt, int64_t n_schur, const int32_t* schur_target,
                           const int32_t* schur_group, int64_t n_aux, const int64_t* aux_blk_size,
                           dd_aux_handle_t* out) {
  if (!out) return fail(-12, "out is NULL");
  if (nblk <= 0) return fail(-1, "nblk must be > 0");
  if (!blk_size) return fail(-2, "blk_size is NULL");
  if (n_schur < 1 || n_schur >= nblk) return fail(-7, "n_schur must be in [1, nblk)");
  if (!schur_target) return fail(-8, "schur_target is NULL");
  if (!schur_group) return fail(-9, "schur_group is NULL");
  if (n_aux < 1) return fail(-10, "n_aux must be >= 1");
  if (!aux_blk_size) return fail(-11, "aux_blk_size is NULL");
  for (int64_t k = 0; k < n_schur; ++k) {
    const int32_t I = schur_target[k];
    if (I < 0 || I >= n_aux) return fail(-8, "schur_target out of range");
    if (schur_group[k] < 0) return fail(-9, "schur_group must be >= 0");
    if (aux_blk_size[I] != blk_size[nblk - n_schur + k])
      return fail(-11, "kept block " + std::to_string(nblk - n_schur + k) + " and its target auxiliary block " +
                           std::to_string(I) + " differ in size");
  }
  dd_aux_handle_t h = nullptr;
  const SchurIn sin{schur_target, schur_group, n_aux, aux_blk_size};
  const int rc = analyze_impl(nblk, blk_size, colptr, rowidx, dtype, opt, n_schur, &sin, &h);
  if (rc) return rc;
  *out = h;
  return DD_OK;
}

int dd_aux_schur_cliques(dd_aux_handle_t h, int64_t* ngroups, int64_t* clq_ptr, int32_t* clq_blk) {
  if (!h) return fail(-1, "handle is NULL");
  if (h->n_schur == 0) return fail(-1, "not a Schur-mode handle");
  const int64_t ng = (int64_t)h->grp_ptr.size() - 1;
  if (ngroups) *ngroups = ng;
  if (clq_ptr)
    for (int64_t g = 0; g <= ng; ++g) clq_ptr[g] = h->grp_ptr[g];
  if (clq_blk)
    for (int64_t q = 0; q < h->n_schur; ++q) clq_blk[q] = h->schur_target[h->grp_kept[q]];
  return DD_OK;
}

int dd_aux_schur_export(dd_aux_handle_t h, const void* d_factor, void* d_S, const int64_t* S_offset, void* stream) {
  if (!h) return fail(-1, "handle is NULL");
  if (h->n_schur == 0) return fail(-1, "not a Schur-mode handle");
  if (!d_factor) return fail(-2, "d_factor is NULL");
  if (!d_S) return fail(-3, "d_S is NULL");
  if (!S_offset) return fail(-4, "S_offset is NULL");
  if (!h->factored || h->factored_ptr != d_factor) return fail(DD_ERR_NOT_FACTORED, "not factored");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ng = (int64_t)h->grp_ptr.size() - 1;
  h->soff_host.assign(S_offset, S_offset + ng);  // kept alive until the next call (async upload)
  uint8_t* F = (uint8_t*)const_cast<void*>(d_factor);
  CUDA_TRY(cudaMemcpyAsync(F + h->off_soff, h->soff_host.data(), ng * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  SchurExportArgs a{(const SxItem*)(F + h->off_sx_items), (const SxTile*)(F + h->off_sx_tiles),
                    (const double*)(F + h->off_arena), h->cplx ? h->nA : 0, (double*)d_S,
                    (const int64_t*)(F + h->off_soff)};
  {
    TraceScope ts(h, DD_PH_SCHUR, 0.0, st);
    launch_schur_export(h->cplx, a, h->n_sx_tiles, st);
  }
  LAUNCH_CHECK("k_schur_export");
  return DD_OK;
}

}  // extern "C"

// condense (mode 0) / recover (mode 1) of one chunk of <= SOLVE_MAX_COLS columns
static int schur_sweep(dd_aux_handle_t h, int mode, const void* d_factor, int64_t nrhs, const void* d_F, int64_t ldf,
                       void* d_V, int64_t ldv, void* d_X, int64_t ldx, void* d_work, cudaStream_t st) {
  const bool C = h->cplx;
  const int planes = C ? 2 : 1;
  const uint8_t* F = (const uint8_t*)d_factor;
  uint8_t* Wb = (uint8_t*)d_work;
  const int64_t ldy = pad8(h->n_pad);
  double* y = (double*)Wb;
  const int64_t yim = C ? ldy * nrhs : 0;
  double* Bsave = (double*)(Wb + align256((size_t)ldy * nrhs * planes * sizeof(double)));
  double* berr_d = (double*)((uint8_t*)Bsave + align256((size_t)h->n * nrhs * planes * sizeof(double)));
  int* flag_d = (int*)((uint8_t*)berr_d + align256((size_t)nrhs * sizeof(double)));
  double* part = (double*)((uint8_t*)flag_d + 256);
  double* Tbuf = (double*)((uint8_t*)part + align256(bupd_part_bytes(C, (int)nrhs)));
  int* cnt = (int*)((uint8_t*)Tbuf + align256((size_t)pad8(std::max<int64_t>(h->nT, 2)) * nrhs * planes * sizeof(double)));
  CUDA_TRY(cudaMemsetAsync(cnt, 0, bupd_cnt_bytes(C, (int)nrhs), st));
  PermArgs pa{};
  pa.gperm = (const int*)(F + h->off_gperm);
  pa.nrows = h->n_pad;
  pa.rowlim = h->r0;  // kept rows start at zero
  pa.nrhs = (int)nrhs;
  pa.y = y;
  pa.yim = yim;
  pa.ldy = ldy;
  pa.src = (const double*)d_F;
  pa.lds = ldf;
  {
    TraceScope ts(h, DD_PH_PERM, 0.0, st);
    launch_perm_in(C, pa, st);
  }
  LAUNCH_CHECK("k_perm_in");
  SchurVecArgs sv{};
  sv.nd = (const NodeDev*)(F + h->off_nodes);
  sv.contrib = (const int*)(F + h->off_sg_contrib);
  sv.y = y;
  sv.yim = yim;
  sv.ldy = ldy;
  sv.G = (double*)d_V;
  sv.ldg = ldv;
  sv.nrhs = (int)nrhs;
  if (mode == 0) {  // condense: forward sweep, then G += kept rows (fixed order)
    int rc = solve_sweep(h, F, y, yim, ldy, (int)nrhs, st, part, Tbuf, nullptr, SW_FWD);
    if (rc) return rc;
    sv.items = (const SgItem*)(F + h->off_sg_items);
    {
      TraceScope ts(h, DD_PH_SCHUR, 0.0, st);
      launch_schur_gather(C, sv, h->n_sg_items, st);
    }
    LAUNCH_CHECK("k_schur_gather");
    return DD_OK;
  }
  // recover: forward sweep + D, kept rows <- x_b, backward sweep, x = P^T y
  int rc = solve_sweep(h, F, y, yim, ldy, (int)nrhs, st, part, Tbuf, nullptr, SW_FWD | SW_D);
  if (rc) return rc;
  sv.items = (const SgItem*)(F + h->off_ss_items);
  {
    TraceScope ts(h, DD_PH_SCHUR, 0.0, st);
    launch_schur_scatter(C, sv, h->n_ss_items, st);
  }
  LAUNCH_CHECK("k_schur_scatter");
  rc = solve_sweep(h, F, y, yim, ldy, (int)nrhs, st, part, Tbuf, nullptr, SW_BWD, cnt);
  if (rc) return rc;
  pa.dst = (double*)d_X;
  pa.ldd = ldx;
  pa.accumulate = 0;
  {
    TraceScope ts(h, DD_PH_PERM, 0.0, st);
    launch_perm_out(C, pa, st);
  }
  LAUNCH_CHECK("k_perm_out");
  return DD_OK;
}

static int schur_call(dd_aux_handle_t h, int mode, const void* d_factor, int64_t nrhs, const void* d_F, int64_t ldf,
                      void* d_V, int64_t ldv, void* d_X, int64_t ldx, void* d_work, void* stream) {
  if (!h) return fail(-1, "handle is NULL");
  if (h->n_schur == 0) return fail(-1, "not a Schur-mode handle (dd_aux_analyze_partial)");
  if (!d_factor) return fail(-2, "d_factor is NULL");
  if (nrhs < 0) return fail(-3, "nrhs must be >= 0");
  if (nrhs == 0) return DD_OK;
  if (!d_F) return fail(-4, "d_F is NULL");
  if (ldf < h->n) return fail(-5, "ldf < n");
  if (!d_V) return fail(-6, mode ? "d_Xb is NULL" : "d_G is NULL");
  if (ldv < h->n_aux_dof) return fail(-7, "leading dimension of the auxiliary block < n_aux DoFs");
  if (mode == 1 && !d_X) return fail(-8, "d_X is NULL");
  if (mode == 1 && ldx < h->n) return fail(-9, "ldx < n");
  if (!d_work || ((uintptr_t)d_work & 255)) return fail(-10, "d_work is NULL or not 256-byte aligned");
  if (!h->factored || h->factored_ptr != d_factor) return fail(DD_ERR_NOT_FACTORED, "not factored");
  if (h->singular) return fail(DD_ERR_SINGULAR, "the partial factorization reported a zero pivot");
  const size_t es = h->cplx ? 16 : 8;
  for (int64_t c0 = 0; c0 < nrhs; c0 += SOLVE_MAX_COLS) {
    const int64_t w = std::min(SOLVE_MAX_COLS, nrhs - c0);
    const int rc = schur_sweep(h, mode, d_factor, w, (const uint8_t*)d_F + (size_t)c0 * ldf * es, ldf,
                               (uint8_t*)d_V + (size_t)c0 * ldv * es, ldv,
                               d_X ? (uint8_t*)d_X + (size_t)c0 * ldx * es : nullptr, ldx, d_work, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return DD_OK;
}

extern "C" {

int dd_aux_condense(dd_aux_handle_t h, const void* d_factor, int64_t nrhs, const void* d_F, int64_t ldf, void* d_G,
                    int64_t ldg, void* d_work, void* stream) {
  return schur_call(h, 0, d_factor, nrhs, d_F, ldf, d_G, ldg, nullptr, 0, d_work, stream);
}

int dd_aux_recover(dd_aux_handle_t h, const void* d_factor, int64_t nrhs, const void* d_F, int64_t ldf,
                   const void* d_Xb, int64_t ldxb, void* d_X, int64_t ldx, void* d_work, void* stream) {
  return schur_call(h, 1, d_factor, nrhs, d_F, ldf, const_cast<void*>(d_Xb), ldxb, d_X, ldx, d_work, stream);
}

}  // extern "C"

extern "C" {

// R = B - A X over the handle's ORIGINAL blocks (both triangles), original DoF order (a8's
// residual, K6, exposed for callers that refine across several handles, e.g. f4).
int dd_aux_residual(dd_aux_handle_t h, const void* d_factor, const void* d_vals, int64_t nrhs, const void* d_B,
                    int64_t ldb, const void* d_X, int64_t ldx, void* d_R, int64_t ldr, void* d_work, void* stream) {
  if (!h) return fail(-1, "handle is NULL");
  if (!d_factor) return fail(-2, "d_factor is NULL");
  if (!d_vals) return fail(-3, "d_vals is NULL");
  if (nrhs < 0) return fail(-4, "nrhs must be >= 0");
  if (nrhs == 0) return DD_OK;
  if (!d_B || ldb < h->n) return fail(-5, "d_B is NULL or ldb < n");
  if (!d_X || ldx < h->n) return fail(-7, "d_X is NULL or ldx < n");
  if (!d_R || ldr < h->n) return fail(-9, "d_R is NULL or ldr < n");
  if (!d_work || ((uintptr_t)d_work & 255)) return fail(-11, "d_work is NULL or not 256-byte aligned");
  if (!h->factored || h->factored_ptr != d_factor) return fail(DD_ERR_NOT_FACTORED, "not factored (row maps)");
  if (nrhs > SOLVE_MAX_COLS) {
    const size_t es = h->cplx ? 16 : 8;
    for (int64_t c0 = 0; c0 < nrhs; c0 += SOLVE_MAX_COLS) {
      const int rc = dd_aux_residual(h, d_factor, d_vals, std::min(SOLVE_MAX_COLS, nrhs - c0),
                                     (const uint8_t*)d_B + (size_t)c0 * ldb * es, ldb,
                                     (const uint8_t*)d_X + (size_t)c0 * ldx * es, ldx,
                                     (uint8_t*)d_R + (size_t)c0 * ldr * es, ldr, d_work, stream);
      if (rc) return rc;
    }
    return DD_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const bool C = h->cplx;
  const uint8_t* F = (const uint8_t*)d_factor;
  const int64_t ldy = pad8(h->n_pad);
  double* y = (double*)d_work;
  const int64_t yim = C ? ldy * nrhs : 0;
  SpmvArgs sa{};
  sa.rows = (const SpRow*)(F + h->off_sprows);
  sa.segs = (const SpSeg*)(F + h->off_spsegs);
  sa.blk_size = (const int64_t*)(F + h->off_blksize);
  sa.odof = (const int64_t*)(F + h->off_odof);
  sa.vals = (const double*)d_vals;
  sa.X = (const double*)d_X;
  sa.ldx = ldx;
  sa.Bsave = (const double*)d_B;
  sa.ldb = ldb;
  sa.ginv = (const int*)(F + h->off_ginv);
  sa.y = y;
  sa.yim = yim;
  sa.ldy = ldy;
  sa.nrhs = (int)nrhs;
  {
    TraceScope ts(h, DD_PH_SPMV, (C ? 8.0 : 2.0) * h->nnz_full * (double)nrhs, st);
    launch_spmv(C, sa, h->n_sprows, st);
  }
  LAUNCH_CHECK("k_spmv");
  PermArgs pa{};
  pa.gperm = (const int*)(F + h->off_gperm);
  pa.nrows = h->n_pad;
  pa.nrhs = (int)nrhs;
  pa.y = y;
  pa.yim = yim;
  pa.ldy = ldy;
  pa.dst = (double*)d_R;
  pa.ldd = ldr;
  {
    TraceScope ts(h, DD_PH_PERM, 0.0, st);
    launch_perm_out(C, pa, st);
  }
  LAUNCH_CHECK("k_perm_out");
  return DD_OK;
}

}  // extern "C"

extern "C" {

// Per-column backward error ||b - A x||_inf / (||A||_inf ||x||_inf) on the device (K6 residual,
// ||A||_inf and k_berr; reading L6), copied to the host: a convergence report for any solve.
int dd_aux_backward_error(dd_aux_handle_t h, const void* d_factor, const void* d_vals, int64_t nrhs, const void* d_B,
                          int64_t ldb, const void* d_X, int64_t ldx, void* d_work, double* berr, void* stream) {
  if (!h) return fail(-1, "handle is NULL");
  if (!d_factor) return fail(-2, "d_factor is NULL");
  if (!d_vals) return fail(-3, "d_vals is NULL");
  if (nrhs < 0 || nrhs > SOLVE_MAX_COLS) return fail(-4, "nrhs must be in [0, 32768]");
  if (nrhs == 0) return DD_OK;
  if (!d_B || ldb < h->n) return fail(-5, "d_B is NULL or ldb < n");
  if (!d_X || ldx < h->n) return fail(-7, "d_X is NULL or ldx < n");
  if (!d_work || ((uintptr_t)d_work & 255)) return fail(-9, "d_work is NULL or not 256-byte aligned");
  if (!berr) return fail(-10, "berr is NULL");
  if (!h->factored || h->factored_ptr != d_factor) return fail(DD_ERR_NOT_FACTORED, "not factored (row maps)");
  cudaStream_t st = (cudaStream_t)stream;
  const bool C = h->cplx;
  const int planes = C ? 2 : 1;
  uint8_t* F = (uint8_t*)const_cast<void*>(d_factor);
  uint8_t* Wb = (uint8_t*)d_work;
  const int64_t ldy = pad8(h->n_pad);
  double* y = (double*)Wb;
  const int64_t yim = C ? ldy * nrhs : 0;
  double* Bsave = (double*)(Wb + align256((size_t)ldy * nrhs * planes * sizeof(double)));
  double* berr_d = (double*)((uint8_t*)Bsave + align256((size_t)h->n * nrhs * planes * sizeof(double)));
  int* flag_d = (int*)((uint8_t*)berr_d + align256((size_t)nrhs * sizeof(double)));
  unsigned long long* norm_d = (unsigned long long*)(F + h->off_norm);
  SpmvArgs sa{};
  sa.rows = (const SpRow*)(F + h->off_sprows);
  sa.segs = (const SpSeg*)(F + h->off_spsegs);
  sa.blk_size = (const int64_t*)(F + h->off_blksize);
  sa.odof = (const int64_t*)(F + h->off_odof);
  sa.vals = (const double*)d_vals;
  sa.X = (const double*)d_X;
  sa.ldx = ldx;
  sa.Bsave = (const double*)d_B;
  sa.ldb = ldb;
  sa.ginv = (const int*)(F + h->off_ginv);
  sa.y = y;
  sa.yim = yim;
  sa.ldy = ldy;
  sa.nrhs = (int)nrhs;
  launch_spmv(C, sa, h->n_sprows, st);
  LAUNCH_CHECK("k_spmv");
  CUDA_TRY(cudaMemsetAsync(norm_d, 0, sizeof(unsigned long long), st));
  launch_norm_a(C, sa, h->n_sprows, norm_d, st);
  LAUNCH_CHECK("k_norm_a");
  CUDA_TRY(cudaMemsetAsync(flag_d, 0, sizeof(int), st));
  launch_berr(C, y, yim, ldy, h->n_pad, (const double*)d_X, ldx, h->n, (int)nrhs, norm_d, 0.0, berr_d, flag_d, st);
  LAUNCH_CHECK("k_berr");
  h->norm_valid = false;
  CUDA_TRY(cudaMemcpyAsync(berr, berr_d, (size_t)nrhs * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DD_OK;
}

}  // extern "C"

// ============================================================================ table validation
// compute-sanitizer is closed on the GPU pool, so every descriptor the kernels index through is
// checked on the host instead: each access a kernel derives from a table entry must fall inside
// its buffer (arena, W / K1 workspace, solve rows).  Integer work only; used by the CPU test suite
// on many random patterns and in Schur mode.
template <class T>
static const T* blob_at(dd_aux_handle_t h, size_t off) {
  return (const T*)(h->blob.data.data() + off);
}

extern "C" int dd_aux_validate(dd_aux_handle_t h) {
  if (!h) return fail(-1, "handle is NULL");
  const int N = h->S.nblk;
  auto bad = [&](const std::string& m) { return fail(DD_ERR_INTERNAL, "validate: " + m); };
  // panels, inverse tiles, full inverses: in bounds and disjoint
  std::vector<std::pair<int64_t, int64_t>> reg;
  for (int t = 0; t < N; ++t) {
    const NodeDev& nd = h->nodes[t];
    if (nd.s <= 0 || nd.sp < nd.s || nd.ld < nd.sp + nd.rp || nd.ld % 8) return bad("panel shape of node " + std::to_string(t));
    reg.push_back({nd.panel, nd.panel + (int64_t)nd.ld * nd.s});
    reg.push_back({nd.linv, nd.linv + (int64_t)((nd.s + TB - 1) / TB) * TB * TB});
    reg.push_back({nd.inv, nd.inv + (int64_t)nd.ldi * nd.s});
    if (nd.ydof + nd.sp > h->n_pad) return bad("ydof of node " + std::to_string(t));
    int64_t ro = nd.sp;
    for (int q = 0; q < nd.nst; ++q) {
      const int u = h->S.st[t][q];
      if (u <= t || u >= N) return bad("struct order of node " + std::to_string(t));
      ro += pad2(h->nodes[u].s);
    }
    if (ro != nd.sp + nd.rp) return bad("struct rows of node " + std::to_string(t));
  }
  reg.push_back({h->d_off, h->d_off + h->n_pad});
  reg.push_back({h->e_off, h->e_off + h->n_pad});
  std::sort(reg.begin(), reg.end());
  for (size_t q = 0; q < reg.size(); ++q) {
    if (reg[q].first < 0 || reg[q].second > h->nA) return bad("arena region out of bounds");
    if (q && reg[q].first < reg[q - 1].second) return bad("arena regions overlap");
  }
  // per-level workspace (W, K1 scratch)
  for (const auto& L : h->S.level_nodes)
    for (int t : L) {
      const NodeDev& nd = h->nodes[t];
      if (nd.w + (int64_t)nd.ldw * nd.s > h->nW || nd.ldw < nd.rp) return bad("W of node " + std::to_string(t));
      if (nd.k1w + (int64_t)nd.sp * K1NB_MAX > h->nK1) return bad("K1 scratch of node " + std::to_string(t));
    }
  // Schur update targets / contributors
  const UpdTarget* tg = blob_at<UpdTarget>(h, h->off_targets);
  const UpdContrib* uc = blob_at<UpdContrib>(h, h->off_contribs);
  const size_t ntg = (h->off_contribs - h->off_targets) / sizeof(UpdTarget);
  for (const LevelRanges& R : h->lv) {
    if (R.t1 < R.t0 || (size_t)R.t1 > ntg) return bad("target range");
    for (int q = R.t0; q < R.t1; ++q) {
      const UpdTarget& T = tg[q];
      if (T.j < 0 || T.j >= N) return bad("target panel");
      const NodeDev& nj = h->nodes[T.j];
      if (T.N != nj.s || T.ro + T.M > nj.ld || (T.diag && (T.ro != 0 || T.M != T.N))) return bad("target rows");
      for (int c = T.c0; c < T.c1; ++c) {
        const NodeDev& nk = h->nodes[uc[c].k];
        if (uc[c].k < 0 || uc[c].k >= T.j) return bad("contributor not eliminated before its target panel");
        if (uc[c].arow < 0 || uc[c].arow + T.M > nk.rp) return bad("contributor W rows");
        if (uc[c].brow < nk.sp || uc[c].brow + T.N > nk.ld) return bad("contributor L rows");
      }
    }
  }
  // forward-solve targets
  const SolveTarget* ft = blob_at<SolveTarget>(h, h->off_ftargets);
  const SolveContrib* fc = blob_at<SolveContrib>(h, h->off_fcontribs);
  for (const LevelRanges& R : h->lv)
    for (int q = R.f0; q < R.f1; ++q) {
      const NodeDev& ni = h->nodes[ft[q].i];
      if (ft[q].tm * solve_bm(h->cplx) >= ni.s) return bad("forward tile");
      for (int c = ft[q].c0; c < ft[q].c1; ++c)
        if (fc[c].ro + ni.s > h->nodes[fc[c].k].ld) return bad("forward contributor rows");
    }
  // Schur mode: export items within the arena, gather/scatter rows within the solve vector
  if (h->n_schur > 0) {
    const SxItem* it = blob_at<SxItem>(h, h->off_sx_items);
    const size_t nit = (h->off_sx_tiles - h->off_sx_items) / sizeof(SxItem);
    for (size_t q = 0; q < nit; ++q) {
      if (it[q].mode == 3) continue;
      const int64_t last = it[q].mode == 1 ? it[q].src + (it[q].cols - 1) + (int64_t)(it[q].rows - 1) * it[q].ld
                                           : it[q].src + (it[q].rows - 1) + (int64_t)(it[q].cols - 1) * it[q].ld;
      if (it[q].src < 0 || last >= h->nA) return bad("export item out of the arena");
      if (it[q].dst + (it[q].rows - 1) + (int64_t)(it[q].cols - 1) * it[q].m >= (int64_t)it[q].m * it[q].m)
        return bad("export item out of its S_g");
    }
    const SgItem* ss = blob_at<SgItem>(h, h->off_ss_items);
    for (int q = 0; q < h->n_ss_items; ++q) {
      const NodeDev& nd = h->nodes[ss[q].c0];
      if (ss[q].c0 < h->n_elim || nd.s != ss[q].s || ss[q].aux_row + ss[q].s > h->n_aux_dof) return bad("scatter item");
    }
  }
  return DD_OK;
}
