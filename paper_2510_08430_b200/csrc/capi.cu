// capi.cu — extern "C" entry points of libsrblock.so (declared in include/sr_block.h).
// Argument checking, workspace carving and stage sequencing only; every arithmetic step
// of the path runs in the kernels of mlp.cu, center.cu, gram.cuh and chol.cu.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "chol.cuh"
#include "gram.cuh"
#include "net.cuh"
#include "ozaki.cuh"

namespace sr {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
void set_error(const std::string& m) { g_err = m; }
void count_launch(int n) { g_launches += n; }
int g_gram_engine = SR_GRAM_INT8;   // default: int8 tcgen05 digit slices (R10)
int gram_engine() { return g_gram_engine; }

struct TimedLaunch {
  std::string name;
  cudaEvent_t a, b;
  cudaStream_t st;
};
bool g_timer = false;
std::vector<TimedLaunch> g_timed;
std::vector<cudaEvent_t> g_event_pool;
bool g_timer_open = false;

cudaEvent_t timer_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void timer_begin(const char* kernel, cudaStream_t st) {
  g_timer_open = false;
  if (!g_timer) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone) return;
  TimedLaunch t{kernel, timer_event(), timer_event(), st};
  cudaEventRecord(t.a, st);
  g_timed.push_back(t);
  g_timer_open = true;
}
void timer_end(cudaStream_t st) {
  if (!g_timer_open) return;
  cudaEventRecord(g_timed.back().b, st);
  g_timer_open = false;
}

sr_status jacobian_impl(const NetDesc&, const double*, const int8_t*, long long, double*, double*, long long,
                        void*, size_t, cudaStream_t);
size_t jacobian_ws(const NetDesc&, long long);
size_t local_energy_ws(const NetDesc&, long long, long long);
sr_status local_energy_impl(const NetDesc&, const double*, long long, const int32_t*, const double*,
                            const int8_t*, long long, const double*, double*, void*, size_t, cudaStream_t);
size_t center_force_ws(long long, long long);
sr_status center_force_impl(long long, long long, double*, long long, const double*, const double*, double*,
                            double*, double*, void*, size_t, cudaStream_t);
size_t aHv_ws(long long, long long);
sr_status column_moments_impl(long long, long long, long long, const double*, long long, const double*, const double*,
                              double*, void*, size_t, cudaStream_t);
sr_status center_force_global_impl(long long, long long, long long, double*, long long, const double*,
                                   const double*, int, const double*, double*, double*, double*, void*, size_t,
                                   cudaStream_t);
sr_status aHv_impl(long long, long long, const double2*, long long, const double2*, double, double2*, void*,
                   size_t, cudaStream_t);

namespace {

__global__ void copy_unpad(const double2* __restrict__ src, long long lds, double2* __restrict__ dst,
                           long long ldd, long long rows, long long cols) {
  const long long total = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols, c = e % cols;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

sr_status copy_matrix(const double2* src, long long lds, double2* dst, long long ldd, long long rows,
                      long long cols, cudaStream_t st) {
  if (rows * cols == 0) return SR_OK;
  const unsigned g = (unsigned)std::min<long long>((rows * cols + 255) / 256, 8 * kNumSMs);
  copy_unpad<<<g, 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  SR_LAUNCHED();
  return SR_OK;
}

bool valid_offsets(int nblk, const int64_t* offs) {
  if (nblk < 1 || nblk > kMaxBlocks || offs == nullptr || offs[0] != 0) return false;
  for (int b = 0; b < nblk; b++)
    if (offs[b + 1] <= offs[b]) return false;
  return true;
}

size_t block_solve_ws(int nblk, const int64_t* offs) {
  std::vector<long long> sizes(nblk);
  for (int b = 0; b < nblk; b++) sizes[b] = offs[b + 1] - offs[b];
  Arena a(nullptr, 0);
  CholSet cs{};
  carve_chol(a, cs, sizes.data(), nblk);
  return a.used;
}

// FP64 engine's QGT Grams with TMA-staged K-slabs (SR_FP64_TMA=0: the cp.async kernel).
bool fp64_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_FP64_TMA");
    v = e ? atoi(e) != 0 : 1;
  }
  return v != 0;
}

sr_status block_qgt_impl(long long ns, int nblk, const int64_t* offs, const double2* A, long long lda,
                         double2* S, cudaStream_t st) {
  gram::ProbSet ps{};
  long long soff = 0;
  for (int b = 0; b < nblk; b++) {
    const long long n = offs[b + 1] - offs[b];
    gram::add_prob(ps, A + offs[b], lda, A + offs[b], lda, S + soff, n, (int)n, (int)n, ns, true);
    soff += n * n;
  }
  timer_begin("gram_tn", st);
  // every block is a column range of A: K-slabs staged by TMA (gram::tn_tma_kernel)
  const sr_status r = fp64_tma() && ns > 0
                          ? gram::launch_tn_tma<gram::HERM_STORE>(ps, A, lda, offs[nblk], ns, st)
                          : gram::launch<gram::TN, gram::HERM_STORE>(ps, st);
  timer_end(st);
  return r;
}

sr_status block_solve_impl(int nblk, const int64_t* offs, const double2* S, const double2* F, double lam,
                           double2* dtheta, int* info, void* ws, size_t bytes, cudaStream_t st) {
  std::vector<long long> sizes(nblk);
  for (int b = 0; b < nblk; b++) sizes[b] = offs[b + 1] - offs[b];
  Arena a(ws, bytes);
  CholSet cs{};
  cs.info = info;
  carve_chol(a, cs, sizes.data(), nblk);
  if (!a.ok()) {
    set_error("sr_block_solve: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  long long soff = 0;
  for (int b = 0; b < nblk; b++) {
    cs.b[b].S = S + soff;
    cs.b[b].F = F + offs[b];
    cs.b[b].out = dtheta + offs[b];
    soff += sizes[b] * sizes[b];
  }
  return chol_solve(cs, lam, false, -1.0, st);
}

// The comparison solves' Grams run on the selected engine (sr_set_gram_engine); the int8
// engine's digit slices follow the Cholesky workspace.
size_t full_i8_ws(long long ns, long long n_p) {
  if (ns < 1) return 0;
  const int64_t o[2] = {0, n_p};
  return oz::workspace_bytes(ns, 1, o);
}

size_t full_qgt_ws(long long ns, long long n_p) {
  long long sz = n_p;
  Arena a(nullptr, 0);
  CholSet cs{};
  carve_chol(a, cs, &sz, 1);
  return round256(a.used) + full_i8_ws(ns, n_p);
}

// S = A^H A (n x n, the n columns of A at lda) formed straight into the padded Cholesky
// matrix on the selected Gram engine, then (S + lambda I) out = -F.  keep_info: *info is
// not reset (blocks solved one call at a time report the first failure); row_base: the
// global row of column 0 in the reported pivot.
sr_status gram_solve_one(long long ns, long long n, const double2* A, long long lda, const double2* F, double lam,
                         double2* out, double2* S_out, int* info, bool keep_info, long long row_base, void* ws,
                         size_t bytes, cudaStream_t st) {
  long long sz = n;
  Arena a(ws, bytes);
  CholSet cs{};
  cs.info = info;
  cs.keep_info = keep_info;
  carve_chol(a, cs, &sz, 1);
  if (!a.ok()) {
    set_error("gram + solve: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  CholBlock& B = cs.b[0];
  B.row_base = row_base;
  if (g_gram_engine == SR_GRAM_INT8 && ns > 0) {   // S straight into the padded factor matrix
    const size_t used = round256(a.used);
    const int64_t o[2] = {0, n};
    SR_TRY(oz::block_qgt_i8(ns, 1, o, A, lda, B.Fm, static_cast<char*>(ws) + used, bytes > used ? bytes - used : 0,
                            st, B.npad));
  } else {
    gram::ProbSet ps{};
    gram::add_prob(ps, A, lda, A, lda, B.Fm, B.npad, (int)n, (int)n, ns, true);
    timer_begin("gram_tn", st);
    const sr_status r = fp64_tma() && ns > 0 ? gram::launch_tn_tma<gram::HERM_STORE>(ps, A, lda, n, ns, st)
                                             : gram::launch<gram::TN, gram::HERM_STORE>(ps, st);
    timer_end(st);
    SR_TRY(r);
  }
  if (S_out) SR_TRY(copy_matrix(B.Fm, B.npad, S_out, n, n, n, st));
  B.F = F;
  B.out = out;
  return chol_solve(cs, lam, true, -1.0, st);
}

// Stages (4)+(5) per block: block b's S_b is formed in its padded factor matrix and solved
// before block b+1's Gram, so the workspace holds one block (the largest) instead of every
// S_b plus its factor copy (sr_block_qgt_solve, the SR_SCHED_PER_BLOCK step schedule).
size_t qgt_solve_ws(long long ns, int nblk, const int64_t* offs) {
  size_t mx = 0;
  for (int b = 0; b < nblk; b++) mx = std::max(mx, full_qgt_ws(ns, offs[b + 1] - offs[b]));
  return round256(sizeof(int)) + mx;
}

sr_status qgt_solve_impl(long long ns, int nblk, const int64_t* offs, const double2* A, long long lda,
                         const double2* F, double lam, double2* dtheta, int* info, void* ws, size_t bytes,
                         cudaStream_t st) {
  if (bytes < qgt_solve_ws(ns, nblk, offs)) {
    set_error("sr_block_qgt_solve: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  if (info) SR_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
  char* rest = static_cast<char*>(ws) + round256(sizeof(int));
  const size_t rbytes = bytes - round256(sizeof(int));
  for (int b = 0; b < nblk; b++)
    SR_TRY(gram_solve_one(ns, offs[b + 1] - offs[b], A + offs[b], lda, F + offs[b], lam, dtheta + offs[b], nullptr,
                          info, true, offs[b], rest, rbytes, st));
  return SR_OK;
}

int g_step_schedule = SR_SCHED_BATCHED;

struct StepLayout {
  NetDesc net;
  std::vector<int64_t> offs;
  size_t log_psi, O, e_loc, energy, e_tilde, F, S, scratch, scratch_bytes, total, chol_off;
  bool per_block;
  size_t h_theta, h_spins, h_bij, h_bj, h_dtheta, h_energy, host_total;
};

std::vector<int64_t> largest_block(const std::vector<int64_t>& offs) {
  int64_t mx = 0;
  for (size_t b = 0; b + 1 < offs.size(); b++) mx = std::max(mx, offs[b + 1] - offs[b]);
  return {0, mx};
}

// Pipelined step (int8 engine, SR_PIPE=1): the Grams of the blocks run one after another on
// the step stream, largest first, and block b's Cholesky starts on its side stream as soon
// as S_b is complete, so the panel chains overlap the remaining Grams.  Off by default: the
// step is power-bound, and the per-block Gram launches cost more than the overlap gains
// (configs[1] graph 36.2-36.3 vs 35.8-35.9 ms).
bool pipe_step() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_PIPE");
    v = e ? atoi(e) != 0 : 0;
  }
  return v != 0;
}

sr_status pipelined_qgt_solve(int nblk, const int64_t* offs, long long ns, const double2* A, long long lda,
                              double2* S, const double2* F, double lam, double2* dtheta, char* scr,
                              size_t scr_bytes, size_t chol_off, cudaStream_t st) {
  static cudaEvent_t ready[kMaxBlocks];
  static bool made = false;
  if (!made) {
    for (int b = 0; b < kMaxBlocks; b++) SR_CUDA(cudaEventCreateWithFlags(&ready[b], cudaEventDisableTiming));
    made = true;
  }
  std::vector<long long> sizes(nblk), soff(nblk);
  std::vector<int> order(nblk);
  long long so = 0;
  for (int b = 0; b < nblk; b++) {
    sizes[b] = offs[b + 1] - offs[b];
    soff[b] = so;
    so += sizes[b] * sizes[b];
    order[b] = b;
  }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sizes[x] > sizes[y]; });
  Arena a(scr + chol_off, scr_bytes - chol_off);
  CholSet cs{};
  cs.info = nullptr;
  carve_chol(a, cs, sizes.data(), nblk);
  if (!a.ok()) {
    set_error("sr_step: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  for (int b = 0; b < nblk; b++) {
    cs.b[b].S = S + soff[b];
    cs.b[b].F = F + offs[b];
    cs.b[b].out = dtheta + offs[b];
  }
  for (int b : order) {
    const int64_t o1[2] = {0, sizes[b]};
    SR_TRY(oz::block_qgt_i8(ns, 1, o1, A + offs[b], lda, S + soff[b], scr, chol_off, st));
    SR_CUDA(cudaEventRecord(ready[b], st));
  }
  return chol_solve(cs, lam, false, -1.0, st, ready);
}

sr_status step_layout(int n_layers, const int32_t* widths, long long ns, long long nb, StepLayout* L) {
  SR_TRY(make_net(n_layers, widths, &L->net));
  const NetDesc& net = L->net;
  L->offs.assign(n_layers + 1, 0);
  for (int l = 0; l < n_layers; l++) L->offs[l + 1] = L->offs[l] + (int64_t)net.w[l + 1] * (net.w[l] + 1);
  long long s_elems = 0;
  for (int l = 0; l < n_layers; l++) s_elems += (L->offs[l + 1] - L->offs[l]) * (L->offs[l + 1] - L->offs[l]);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += round256(bytes);
    return o;
  };
  const size_t c16 = sizeof(double2);
  L->log_psi = take(ns * c16);
  L->O = take((size_t)ns * net.n_p * c16);
  L->e_loc = take(ns * c16);
  L->energy = take(c16);
  L->e_tilde = take(ns * c16);
  L->F = take(net.n_p * c16);
  const bool per_block = g_step_schedule == SR_SCHED_PER_BLOCK;
  L->per_block = per_block;
  L->S = take(per_block ? 0 : (size_t)s_elems * c16);
  size_t scr = jacobian_ws(net, ns);
  scr = std::max(scr, local_energy_ws(net, ns, nb));
  scr = std::max(scr, center_force_ws(ns, net.n_p));
  if (per_block) {
    L->chol_off = 0;
    scr = std::max(scr, qgt_solve_ws(ns, n_layers, L->offs.data()));
  } else {
    scr = std::max(scr, block_solve_ws(n_layers, L->offs.data()));
    scr = std::max(scr, oz::workspace_bytes(ns, n_layers, L->offs.data()));
    // pipelined int8 step: the digit slices of one block and the Cholesky workspace of all
    // blocks are live at once
    L->chol_off = round256(oz::workspace_bytes(ns, 1, largest_block(L->offs).data()));
    scr = std::max(scr, L->chol_off + block_solve_ws(n_layers, L->offs.data()));
  }
  L->scratch_bytes = round256(scr);
  L->scratch = take(L->scratch_bytes);
  L->total = off;
  L->h_theta = take(net.n_p * c16);
  L->h_spins = take((size_t)ns * net.w[0]);
  L->h_bij = take((size_t)nb * 2 * sizeof(int32_t));
  L->h_bj = take((size_t)nb * sizeof(double));
  L->h_dtheta = take(net.n_p * c16);
  L->h_energy = take(c16);
  L->host_total = off - L->total;
  return SR_OK;
}

sr_status step_impl(const StepLayout& L, const double* theta, const int8_t* spins, long long ns, long long nb,
                    const int32_t* bij, const double* bj, double lam, double* dtheta, double* energy, char* ws,
                    cudaStream_t st) {
  const NetDesc& net = L.net;
  double* log_psi = reinterpret_cast<double*>(ws + L.log_psi);
  double* O = reinterpret_cast<double*>(ws + L.O);
  double* e_loc = reinterpret_cast<double*>(ws + L.e_loc);
  double* e_tilde = reinterpret_cast<double*>(ws + L.e_tilde);
  double* F = reinterpret_cast<double*>(ws + L.F);
  double2* S = reinterpret_cast<double2*>(ws + L.S);
  void* scr = ws + L.scratch;
  SR_TRY(jacobian_impl(net, theta, spins, ns, log_psi, O, net.n_p, scr, L.scratch_bytes, st));
  SR_TRY(local_energy_impl(net, theta, nb, bij, bj, spins, ns, log_psi, e_loc, scr, L.scratch_bytes, st));
  SR_TRY(center_force_impl(ns, net.n_p, O, net.n_p, nullptr, e_loc, energy, e_tilde, F, scr, L.scratch_bytes, st));
  if (L.per_block)
    return qgt_solve_impl(ns, net.L, L.offs.data(), reinterpret_cast<const double2*>(O), net.n_p,
                          reinterpret_cast<const double2*>(F), lam, reinterpret_cast<double2*>(dtheta), nullptr, scr,
                          L.scratch_bytes, st);
  if (g_gram_engine == SR_GRAM_INT8 && pipe_step())
    return pipelined_qgt_solve(net.L, L.offs.data(), ns, reinterpret_cast<const double2*>(O), net.n_p, S,
                               reinterpret_cast<const double2*>(F), lam, reinterpret_cast<double2*>(dtheta),
                               reinterpret_cast<char*>(scr), L.scratch_bytes, L.chol_off, st);
  if (g_gram_engine == SR_GRAM_INT8)
    SR_TRY(oz::block_qgt_i8(ns, net.L, L.offs.data(), reinterpret_cast<const double2*>(O), net.n_p, S, scr,
                            L.scratch_bytes, st));
  else
    SR_TRY(block_qgt_impl(ns, net.L, L.offs.data(), reinterpret_cast<const double2*>(O), net.n_p, S, st));
  SR_TRY(block_solve_impl(net.L, L.offs.data(), S, reinterpret_cast<const double2*>(F), lam,
                          reinterpret_cast<double2*>(dtheta), nullptr, scr, L.scratch_bytes, st));
  return SR_OK;
}

// CUDA-graph cache of sr_step_host: the ~900 launches of a step are captured once per
// (workspace, shapes, lambda, engine) and replayed, so the host-buffer path pays one graph
// launch instead of the per-kernel launch overhead.  The step reads its inputs from fixed
// places in the workspace (sr_step_host copies them there first), so a replay is exact.
// SR_STEP_GRAPH=0 turns it off.
struct StepGraphKey {
  const void* ws;
  std::vector<int32_t> widths;
  long long ns, nb;
  double lam;
  int engine, schedule;
  bool operator==(const StepGraphKey& o) const {
    return ws == o.ws && widths == o.widths && ns == o.ns && nb == o.nb && lam == o.lam && engine == o.engine &&
           schedule == o.schedule;
  }
};
struct StepGraph {
  StepGraphKey key;
  cudaGraphExec_t exec;
};
std::vector<StepGraph> g_step_graphs;
bool step_graph_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_STEP_GRAPH");
    v = e ? atoi(e) != 0 : 1;
  }
  return v != 0;
}

sr_status step_graphed(const StepLayout& L, const StepGraphKey& key, const double* theta, const int8_t* spins,
                       long long ns, long long nb, const int32_t* bij, const double* bj, double lam, double* dtheta,
                       double* energy, char* ws, cudaStream_t st) {
  if (!step_graph_enabled())
    return step_impl(L, theta, spins, ns, nb, bij, bj, lam, dtheta, energy, ws, st);
  for (StepGraph& g : g_step_graphs)
    if (g.key == key) {
      SR_CUDA(cudaGraphLaunch(g.exec, st));
      return SR_OK;
    }
  static cudaStream_t cap = nullptr;
  if (!cap) SR_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  SR_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  const sr_status r = step_impl(L, theta, spins, ns, nb, bij, bj, lam, dtheta, energy, ws, cap);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cap, &graph);
  cudaGraphExec_t exec = nullptr;
  if (r != SR_OK || ec != cudaSuccess ||
      cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (r != SR_OK) return r;
    set_error(std::string("sr_step_host: graph capture failed: ") + cudaGetErrorString(ec));
    return SR_ERR_CUDA;
  }
  cudaGraphDestroy(graph);
  if (g_step_graphs.size() >= 4) {
    cudaGraphExecDestroy(g_step_graphs.front().exec);
    g_step_graphs.erase(g_step_graphs.begin());
  }
  g_step_graphs.push_back({key, exec});
  SR_CUDA(cudaGraphLaunch(exec, st));
  return SR_OK;
}

}  // namespace
}  // namespace sr

using namespace sr;

extern "C" {

SR_API int sr_version(void) { return 100; }
SR_API const char* sr_last_error(void) { return g_err.c_str(); }
SR_API int64_t sr_launch_count(void) { return g_launches; }
SR_API void sr_reset_launch_count(void) { g_launches = 0; }

SR_API size_t sr_jacobian_workspace_bytes(int n_layers, const int32_t* widths, int64_t n_samples) {
  NetDesc net;
  if (make_net(n_layers, widths, &net) != SR_OK || n_samples < 0) return 0;
  return jacobian_ws(net, n_samples);
}

SR_API sr_status sr_jacobian(int n_layers, const int32_t* widths, const double* theta, const int8_t* spins,
                             int64_t n_samples, double* log_psi, double* O, int64_t ldo, void* workspace,
                             size_t workspace_bytes, void* stream) {
  NetDesc net;
  SR_TRY(make_net(n_layers, widths, &net));
  SR_CHECK_ARG(n_samples >= 0, "n_samples < 0");
  SR_CHECK_ARG(ldo >= net.n_p, "ldo < n_p");
  SR_CHECK_ARG(n_samples == 0 || (theta && spins && log_psi && O && workspace), "null pointer");
  return jacobian_impl(net, theta, spins, n_samples, log_psi, O, ldo, workspace, workspace_bytes,
                       (cudaStream_t)stream);
}

SR_API size_t sr_local_energy_workspace_bytes(int n_layers, const int32_t* widths, int64_t n_samples,
                                              int64_t n_bonds) {
  NetDesc net;
  if (make_net(n_layers, widths, &net) != SR_OK || n_samples < 0 || n_bonds < 0) return 0;
  return local_energy_ws(net, n_samples, n_bonds);
}

SR_API sr_status sr_local_energy(int n_layers, const int32_t* widths, const double* theta, int64_t n_bonds,
                                 const int32_t* bonds_ij, const double* bond_j, const int8_t* spins,
                                 int64_t n_samples, const double* log_psi, double* e_loc, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  NetDesc net;
  SR_TRY(make_net(n_layers, widths, &net));
  SR_CHECK_ARG(n_samples >= 0 && n_bonds >= 0, "negative size");
  SR_CHECK_ARG(n_samples == 0 || (theta && spins && log_psi && e_loc && workspace), "null pointer");
  SR_CHECK_ARG(n_bonds == 0 || (bonds_ij && bond_j), "null bond arrays");
  return local_energy_impl(net, theta, n_bonds, bonds_ij, bond_j, spins, n_samples, log_psi, e_loc, workspace,
                           workspace_bytes, (cudaStream_t)stream);
}

SR_API size_t sr_center_force_workspace_bytes(int64_t n_samples, int64_t n_p) {
  if (n_samples < 0 || n_p < 0) return 0;
  return center_force_ws(n_samples, n_p);
}

SR_API sr_status sr_center_force(int64_t n_samples, int64_t n_p, double* O, int64_t ldo, const double* weights,
                                 const double* e_loc, double* energy, double* e_tilde, double* F, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_samples >= 1 && n_p >= 1, "n_samples and n_p must be >= 1");
  SR_CHECK_ARG(ldo >= n_p, "ldo < n_p");
  SR_CHECK_ARG(O && e_loc && e_tilde && F && workspace, "null pointer");
  return center_force_impl(n_samples, n_p, O, ldo, weights, e_loc, energy, e_tilde, F, workspace, workspace_bytes,
                           (cudaStream_t)stream);
}

SR_API size_t sr_column_moments_workspace_bytes(int64_t n_local, int64_t n_p) {
  if (n_local < 0 || n_p < 0) return 0;
  return center_force_ws(n_local, n_p);
}

SR_API sr_status sr_column_moments(int64_t n_local, int64_t n_total, int64_t n_p, const double* O, int64_t ldo,
                                   const double* weights, const double* e_loc, double* moments, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_local >= 1 && n_total >= n_local && n_p >= 1, "bad sizes");
  SR_CHECK_ARG(ldo >= n_p, "ldo < n_p");
  SR_CHECK_ARG(O && e_loc && moments && workspace, "null pointer");
  return column_moments_impl(n_local, n_total, n_p, O, ldo, weights, e_loc, moments, workspace, workspace_bytes,
                             (cudaStream_t)stream);
}

SR_API sr_status sr_center_force_global(int64_t n_local, int64_t n_total, int64_t n_p, double* O, int64_t ldo,
                                        const double* weights, const double* e_loc, int n_parts,
                                        const double* moments, double* energy, double* e_tilde, double* F_partial,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_local >= 1 && n_total >= n_local && n_p >= 1 && n_parts >= 1, "bad sizes");
  SR_CHECK_ARG(ldo >= n_p, "ldo < n_p");
  SR_CHECK_ARG(O && e_loc && moments && e_tilde && F_partial && workspace, "null pointer");
  return center_force_global_impl(n_local, n_total, n_p, O, ldo, weights, e_loc, n_parts, moments, energy, e_tilde,
                                  F_partial, workspace, workspace_bytes, (cudaStream_t)stream);
}

SR_API size_t sr_block_qgt_workspace_bytes(int n_blocks, const int64_t* block_offsets) {
  (void)n_blocks;
  (void)block_offsets;
  return 0;
}

SR_API sr_status sr_block_qgt(int64_t n_samples, int n_blocks, const int64_t* block_offsets, const double* A,
                              int64_t lda, double* S, void* workspace, size_t workspace_bytes, void* stream) {
  (void)workspace;
  (void)workspace_bytes;
  SR_CHECK_ARG(valid_offsets(n_blocks, block_offsets), "block_offsets must start at 0 and increase; 1..24 blocks");
  SR_CHECK_ARG(n_samples >= 0 && lda >= block_offsets[n_blocks], "lda < n_p");
  for (int b = 0; b < n_blocks; b++)
    SR_CHECK_ARG(block_offsets[b + 1] - block_offsets[b] < (1LL << 31), "block too large");
  SR_CHECK_ARG(S && (A || n_samples == 0), "null pointer");
  return block_qgt_impl(n_samples, n_blocks, block_offsets, reinterpret_cast<const double2*>(A), lda,
                        reinterpret_cast<double2*>(S), (cudaStream_t)stream);
}

SR_API size_t sr_block_qgt_i8_workspace_bytes(int64_t n_samples, int n_blocks, const int64_t* block_offsets) {
  if (n_samples < 0 || !valid_offsets(n_blocks, block_offsets)) return 0;
  return oz::workspace_bytes(n_samples, n_blocks, block_offsets);
}

SR_API sr_status sr_block_qgt_i8(int64_t n_samples, int n_blocks, const int64_t* block_offsets, const double* A,
                                 int64_t lda, double* S, void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(valid_offsets(n_blocks, block_offsets), "block_offsets must start at 0 and increase; 1..24 blocks");
  SR_CHECK_ARG(n_samples >= 0 && lda >= block_offsets[n_blocks], "lda < n_p");
  SR_CHECK_ARG(block_offsets[n_blocks] < (1LL << 31) / oz::kSlices, "n_p too large for the slice tensor map");
  SR_CHECK_ARG(n_samples <= (1LL << 31) / 8, "n_samples too large");
  SR_CHECK_ARG(S && (A || n_samples == 0), "null pointer");
  return oz::block_qgt_i8(n_samples, n_blocks, block_offsets, reinterpret_cast<const double2*>(A), lda,
                          reinterpret_cast<double2*>(S), workspace, workspace_bytes, (cudaStream_t)stream);
}

SR_API sr_status sr_block_qgt_i8_acc(int64_t n_samples, int n_blocks, const int64_t* block_offsets, const double* A,
                                     int64_t lda, double* S, void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(valid_offsets(n_blocks, block_offsets), "block_offsets must start at 0 and increase; 1..24 blocks");
  SR_CHECK_ARG(n_samples >= 0 && lda >= block_offsets[n_blocks], "lda < n_p");
  SR_CHECK_ARG(block_offsets[n_blocks] < (1LL << 31) / oz::kSlices, "n_p too large for the slice tensor map");
  SR_CHECK_ARG(n_samples <= (1LL << 31) / 8, "n_samples too large");
  SR_CHECK_ARG(S && (A || n_samples == 0), "null pointer");
  return oz::block_qgt_i8(n_samples, n_blocks, block_offsets, reinterpret_cast<const double2*>(A), lda,
                          reinterpret_cast<double2*>(S), workspace, workspace_bytes, (cudaStream_t)stream, 0, true);
}

SR_API void sr_kernel_timer(int enable) { g_timer = enable != 0; }

SR_API sr_status sr_gram_nh(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                            int64_t ldb, double* C, int64_t ldc, void* stream) {
  SR_CHECK_ARG(m >= 0 && n >= 0 && k >= 0 && m < (1LL << 31) && n < (1LL << 31), "bad sizes");
  SR_CHECK_ARG(lda >= k && ldb >= k && ldc >= n, "leading dimension too small");
  if (m == 0 || n == 0) return SR_OK;
  SR_CHECK_ARG(C && ((A && B) || k == 0), "null pointer");
  gram::ProbSet ps{};
  gram::add_prob(ps, reinterpret_cast<const double2*>(A), lda, reinterpret_cast<const double2*>(B), ldb,
                 reinterpret_cast<double2*>(C), ldc, (int)m, (int)n, k, false);
  return gram::launch<gram::NH, gram::STORE>(ps, (cudaStream_t)stream);
}

SR_API size_t sr_aHv_workspace_bytes(int64_t n_rows, int64_t n_p) {
  if (n_rows < 1 || n_p < 1) return 0;
  return aHv_ws(n_rows, n_p);
}

SR_API sr_status sr_aHv(int64_t n_rows, int64_t n_p, const double* A, int64_t lda, const double* v, double alpha,
                        double* out, void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_rows >= 1 && n_p >= 1 && lda >= n_p, "bad sizes");
  SR_CHECK_ARG(A && v && out && workspace, "null pointer");
  return aHv_impl(n_rows, n_p, reinterpret_cast<const double2*>(A), lda, reinterpret_cast<const double2*>(v), alpha,
                  reinterpret_cast<double2*>(out), workspace, workspace_bytes, (cudaStream_t)stream);
}

SR_API sr_status sr_graph_capture_begin(void* stream) {
  SR_CHECK_ARG(stream != nullptr, "capture needs a non-default stream");
  SR_CUDA(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return SR_OK;
}

SR_API sr_status sr_graph_capture_end(void* stream, void** graph_exec) {
  SR_CHECK_ARG(stream != nullptr && graph_exec != nullptr, "null pointer");
  cudaGraph_t g = nullptr;
  SR_CUDA(cudaStreamEndCapture((cudaStream_t)stream, &g));
  cudaGraphExec_t e = nullptr;
  const cudaError_t r = cudaGraphInstantiateWithFlags(&e, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  SR_CUDA(r);
  *graph_exec = e;
  return SR_OK;
}

SR_API sr_status sr_graph_launch(void* graph_exec, void* stream) {
  SR_CHECK_ARG(graph_exec != nullptr, "null graph");
  SR_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream));
  return SR_OK;
}

SR_API sr_status sr_graph_destroy(void* graph_exec) {
  if (graph_exec) SR_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)graph_exec));
  return SR_OK;
}

SR_API sr_status sr_trace_buffer(void* records, int64_t capacity) {
  SR_CHECK_ARG(records == nullptr || capacity >= 2, "capacity must be >= 2 records");
  TraceDev t{static_cast<TraceRec*>(records), records ? capacity : 0};
  SR_CUDA(trace_install_chol(t));
  SR_CUDA(trace_install_ozaki(t));
  return SR_OK;
}

SR_API size_t sr_kernel_timeline(char* buf, size_t bytes) {
  std::string out;
  std::vector<cudaStream_t> streams;
  cudaEvent_t origin = g_timed.empty() ? nullptr : g_timed.front().a;
  for (TimedLaunch& t : g_timed) {
    cudaEventSynchronize(t.b);
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, origin, t.a);
    cudaEventElapsedTime(&b, origin, t.b);
    size_t sid = std::find(streams.begin(), streams.end(), t.st) - streams.begin();
    if (sid == streams.size()) streams.push_back(t.st);
    char line[160];
    snprintf(line, sizeof line, "%s %zu %.4f %.4f\n", t.name.c_str(), sid, a, b);
    out += line;
  }
  if (buf && bytes) {   // records are consumed only when they are returned
    for (TimedLaunch& t : g_timed) {
      g_event_pool.push_back(t.a);
      g_event_pool.push_back(t.b);
    }
    g_timed.clear();
    const size_t n = std::min(bytes - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return out.size() + 1;
}

SR_API double sr_kernel_time_ms(const char* kernel, int64_t* launches) {
  double ms = 0.0;
  int64_t n = 0;
  std::vector<TimedLaunch> keep;
  for (TimedLaunch& t : g_timed) {
    if (kernel && t.name == kernel) {
      float x = 0.f;
      cudaEventSynchronize(t.b);
      if (cudaEventElapsedTime(&x, t.a, t.b) == cudaSuccess) {
        ms += x;
        n++;
      }
      g_event_pool.push_back(t.a);
      g_event_pool.push_back(t.b);
    } else {
      keep.push_back(t);
    }
  }
  g_timed.swap(keep);
  if (launches) *launches = n;
  return ms;
}

SR_API int sr_set_gram_engine(int engine) {
  if (engine != SR_GRAM_FP64 && engine != SR_GRAM_INT8) return -1;
  const int prev = g_gram_engine;
  g_gram_engine = engine;
  return prev;
}
SR_API int sr_get_gram_engine(void) { return g_gram_engine; }

SR_API size_t sr_block_solve_workspace_bytes(int n_blocks, const int64_t* block_offsets) {
  if (!valid_offsets(n_blocks, block_offsets)) return 0;
  return block_solve_ws(n_blocks, block_offsets);
}

SR_API sr_status sr_block_solve(int n_blocks, const int64_t* block_offsets, const double* S, const double* F,
                                double lambda, double* dtheta, int32_t* info, void* workspace,
                                size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(valid_offsets(n_blocks, block_offsets), "block_offsets must start at 0 and increase; 1..24 blocks");
  SR_CHECK_ARG(S && F && dtheta && workspace, "null pointer");
  SR_CHECK_ARG(lambda >= 0.0, "lambda < 0");
  return block_solve_impl(n_blocks, block_offsets, reinterpret_cast<const double2*>(S),
                          reinterpret_cast<const double2*>(F), lambda, reinterpret_cast<double2*>(dtheta), info,
                          workspace, workspace_bytes, (cudaStream_t)stream);
}

SR_API size_t sr_full_qgt_solve_workspace_bytes(int64_t n_samples, int64_t n_p) {
  if (n_p < 1 || n_samples < 0) return 0;
  return full_qgt_ws(n_samples, n_p);
}

SR_API sr_status sr_full_qgt_solve(int64_t n_samples, int64_t n_p, const double* A, int64_t lda, const double* F,
                                   double lambda, double* dtheta, double* S_out, int32_t* info, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_samples >= 0 && n_p >= 1 && n_p < (1LL << 31), "bad sizes");
  SR_CHECK_ARG(lda >= n_p, "lda < n_p");
  SR_CHECK_ARG(A && F && dtheta && workspace, "null pointer");
  SR_CHECK_ARG(lambda >= 0.0, "lambda < 0");
  return gram_solve_one(n_samples, n_p, reinterpret_cast<const double2*>(A), lda, reinterpret_cast<const double2*>(F),
                        lambda, reinterpret_cast<double2*>(dtheta), reinterpret_cast<double2*>(S_out), info, false, 0,
                        workspace, workspace_bytes, (cudaStream_t)stream);
}

SR_API size_t sr_block_qgt_solve_workspace_bytes(int64_t n_samples, int n_blocks, const int64_t* block_offsets) {
  if (n_samples < 0 || !valid_offsets(n_blocks, block_offsets)) return 0;
  return qgt_solve_ws(n_samples, n_blocks, block_offsets);
}

SR_API sr_status sr_block_qgt_solve(int64_t n_samples, int n_blocks, const int64_t* block_offsets, const double* A,
                                    int64_t lda, const double* F, double lambda, double* dtheta, int32_t* info,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(valid_offsets(n_blocks, block_offsets), "block_offsets must start at 0 and increase; 1..24 blocks");
  SR_CHECK_ARG(n_samples >= 0 && lda >= block_offsets[n_blocks], "lda < n_p");
  SR_CHECK_ARG(block_offsets[n_blocks] < (1LL << 31) / oz::kSlices, "n_p too large for the slice tensor map");
  SR_CHECK_ARG(A && F && dtheta && workspace, "null pointer");
  SR_CHECK_ARG(lambda >= 0.0, "lambda < 0");
  return qgt_solve_impl(n_samples, n_blocks, block_offsets, reinterpret_cast<const double2*>(A), lda,
                        reinterpret_cast<const double2*>(F), lambda, reinterpret_cast<double2*>(dtheta), info,
                        workspace, workspace_bytes, (cudaStream_t)stream);
}

SR_API int sr_set_step_schedule(int schedule) {
  if (schedule != SR_SCHED_BATCHED && schedule != SR_SCHED_PER_BLOCK) return -1;
  const int prev = g_step_schedule;
  g_step_schedule = schedule;
  return prev;
}
SR_API int sr_get_step_schedule(void) { return g_step_schedule; }

SR_API size_t sr_ntk_solve_workspace_bytes(int64_t n_samples, int64_t n_p) {
  if (n_samples < 1 || n_p < 1) return 0;
  long long sz = n_samples;
  Arena a(nullptr, 0);
  CholSet cs{};
  carve_chol(a, cs, &sz, 1);
  a.take<double2>(n_samples);
  return a.used + std::max(aHv_ws(n_samples, n_p), round256(oz::rows_workspace_bytes(n_samples, n_p)));
}

SR_API sr_status sr_ntk_solve(int64_t n_samples, int64_t n_p, const double* A, int64_t lda, const double* e_tilde,
                              double lambda, double* dtheta, double* T_out, int32_t* info, void* workspace,
                              size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_samples >= 1 && n_samples < (1LL << 31) && n_p >= 1, "bad sizes");
  SR_CHECK_ARG(lda >= n_p, "lda < n_p");
  SR_CHECK_ARG(A && e_tilde && dtheta && workspace, "null pointer");
  SR_CHECK_ARG(lambda >= 0.0, "lambda < 0");
  cudaStream_t st = (cudaStream_t)stream;
  long long sz = n_samples;
  Arena a(workspace, workspace_bytes);
  CholSet cs{};
  cs.info = info;
  carve_chol(a, cs, &sz, 1);
  double2* y = a.take<double2>(n_samples);
  const size_t rest = a.ok() ? workspace_bytes - a.used : 0;
  if (!a.ok() || rest < aHv_ws(n_samples, n_p)) {
    set_error("sr_ntk_solve: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  CholBlock& B = cs.b[0];
  const double2* Ad = reinterpret_cast<const double2*>(A);
  if (g_gram_engine == SR_GRAM_INT8) {   // T = A A^H on the int8 engine (rows split), scratch after y
    SR_TRY(oz::gram_rows_i8(Ad, lda, n_samples, n_p, B.Fm, B.npad, a.base + a.used, rest, st));
  } else {
    gram::ProbSet ps{};
    gram::add_prob(ps, Ad, lda, Ad, lda, B.Fm, B.npad, (int)n_samples, (int)n_samples, n_p, true);
    SR_TRY((gram::launch<gram::NH, gram::HERM_STORE>(ps, st)));
  }
  if (T_out)
    SR_TRY(copy_matrix(B.Fm, B.npad, reinterpret_cast<double2*>(T_out), n_samples, n_samples, n_samples, st));
  B.F = reinterpret_cast<const double2*>(e_tilde);
  B.out = y;
  SR_TRY(chol_solve(cs, lambda, true, 1.0, st));
  return aHv_impl(n_samples, n_p, Ad, lda, y, -1.0, reinterpret_cast<double2*>(dtheta), a.base + a.used, rest, st);
}

SR_API size_t sr_step_workspace_bytes(int n_layers, const int32_t* widths, int64_t n_samples, int64_t n_bonds) {
  StepLayout L;
  if (n_samples < 1 || n_bonds < 0 || step_layout(n_layers, widths, n_samples, n_bonds, &L) != SR_OK) return 0;
  return L.total;
}

SR_API size_t sr_step_s_offset(int n_layers, const int32_t* widths, int64_t n_samples, int64_t n_bonds) {
  StepLayout L;
  if (n_samples < 1 || n_bonds < 0 || step_layout(n_layers, widths, n_samples, n_bonds, &L) != SR_OK) return 0;
  return L.per_block ? SIZE_MAX : L.S;
}

SR_API sr_status sr_step(int n_layers, const int32_t* widths, const double* theta, const int8_t* spins,
                         int64_t n_samples, int64_t n_bonds, const int32_t* bonds_ij, const double* bond_j,
                         double lambda, double* dtheta, double* energy, void* workspace, size_t workspace_bytes,
                         void* stream) {
  SR_CHECK_ARG(n_samples >= 1 && n_bonds >= 0, "bad sizes");
  StepLayout L;
  SR_TRY(step_layout(n_layers, widths, n_samples, n_bonds, &L));
  SR_CHECK_ARG(theta && spins && dtheta && workspace, "null pointer");
  SR_CHECK_ARG(n_bonds == 0 || (bonds_ij && bond_j), "null bond arrays");
  SR_CHECK_ARG(lambda >= 0.0, "lambda < 0");
  if (workspace_bytes < L.total) {
    set_error("sr_step: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  double* e = energy ? energy : reinterpret_cast<double*>(static_cast<char*>(workspace) + L.energy);
  return step_impl(L, theta, spins, n_samples, n_bonds, bonds_ij, bond_j, lambda, dtheta, e,
                   static_cast<char*>(workspace), (cudaStream_t)stream);
}

SR_API size_t sr_step_host_extra_bytes(int n_layers, const int32_t* widths, int64_t n_samples, int64_t n_bonds) {
  StepLayout L;
  if (n_samples < 1 || n_bonds < 0 || step_layout(n_layers, widths, n_samples, n_bonds, &L) != SR_OK) return 0;
  return L.host_total;
}

SR_API sr_status sr_step_host(int n_layers, const int32_t* widths, const double* theta_h, const int8_t* spins_h,
                              int64_t n_samples, int64_t n_bonds, const int32_t* bonds_ij_h, const double* bond_j_h,
                              double lambda, double* dtheta_h, double* energy_h, void* workspace,
                              size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_samples >= 1 && n_bonds >= 0, "bad sizes");
  StepLayout L;
  SR_TRY(step_layout(n_layers, widths, n_samples, n_bonds, &L));
  SR_CHECK_ARG(theta_h && spins_h && dtheta_h && workspace, "null pointer");
  SR_CHECK_ARG(n_bonds == 0 || (bonds_ij_h && bond_j_h), "null bond arrays");
  if (workspace_bytes < L.total + L.host_total) {
    set_error("sr_step_host: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);
  const size_t c16 = sizeof(double2);
  const long long np = L.net.n_p;
  double* theta = reinterpret_cast<double*>(ws + L.h_theta);
  int8_t* spins = reinterpret_cast<int8_t*>(ws + L.h_spins);
  int32_t* bij = reinterpret_cast<int32_t*>(ws + L.h_bij);
  double* bj = reinterpret_cast<double*>(ws + L.h_bj);
  double* dtheta = reinterpret_cast<double*>(ws + L.h_dtheta);
  double* energy = reinterpret_cast<double*>(ws + L.h_energy);
  SR_CUDA(cudaMemcpyAsync(theta, theta_h, np * c16, cudaMemcpyHostToDevice, st));
  SR_CUDA(cudaMemcpyAsync(spins, spins_h, (size_t)n_samples * L.net.w[0], cudaMemcpyHostToDevice, st));
  if (n_bonds) {
    SR_CUDA(cudaMemcpyAsync(bij, bonds_ij_h, (size_t)n_bonds * 2 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    SR_CUDA(cudaMemcpyAsync(bj, bond_j_h, (size_t)n_bonds * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  StepGraphKey key{workspace, std::vector<int32_t>(widths, widths + n_layers + 1), n_samples, n_bonds, lambda,
                   g_gram_engine, g_step_schedule};
  SR_TRY(step_graphed(L, key, theta, spins, n_samples, n_bonds, bij, bj, lambda, dtheta, energy, ws, st));
  SR_CUDA(cudaMemcpyAsync(dtheta_h, dtheta, np * c16, cudaMemcpyDeviceToHost, st));
  if (energy_h) SR_CUDA(cudaMemcpyAsync(energy_h, energy, c16, cudaMemcpyDeviceToHost, st));
  SR_CUDA(cudaStreamSynchronize(st));
  return SR_OK;
}

}  // extern "C"
