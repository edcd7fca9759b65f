// chol.cu — stage (5): batched, blocked, right-looking Cholesky solve of
// (S_b + lambda I) x_b = F_b for all layer blocks at once (§2: "Each block S_l
// is inverted independently, using a uniform diagonal shift lambda"), also used by the
// full-QGT and NTK comparison paths with a single "block".
//
// Each block is copied into a padded factor matrix (n_pad = 64*ceil(n/64), identity in
// the padding so the padded system decouples).  Panel step p (all blocks with
// p < P_b advance together, one launch per kernel):
//   chol_diag        factor the 64x64 diagonal tile in shared memory, form its inverse
//                    Linv_p, and y_p = Linv_p b_p (forward substitution folded in)
//   trsm (engine)    L_ip = A_ip Linv_p^H for every row tile i > p      (DMMA, NH/STORE)
//   (chol_diag also subtracts the strip's earlier panels from its own 64 rows of b)
//   inner (engine)   A_ij -= L_ip L_jp^H for the strip's later columns j (DMMA, NH/SUB)
// and after every strip of kStrip panels chol_rhs_update (b_i -= L_i,strip y_strip for the rows
// below) and one deferred trailing update with K = 64 kStrip:
//   trail (engine)   A_ij -= L_i,strip L_j,strip^H for i >= j beyond the strip (NH/SUB)
// then back substitution L^H x = y strip by strip (x_p = Linv_p^H y_p inside the strip,
// then y_{<strip} -= L_strip,<^H x_strip) and dtheta = -x.
#include <cooperative_groups.h>
#include <cstdlib>

#include "chol.cuh"
#include "chol_diag.cuh"
#include "gram.cuh"
#include "ozaki.cuh"

namespace sr {
namespace {

#ifndef SR_KSTRIP
#define SR_KSTRIP 8   // measured best of 2, 4, 8, 12, 16 at configs[1] (3-block solve 25.9 -> 24.0 ms)
#endif
using cholk::NB;
using cholk::chol_diag;
using cholk::kDiagSmem;
constexpr int kStrip = SR_KSTRIP;   // panels per back-substitution strip (one cluster CTA each)
#ifndef SR_SIDE_TM
#define SR_SIDE_TM 16   // rows per CTA of the off-chain skinny launches (the chain's stay at 16)
#endif
constexpr int kSideTM = SR_SIDE_TM;
// Panels per factorisation strip (deferred trailing update with K = 64 x strip), by block
// size: 8 below 20000 rows (chain-bound blocks: the strip's panels are on the chain), 16 from
// 20000 (throughput-bound: half the read-modify-write passes over the trailing matrix).
// Measured: configs[4]'s 25760 blocks 4350 -> 4146 ms per step at 16 (4207 at 12); configs[3]
// (16512) and configs[1] (6480) equal or slower at 12/16.  SR_KSTRIP_F forces one value.
constexpr int kFStripMax = 16;
int fstrip(long long n) {
  static int forced = -2;
  if (forced == -2) {
    const char* e = getenv("SR_KSTRIP_F");
    forced = e ? std::max(1, std::min(kFStripMax, atoi(e))) : -1;
  }
  if (forced > 0) return forced;
  return n >= 20000 ? 16 : kStrip;
}

__global__ void chol_init(CholSet cs, double lam, int inplace, int b0) {
  TraceScope trace_(TR_INIT, b0);
  const int b = b0 + blockIdx.y;
  const CholBlock& B = cs.b[b];
  const long long n = B.n, np = B.npad;
  const long long total = np * np;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / np, c = e % np;
    if (r < n && c < n) {
      if (inplace) {
        if (r == c) B.Fm[e].x += lam;
      } else {
        double2 v = B.S[r * n + c];
        if (r == c) v.x += lam;
        B.Fm[e] = v;
      }
    } else {
      B.Fm[e] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
  }
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < np;
       r += (long long)gridDim.x * blockDim.x)
    B.rhs[r] = r < n ? B.F[r] : make_double2(0.0, 0.0);
}

// b_i -= sum_{c in [c0, c1)} L[i][c] y[c] for rows i >= c1 (the strip's panels applied to the
// right-hand side of every later row at once; one warp per row).
__global__ void chol_rhs_update(const CholBlock B, long long c0, long long c1) {
  TraceScope trace_(TR_RHS, (int)(B.row_base / 64) * 4096 + (int)(c0 / 64));
  const long long np = B.npad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long r = c1 + (long long)blockIdx.x * 8 + warp; r < np; r += (long long)gridDim.x * 8) {
    const double2* row = B.Fm + r * np;
    double2 sa[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    for (long long c = c0 + lane; c < c1; c += 128) {   // c1 - c0 is a multiple of 64
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (c + 32 * u < c1) cfma(sa[u], row[c + 32 * u], B.rhs[c + 32 * u]);
    }
    double2 s = cadd(cadd(sa[0], sa[1]), cadd(sa[2], sa[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) B.rhs[r] = csub(B.rhs[r], s);
  }
}

// Back substitution L^H x = y by strips of panels [p0, pend), two launches per strip:
// chol_back_strip, a cluster of kStrip CTAs, CTA j owning panel q = p0 + j and its y_q in
// shared memory: step p = pend-1 .. p0 the owner of p forms x_p = Linv_p^H y_p and writes
// it into the shared memory of the CTAs j < p - p0 (distributed shared memory), one
// cluster barrier, then each of those applies y_q -= L_pq^H x_p.  Every CTA streams the
// 64x64 blocks it needs (L_pq for p = pend-1 .. q+1, then Linv_q) through a double buffer
// with cp.async, a step ahead of use, so a step is two shared-memory GEMVs and a barrier
// instead of a round trip to HBM per block on one SM.
// chol_back_rest (one CTA per 32 columns c < 64 p0): y_c -= sum_{r in strip} conj(L[r][c]) x_r.
// Reductions run in a fixed order (deterministic).
static_assert(kStrip <= 8, "the back-substitution cluster holds one CTA per strip panel (portable size 8)");
constexpr size_t kBackSmem = (size_t)2 * NB * NB * sizeof(double2);   // 128 KB

__global__ void __cluster_dims__(kStrip, 1, 1) __launch_bounds__(256) chol_back_strip(const CholBlock B, int p0, int pend) {
  TraceScope trace_(TR_BACK, (int)(B.row_base / 64) * 4096 + p0);
  extern __shared__ __align__(16) double2 bsm[];   // [2][64][64] streamed blocks
  __shared__ double2 xb[2][NB];
  __shared__ double2 ys[NB];
  __shared__ double2 red[4][NB];
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int j = (int)cl.block_rank();
  const int nps = pend - p0, q = p0 + j;
  const bool act = j < nps;
  const int nblk = act ? nps - j : 0;   // L_pq for p = pend-1 .. q+1, then Linv_q
  const long long np = B.npad;
  const int t = threadIdx.x, c = t & 63, rq = t >> 6;
  auto issue = [&](int i) {
    double2* dst = bsm + (size_t)(i & 1) * NB * NB;
    const bool lin = i == nblk - 1;
    const double2* src = lin ? B.linv + (long long)q * NB * NB : B.Fm + (long long)(pend - 1 - i) * NB * np + (long long)q * NB;
    const long long ld = lin ? NB : np;
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int e = t + 256 * u, r = e >> 6, cc = e & 63;
      gram::cp_async16(dst + r * NB + cc, src + (long long)r * ld + cc, true);
    }
    gram::cp_commit();
  };
  // y_blk = sum_r conj(Blk[r][c]) v[r] over the 64 rows, 4 row groups then a fixed-order sum
  auto gemv = [&](const double2* blk, const double2* v) {
    double2 sa[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
    for (int i = 0; i < 16; i++) cfma_conj(sa[i & 3], blk[(rq + 4 * i) * NB + c], v[rq + 4 * i]);
    red[rq][c] = cadd(cadd(sa[0], sa[1]), cadd(sa[2], sa[3]));
    __syncthreads();
    return cadd(cadd(red[0][c], red[1][c]), cadd(red[2][c], red[3][c]));
  };
  if (act) {
    if (t < NB) ys[t] = B.rhs[(long long)q * NB + t];
    issue(0);
    if (nblk > 1) issue(1);
  }
  int cur = 0;
  for (int st = 0; st < nps; st++) {
    const int jp = nps - 1 - st;   // owner of panel p = pend - 1 - st
    if (j == jp) {                 // x_p = Linv_p^H y_p (Linv is this CTA's last block)
      gram::cp_wait<0>();
      __syncthreads();
      const double2 x = gemv(bsm + (size_t)(cur & 1) * NB * NB, ys);
      if (t < NB) {
        B.xout[(long long)(p0 + jp) * NB + t] = x;
        for (int jj = 0; jj < jp; jj++) cl.map_shared_rank(&xb[st & 1][0], jj)[t] = x;
      }
    }
    cl.sync();
    if (j < jp) {   // y_q -= L_pq^H x_p
      if (cur + 1 < nblk) gram::cp_wait<1>();
      else gram::cp_wait<0>();
      __syncthreads();
      const double2 v = gemv(bsm + (size_t)(cur & 1) * NB * NB, &xb[st & 1][0]);
      if (t < NB) ys[t] = csub(ys[t], v);
      __syncthreads();   // the buffer of block cur is free, ys updated
      cur++;
      if (cur + 1 < nblk) issue(cur + 1);
    }
  }
}

// One CTA per 32 columns: warp w sums rows w, w + 8, ... of the strip (8 loads in flight
// per thread: the column GEMV is latency-bound with fewer), then a fixed-order reduction.
__global__ void __launch_bounds__(256) chol_back_rest(const CholBlock B, int p0, int pend) {
  TraceScope trace_(TR_BACK_REST, (int)(B.row_base / 64) * 4096 + p0);
  __shared__ double2 xs[kStrip * NB];
  __shared__ double2 red[8][33];
  const long long np = B.npad;
  const int t = threadIdx.x, cl = t & 31, rq = t >> 5;
  const int nr = (pend - p0) * NB;
  for (int e = t; e < nr; e += 256) xs[e] = B.xout[(long long)p0 * NB + e];
  __syncthreads();
  const long long ncol = (long long)p0 * NB;
  for (long long cb = (long long)blockIdx.x * 32; cb < ncol; cb += (long long)gridDim.x * 32) {
    const long long c = cb + cl;
    double2 sa[8];
#pragma unroll
    for (int u = 0; u < 8; u++) sa[u] = make_double2(0.0, 0.0);
    const double2* col = B.Fm + ((long long)p0 * NB) * np + c;
    for (int r0 = rq; r0 < nr; r0 += 64) {   // nr is a multiple of 64
#pragma unroll
      for (int u = 0; u < 8; u++) cfma_conj(sa[u], col[(long long)(r0 + 8 * u) * np], xs[r0 + 8 * u]);
    }
    red[rq][cl] = cadd(cadd(cadd(sa[0], sa[1]), cadd(sa[2], sa[3])), cadd(cadd(sa[4], sa[5]), cadd(sa[6], sa[7])));
    __syncthreads();
    if (rq == 0) {
      double2 v = red[0][cl];
#pragma unroll
      for (int w = 1; w < 8; w++) v = cadd(v, red[w][cl]);
      B.rhs[c] = csub(B.rhs[c], v);
    }
    __syncthreads();
  }
}

__global__ void chol_output(CholSet cs, double sign) {
  TraceScope trace_(TR_OUTPUT, 0);
  const CholBlock& B = cs.b[blockIdx.y];
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < B.n;
       r += (long long)gridDim.x * blockDim.x)
    B.out[r] = cscale(B.xout[r], sign);
}

}  // namespace

void carve_chol(Arena& a, CholSet& cs, const long long* sizes, int nblk) {
  cs.count = nblk;
  long long row_base = 0;
  for (int b = 0; b < nblk; b++) {
    CholBlock& B = cs.b[b];
    B.n = sizes[b];
    B.P = (int)((B.n + NB - 1) / NB);
    B.npad = (long long)B.P * NB;
    B.row_base = row_base;
    row_base += B.n;
    B.Fm = a.take<double2>((size_t)B.npad * B.npad);
    B.rhs = a.take<double2>(B.npad);
    B.xout = a.take<double2>(B.npad);
    B.linv = a.take<double2>((size_t)B.P * NB * NB);
    B.tws_bytes = oz::trail_workspace_bytes(B.npad, (long long)fstrip(B.n) * NB);
    B.tws = a.take<char>(B.tws_bytes);
  }
}

namespace {

// Persistent-grid cap of the int8 trailing update: with several blocks in flight, leave SMs
// for the other blocks' latency-bound panel chains (SR_TRAIL_CTAS overrides, for tuning).
int trail_ctas(int nblocks) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SR_TRAIL_CTAS");
    env = e ? atoi(e) : -1;
  }
  if (env >= 0) return env;
  (void)nblocks;
  return 0;   // measured: capping the grid slows the 3-block solve (trailing throughput bound)
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// In-strip updates of the columns beyond the two-column lookahead: left-looking (one K =
// 64 (p - p0 + 1) update of column p+3 per step on s2, SR_INSTRIP_LEFT=1) or right-looking
// (every panel updating all later columns, SR_INSTRIP_LEFT=0).
bool instrip_left() {
  static const int v = env_int("SR_INSTRIP_LEFT", 1);
  return v != 0;
}

// Split TRSM (see solve_block); SR_TRSM_SPLIT=0 restores the whole TRSM on the chain.
bool trsm_split() {
  static const int v = env_int("SR_TRSM_SPLIT", 1);
  return v != 0;
}

// Trailing-update lookahead (see solve_block); SR_LOOKAHEAD=0 turns it off, SR_TRAIL_B_TPC
// sets the tiles per CTA of the off-chain part.
// Default: on for a single block (an owner's solve in the sharded step, the full-QGT and
// NTK solves), where the chain leaves SMs idle (6480 block: graph 10.56 -> 10.07 ms with (b)
// on 120 persistent CTAs; 16240: 94.4 -> 92.9 ms); off for several concurrent blocks, which
// fill the GPU already (configs[1] step 35.3 vs 34.6 ms).
bool lookahead(int nblocks) {
  static const int v = env_int("SR_LOOKAHEAD", -1);
  return v < 0 ? nblocks == 1 : v != 0;
}
int trail_b_tpc() {
  static const int v = std::max(1, env_int("SR_TRAIL_B_TPC", 2));
  return v;
}

// Programmatic dependent launch along the panel chain (diag -> TRSM -> next tile -> diag);
// SR_PDL=0 turns it off (A/B measurements).
bool pdl_chain() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_PDL");
    v = e ? atoi(e) != 0 : 1;
  }
  return v != 0;
}

// Factorisation + substitutions of ONE block on one stream (two-level blocking, see header).
// Side streams of the block: Q.s2 / Q.s3 with events Q.ea / Q.eb / Q.ec.  Within a strip the
// panel chain on `st` runs diag(p) -> TRSM(p) -> the update of the next DIAGONAL tile
// (p+1, p+1) by panel p -> diag(p+1): that tile is all diag(p+1) reads.  Panel p's other
// in-strip updates run off the chain: on s3 the rest of column p+1 and all of column p+2
// (joined into st before TRSM(p+1)), on s2 the columns >= p+3.  Ordering of the writers of
// one column: s3's job(p) waits for the last s2 job (which wrote columns >= p+2), and the
// chain reaches every column through s3 (ec before each TRSM), so the chain itself never
// waits on s2 -- s2's job(p-1) has two panel steps to finish before s3's job(p+1) needs it.
struct BlockStreams {
  cudaStream_t s2, s3, s4;
  cudaEvent_t ea, eb, ec, ed, er, es, et;
};
// Stagger of equal-size blocks (SR_STAGGER=k, k >= 1): block b starts once the previous
// block of the same size has factored k panels, so their strip-end trailing updates (full-
// GPU kernels on the chain) alternate instead of coinciding.  0 = off.
int stagger_panels() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_STAGGER");
    v = e ? atoi(e) : 0;
  }
  return v;
}

sr_status solve_block(CholSet& cs, int b, cudaStream_t st, const BlockStreams& Q, cudaEvent_t stagger_rec = nullptr) {
  const CholBlock& B = cs.b[b];
  // Two-level blocking: strips of kStrip panels.  Inside a strip each panel p is factored
  // (chol_diag), its column solved (TRSM), the RHS updated, and only the strip's own later
  // columns updated (K = 64); the rest of the trailing matrix receives one deferred update
  // per strip with K = 64 * kStrip, which is where the flops are (4x the arithmetic
  // intensity of a per-panel update, 4x fewer passes over the trailing matrix).
  const bool i8 = gram_engine() == SR_GRAM_INT8;
  bool pending_b = false;   // a lookahead (b) update on s4 not yet joined into st
  // ec / eb are waited on only once recorded by this call (inside a CUDA-graph capture, a
  // wait on an event last recorded outside it is an error, not a no-op)
  bool ec_rec = false, eb_rec = false;
  const int kFStrip = fstrip(B.n);
  for (int p0 = 0; p0 < B.P; p0 += kFStrip) {
    const int pend = std::min(p0 + kFStrip, B.P);
    for (int p = p0; p < pend; p++) {
      timer_begin("chol_diag", st);
      if (pdl_chain()) SR_CUDA(launch_pdl(chol_diag, dim3(1), dim3(256), kDiagSmem, st, B, cs.info, p, p0));
      else chol_diag<<<1, 256, kDiagSmem, st>>>(B, cs.info, p, p0);
      timer_end(st);
      SR_LAUNCHED();
      if (stagger_rec && p + 1 == stagger_panels()) SR_CUDA(cudaEventRecord(stagger_rec, st));
      // the previous panel's update of this column below the diagonal tile (s3) must be
      // complete before TRSM(p) (and joined into st in any case)
      if (p > p0 && ec_rec) SR_CUDA(cudaStreamWaitEvent(st, Q.ec, 0));
      const long long m = B.npad - (long long)(p + 1) * NB;
      if (m <= 0) continue;
      gram::ProbSet trsm{}, trsm_rest{}, next_tile{}, next_rows{}, next_rows2{}, inner_rest{};
      bool ec_now = false;
      double2* panel = B.Fm + (long long)(p + 1) * NB * B.npad + (long long)p * NB;
      const double2* linv_p = B.linv + (long long)p * NB * NB;
      // Split TRSM: the chain solves only the next panel's row block (all that the next-tile
      // update and chol_diag(p+1) read); the rows below go to s3 ahead of its update job.
      const bool split = trsm_split() && p + 1 < pend && m > NB;
      if (split) {
        gram::add_prob(trsm, panel, B.npad, linv_p, NB, panel, B.npad, NB, NB, NB, false);
        gram::add_prob(trsm_rest, panel + (long long)NB * B.npad, B.npad, linv_p, NB, panel + (long long)NB * B.npad,
                       B.npad, (int)(m - NB), NB, NB, false);
      } else {
        gram::add_prob(trsm, panel, B.npad, linv_p, NB, panel, B.npad, (int)m, NB, NB, false);
      }
      const bool left = instrip_left();
      for (int jj = p + 1; jj < pend; jj++) {   // later columns of the strip, rows i >= jj
        const double2* lrows = B.Fm + (long long)jj * NB * B.npad + (long long)p * NB;
        double2* cblk = B.Fm + (long long)jj * NB * B.npad + (long long)jj * NB;
        const int rows = (int)(B.npad - (long long)jj * NB);
        if (jj == p + 1) {
          gram::add_prob(next_tile, lrows, B.npad, lrows, B.npad, cblk, B.npad, NB, NB, NB, false);
          if (rows > NB)
            gram::add_prob(next_rows, lrows + (long long)NB * B.npad, B.npad, lrows, B.npad,
                           cblk + (long long)NB * B.npad, B.npad, rows - NB, NB, NB, false);
        } else if (jj == p + 2) {   // two-column lookahead on s3 (see the ordering note above);
          // left-looking after the first step: its own launch, behind the s2 job it waits for
          gram::add_prob(left && p > p0 ? next_rows2 : next_rows, lrows, B.npad, lrows, B.npad, cblk, B.npad, rows,
                         NB, NB, false);
        } else if (left) {
          if (jj == p + 3) {   // left-looking: column p+3 by all of the strip's panels p0..p at once
            const double2* lk = B.Fm + (long long)jj * NB * B.npad + (long long)p0 * NB;
            gram::add_prob(inner_rest, lk, B.npad, lk, B.npad, cblk, B.npad, rows, NB, (long long)(p - p0 + 1) * NB,
                           false);
          }
        } else {
          gram::add_prob(inner_rest, lrows, B.npad, lrows, B.npad, cblk, B.npad, rows, NB, NB, false);
        }
      }
      timer_begin("chol_trsm", st);
      static const bool pdl_trsm = env_int("SR_PDL_TRSM", 1) != 0;
      SR_TRY((gram::launch_skinny<gram::STORE>(trsm, st, pdl_chain() && pdl_trsm)));
      timer_end(st);
      const bool side = next_tile.count > 0;
      if (side) SR_CUDA(cudaEventRecord(Q.ea, st));           // L column p ready for s2 / s3
      timer_begin("chol_inner", st);
      if (side) SR_TRY((gram::launch_skinny<gram::SUB>(next_tile, st, pdl_chain())));
      timer_end(st);
      // The off-chain jobs start after the next-tile update, so the next chol_diag is already
      // pending (at the chain's higher priority) when their CTAs flood the SMs.
      static const bool after_next = env_int("SR_SIDE_AFTER_NEXT", 1) != 0;
      const cudaEvent_t side_go = after_next ? Q.ed : Q.ea;
      if (side && after_next) SR_CUDA(cudaEventRecord(Q.ed, st));
      if (side && (next_rows.count || next_rows2.count)) {
        SR_CUDA(cudaStreamWaitEvent(Q.s3, side_go, 0));
        if (p > p0 && !left && eb_rec) SR_CUDA(cudaStreamWaitEvent(Q.s3, Q.eb, 0));
        if (split) {
          timer_begin("chol_trsm_rest", Q.s3);
          SR_TRY((gram::launch_skinny<gram::STORE, kSideTM>(trsm_rest, Q.s3)));
          timer_end(Q.s3);
          SR_CUDA(cudaEventRecord(Q.er, Q.s3));   // all of L column p: the s2 job may start
        }
        timer_begin("chol_next_rows", Q.s3);
        if (next_rows.count) SR_TRY((gram::launch_skinny<gram::SUB, kSideTM>(next_rows, Q.s3)));
        // left-looking: column p+2 first takes the s2 job of the previous step (panels
        // p0..p-1), which began right after that step's TRSM
        if (next_rows2.count && eb_rec) SR_CUDA(cudaStreamWaitEvent(Q.s3, Q.eb, 0));
        if (next_rows2.count) SR_TRY((gram::launch_skinny<gram::SUB, kSideTM>(next_rows2, Q.s3)));
        timer_end(Q.s3);
        SR_CUDA(cudaEventRecord(Q.ec, Q.s3));
        ec_rec = true;
        ec_now = true;
      }
      if (inner_rest.count) {
        // SR_S2_AFTER_S3=1: the left-looking job (needed two panels later) starts only after
        // this step's s3 jobs (needed by the next TRSM), so it does not take their SMs
        static const bool s2_after_s3 = env_int("SR_S2_AFTER_S3", 0) != 0;
        if (s2_after_s3 && ec_now) SR_CUDA(cudaStreamWaitEvent(Q.s2, Q.ec, 0));
        if (left) SR_CUDA(cudaStreamWaitEvent(Q.s2, split ? Q.er : Q.ea, 0));
        else SR_CUDA(cudaStreamWaitEvent(Q.s2, side_go, 0));
        if (split && !left) SR_CUDA(cudaStreamWaitEvent(Q.s2, Q.er, 0));
        timer_begin("chol_inner_rest", Q.s2);
        SR_TRY((gram::launch_skinny<gram::SUB, kSideTM>(inner_rest, Q.s2)));
        timer_end(Q.s2);
        SR_CUDA(cudaEventRecord(Q.eb, Q.s2));
        eb_rec = true;
      }
    }
    const long long m = B.npad - (long long)pend * NB;
    if (m > 0) {   // the strip's y applied to the right-hand side of all later rows
      dim3 g((unsigned)std::min<long long>((m + 7) / 8, 4 * kNumSMs), 1);
      timer_begin("chol_rhs", st);
      chol_rhs_update<<<g, 256, 0, st>>>(B, (long long)p0 * NB, (long long)pend * NB);
      timer_end(st);
      SR_LAUNCHED();
    }
    if (m > 0) {   // deferred trailing update of the strip, K = 64 * (pend - p0)
      const double2* lp = B.Fm + (long long)pend * NB * B.npad + (long long)p0 * NB;
      double2* trailing = B.Fm + (long long)pend * NB * B.npad + (long long)pend * NB;
      const long long K = (long long)(pend - p0) * NB;
      const long long look = (long long)kFStrip * NB;   // the next strip's columns
      if (i8 && lookahead(cs.count) && m > look) {
        // Lookahead: the chain needs only the next strip's columns (a), so the rest of the
        // trailing matrix (b) is updated on s4 (lowest priority, non-persistent grid) while
        // the next strip factors.  (b) reads the digit slices and writes columns beyond the
        // next strip, so the next strip-end split waits for it (et), which also keeps one
        // addend per element per launch in a fixed order (deterministic).
        if (pending_b) SR_CUDA(cudaStreamWaitEvent(st, Q.et, 0));
        SR_TRY(oz::trail_split_i8(lp, B.npad, m, K, B.tws, B.tws_bytes, st));
        SR_CUDA(cudaEventRecord(Q.es, st));
        SR_TRY(oz::trail_apply_i8(m, K, trailing, B.npad, B.tws, 0, kFStrip, trail_ctas(cs.count), st));
        SR_CUDA(cudaStreamWaitEvent(Q.s4, Q.es, 0));
        static const int b_ctas = env_int("SR_TRAIL_B_CTAS", 120);   // > 0: persistent (b) on that many CTAs
        SR_TRY(oz::trail_apply_i8(m, K, trailing, B.npad, B.tws, look, 0, b_ctas > 0 ? b_ctas : -trail_b_tpc(), Q.s4));
        SR_CUDA(cudaEventRecord(Q.et, Q.s4));
        pending_b = true;
      } else if (i8) {   // int8 digit-slice tcgen05 engine (ozaki.cu), lower triangle
        if (pending_b) SR_CUDA(cudaStreamWaitEvent(st, Q.et, 0));
        pending_b = false;
        SR_TRY(oz::trail_update_i8(lp, B.npad, m, (long long)(pend - p0) * NB, trailing, B.npad, B.tws, B.tws_bytes,
                                   trail_ctas(cs.count), st));
      } else {
        gram::ProbSet trail{};
        gram::add_prob(trail, lp, B.npad, lp, B.npad, trailing, B.npad, (int)m, (int)m,
                       (long long)(pend - p0) * NB, true);
        timer_begin("trail_dmma", st);
        SR_TRY((gram::launch<gram::NH, gram::SUB>(trail, st)));
        timer_end(st);
      }
    }
  }
  if (pending_b) SR_CUDA(cudaStreamWaitEvent(st, Q.et, 0));
  for (int p0 = (B.P - 1) / kStrip * kStrip; p0 >= 0; p0 -= kStrip) {
    const int pend = std::min(p0 + kStrip, B.P);
    timer_begin("chol_back", st);
    chol_back_strip<<<kStrip, 256, kBackSmem, st>>>(B, p0, pend);
    SR_LAUNCHED();
    timer_end(st);
    if (p0 > 0) {
      timer_begin("chol_back_rest", st);
      chol_back_rest<<<(unsigned)std::min(2 * p0, 4 * kNumSMs), 256, 0, st>>>(B, p0, pend);
      SR_LAUNCHED();
      timer_end(st);
    }
  }
  return SR_OK;
}

// Side streams for independent blocks (created once per process; high priority so the
// latency-bound panel chain of one block is scheduled ahead of another block's big update).
constexpr int kSideStreams = 8;
struct SidePool {
  cudaStream_t s[kSideStreams];
  BlockStreams q[kSideStreams];
  cudaEvent_t fork, join[kSideStreams], stag[kSideStreams];
  bool ok = false;
};
sr_status side_pool(SidePool*& out) {
  static SidePool pool;
  if (!pool.ok) {
    int lo = 0, hi = 0;
    SR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < kSideStreams; i++) {
      BlockStreams& q = pool.q[i];
      // the panel chain (s) ahead of the block's off-chain in-strip updates (s3, then s2):
      // when an SM frees up, the chain's next kernel is placed first
      const int side_prio = env_int("SR_SIDE_PRIO", 1);
      SR_CUDA(cudaStreamCreateWithPriority(&pool.s[i], cudaStreamNonBlocking, hi));
      SR_CUDA(cudaStreamCreateWithPriority(&q.s2, cudaStreamNonBlocking, side_prio ? std::min(lo, hi + 2) : hi));
      SR_CUDA(cudaStreamCreateWithPriority(&q.s3, cudaStreamNonBlocking, side_prio ? std::min(lo, hi + 1) : hi));
      SR_CUDA(cudaStreamCreateWithPriority(&q.s4, cudaStreamNonBlocking, lo));
      SR_CUDA(cudaEventCreateWithFlags(&q.es, cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&q.ed, cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&q.er, cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&q.et, cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&pool.join[i], cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&pool.stag[i], cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&q.ea, cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&q.eb, cudaEventDisableTiming));
      SR_CUDA(cudaEventCreateWithFlags(&q.ec, cudaEventDisableTiming));
    }
    SR_CUDA(cudaEventCreateWithFlags(&pool.fork, cudaEventDisableTiming));
    pool.ok = true;
  }
  out = &pool;
  return SR_OK;
}

}  // namespace

sr_status chol_solve(CholSet& cs, double lam, bool inplace, double sign, cudaStream_t st,
                     const cudaEvent_t* ready) {
  if (ready && cs.info) {   // the reset on st would race with blocks already released by ready[b]
    set_error("chol_solve: info must be null with ready events");
    return SR_ERR_INVALID;
  }
  if (cs.info && !cs.keep_info) SR_CUDA(cudaMemsetAsync(cs.info, 0, sizeof(int), st));
  auto init_grid = [](const CholBlock& B, int nb) {
    return dim3((unsigned)std::min<long long>((B.npad * B.npad + 255) / 256, 2 * kNumSMs), (unsigned)nb);
  };
  if (!ready) {
    long long mx = 0;
    for (int b = 0; b < cs.count; b++) mx = std::max(mx, cs.b[b].npad * cs.b[b].npad);
    dim3 g((unsigned)std::min<long long>((mx + 255) / 256, 2 * kNumSMs), (unsigned)cs.count);
    chol_init<<<g, 256, 0, st>>>(cs, lam, inplace ? 1 : 0, 0);
    SR_LAUNCHED();
  }
  static unsigned long long diag_attr = 0;
  if (first_on_device(diag_attr)) {
    SR_CUDA(cudaFuncSetAttribute(chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem));
    SR_CUDA(cudaFuncSetAttribute(chol_back_strip, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBackSmem));
  }
  SidePool* pool;
  SR_TRY(side_pool(pool));
  SR_CUDA(cudaEventRecord(pool->fork, st));
  if (cs.count == 1 && !ready) {
    SR_CUDA(cudaStreamWaitEvent(pool->q[0].s2, pool->fork, 0));
    SR_CUDA(cudaStreamWaitEvent(pool->q[0].s3, pool->fork, 0));
    SR_CUDA(cudaStreamWaitEvent(pool->q[0].s4, pool->fork, 0));
    SR_TRY(solve_block(cs, 0, st, pool->q[0]));
  } else {
    // independent blocks on side streams, forked from and joined back into `st`
    bool prev_stagger = false;
    for (int b = 0; b < cs.count; b++) {
      const int i = b % kSideStreams;
      cudaStream_t sb = pool->s[i];
      // pipelined: block b's S (and everything queued on st before it) is complete once
      // ready[b] fires; otherwise everything queued on st before this call
      const cudaEvent_t go = ready ? ready[b] : pool->fork;
      SR_CUDA(cudaStreamWaitEvent(sb, go, 0));
      SR_CUDA(cudaStreamWaitEvent(pool->q[i].s2, go, 0));
      SR_CUDA(cudaStreamWaitEvent(pool->q[i].s3, go, 0));
      SR_CUDA(cudaStreamWaitEvent(pool->q[i].s4, go, 0));
      if (ready) {
        chol_init<<<init_grid(cs.b[b], 1), 256, 0, sb>>>(cs, lam, inplace ? 1 : 0, b);
        SR_LAUNCHED();
      }
      // stagger: wait for the previous equal-size block's first panels (see stagger_panels)
      const bool stag = stagger_panels() > 0 && b + 1 < cs.count && cs.b[b + 1].npad == cs.b[b].npad &&
                        cs.b[b].P > stagger_panels();
      if (b > 0 && prev_stagger) SR_CUDA(cudaStreamWaitEvent(sb, pool->stag[(b - 1) % kSideStreams], 0));
      SR_TRY(solve_block(cs, b, sb, pool->q[i], stag ? pool->stag[b % kSideStreams] : nullptr));
      prev_stagger = stag;
    }
    for (int i = 0; i < std::min(cs.count, kSideStreams); i++) {
      SR_CUDA(cudaEventRecord(pool->join[i], pool->s[i]));
      SR_CUDA(cudaStreamWaitEvent(st, pool->join[i], 0));
    }
  }
  {
    long long mx = 0;
    for (int b = 0; b < cs.count; b++) mx = std::max(mx, cs.b[b].n);
    dim3 g((unsigned)std::max<long long>(1, std::min<long long>((mx + 255) / 256, 4 * kNumSMs)),
           (unsigned)cs.count);
    chol_output<<<g, 256, 0, st>>>(cs, sign);
    SR_LAUNCHED();
  }
  return SR_OK;
}

cudaError_t trace_install_chol(TraceDev t) { return trace_install_local(t); }

}  // namespace sr
