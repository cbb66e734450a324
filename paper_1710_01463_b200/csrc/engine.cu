// Host-side orchestration of the B200 RSVD pipeline and the C ABI
// (include/rsvd_c.h).
//
// One call runs the reference's rsvd (factorize.cpp:76-95) for a whole batch
// of equally shaped matrices, every stage a batched kernel over all items:
//
//   Omega      = CounterRng(seed_b) Gaussians            rng.cu       (factorize.cpp:61-63)
//   Y          = A Omega                                  gemm NN      (:68)
//   Q          = orth(Y)                                  CholeskyQR2  (lapack.cpp:180-201)
//   q times:   Z = A^T Q; Q' = orth(Z); Y = A Q'; Q = orth(Y)           (:69-72)
//   B^T        = A^T Q            (B = Q^T A, :86, never formed)
//   B^T        = Qb Rt                                    CholeskyQR2 with R
//   H = Rt^T;  H J = U~ Sigma                             one-sided Jacobi (lapack.cpp:112-128)
//   rank cut, discarded weight                            (:17-38, :91)
//   U = Q U~[:, :r];  Vt = (Qb J[:, :r])^T                gemm NN      (:92)
//
// orth() is CholeskyQR2 with a diagonally pivoted first Cholesky: columns
// whose pivot falls below tau * max pivot (rank deficiency) are replaced by
// a deterministic Gaussian completion that the second pass orthonormalises,
// so the result always has l orthonormal columns (lapack.hpp:18-20).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <initializer_list>
#include <map>
#include <tuple>
#include <vector>

#include "../../include/rsvd_c.h"
#include "common.cuh"

namespace rsvd {
namespace {

constexpr double kPivotTau = 1e-13;   // relative pivot floor of the CholeskyQR Gram
// Widest l x l factor the GPU path takes (the row-streamed Jacobi kernel has
// no l-dependent shared memory; the bound keeps int32 element offsets of the
// l x l work matrices safe and the workspace within one device).
constexpr int64_t kTsvdMaxDim = 16384;
constexpr int kMaxSweeps = 40;        // one-sided Jacobi sweep cap
constexpr uint64_t kCompletionTag = 0x436f6d706c657465ull;  // "Complete"

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// Grow-only device arena, the analogue of the reference's thread_local
// LAPACK workspace (lapack.cpp:23-50).  Contents do not persist across calls.
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  void reserve(size_t bytes) {
    if (bytes <= cap) return;
    if (base) RSVD_CUDA(cudaFree(base));
    base = nullptr;
    cap = 0;
    RSVD_CUDA(cudaMalloc(&base, bytes));
    cap = bytes;
  }
  void release() {
    if (base) cudaFree(base);
    base = nullptr;
    cap = 0;
  }
};

// Two-phase carve: measure with base == nullptr, then allocate and carve.
struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

}  // namespace

std::atomic<uint64_t> g_kernel_launches{0};

// Per-stage device-time accounting (CUDA events on the launching stream),
// enabled by rsvd_profile_enable; read back with rsvd_profile_read.
enum Stage : int {
  kStOmega = 0,   // Omega generation
  kStApassNN,     // Y = A X               (A-pass, NN)
  kStApassTN,     // Z = A^T Y             (A-pass, TN)
  kStGram,        // G = Y^T Y             (CholeskyQR Gram)
  kStChol,        // pivoted Cholesky + triangular inverse
  kStApply,       // Y T, completion, Rf2 Rf1
  kStJacobi,      // one-sided Jacobi on the l x l factor
  kStLift,        // spectrum, gathers, U = Q U~, V = Qb J, transposes
  kStSlice,       // INT8 slicing of A and of the A-pass right operands (nested
                  // inside apass_nn / apass_tn: subtract it for the GEMM alone)
  kNumStages
};
const char* const kStageNames[kNumStages] = {"omega", "apass_nn", "apass_tn", "gram",
                                             "chol",  "apply",    "jacobi",   "lift", "apass_slice"};

struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> marks;  // (stage, index of start event)
  double ms[kNumStages] = {};
  int64_t calls[kNumStages] = {};
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      RSVD_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
  // Call after the stream has been synchronized.
  void collect() {
    for (auto& [st, i] : marks) {
      float t = 0.f;
      RSVD_CUDA(cudaEventElapsedTime(&t, pool[i], pool[i + 1]));
      ms[st] += t;
      calls[st] += 1;
    }
    marks.clear();
    used = 0;
  }
  void reset() {
    for (int i = 0; i < kNumStages; ++i) ms[i] = 0.0, calls[i] = 0;
  }
  void destroy() {
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
  }
};

struct Scope {
  Prof* p;
  cudaStream_t st;
  size_t idx = 0;
  Scope(Prof* prof, int stage, cudaStream_t s) : p(prof && prof->on ? prof : nullptr), st(s) {
    if (!p) return;
    idx = p->used;
    RSVD_CUDA(cudaEventRecord(p->get(), st));
    p->get();
    p->marks.emplace_back(stage, idx);
  }
  ~Scope() {
    if (p) cudaEventRecord(p->pool[idx + 1], st);
  }
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  bool failed = false;
  uint64_t launches = 0;  // engine kernels captured in the graph (added on every replay)
  int seen = 0;           // calls with this key so far
};

// Pinned host staging for the per-call scalars (seeds in; ranks, sweeps,
// discarded weights out): stable addresses, so captured graphs can replay.
struct Pinned {
  uint64_t* seeds = nullptr;
  int* ints = nullptr;
  double* dbls = nullptr;
  int64_t cap = 0;
  bool reserve(int64_t n) {  // true when the buffers moved
    if (n <= cap) return false;
    release();
    const int64_t c = std::max<int64_t>(n, 64);
    RSVD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&seeds), sizeof(uint64_t) * c, 0));
    RSVD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ints), sizeof(int) * 2 * c, 0));
    RSVD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&dbls), sizeof(double) * c, 0));
    cap = c;
    return true;
  }
  void release() {
    if (seeds) cudaFreeHost(seeds);
    if (ints) cudaFreeHost(ints);
    if (dbls) cudaFreeHost(dbls);
    seeds = nullptr, ints = nullptr, dbls = nullptr, cap = 0;
  }
};

bool graphs_enabled() {
  static const bool v = std::getenv("RSVD_NO_GRAPH") == nullptr;
  return v;
}

}  // namespace rsvd

struct rsvd_context {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  rsvd::Arena arena;
  rsvd::Prof prof;
  rsvd::Pinned pin;
  rsvd::Arena tab;  // device copies of the TEBD job tables (rsvd_combine_blocks & co.)
  rsvd::Arena blk;  // sector staging of rsvd_block_factorize_f64 (outside the engine arena)
  std::unordered_map<std::string, rsvd::GraphEntry> graphs;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::unique_ptr<rsvd::Reducer> red;  // row-sharded calls (NCCL or in-process group)
  // Host-pointer pipelining: copy-in / copy-out streams and per-slot events.
  cudaStream_t s_in = nullptr, s_out = nullptr, s_c2 = nullptr, s_c3 = nullptr, s_c4 = nullptr;
  static constexpr int kMaxChunks = 16;
  cudaEvent_t ev_slot_in[kMaxChunks] = {}, ev_slot_comp[kMaxChunks] = {},
              ev_slot_out[kMaxChunks] = {};
  void ensure_pipeline() {
    if (s_in) return;
    RSVD_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    RSVD_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    RSVD_CUDA(cudaStreamCreateWithFlags(&s_c2, cudaStreamNonBlocking));
    RSVD_CUDA(cudaStreamCreateWithFlags(&s_c3, cudaStreamNonBlocking));
    RSVD_CUDA(cudaStreamCreateWithFlags(&s_c4, cudaStreamNonBlocking));
    for (int i = 0; i < kMaxChunks; ++i) {
      RSVD_CUDA(cudaEventCreateWithFlags(&ev_slot_in[i], cudaEventDisableTiming));
      RSVD_CUDA(cudaEventCreateWithFlags(&ev_slot_comp[i], cudaEventDisableTiming));
      RSVD_CUDA(cudaEventCreateWithFlags(&ev_slot_out[i], cudaEventDisableTiming));
    }
  }
  void destroy_pipeline() {
    if (!s_in) return;
    cudaStreamDestroy(s_in);
    cudaStreamDestroy(s_out);
    cudaStreamDestroy(s_c2);
    cudaStreamDestroy(s_c3);
    cudaStreamDestroy(s_c4);
    for (int i = 0; i < kMaxChunks; ++i) {
      cudaEventDestroy(ev_slot_in[i]);
      cudaEventDestroy(ev_slot_comp[i]);
      cudaEventDestroy(ev_slot_out[i]);
    }
    s_in = s_out = nullptr;
  }
  int last_sweeps = 0;
  int last_gemm_path = 0;  // 1: the last rsvd's A-passes ran on the emulated-FP64 INT8 path
  void drop_graphs() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
};

namespace rsvd {
namespace {

struct Shape {
  int64_t m, n, batch, k, ell, ellp, q;
  // Row sharding: this rank holds rows [row_off, row_off + m) of m_global.
  int64_t m_global = 0, row_off = 0;
  int64_t mg() const { return m_global > 0 ? m_global : m; }
};

struct Buffers {
  uint64_t* seeds;
  double *X, *X2, *Y, *Y2;
  double *G, *G0, *T, *Rf1, *Rf2, *Rt, *H, *Jm, *cscratch;
  int* ill;  // per item: the current orth took the ill-conditioned fallback
  double *Ut, *Jr, *Vb;
  double* sig;
  double* dw;
  double* scale;  // per item: exact power-of-two input scaling (1 = none)
  bool scaled;    // scale[] chosen for this call
  int *rank1, *rank2, *rankF, *perm, *permS, *sweeps;
  unsigned* jflags;
  double* partial;
  int64_t partial_cap;
  // Emulated-FP64 A-passes (ozaki.cu): slices of A in both K-major layouts,
  // slices of the right operand, exponents (rows of A, columns of A, columns
  // of the right operand).  ozR == nullptr: the A-passes run on DMMA.
  int8_t *ozR, *ozC, *ozB;
  int *ozErow, *ozEcol, *ozEb;
  bool oz_ready;  // A sliced for this call
  // staging for host-pointer calls
  double *Ah, *Uh, *Vth, *Sh;
  Prof* prof;
  Reducer* red;  // non-null for a row-sharded call
};

int64_t partial_need(const Shape& s) {
  const int64_t b = s.batch, lp = s.ellp;
  int64_t need = 0;
  auto upd = [&](bool t, int64_t M, int64_t N, int64_t K) {
    need = std::max(need, dgemm_partial_elems(t, M, N, K, b));
  };
  upd(false, s.m, lp, s.n);
  upd(true, lp, lp, s.m);
  upd(true, lp, lp, s.n);
  upd(false, s.m, lp, lp);
  upd(false, s.n, lp, lp);
  upd(true, s.n, lp, s.m);
  upd(false, lp, lp, lp);
  upd(false, s.m, s.k, lp);
  upd(false, s.n, s.k, lp);
  return need;
}

// The A-passes run on the INT8 tensor cores (Ozaki slices, ozaki.cu) when
// the one-CTA-per-SM output tiles of both directions keep >= 72% of their
// SM-waves busy (128 x 64 tiles, or 128 x 32 for grids of one or two thin
// waves: C3, C4, C5, C4 chunks of >= 2 items) and both K extents are >= 1024
// (a tile's prologue / TMEM drain is ~10 K steps: C2's K = 256 measured 22.2k
// against 25.4k trunc/s on DMMA).  C1 (24 tiles) and C2 stay on the split-K
// DMMA GEMM.  RSVD_FP64_GEMM=dmma forces the DMMA path (tests compare both).
bool oz_wanted(const Shape& s) {
  static const bool off = [] {
    const char* e = std::getenv("RSVD_FP64_GEMM");
    return e && std::string(e) == "dmma";
  }();
  if (off || !oz_supported(s.m, s.n, s.ellp) || s.m > 65536 || s.n > 65536) return false;
  if (s.m < 1024 || s.n < 1024) return false;
  // The slice copies (14 bytes per entry of A + the thin operand's) must leave
  // room for the input and the rest of the workspace: beyond half of the
  // device's memory the call stays on DMMA instead of failing its allocation.
  const int64_t need = 2 * oz_slice_bytes(s.m, s.n, s.batch) +
                       oz_slice_bytes(std::max(s.m, s.n), s.ellp, s.batch);
  if (need > device_total_memory() / 2) return false;
  return oz_grid_efficiency(s.m, s.ellp, s.batch) >= 0.72 &&
         oz_grid_efficiency(s.n, s.ellp, s.batch) >= 0.72;
}

Buffers carve(Carver& c, const Shape& s, bool host_io, bool want_svd) {
  Buffers B{};
  const int64_t b = s.batch, lp = s.ellp;
  if (oz_wanted(s)) {
    B.ozR = c.take<int8_t>(oz_slice_bytes(s.m, s.n, b));
    B.ozC = c.take<int8_t>(oz_slice_bytes(s.m, s.n, b));
    B.ozB = c.take<int8_t>(oz_slice_bytes(std::max(s.m, s.n), lp, b));
    B.ozErow = c.take<int>(s.m * b);
    B.ozEcol = c.take<int>(s.n * b);
    B.ozEb = c.take<int>(lp * b);
  }
  B.seeds = c.take<uint64_t>(b);
  B.scale = c.take<double>(b);
  B.X = c.take<double>(b * s.n * lp);
  B.X2 = c.take<double>(b * s.n * lp);
  B.Y = c.take<double>(b * s.m * lp);
  B.Y2 = c.take<double>(b * s.m * lp);
  B.G = c.take<double>(b * lp * lp);
  B.G0 = c.take<double>(b * lp * lp);
  B.ill = c.take<int>(b);
  B.T = c.take<double>(b * lp * lp);
  B.Rf1 = c.take<double>(b * lp * lp);
  B.Rf2 = c.take<double>(b * lp * lp);
  // Cholesky scratch; also the fused CholeskyQR's cluster exchange (l_p <= 160)
  B.cscratch = c.take<double>(std::max(pchol_scratch_elems(lp, b),
                                       lp <= 160 ? fcqr_xscratch_elems(lp, b) : int64_t(0)));
  B.rank1 = c.take<int>(b);
  B.rank2 = c.take<int>(b);
  B.perm = c.take<int>(b * lp);
  if (want_svd) {
    B.Rt = c.take<double>(b * lp * lp);
    B.H = c.take<double>(b * lp * lp);
    B.Jm = c.take<double>(b * lp * lp);
    B.Ut = c.take<double>(b * lp * s.k);
    B.Jr = c.take<double>(b * lp * s.k);
    B.Vb = c.take<double>(b * s.n * s.k);
    B.sig = c.take<double>(b * s.k);
    B.dw = c.take<double>(b);
    B.rankF = c.take<int>(b);
    B.permS = c.take<int>(b * lp);
    B.sweeps = c.take<int>(b);
    B.jflags = c.take<unsigned>(jacobi_flag_elems(b, lp));
  }
  B.partial_cap = partial_need(s);
  B.partial = c.take<double>(std::max<int64_t>(B.partial_cap, 1));
  if (host_io) {
    B.Ah = c.take<double>(b * s.m * s.n);
    B.Uh = c.take<double>(b * s.m * std::max<int64_t>(s.k, s.ell));
    if (want_svd) {
      B.Vth = c.take<double>(b * s.k * s.n);
      B.Sh = c.take<double>(b * s.k);
    }
  }
  return B;
}

// CholeskyQR of Y (rows x ellp per item): `passes` = 2 is CholeskyQR2 (the
// result is orthonormal to working precision); 1 pass gives Q1 = (Y P) R11^-1,
// an exact-span, well-conditioned basis (kappa(Q1)^2 - 1 = O(u kappa(Y)^2) with
// kappa(Y) <= tau^-1/2), which is all an intermediate power-iteration step
// consumes: the next product only sees span(Q).  The result is left in *Yb
// (the two buffers are swapped when passes is odd).  When Rt is given, also
// Rt = R_last ... R_1 with Y_in ~= Y_out * Rt.
// m_side: Y has the (possibly row-sharded) m rows of A; its Gram is then
// all-reduced across ranks and the completion uses global row indices.
//
// Ill-conditioned fallback (the north star's "TSQR fallback for ill-conditioned
// Y", as shifted CholeskyQR, Fukaya et al. 2020): an item whose first
// factorization stops below full rank (kappa(Y) > tau^-1/2 ~ 3e6, or a rank-
// deficient Y) is refactored from the saved Gram as G + sI,
// s = 11 (rows l + l (l + 1)) u tr(G), unpivoted and without truncation, and
// gets one extra CholeskyQR pass (masked to those items).  Directions down to
// sigma ~ u ||Y|| keep their true components, as with the reference's
// Householder QR (lapack.cpp:146-201), instead of a random completion -- the
// sampled tail (discarded weight) of steep spectra depends on them.  Items
// that never truncate pay only the no-op launches.
// cplx: Y is a complex basis in P-layout (zkern.cu; s.ell / s.ellp are the
// realified 2l / 2lp) and every Gram is replaced by the realified complex Gram
// before the Cholesky (launch_hermitize): the same passes then compute the
// complex CholeskyQR.
void orth(const Shape& s, Buffers& B, double*& Yb, double*& Tmp, int64_t rows, double* Rt,
          uint64_t tag, int passes, bool m_side, cudaStream_t st, bool cplx = false) {
  const int64_t lp = s.ellp, b = s.batch;
  const bool sharded = m_side && B.red;
  const int64_t row_off = m_side ? s.row_off : 0, rows_global = m_side ? s.mg() : rows;
  const MatRef Y{Yb, rows, rows * lp}, Tm{Tmp, rows, rows * lp};
  const MatRef G{B.G, lp, lp * lp}, T{B.T, lp, lp * lp};
  Prof* P = B.prof;
  // Small real bases: one fused CholeskyQR kernel per pass (chol.cu
  // fcqr_kernel: one CTA per item for batches, a row-split cluster of up to 8
  // CTAs per item for single / few items).
  const bool fused = !cplx && !sharded && lp <= 160;
  auto gram = [&](const MatRef& in, const int* mask) {
    Scope sc(P, kStGram, st);
    GemmOpts sym;
    sym.c_upper = true;
    sym.item_mask = mask;
    dgemm_ex(true, lp, lp, rows, in, in, G, b, B.partial, B.partial_cap, sym, st);
    if (sharded) B.red->allreduce_sum(B.G, b * lp * lp, st);  // G = sum_p Y_p^T Y_p
    if (cplx) launch_hermitize(B.G, lp / 2, mask, b, st);
  };
  auto apply = [&](const MatRef& in, const MatRef& out, const int* mask, bool pivoted) {
    // out = (in P) R11^{-1}: pivot-gathered columns (only when this pass
    // pivoted; without the column map the TMA GEMM takes it), upper-triangular
    // right factor.
    GemmOpts tri;
    tri.colmapA = pivoted ? B.perm : nullptr;
    tri.colmap_stride = lp;
    tri.b_upper = true;
    tri.item_mask = mask;
    dgemm_ex(false, rows, lp, lp, in, T, out, b, B.partial, B.partial_cap, tri, st);
  };
  for (int pass = 0; pass < passes; ++pass) {
    const MatRef& in = pass == 0 ? Y : Tm;
    const MatRef& out = pass == 0 ? Tm : Y;
    double* Rf = Rt ? (pass == 0 ? B.Rf1 : B.Rf2) : nullptr;
    int* rk = pass == 0 ? B.rank1 : B.rank2;
    const bool pivot = false;
    auto shifted_retry = [&] {  // the items that stopped short of full rank
      CholOpts o;
      o.gate_rank = rk;
      o.ill_out = B.ill;
      o.Gsrc = B.G0;
      o.shift_coef = 11.0 *
                     (static_cast<double>(rows_global) * s.ell +
                      static_cast<double>(s.ell) * (s.ell + 1)) *
                     1.1102230246251565e-16;
      launch_pchol(B.G, B.T, Rf, B.cscratch, rk, B.perm, s.ell, lp, kPivotTau, false, b, st, &o);
    };
    if (fused) {
      // One fused kernel per pass (Gram, Cholesky, Q = Y R^-1; G0 saved on the
      // first pass); the ill items are then redone from G0 as before.
      {
        Scope sc(P, kStChol, st);
        if (!launch_fused_cqr(in.base, rows, rows * lp, out.base, rows, rows * lp,
                              pass == 0 ? B.G0 : nullptr, Rf, B.cscratch, rk, rows, s.ell, lp, kPivotTau,
                              b, st, pass > 0))
          throw CudaError("orth: fused CholeskyQR does not fit this shape");
        if (pass == 0) shifted_retry();
      }
      Scope sc(P, kStApply, st);
      if (pass == 0) apply(in, out, B.ill, pivot);
      launch_complete_basis(out, rows, s.ell, rk, B.seeds, tag + pass, b, row_off, rows_global,
                            st);
    } else {
      gram(in, nullptr);
      {
        Scope sc(P, kStChol, st);
        if (pass == 0)
          RSVD_CUDA(cudaMemcpyAsync(B.G0, B.G, sizeof(double) * b * lp * lp,
                                    cudaMemcpyDeviceToDevice, st));
        // Unpivoted everywhere (grid-parallel gchol; breakdown -> numerical
        // rank).  Pivoting the first pass on B^T (QRCP grading of Rt for the
        // Jacobi) measured no fewer sweeps (r01 and r02, C2 8 / C4 7 sweeps).
        // Repeat passes: first-order factor for the items already orthonormal
        // to ~1e-8 (chol.cu kLinTol2), exact gchol for the rest.
        CholOpts lo;
        lo.lin = pass > 0 && !cplx;
        launch_pchol(B.G, B.T, Rf, B.cscratch, rk, B.perm, s.ell, lp, kPivotTau, pivot, b, st,
                     lo.lin ? &lo : nullptr);
        if (pass == 0) shifted_retry();
      }
      Scope sc(P, kStApply, st);
      apply(in, out, nullptr, pivot);
      launch_complete_basis(out, rows, s.ell, rk, B.seeds, tag + pass, b, row_off, rows_global,
                            st);
    }
    if (pass == 0) {
      // Extra CholeskyQR pass for the ill items: out -> in (free now) -> out.
      gram(out, B.ill);
      {
        Scope sc(P, kStChol, st);
        // Pivoted (dpstrf semantics): the shifted pass leaves exact-null
        // directions as tiny columns at arbitrary positions, and an unpivoted
        // factorization would stop at the first and drop every later column.
        CholOpts o;
        o.mask = B.ill;
        o.pairs = cplx;
        launch_pchol(B.G, B.T, Rt ? B.Rf2 : nullptr, B.cscratch, B.rank2, B.perm, s.ell, lp,
                     kPivotTau, true, b, st, &o);
      }
      Scope sc(P, kStApply, st);
      apply(out, in, B.ill, true);
      launch_complete_basis(in, rows, s.ell, B.rank2, B.seeds, tag + 0x40, b, row_off, rows_global,
                            st, B.ill);
      launch_masked_copy(B.ill, in, out, rows, lp, b, st);
      if (Rt) {  // R1 <- R_extra R1 for the ill items (Rt is scratch until the end)
        GemmOpts mk;
        mk.item_mask = B.ill;
        dgemm_ex(false, lp, lp, lp, MatRef{B.Rf2, lp, lp * lp}, MatRef{B.Rf1, lp, lp * lp},
                 MatRef{Rt, lp, lp * lp}, b, B.partial, B.partial_cap, mk, st);
        launch_masked_copy(B.ill, MatRef{Rt, lp, lp * lp}, MatRef{B.Rf1, lp, lp * lp}, lp, lp, b,
                           st);
      }
    }
  }
  if (Rt) {
    Scope sc(P, kStApply, st);
    if (passes >= 2)
      dgemm(false, lp, lp, lp, MatRef{B.Rf2, lp, lp * lp}, MatRef{B.Rf1, lp, lp * lp},
            MatRef{Rt, lp, lp * lp}, b, B.partial, B.partial_cap, st);
    else
      launch_copy_matrix(MatRef{B.Rf1, lp, lp * lp}, lp, lp, MatRef{Rt, lp, lp * lp}, b, st);
  }
  if (passes % 2 == 1) std::swap(Yb, Tmp);
}

// A-pass with the caller's A: C = A X (NN: m x l_p, K = n) or C = A^T Y (TN:
// n x l_p, K = m).  On the emulated-FP64 path A is sliced once per call, at
// its first pass.  (A null slice buffer in a chunk's Buffers is the host
// pipeline's measuring carve: never launched.)
void apass(const Shape& s, Buffers& B, CMatRef A, bool trans, CMatRef R, MatRef C, cudaStream_t st) {
  const int64_t lp = s.ellp, b = s.batch;
  if (B.ozR) {
    const int64_t M = trans ? s.n : s.m, K = trans ? s.m : s.n;
    {
      Scope sc(B.prof, kStSlice, st);
      if (!B.oz_ready) {
        oz_prepare_a(A, s.m, s.n, b, B.ozR, B.ozC, B.ozErow, B.ozEcol, st);
        B.oz_ready = true;
      }
      oz_slice_b(R, K, lp, b, B.ozB, B.ozEb, st);
    }
    oz_gemm(M, lp, K, trans ? B.ozC : B.ozR, trans ? B.ozEcol : B.ozErow, B.ozB, B.ozEb, C, b, st);
    return;
  }
  if (trans) dgemm(true, s.n, lp, s.m, A, R, C, b, B.partial, B.partial_cap, st);
  else dgemm(false, s.m, lp, s.n, A, R, C, b, B.partial, B.partial_cap, st);
}

// randomized_range (factorize.cpp:52-74): leaves Q (orthonormal) in B.Y.
void range_finder(const Shape& s, Buffers& B, CMatRef A, cudaStream_t st) {
  const int64_t lp = s.ellp, b = s.batch;
  Prof* P = B.prof;
  {
    Scope sc(P, kStOmega, st);
    launch_fill_gaussian(MatRef{B.X, s.n, s.n * lp}, s.n, lp, s.ell, B.seeds, b, st);
  }
  // Extreme-magnitude items run on 2^-e A (exact): the scale is chosen from
  // the first product Y = A Omega (|Y| tracks sigma_max(A)) and applied to
  // every A-pass output; sigma and the discarded weight are scaled back at the
  // end.  Row-sharded calls are not scaled (a per-rank max would disagree).
  const bool do_scale = !B.red;
  auto nn = [&] {
    Scope sc(P, kStApassNN, st);
    apass(s, B, A, false, MatRef{B.X, s.n, s.n * lp}, MatRef{B.Y, s.m, s.m * lp}, st);
    if (do_scale) {
      if (!B.scaled) {
        launch_choose_scale(MatRef{B.Y, s.m, s.m * lp}, s.m, s.ell, B.scale, b, st);
        B.scaled = true;
      }
      launch_apply_scale(MatRef{B.Y, s.m, s.m * lp}, s.m, lp, B.scale, 0, b, st);
    }
  };
  auto tn = [&] {
    Scope sc(P, kStApassTN, st);
    apass(s, B, A, true, MatRef{B.Y, s.m, s.m * lp}, MatRef{B.X, s.n, s.n * lp}, st);
    if (B.red) B.red->allreduce_sum(B.X, b * s.n * lp, st);  // Z = sum_p A_p^T Q_p
    if (do_scale) launch_apply_scale(MatRef{B.X, s.n, s.n * lp}, s.n, lp, B.scale, 0, b, st);
  };
  B.scaled = false;
  B.oz_ready = false;
  nn();
  uint64_t tag = kCompletionTag;
  // Only the last orthonormalisation feeds B = Q^T A and U = Q U~; the
  // intermediate ones need a well-conditioned basis of the span (one pass).
  orth(s, B, B.Y, B.Y2, s.m, nullptr, tag, s.q == 0 ? 2 : 1, true, st);
  tag += 2;
  for (int64_t t = 0; t < s.q; ++t) {
    tn();
    orth(s, B, B.X, B.X2, s.n, nullptr, tag, 1, false, st);
    tag += 2;
    nn();
    orth(s, B, B.Y, B.Y2, s.m, nullptr, tag, t + 1 == s.q ? 2 : 1, true, st);
    tag += 2;
  }
}

// Projection + small SVD + lift (factorize.cpp:86-93).  Outputs go to
// U (m x k), S (k per item, contiguous stride sS), Vt (k x n).
// exact_h (tsvd, Q = I): the Jacobi input is recomputed as H = A Qb instead of
// Rt^T.  A annihilates the part of Qb outside range(A^T), so sigma(H) carries
// only the O(u) departure of Qb from orthonormality: absolute errors
// O(u ||A||) like LAPACK's gesdd, where Rt = R2 R1 alone inherits the
// O(u kappa) residual of the first CholeskyQR pass on ill-conditioned blocks.
void svd_stage(const Shape& s, Buffers& B, CMatRef A, MatRef U, double* S, int64_t sS, MatRef Vt,
               cudaStream_t st, bool exact_h = false) {
  const int64_t lp = s.ellp, b = s.batch, k = s.k;
  const MatRef X{B.X, s.n, s.n * lp}, Y{B.Y, s.m, s.m * lp};
  Prof* P = B.prof;
  // B^T = A^T Q (n x ellp), then B^T = Qb Rt.
  {
    Scope sc(P, kStApassTN, st);
    apass(s, B, A, true, Y, X, st);
    if (B.red) B.red->allreduce_sum(B.X, b * s.n * lp, st);  // B^T = sum_p A_p^T Q_p
    if (!B.red) {
      if (!B.scaled) {  // tsvd (Q = I): choose the scale from B^T = A_e^T
        launch_choose_scale(X, s.n, s.ell, B.scale, b, st);
        B.scaled = true;
      }
      launch_apply_scale(X, s.n, lp, B.scale, 0, b, st);
    }
  }
  orth(s, B, B.X, B.X2, s.n, B.Rt, kCompletionTag + 0x1000, 2, false, st);
  const MatRef Qb{B.X, s.n, s.n * lp};  // orth may have swapped B.X and B.X2
  {
    Scope sc(P, kStJacobi, st);
    if (exact_h) {
      RSVD_CUDA(cudaMemsetAsync(B.H, 0, sizeof(double) * b * lp * lp, st));
      apass(s, B, A, false, Qb, MatRef{B.H, lp, lp * lp}, st);
      if (!B.red && B.scaled) launch_apply_scale(MatRef{B.H, lp, lp * lp}, s.m, lp, B.scale, 0, b, st);
    } else {
      launch_transpose(MatRef{B.Rt, lp, lp * lp}, lp, lp, MatRef{B.H, lp, lp * lp}, b, st);
    }
    launch_jacobi(B.H, B.Jm, s.ell, lp, kMaxSweeps, B.sweeps, B.jflags, b, st);
  }
  Scope sc(P, kStLift, st);
  launch_finalize_spectrum(B.H, lp, s.ell, k, s.mg(), s.n, B.sig, B.permS, B.rankF, B.dw, b, st);
  // U~ = W Sigma^{-1} restricted to the kept columns, then U = Q U~.
  launch_gather_scale_columns(B.H, lp, lp * lp, B.permS, lp, B.sig, k, B.rankF, lp, k, B.Ut, lp,
                              lp * k, b, st);
  dgemm(false, s.m, k, lp, Y, MatRef{B.Ut, lp, lp * k}, U, b, B.partial, B.partial_cap, st);
  // V = Qb J[:, perm[:r]], Vt = V^T.
  launch_gather_scale_columns(B.Jm, lp, lp * lp, B.permS, lp, nullptr, k, B.rankF, lp, k, B.Jr,
                              lp, lp * k, b, st);
  dgemm(false, s.n, k, lp, Qb, MatRef{B.Jr, lp, lp * k}, MatRef{B.Vb, s.n, s.n * k}, b, B.partial,
        B.partial_cap, st);
  launch_transpose(MatRef{B.Vb, s.n, s.n * k}, s.n, k, Vt, b, st);
  if (!B.red && B.scaled) {  // back to the caller's scale (exact powers of two)
    launch_apply_scale(MatRef{B.sig, k, k}, k, 1, B.scale, 1, b, st);
    launch_apply_scale(MatRef{B.dw, 1, 1}, 1, 1, B.scale, 2, b, st);
  }
  launch_copy_matrix(MatRef{B.sig, k, k}, k, 1, MatRef{S, k, sS}, b, st);
}

// ------------------------------------------------------------ validation
// Same checks, order and messages as the reference.
void validate_rsvd(int64_t m, int64_t n, int64_t rank, int64_t oversample, int power,
                   int64_t& ell) {
  if (m <= 0 || n <= 0) throw InvalidArgument("rsvd: empty matrix");              // :79
  if (rank < 1) throw InvalidArgument("rsvd: rank must be >= 1");                 // :80
  ell = oversample;
  if (ell == 0) ell = std::min(2 * rank, std::min(m, n));                         // :82
  if (ell < rank) throw InvalidArgument("rsvd: oversample must be >= rank");      // :83
  if (ell < 1 || ell > std::min(m, n))                                            // :57-58
    throw InvalidArgument("randomized_range: need 1 <= ell <= min(m, n)");
  if (power < 0) throw InvalidArgument("randomized_range: power must be >= 0");   // :59
}

void validate_range(int64_t m, int64_t n, int64_t ell, int power) {
  if (m <= 0 || n <= 0) throw InvalidArgument("randomized_range: empty matrix");
  if (ell < 1 || ell > std::min(m, n))
    throw InvalidArgument("randomized_range: need 1 <= ell <= min(m, n)");
  if (power < 0) throw InvalidArgument("randomized_range: power must be >= 0");
}

void check_flags(int flags) {
  if (flags != RSVD_PTR_HOST && flags != RSVD_PTR_DEVICE)
    throw InvalidArgument("rsvd: flags must be RSVD_PTR_HOST or RSVD_PTR_DEVICE");
}

void copy_2d(void* dst, int64_t dpitch_elems, const void* src, int64_t spitch_elems, int64_t rows,
             int64_t cols, cudaMemcpyKind kind, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  if (dpitch_elems == rows && spitch_elems == rows) {  // contiguous: one linear DMA
    RSVD_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols, kind, st));
    return;
  }
  RSVD_CUDA(cudaMemcpy2DAsync(dst, dpitch_elems * sizeof(double), src,
                              spitch_elems * sizeof(double), rows * sizeof(double), cols, kind,
                              st));
}

// A strided batch of column-major items: one linear copy when the items are
// packed back to back in both buffers, per-item (2-D) copies otherwise.
void copy_batch(void* dst, int64_t dld, int64_t dstride, const void* src, int64_t sld,
                int64_t sstride, int64_t rows, int64_t cols, int64_t count, cudaMemcpyKind kind,
                cudaStream_t st) {
  if (count <= 0) return;
  if (dld == rows && sld == rows && dstride == rows * cols && sstride == rows * cols) {
    RSVD_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols * count, kind, st));
    return;
  }
  for (int64_t b = 0; b < count; ++b)
    copy_2d(static_cast<double*>(dst) + b * dstride, dld, static_cast<const double*>(src) + b * sstride,
            sld, rows, cols, kind, st);
}

// Number of chunks for the host-pointer path (overlap of the PCIe copies
// with compute); RSVD_HOST_CHUNKS overrides.
int64_t host_chunks(int64_t batch, int64_t m, int64_t n) {
  if (const char* e = std::getenv("RSVD_HOST_CHUNKS"))
    return std::min<int64_t>(rsvd_context::kMaxChunks, std::max<int64_t>(1, std::atoi(e)));
  // Each chunk has its own staging, so the H2D stream never waits for a slot.
  // C4 (4.3 GB): 7 chunks (5,5,5,5,5,5,2) on three compute streams measured
  // 319 trunc/s against 295 for 4 chunks on two (tools/probe/e2e_probe.py).
  // C2 (256 x 256^2, 134 MB): 2 chunks 18.7k trunc/s against 16.0k unchunked
  // (3: 18.4k, 4: 15.6k).
  const int64_t per = m * n * 8;
  if (batch < 2 || per * batch < (int64_t(64) << 20)) return 1;
  const int64_t by_size = std::max<int64_t>(1, per * batch / (int64_t(512) << 20));
  return std::max<int64_t>(2, std::min<int64_t>({by_size, batch, 7}));
}

// Host-pointer batched rsvd with the PCIe transfers overlapped: chunk c's H2D
// (stream s_in) runs while earlier chunks compute; chunks alternate between
// two compute streams, so one chunk's latency-bound stages (Cholesky, Jacobi)
// overlap the next chunk's GEMMs; factors return on s_out.  Every chunk has
// its own device staging and workspace (no slot reuse, no copy-engine stalls).
void rsvd_host_pipelined(rsvd_context* h, const Shape& full, int64_t nchunks, const double* A,
                         int64_t lda, int64_t strideA, double* U, int64_t ldu, int64_t strideU,
                         double* S, int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt) {
  const int64_t batch = full.batch, m = full.m, n = full.n, k = full.k;
  // Equal chunk sizes (a shorter last chunk measured no better on C4: the
  // GPU, not the tail, is the limit).
  std::vector<int64_t> sizes;
  {
    const int64_t cb = ceil_div(batch, nchunks);
    for (int64_t tot = 0; tot < batch; tot += cb) sizes.push_back(std::min(cb, batch - tot));
  }
  nchunks = static_cast<int64_t>(std::min<size_t>(sizes.size(), rsvd_context::kMaxChunks));
  std::vector<int64_t> off(nchunks + 1, 0);
  for (int64_t c = 0; c < nchunks; ++c) off[c + 1] = off[c] + sizes[c];
  const int64_t cb = *std::max_element(sizes.begin(), sizes.begin() + nchunks);
  h->ensure_pipeline();
  cudaStream_t st = h->stream;
  Shape sc = full;
  sc.batch = cb;
  std::vector<Buffers> B(nchunks);
  std::vector<double*> Ah(nchunks), Uh(nchunks), Sh(nchunks), Vh(nchunks);
  auto layout = [&](Carver& c) {
    for (int64_t q = 0; q < nchunks; ++q) {
      B[q] = carve(c, sc, false, true);
      Ah[q] = c.take<double>(cb * m * n);
      Uh[q] = c.take<double>(cb * m * k);
      Sh[q] = c.take<double>(cb * k);
      Vh[q] = c.take<double>(cb * k * n);
    }
  };
  Carver meas{nullptr};
  layout(meas);
  char* const before = h->arena.base;
  h->arena.reserve(meas.off + 256);
  if (h->arena.base != before) h->drop_graphs();
  Carver cv{h->arena.base};
  layout(cv);
  h->last_gemm_path = B[0].ozR ? 1 : 0;
  cudaStream_t cs[4] = {st, h->s_c2, h->s_c3, h->s_c4};
  // 3 compute streams measured best on C4 (2: 295, 3: 319 trunc/s); uneven
  // chunk sizes (small first / last chunks) and 4 streams measured no better
  // (100.5-103.5 ms against 100.9 per call): the chunked GPU work, not the
  // pipeline fill, is the limit (tools/probe/e2e_probe.py).
  constexpr int nstreams = 3;
  // Order the side streams after whatever the caller queued on its stream.
  RSVD_CUDA(cudaEventRecord(h->ev_in, st));
  RSVD_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_in, 0));
  RSVD_CUDA(cudaStreamWaitEvent(h->s_out, h->ev_in, 0));
  RSVD_CUDA(cudaStreamWaitEvent(h->s_c2, h->ev_in, 0));
  RSVD_CUDA(cudaStreamWaitEvent(h->s_c3, h->ev_in, 0));
  RSVD_CUDA(cudaStreamWaitEvent(h->s_c4, h->ev_in, 0));
  // All H2D copies first (one stream, back to back), then the compute chain.
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t b0 = off[c], nb = sizes[c];
    copy_batch(Ah[c], m, m * n, A + b0 * strideA, lda, strideA, m, n, nb, cudaMemcpyHostToDevice,
               h->s_in);
    RSVD_CUDA(cudaEventRecord(h->ev_slot_in[c], h->s_in));
  }
#ifdef RSVD_PIPE_TRACE
  // Timeline of the chunks (make EXTRA=-DRSVD_PIPE_TRACE; tools/probe/e2e_probe.py).
  std::vector<cudaEvent_t> tev(4 * nchunks + 1);
  for (auto& e : tev) cudaEventCreate(&e);
  cudaEventRecord(tev[0], h->s_in);
#endif
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t b0 = off[c], nb = sizes[c];
    cudaStream_t q = cs[c % nstreams];
    RSVD_CUDA(cudaStreamWaitEvent(q, h->ev_slot_in[c], 0));
#ifdef RSVD_PIPE_TRACE
    cudaEventRecord(tev[1 + 4 * c], q);
#endif
    Shape s = sc;
    s.batch = nb;
    Buffers Bq = B[c];
    Bq.prof = (c == 0) ? &h->prof : nullptr;
    Bq.red = nullptr;
    RSVD_CUDA(cudaMemcpyAsync(Bq.seeds, h->pin.seeds + b0, sizeof(uint64_t) * nb,
                              cudaMemcpyHostToDevice, q));
    const CMatRef Ad{Ah[c], m, m * n};
    range_finder(s, Bq, Ad, q);
#ifdef RSVD_PIPE_TRACE
    cudaEventRecord(tev[2 + 4 * c], q);
#endif
    svd_stage(s, Bq, Ad, MatRef{Uh[c], m, m * k}, Sh[c], k, MatRef{Vh[c], k, k * n}, q);
#ifdef RSVD_PIPE_TRACE
    cudaEventRecord(tev[3 + 4 * c], q);
#endif
    RSVD_CUDA(cudaMemcpyAsync(h->pin.ints + b0, B[c].rankF, sizeof(int) * nb,
                              cudaMemcpyDeviceToHost, q));
    RSVD_CUDA(cudaMemcpyAsync(h->pin.ints + batch + b0, B[c].sweeps, sizeof(int) * nb,
                              cudaMemcpyDeviceToHost, q));
    RSVD_CUDA(cudaMemcpyAsync(h->pin.dbls + b0, B[c].dw, sizeof(double) * nb,
                              cudaMemcpyDeviceToHost, q));
    RSVD_CUDA(cudaEventRecord(h->ev_slot_comp[c], q));
    RSVD_CUDA(cudaStreamWaitEvent(h->s_out, h->ev_slot_comp[c], 0));
    copy_batch(U + b0 * strideU, ldu, strideU, Uh[c], m, m * k, m, k, nb, cudaMemcpyDeviceToHost,
               h->s_out);
    copy_batch(Vt + b0 * strideVt, ldvt, strideVt, Vh[c], k, k * n, k, n, nb,
               cudaMemcpyDeviceToHost, h->s_out);
    copy_batch(S + b0 * strideS, k, strideS, Sh[c], k, k, k, 1, nb, cudaMemcpyDeviceToHost,
               h->s_out);
#ifdef RSVD_PIPE_TRACE
    cudaEventRecord(tev[4 + 4 * c], h->s_out);
#endif
  }
  RSVD_CUDA(cudaStreamSynchronize(h->s_out));
#ifdef RSVD_PIPE_TRACE
  cudaDeviceSynchronize();
  for (int64_t c = 0; c < nchunks; ++c) {
    float t[4];
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[1 + 4 * c + i]);
    std::fprintf(stderr, "chunk %lld (%lld items): in %.1f  range %.1f  svd %.1f  out %.1f ms\n",
                 static_cast<long long>(c), static_cast<long long>(sizes[c]), t[0], t[1], t[2], t[3]);
  }
  for (auto& e : tev) cudaEventDestroy(e);
#endif
  RSVD_CUDA(cudaStreamSynchronize(st));
  RSVD_CUDA(cudaStreamSynchronize(h->s_c2));
  RSVD_CUDA(cudaStreamSynchronize(h->s_c3));
  RSVD_CUDA(cudaStreamSynchronize(h->s_c4));
  RSVD_CUDA(cudaStreamSynchronize(h->s_in));
}

// True when every host buffer is page-locked right now.  A captured host-copy
// graph is keyed on raw addresses: a caller that frees a pinned buffer and
// gets pageable memory back at the same address must not replay copies bound
// to the old pinned allocation, so the check runs before every replay.
bool all_pinned(std::initializer_list<const void*> ptrs) {
  for (const void* p : ptrs) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;
  }
  return true;
}

// Replay a captured CUDA graph of `enqueue` (one host launch per call), keyed
// by everything the captured pointers and shapes depend on; captured on the
// handle's own stream and ordered after / before the caller's stream with
// events.  Falls back to a direct enqueue when capture fails.
template <class F>
void run_graph(rsvd_context* h, const std::string& key, cudaStream_t st, F&& enqueue) {
    // Keys include the caller's buffers: callers that allocate fresh outputs
    // every call (instead of reusing them) would grow the cache without bound.
    if (h->graphs.size() >= 64 && h->graphs.find(key) == h->graphs.end()) h->drop_graphs();
    GraphEntry& ge = h->graphs[key];
    // Capture on the second call with the same key: a caller that passes fresh
    // output buffers every call (a new key each time) never pays a capture.
    if (ge.seen++ == 0) {
      enqueue(st);
      RSVD_CUDA(cudaStreamSynchronize(st));
      return;
    }
    if (!ge.exec && !ge.failed) {
      cudaGraph_t g = nullptr;
      RSVD_CUDA(cudaStreamBeginCapture(h->own, cudaStreamCaptureModeThreadLocal));
      const uint64_t l0 = g_kernel_launches.load();
      try {
        enqueue(h->own);
        // Capture does not run the kernels: count them once per replay instead.
        ge.launches = g_kernel_launches.load() - l0;
        g_kernel_launches.fetch_sub(ge.launches);
      } catch (...) {
        cudaStreamEndCapture(h->own, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        ge.failed = true;
      }
      if (!ge.failed) {
        const cudaError_t e = cudaStreamEndCapture(h->own, &g);
        if (e != cudaSuccess || !g || cudaGraphInstantiate(&ge.exec, g, 0) != cudaSuccess) {
          ge.failed = true;
          ge.exec = nullptr;
          cudaGetLastError();
        }
        if (g) cudaGraphDestroy(g);
      }
    }
    if (ge.exec) {
      RSVD_CUDA(cudaEventRecord(h->ev_in, st));
      RSVD_CUDA(cudaStreamWaitEvent(h->own, h->ev_in, 0));
      RSVD_CUDA(cudaGraphLaunch(ge.exec, h->own));
      g_kernel_launches.fetch_add(ge.launches);
      RSVD_CUDA(cudaEventRecord(h->ev_out, h->own));
      RSVD_CUDA(cudaStreamWaitEvent(st, h->ev_out, 0));
      RSVD_CUDA(cudaStreamSynchronize(h->own));
    } else {
      enqueue(st);
      RSVD_CUDA(cudaStreamSynchronize(st));
    }
}

void rsvd_batched_impl(rsvd_context* h, int64_t batch, const double* A, int64_t m, int64_t n,
                       int64_t lda, int64_t strideA, int64_t rank, int64_t oversample, int power,
                       const uint64_t* seeds, double* U, int64_t ldu, int64_t strideU, double* S,
                       int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt,
                       int64_t* out_rank, double* dw, int flags, int64_t m_global = 0,
                       int64_t row_off = 0, bool sharded = false) {
  check_flags(flags);
  int64_t ell = 0;
  validate_rsvd(sharded ? m_global : m, n, rank, oversample, power, ell);
  if (sharded) {
    if (!h->red) throw InvalidArgument("rsvd_rowsharded: no group / communicator attached");
    if (m < 1 || row_off < 0 || row_off + m > m_global)
      throw InvalidArgument("rsvd_rowsharded: local rows out of range");
  }
  if (batch < 0) throw InvalidArgument("rsvd: batch must be >= 0");
  if (batch == 0) return;
  if (!A || !U || !S || !Vt || !seeds || !out_rank || !dw)
    throw InvalidArgument("rsvd: null pointer argument");
  if (lda < m || ldu < m || ldvt < rank) throw InvalidArgument("rsvd: leading dimension too small");
  if (ell > kTsvdMaxDim) throw InvalidArgument("rsvd: l > 16384 is not supported by the GPU path");
  const bool host = flags == RSVD_PTR_HOST;
  RSVD_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;

  Shape s{m, n, batch, rank, ell, round_up(ell, 32), power};
  if (sharded) s.m_global = m_global, s.row_off = row_off;
  if (host && !sharded) {
    const int64_t nchunks = host_chunks(batch, m, n);
    if (nchunks > 1) {
      if (h->pin.reserve(batch)) h->drop_graphs();
      std::memcpy(h->pin.seeds, seeds, sizeof(uint64_t) * batch);
      rsvd_host_pipelined(h, s, nchunks, A, lda, strideA, U, ldu, strideU, S, strideS, Vt, ldvt,
                          strideVt);
      if (h->prof.on) h->prof.collect();
      h->last_sweeps = 0;
      for (int64_t b = 0; b < batch; ++b) {
        out_rank[b] = h->pin.ints[b];
        dw[b] = h->pin.dbls[b];
        h->last_sweeps = std::max(h->last_sweeps, h->pin.ints[batch + b]);
      }
      return;
    }
  }
  Carver meas{nullptr};
  carve(meas, s, host, true);
  char* const arena_before = h->arena.base;
  h->arena.reserve(meas.off + 256);
  if (h->arena.base != arena_before) h->drop_graphs();
  Carver cv{h->arena.base};
  Buffers B = carve(cv, s, host, true);
  h->last_gemm_path = B.ozR ? 1 : 0;

  if (h->pin.reserve(batch)) h->drop_graphs();
  std::memcpy(h->pin.seeds, seeds, sizeof(uint64_t) * batch);
  CMatRef Ad{A, lda, strideA};
  MatRef Ud{U, ldu, strideU}, Vtd{Vt, ldvt, strideVt};
  double* Sd = S;
  int64_t sS = strideS;
  if (host) {
    Ad = CMatRef{B.Ah, m, m * n};
    Ud = MatRef{B.Uh, m, m * rank};
    Vtd = MatRef{B.Vth, rank, rank * n};
    Sd = B.Sh;
    sS = rank;
  }
  B.prof = &h->prof;
  B.red = sharded ? h->red.get() : nullptr;
  // The device part of the call: pinned seeds in, pipeline, small results out.
  auto enqueue = [&](cudaStream_t q) {
    RSVD_CUDA(cudaMemcpyAsync(B.seeds, h->pin.seeds, sizeof(uint64_t) * batch,
                              cudaMemcpyHostToDevice, q));
    Buffers Bq = B;  // range_finder swaps ping-pong buffers in its copy
    range_finder(s, Bq, Ad, q);
    svd_stage(s, Bq, Ad, Ud, Sd, sS, Vtd, q);
    RSVD_CUDA(cudaMemcpyAsync(h->pin.ints, B.rankF, sizeof(int) * batch, cudaMemcpyDeviceToHost, q));
    RSVD_CUDA(cudaMemcpyAsync(h->pin.ints + batch, B.sweeps, sizeof(int) * batch,
                              cudaMemcpyDeviceToHost, q));
    RSVD_CUDA(cudaMemcpyAsync(h->pin.dbls, B.dw, sizeof(double) * batch, cudaMemcpyDeviceToHost, q));
  };

  if (host) {
    // Copies in, pipeline, factors out: one graph when the caller's host
    // buffers are page-locked and reused (a pageable buffer fails the capture
    // and the call runs directly).
    auto enqueue_host = [&](cudaStream_t q) {
      // one linear copy per operand when the items are packed (copy_batch)
      copy_batch(B.Ah, m, m * n, A, lda, strideA, m, n, batch, cudaMemcpyHostToDevice, q);
      enqueue(q);
      copy_batch(U, ldu, strideU, B.Uh, m, m * rank, m, rank, batch, cudaMemcpyDeviceToHost, q);
      copy_batch(Vt, ldvt, strideVt, B.Vth, rank, rank * n, rank, n, batch, cudaMemcpyDeviceToHost,
                 q);
      copy_batch(S, rank, strideS, B.Sh, rank, rank, rank, 1, batch, cudaMemcpyDeviceToHost, q);
    };
    if (!h->prof.on && graphs_enabled() && !sharded && all_pinned({A, U, S, Vt})) {
      char keybuf[512];
      std::snprintf(keybuf, sizeof(keybuf),
                    "h|%p|%p|%p|%p|%p|%p|%p|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%d",
                    (const void*)A, (void*)U, (void*)S, (void*)Vt, (void*)h->arena.base,
                    (void*)h->pin.seeds, (void*)h->pin.ints, (long long)m, (long long)n,
                    (long long)lda, (long long)strideA, (long long)batch, (long long)rank,
                    (long long)ell, (long long)ldu, (long long)strideU, (long long)strideS,
                    (long long)ldvt * 1000003LL + strideVt, power);
      run_graph(h, std::string(keybuf), st, enqueue_host);
    } else {
      enqueue_host(st);
      RSVD_CUDA(cudaStreamSynchronize(st));
    }
  } else if (!h->prof.on && graphs_enabled() && (!B.red || B.red->capturable())) {
    // Replay a captured CUDA graph of the whole pipeline (one host launch per
    // call); captured on the handle's own stream and ordered after / before the
    // caller's stream with events.
    char keybuf[512];
    std::snprintf(keybuf, sizeof(keybuf),
                  "%p|%p|%p|%p|%p|%p|%p|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%d|%p|%lld|%lld",
                  (const void*)A, (void*)U, (void*)S, (void*)Vt, (void*)h->arena.base,
                  (void*)h->pin.seeds, (void*)h->pin.ints, (long long)m, (long long)n,
                  (long long)lda, (long long)strideA, (long long)batch, (long long)rank,
                  (long long)ell, (long long)ldu, (long long)strideU, (long long)strideS,
                  (long long)ldvt * 1000003LL + strideVt, power, (void*)B.red,
                  (long long)s.m_global, (long long)s.row_off);
    run_graph(h, std::string(keybuf), st, enqueue);
  } else {
    enqueue(st);
    RSVD_CUDA(cudaStreamSynchronize(st));
  }
  if (h->prof.on) h->prof.collect();
  h->last_sweeps = 0;
  for (int64_t b = 0; b < batch; ++b) {
    out_rank[b] = h->pin.ints[b];
    dw[b] = h->pin.dbls[b];
    h->last_sweeps = std::max(h->last_sweeps, h->pin.ints[batch + b]);
  }
}

// Deterministic truncated SVD, rlftn::tsvd (factorize.cpp:42-50): the full
// thin SVD then truncation with the exact discarded weight.  With Q = I
// (l = min(m, n)) the RSVD's SVD stage is exact: B^T = A_e^T is factored by
// CholeskyQR2 with R and the l x l factor by one-sided Jacobi.  For m > n the
// engine factors A^T and swaps the factors (A = V S U^T).

uint64_t mix64_host(uint64_t z);

void tsvd_impl(rsvd_context* h, int64_t batch, const double* A, int64_t m, int64_t n, int64_t lda,
               int64_t strideA, int64_t chi, double* U, int64_t ldu, int64_t strideU, double* S,
               int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt, int64_t* out_rank,
               double* dw, int flags) {
  check_flags(flags);
  if (m <= 0 || n <= 0) throw InvalidArgument("tsvd: empty matrix");  // :44
  if (chi < 1) throw InvalidArgument("tsvd: rank must be >= 1");      // :45
  if (batch < 0) throw InvalidArgument("tsvd: batch must be >= 0");
  if (batch == 0) return;
  const int64_t p = std::min(m, n), k = std::min(chi, p);
  if (p > kTsvdMaxDim)
    throw InvalidArgument("tsvd: min(m, n) > 16384 is not supported by the GPU path");
  if (!A || !U || !S || !Vt || !out_rank || !dw) throw InvalidArgument("tsvd: null pointer argument");
  if (lda < m || ldu < m || ldvt < k) throw InvalidArgument("tsvd: leading dimension too small");
  const bool host = flags == RSVD_PTR_HOST;
  const bool tr = m > n;
  const int64_t me = tr ? n : m, ne = tr ? m : n;
  RSVD_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  Shape s{me, ne, batch, k, me, round_up(me, 32), 0};
  auto layout = [&](Carver& c, Buffers& B, double*& Ain, double*& Ae, double*& Ue, double*& Ve,
                    double*& Uo, double*& So, double*& Vo) {
    B = carve(c, s, false, true);
    Ain = host ? c.take<double>(batch * m * n) : nullptr;
    Ae = tr ? c.take<double>(batch * me * ne) : nullptr;
    Ue = c.take<double>(batch * me * k);
    Ve = c.take<double>(batch * k * ne);
    Uo = c.take<double>(batch * m * k);
    So = c.take<double>(batch * k);
    Vo = c.take<double>(batch * k * n);
  };
  Buffers B;
  double *Ain, *Ae, *Ue, *Ve, *Uo, *So, *Vo;
  Carver meas{nullptr};
  layout(meas, B, Ain, Ae, Ue, Ve, Uo, So, Vo);
  char* const before = h->arena.base;
  h->arena.reserve(meas.off + 256);
  if (h->arena.base != before) h->drop_graphs();
  Carver cv{h->arena.base};
  layout(cv, B, Ain, Ae, Ue, Ve, Uo, So, Vo);
  if (h->pin.reserve(batch)) h->drop_graphs();
  for (int64_t b = 0; b < batch; ++b) h->pin.seeds[b] = mix64_host(0x7473766400ull + b);  // completion only
  B.prof = &h->prof;
  B.red = nullptr;
  RSVD_CUDA(cudaMemcpyAsync(B.seeds, h->pin.seeds, sizeof(uint64_t) * batch, cudaMemcpyHostToDevice,
                            st));
  CMatRef Ad{A, lda, strideA};
  if (host) {
    copy_batch(Ain, m, m * n, A, lda, strideA, m, n, batch, cudaMemcpyHostToDevice, st);
    Ad = CMatRef{Ain, m, m * n};
  }
  CMatRef Aeff = Ad;
  if (tr) {
    launch_transpose(Ad, m, n, MatRef{Ae, me, me * ne}, batch, st);
    Aeff = CMatRef{Ae, me, me * ne};
  }
  launch_set_identity_rect(MatRef{B.Y, me, me * s.ellp}, me, s.ellp, batch, st);
  svd_stage(s, B, Aeff, MatRef{Ue, me, me * k}, So, k, MatRef{Ve, k, k * ne}, st, true);
  if (!tr) {
    launch_copy_matrix(CMatRef{Ue, me, me * k}, m, k, MatRef{Uo, m, m * k}, batch, st);
    launch_copy_matrix(CMatRef{Ve, k, k * ne}, k, n, MatRef{Vo, k, k * n}, batch, st);
  } else {
    launch_transpose(CMatRef{Ve, k, k * ne}, k, m, MatRef{Uo, m, m * k}, batch, st);  // U = V_e
    launch_transpose(CMatRef{Ue, me, me * k}, n, k, MatRef{Vo, k, k * n}, batch, st);  // Vt = U_e^T
  }
  const cudaMemcpyKind out = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  copy_batch(U, ldu, strideU, Uo, m, m * k, m, k, batch, out, st);
  copy_batch(Vt, ldvt, strideVt, Vo, k, k * n, k, n, batch, out, st);
  copy_batch(S, k, strideS, So, k, k, k, 1, batch, out, st);
  RSVD_CUDA(cudaMemcpyAsync(h->pin.ints, B.rankF, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
  RSVD_CUDA(cudaMemcpyAsync(h->pin.dbls, B.dw, sizeof(double) * batch, cudaMemcpyDeviceToHost, st));
  RSVD_CUDA(cudaStreamSynchronize(st));
  if (h->prof.on) h->prof.collect();
  for (int64_t b = 0; b < batch; ++b) {
    out_rank[b] = h->pin.ints[b];
    dw[b] = h->pin.dbls[b];
  }
}

void range_impl(rsvd_context* h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t ell,
                int power, uint64_t seed, double* Q, int64_t ldq, int flags) {
  check_flags(flags);
  validate_range(m, n, ell, power);
  if (!A || !Q) throw InvalidArgument("randomized_range: null pointer argument");
  if (lda < m || ldq < m) throw InvalidArgument("randomized_range: leading dimension too small");
  const bool host = flags == RSVD_PTR_HOST;
  RSVD_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  Shape s{m, n, 1, ell, ell, round_up(ell, 32), power};
  Carver meas{nullptr};
  carve(meas, s, host, false);
  h->arena.reserve(meas.off + 256);
  Carver cv{h->arena.base};
  Buffers B = carve(cv, s, host, false);
  RSVD_CUDA(cudaMemcpyAsync(B.seeds, &seed, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  CMatRef Ad{A, lda, 0};
  if (host) {
    copy_2d(B.Ah, m, A, lda, m, n, cudaMemcpyHostToDevice, st);
    Ad = CMatRef{B.Ah, m, m * n};
  }
  B.prof = &h->prof;
  range_finder(s, B, Ad, st);
  copy_2d(Q, ldq, B.Y, m, m, ell, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st);
  RSVD_CUDA(cudaStreamSynchronize(st));
  if (h->prof.on) h->prof.collect();
}

void recon_impl(rsvd_context* h, const double* A, int64_t m, int64_t n, int64_t lda,
                const double* U, int64_t ldu, const double* S, const double* Vt, int64_t ldvt,
                int64_t r, double* out, int flags) {
  check_flags(flags);
  if (m <= 0 || n <= 0) throw InvalidArgument("reconstruction_error: empty matrix");
  if (r < 0) throw InvalidArgument("reconstruction_error: rank must be >= 0");
  if (!A || !out || (r > 0 && (!U || !S || !Vt)))
    throw InvalidArgument("reconstruction_error: null pointer argument");
  const bool host = flags == RSVD_PTR_HOST;
  RSVD_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const int64_t rr = std::max<int64_t>(r, 1);
  const int64_t nparts = 4 * num_sms();
  Carver meas{nullptr};
  auto layout = [&](Carver& c, double*& Ad, double*& Us, double*& Vd, double*& Sd, double*& R,
                    double*& part, double*& pg) {
    Ad = c.take<double>(m * n);
    Us = c.take<double>(m * rr);
    Vd = c.take<double>(rr * n);
    Sd = c.take<double>(rr);
    R = c.take<double>(m * n);
    part = c.take<double>(nparts);
    pg = c.take<double>(std::max<int64_t>(dgemm_partial_elems(false, m, n, rr, 1), 1));
  };
  double *Ad, *Us, *Vd, *Sd, *R, *part, *pg;
  layout(meas, Ad, Us, Vd, Sd, R, part, pg);
  h->arena.reserve(meas.off + 256);
  Carver cv{h->arena.base};
  layout(cv, Ad, Us, Vd, Sd, R, part, pg);
  const cudaMemcpyKind kin = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  copy_2d(Ad, m, A, lda, m, n, kin, st);
  if (r > 0) {
    copy_2d(Us, m, U, ldu, m, r, kin, st);
    copy_2d(Vd, r, Vt, ldvt, r, n, kin, st);
    RSVD_CUDA(cudaMemcpyAsync(Sd, S, sizeof(double) * r, kin, st));
    launch_scale_columns(MatRef{Us, m, 0}, m, r, Sd, st);  // U diag(S)
    dgemm(false, m, n, r, CMatRef{Us, m, 0}, CMatRef{Vd, r, 0}, MatRef{R, m, 0}, 1, pg,
          dgemm_partial_elems(false, m, n, rr, 1), st);
  } else {
    RSVD_CUDA(cudaMemsetAsync(R, 0, sizeof(double) * m * n, st));
  }
  launch_residual_sumsq(CMatRef{Ad, m, 0}, CMatRef{R, m, 0}, m, n, part, nparts, st);
  std::vector<double> hp(nparts);
  RSVD_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * nparts, cudaMemcpyDeviceToHost, st));
  RSVD_CUDA(cudaStreamSynchronize(st));
  double sum = 0.0;
  for (double v : hp) sum += v;
  *out = std::sqrt(sum);
}

template <class F>
int guarded(rsvd_context* h, F&& f) {
  if (!h) return RSVD_ERR_INVALID;
  try {
    f();
    h->err.clear();
    return RSVD_OK;
  } catch (const InvalidArgument& e) {
    h->err = e.what();
    return RSVD_ERR_INVALID;
  } catch (const NumericalError& e) {
    h->err = e.what();
    return RSVD_ERR_NUMERICAL;
  } catch (const CudaError& e) {
    h->err = e.what();
    cudaGetLastError();  // a failed launch / attribute call must not poison the next call
    return RSVD_ERR_CUDA;
  } catch (const std::exception& e) {
    h->err = e.what();
    return RSVD_ERR_CUDA;
  }
}

uint64_t mix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Thin QR through the engine's CholeskyQR2 (orth with R accumulation): the
// product-form factor lapack::qr (mps.cpp:265 -> lapack.cpp:180-201).
void qr_impl(rsvd_context* h, int64_t batch, const double* A, int64_t m, int64_t n, int64_t lda,
             int64_t strideA, double* Q, int64_t ldq, int64_t strideQ, double* R, int64_t ldr,
             int64_t strideR, int flags) {
  check_flags(flags);
  if (batch < 0) throw InvalidArgument("qr: batch must be >= 0");
  if (batch == 0) return;
  if (m <= 0 || n <= 0) throw InvalidArgument("lapack::qr: empty matrix");  // lapack.cpp:184
  if (m < n) throw InvalidArgument("qr: need m >= n (thin QR of a tall matrix)");
  if (!A || !Q || !R) throw InvalidArgument("qr: null pointer argument");
  if (lda < m || ldq < m || ldr < n) throw InvalidArgument("qr: leading dimension too small");
  if (n > kTsvdMaxDim) throw InvalidArgument("qr: n > 16384 is not supported by the GPU path");
  const bool host = flags == RSVD_PTR_HOST;
  RSVD_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  Shape s{m, 1, batch, 1, n, round_up(n, 32), 0};
  Carver meas{nullptr};
  carve(meas, s, false, true);
  h->arena.reserve(meas.off + 256);
  Carver cv{h->arena.base};
  Buffers B = carve(cv, s, false, true);
  B.prof = &h->prof;
  B.red = nullptr;
  if (h->pin.reserve(batch)) h->drop_graphs();
  for (int64_t b = 0; b < batch; ++b) h->pin.seeds[b] = mix64_host(0x7172000000ull + b);  // completion
  RSVD_CUDA(cudaMemcpyAsync(B.seeds, h->pin.seeds, sizeof(uint64_t) * batch, cudaMemcpyHostToDevice,
                            st));
  const int64_t lp = s.ellp;
  const cudaMemcpyKind in = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const cudaMemcpyKind out = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  copy_batch(B.Y, m, m * lp, A, lda, strideA, m, n, batch, in, st);
  if (lp > n)
    RSVD_CUDA(cudaMemset2DAsync(B.Y + m * n, sizeof(double) * m * lp, 0, sizeof(double) * m * (lp - n),
                                batch, st));
  double *Yb = B.Y, *Tmp = B.Y2;
  orth(s, B, Yb, Tmp, m, B.Rt, kCompletionTag + 0x2000, 2, true, st);
  copy_batch(Q, ldq, strideQ, Yb, m, m * lp, m, n, batch, out, st);
  copy_batch(R, ldr, strideR, B.Rt, lp, lp * lp, n, n, batch, out, st);
  if (host) RSVD_CUDA(cudaStreamSynchronize(st));
}

// Copy host job tables into the handle's table arena (stream-ordered).
template <class... P>
void upload_tables(rsvd_context* h, cudaStream_t st, P&... parts) {
  size_t total = 0;
  auto sz = [&](auto& p) { total = (total + 255) & ~size_t(255); total += p.bytes; };
  (sz(parts), ...);
  if (total > h->tab.cap) {
    RSVD_CUDA(cudaStreamSynchronize(st));
    h->tab.reserve(std::max<size_t>(total, 1 << 16));
  }
  size_t off = 0;
  auto put = [&](auto& p) {
    off = (off + 255) & ~size_t(255);
    p.dev = h->tab.base + off;
    if (p.bytes) RSVD_CUDA(cudaMemcpyAsync(p.dev, p.host, p.bytes, cudaMemcpyHostToDevice, st));
    off += p.bytes;
  };
  (put(parts), ...);
}

struct TablePart {
  const void* host;
  size_t bytes;
  char* dev = nullptr;
};

#include "zpath.inc"
#include "blocks.inc"

}  // namespace
}  // namespace rsvd

#pragma GCC visibility push(default)
extern "C" {

const char* rsvd_version(void) { return "rsvd_b200 0.1.0 (sm_100a, FP64 DMMA)"; }

uint64_t rsvd_mix64(uint64_t z) { return rsvd::mix64_host(z); }
uint64_t rsvd_derive_seed(uint64_t seed, uint64_t tag) { return seed ^ rsvd::mix64_host(tag); }

int rsvd_create(rsvd_handle* out, int device) {
  if (!out) return RSVD_ERR_INVALID;
  *out = nullptr;
  auto* h = new rsvd_context();
  h->device = device;
  const int rc = rsvd::guarded(h, [&] {
    int count = 0;
    RSVD_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw rsvd::InvalidArgument("rsvd_create: bad device index");
    RSVD_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    RSVD_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw rsvd::CudaError("rsvd_create: this build targets sm_100a (B200); device is sm_" +
                            std::to_string(prop.major * 10 + prop.minor));
    RSVD_CUDA(cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking));
    RSVD_CUDA(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
    RSVD_CUDA(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
    h->stream = h->own;
  });
  if (rc != RSVD_OK) {
    // Keep the handle so the caller can read the message, then destroy it.
    *out = h;
    return rc;
  }
  *out = h;
  return RSVD_OK;
}

uint64_t rsvd_kernel_launches(void) { return rsvd::g_kernel_launches.load(); }

int rsvd_profile_enable(rsvd_handle h, int on) {
  return rsvd::guarded(h, [&] {
    h->prof.on = on != 0;
    h->prof.reset();
  });
}

int rsvd_profile_read(rsvd_handle h, double* ms, int64_t* calls, int n) {
  if (!h) return -1;
  const int k = std::min<int>(n, rsvd::kNumStages);
  for (int i = 0; i < k; ++i) {
    if (ms) ms[i] = h->prof.ms[i];
    if (calls) calls[i] = h->prof.calls[i];
  }
  return rsvd::kNumStages;
}

const char* rsvd_profile_stage_name(int i) {
  return (i >= 0 && i < rsvd::kNumStages) ? rsvd::kStageNames[i] : "";
}

int rsvd_last_jacobi_sweeps(rsvd_handle h) { return h ? h->last_sweeps : -1; }
int rsvd_last_gemm_path(rsvd_handle h) { return h ? h->last_gemm_path : -1; }

int rsvd_destroy(rsvd_handle h) {
  if (!h) return RSVD_ERR_INVALID;
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->prof.destroy();
  h->drop_graphs();
  h->destroy_pipeline();
  h->pin.release();
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  h->arena.release();
  h->tab.release();
  h->blk.release();
  if (h->own) cudaStreamDestroy(h->own);
  delete h;
  return RSVD_OK;
}

const char* rsvd_last_error(rsvd_handle h) { return h ? h->err.c_str() : "null handle"; }

int rsvd_set_stream(rsvd_handle h, void* stream) {
  // Does not touch the last-error string: callers restore the stream after a
  // failed call and still read its message.
  if (!h) return RSVD_ERR_INVALID;
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own;
  return RSVD_OK;
}

int rsvd_trim(rsvd_handle h) {
  return rsvd::guarded(h, [&] {
    RSVD_CUDA(cudaStreamSynchronize(h->stream));
    h->drop_graphs();
    h->arena.release();
    h->tab.release();
    h->blk.release();
  });
}

int rsvd_fill_gaussian_f64(rsvd_handle h, uint64_t seed, double* out, int64_t count, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::check_flags(flags);
    if (count < 0) throw rsvd::InvalidArgument("fill_gaussian: count must be >= 0");
    if (count == 0) return;
    if (!out) throw rsvd::InvalidArgument("fill_gaussian: null pointer argument");
    RSVD_CUDA(cudaSetDevice(h->device));
    double* dst = out;
    if (flags == RSVD_PTR_HOST) {
      h->arena.reserve(sizeof(double) * count + 256);
      dst = reinterpret_cast<double*>(h->arena.base);
    }
    rsvd::launch_fill_gaussian_flat(dst, count, seed, h->stream);
    if (flags == RSVD_PTR_HOST)
      RSVD_CUDA(cudaMemcpyAsync(out, dst, sizeof(double) * count, cudaMemcpyDeviceToHost,
                                h->stream));
    RSVD_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int rsvd_f64(rsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t rank,
             int64_t oversample, int power, uint64_t seed, double* U, int64_t ldu, double* S,
             double* Vt, int64_t ldvt, int64_t* out_rank, double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::rsvd_batched_impl(h, 1, A, m, n, lda, 0, rank, oversample, power, &seed, U, ldu, 0, S,
                            0, Vt, ldvt, 0, out_rank, discarded_weight, flags);
  });
}

int rsvd_f64_batched(rsvd_handle h, int64_t batch, const double* A, int64_t m, int64_t n,
                     int64_t lda, int64_t strideA, int64_t rank, int64_t oversample, int power,
                     const uint64_t* seeds, double* U, int64_t ldu, int64_t strideU, double* S,
                     int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt,
                     int64_t* out_rank, double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::rsvd_batched_impl(h, batch, A, m, n, lda, strideA, rank, oversample, power, seeds, U,
                            ldu, strideU, S, strideS, Vt, ldvt, strideVt, out_rank,
                            discarded_weight, flags);
  });
}

int rsvd_group_create(rsvd_group* g, int nranks) {
  if (!g) return RSVD_ERR_INVALID;
  try {
    *g = reinterpret_cast<rsvd_group>(rsvd::group_create(nranks));
    return RSVD_OK;
  } catch (...) {
    *g = nullptr;
    return RSVD_ERR_INVALID;
  }
}

int rsvd_group_destroy(rsvd_group g) {
  rsvd::group_destroy(reinterpret_cast<rsvd::Group*>(g));
  return RSVD_OK;
}

int rsvd_attach_group(rsvd_handle h, rsvd_group g, int rank) {
  return rsvd::guarded(h, [&] {
    h->drop_graphs();
    h->red = rsvd::make_group_reducer(reinterpret_cast<rsvd::Group*>(g), rank);
  });
}

int rsvd_nccl_unique_id(unsigned char* id128) {
  if (!id128) return RSVD_ERR_INVALID;
  try {
    rsvd::nccl_unique_id(id128);
    return RSVD_OK;
  } catch (...) {
    return RSVD_ERR_CUDA;
  }
}

int rsvd_attach_nccl(rsvd_handle h, int nranks, int rank, const unsigned char* id128) {
  return rsvd::guarded(h, [&] {
    if (!id128 || nranks < 1 || rank < 0 || rank >= nranks)
      throw rsvd::InvalidArgument("rsvd_attach_nccl: bad arguments");
    RSVD_CUDA(cudaSetDevice(h->device));
    h->drop_graphs();
    h->red = rsvd::make_nccl_reducer(nranks, rank, id128);
  });
}

int rsvd_detach(rsvd_handle h) {
  return rsvd::guarded(h, [&] {
    h->drop_graphs();
    h->red.reset();
  });
}

int rsvd_f64_rowsharded(rsvd_handle h, const double* A_local, int64_t m_local, int64_t n,
                        int64_t lda, int64_t m_global, int64_t row_offset, int64_t rank,
                        int64_t oversample, int power, uint64_t seed, double* U_local, int64_t ldu,
                        double* S, double* Vt, int64_t ldvt, int64_t* out_rank,
                        double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::rsvd_batched_impl(h, 1, A_local, m_local, n, lda, 0, rank, oversample, power, &seed,
                            U_local, ldu, 0, S, 0, Vt, ldvt, 0, out_rank, discarded_weight, flags,
                            m_global, row_offset, true);
  });
}

int rsvd_tsvd_f64(rsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t chi,
                  double* U, int64_t ldu, double* S, double* Vt, int64_t ldvt, int64_t* out_rank,
                  double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::tsvd_impl(h, 1, A, m, n, lda, 0, chi, U, ldu, 0, S, 0, Vt, ldvt, 0, out_rank,
                    discarded_weight, flags);
  });
}

int rsvd_tsvd_f64_batched(rsvd_handle h, int64_t batch, const double* A, int64_t m, int64_t n,
                          int64_t lda, int64_t strideA, int64_t chi, double* U, int64_t ldu,
                          int64_t strideU, double* S, int64_t strideS, double* Vt, int64_t ldvt,
                          int64_t strideVt, int64_t* out_rank, double* discarded_weight,
                          int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::tsvd_impl(h, batch, A, m, n, lda, strideA, chi, U, ldu, strideU, S, strideS, Vt, ldvt,
                    strideVt, out_rank, discarded_weight, flags);
  });
}

int rsvd_randomized_range_f64(rsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                              int64_t ell, int power, uint64_t seed, double* Q, int64_t ldq,
                              int flags) {
  return rsvd::guarded(h, [&] { rsvd::range_impl(h, A, m, n, lda, ell, power, seed, Q, ldq, flags); });
}

int rsvd_validate_params(int64_t m, int64_t n, int64_t rank, int64_t oversample, int power,
                         int64_t* ell_out, char* msg, int64_t msg_len) {
  try {
    int64_t ell = 0;
    rsvd::validate_rsvd(m, n, rank, oversample, power, ell);
    if (ell_out) *ell_out = ell;
    if (msg && msg_len > 0) msg[0] = 0;
    return RSVD_OK;
  } catch (const std::exception& e) {
    if (msg && msg_len > 0) {
      std::strncpy(msg, e.what(), static_cast<size_t>(msg_len - 1));
      msg[msg_len - 1] = 0;
    }
    return RSVD_ERR_INVALID;
  }
}

int rsvd_testing_dgemm(rsvd_handle h, int trans_a, int64_t M, int64_t N, int64_t K,
                       const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                       int64_t strideB, double* C, int64_t ldc, int64_t strideC, int64_t batch) {
  return rsvd::guarded(h, [&] {
    RSVD_CUDA(cudaSetDevice(h->device));
    const int64_t need = rsvd::dgemm_partial_elems(trans_a != 0, M, N, K, batch);
    h->arena.reserve(sizeof(double) * std::max<int64_t>(need, 1) + 256);
    rsvd::dgemm(trans_a != 0, M, N, K, rsvd::CMatRef{A, lda, strideA},
                rsvd::CMatRef{B, ldb, strideB}, rsvd::MatRef{C, ldc, strideC}, batch,
                reinterpret_cast<double*>(h->arena.base), need, h->stream);
    RSVD_CUDA(cudaStreamSynchronize(h->stream));
  });
}

#ifdef RSVD_OZ_TRACE
int rsvd_testing_oz_trace_read(unsigned long long* out, int64_t n) {
  cudaDeviceSynchronize();
  rsvd::oz_trace_read(out, n);
  return 0;
}
#endif

int rsvd_testing_ozaki_gemm(rsvd_handle h, int trans_a, int64_t M, int64_t N, int64_t K,
                            const double* A, int64_t lda, int64_t strideA, const double* B,
                            int64_t ldb, int64_t strideB, double* C, int64_t ldc, int64_t strideC,
                            int64_t batch) {
  return rsvd::guarded(h, [&] {
    RSVD_CUDA(cudaSetDevice(h->device));
    if (!rsvd::oz_supported(M, N, K) || batch < 1)
      throw rsvd::InvalidArgument("ozaki_gemm: M, N, K must be multiples of 16, K <= 65536");
    // stored A: M x K (NN) or K x M (TN)
    const int64_t rows = trans_a ? K : M, cols = trans_a ? M : K;
    const int64_t sa = rsvd::oz_slice_bytes(rows, cols, batch), sb = rsvd::oz_slice_bytes(K, N, batch);
    const int64_t ints = (rows + cols + N) * batch;
    const size_t bytes = 2 * sa + sb + sizeof(int) * ints + 1024;
    h->arena.reserve(bytes);
    char* base = reinterpret_cast<char*>(h->arena.base);
    int8_t* sR = reinterpret_cast<int8_t*>(base);
    int8_t* sC = sR + sa;
    int8_t* sB = sC + sa;
    int* eRow = reinterpret_cast<int*>(base + ((2 * sa + sb + 255) / 256) * 256);
    int* eCol = eRow + rows * batch;
    int* eB = eCol + cols * batch;
    rsvd::oz_prepare_a(rsvd::CMatRef{A, lda, strideA}, rows, cols, batch, sR, sC, eRow, eCol,
                       h->stream);
    rsvd::oz_slice_b(rsvd::CMatRef{B, ldb, strideB}, K, N, batch, sB, eB, h->stream);
    rsvd::oz_gemm(M, N, K, trans_a ? sC : sR, trans_a ? eCol : eRow, sB, eB,
                  rsvd::MatRef{C, ldc, strideC}, batch, h->stream);
    RSVD_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int rsvd_reconstruction_error_f64(rsvd_handle h, const double* A, int64_t m, int64_t n,
                                  int64_t lda, const double* U, int64_t ldu, const double* S,
                                  const double* Vt, int64_t ldvt, int64_t r, double* out,
                                  int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::recon_impl(h, A, m, n, lda, U, ldu, S, Vt, ldvt, r, out, flags);
  });
}

// ---- complex instantiation (rlftn::rsvd<std::complex<double>> etc.) ----

int rsvd_fill_gaussian_z128(rsvd_handle h, uint64_t seed, double* out, int64_t count, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::check_flags(flags);
    if (count < 0) throw rsvd::InvalidArgument("fill_gaussian: count must be >= 0");
    if (count == 0) return;
    if (!out) throw rsvd::InvalidArgument("fill_gaussian: null pointer argument");
    RSVD_CUDA(cudaSetDevice(h->device));
    double* dst = out;
    if (flags == RSVD_PTR_HOST) {
      h->arena.reserve(sizeof(double) * 2 * count + 256);
      dst = reinterpret_cast<double*>(h->arena.base);
    }
    rsvd::launch_zfill_gaussian_flat(dst, count, seed, h->stream);
    if (flags == RSVD_PTR_HOST)
      RSVD_CUDA(cudaMemcpyAsync(out, dst, sizeof(double) * 2 * count, cudaMemcpyDeviceToHost,
                                h->stream));
    RSVD_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int rsvd_z128(rsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t rank,
              int64_t oversample, int power, uint64_t seed, double* U, int64_t ldu, double* S,
              double* Vt, int64_t ldvt, int64_t* out_rank, double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::zrsvd_batched_impl(h, 1, A, m, n, lda, 0, rank, oversample, power, &seed, U, ldu, 0, S,
                             0, Vt, ldvt, 0, out_rank, discarded_weight, flags);
  });
}

int rsvd_z128_batched(rsvd_handle h, int64_t batch, const double* A, int64_t m, int64_t n,
                      int64_t lda, int64_t strideA, int64_t rank, int64_t oversample, int power,
                      const uint64_t* seeds, double* U, int64_t ldu, int64_t strideU, double* S,
                      int64_t strideS, double* Vt, int64_t ldvt, int64_t strideVt,
                      int64_t* out_rank, double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::zrsvd_batched_impl(h, batch, A, m, n, lda, strideA, rank, oversample, power, seeds, U,
                             ldu, strideU, S, strideS, Vt, ldvt, strideVt, out_rank,
                             discarded_weight, flags);
  });
}

int rsvd_tsvd_z128(rsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t chi,
                   double* U, int64_t ldu, double* S, double* Vt, int64_t ldvt, int64_t* out_rank,
                   double* discarded_weight, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::ztsvd_impl(h, 1, A, m, n, lda, 0, chi, U, ldu, 0, S, 0, Vt, ldvt, 0, out_rank,
                     discarded_weight, flags);
  });
}

int rsvd_tsvd_z128_batched(rsvd_handle h, int64_t batch, const double* A, int64_t m, int64_t n,
                           int64_t lda, int64_t strideA, int64_t chi, double* U, int64_t ldu,
                           int64_t strideU, double* S, int64_t strideS, double* Vt, int64_t ldvt,
                           int64_t strideVt, int64_t* out_rank, double* discarded_weight,
                           int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::ztsvd_impl(h, batch, A, m, n, lda, strideA, chi, U, ldu, strideU, S, strideS, Vt, ldvt,
                     strideVt, out_rank, discarded_weight, flags);
  });
}

int rsvd_randomized_range_z128(rsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                               int64_t ell, int power, uint64_t seed, double* Q, int64_t ldq,
                               int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::zrange_impl(h, A, m, n, lda, ell, power, seed, Q, ldq, flags);
  });
}

int rsvd_reconstruction_error_z128(rsvd_handle h, const double* A, int64_t m, int64_t n,
                                   int64_t lda, const double* U, int64_t ldu, const double* S,
                                   const double* Vt, int64_t ldvt, int64_t r, double* out,
                                   int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::zrecon_impl(h, A, m, n, lda, U, ldu, S, Vt, ldvt, r, out, flags);
  });
}

int rsvd_block_factorize_f64(rsvd_handle h, int64_t nsectors, const int64_t* charges,
                             const double* const* blocks, const int64_t* rows, const int64_t* cols,
                             const int64_t* ld, int64_t chi, int policy, int64_t slack, int kind,
                             int64_t oversample, int power, uint64_t seed, int64_t rsvd_min_dim,
                             double* const* U, const int64_t* ldu, double* const* S,
                             double* const* Vt, const int64_t* ldvt, int64_t* out_rank,
                             double* sector_dw, double* total_dw, int* exact, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::block_factorize_impl(h, nsectors, charges, blocks, rows, cols, ld, chi, policy, slack,
                               kind, oversample, power, seed, rsvd_min_dim, U, ldu, S, Vt, ldvt,
                               out_rank, sector_dw, total_dw, exact, flags);
  });
}

int rsvd_qr_f64(rsvd_handle h, int64_t batch, const double* A, int64_t m, int64_t n, int64_t lda,
                int64_t strideA, double* Q, int64_t ldq, int64_t strideQ, double* R, int64_t ldr,
                int64_t strideR, int flags) {
  return rsvd::guarded(h, [&] {
    rsvd::qr_impl(h, batch, A, m, n, lda, strideA, Q, ldq, strideQ, R, ldr, strideR, flags);
  });
}

int rsvd_combine_blocks(rsvd_handle h, int complex_, int64_t njobs, const rsvd_block_job* jobs,
                        int64_t nterms, const rsvd_block_term* terms) {
  return rsvd::guarded(h, [&] {
    if (njobs < 0 || nterms < 0) throw rsvd::InvalidArgument("combine_blocks: negative table size");
    if (njobs == 0) return;
    if (!jobs || (nterms > 0 && !terms)) throw rsvd::InvalidArgument("combine_blocks: null table");
    std::vector<int64_t> start(static_cast<size_t>(njobs) + 1, 0);
    for (int64_t j = 0; j < njobs; ++j) {
      const rsvd_block_job& jb = jobs[j];
      if (jb.rows < 0 || jb.cols < 0 || jb.term_begin < 0 || jb.term_count < 0 ||
          jb.term_begin + jb.term_count > nterms || (jb.rows * jb.cols > 0 && !jb.dst))
        throw rsvd::InvalidArgument("combine_blocks: malformed job");
      start[j + 1] = start[j] + jb.rows * jb.cols;
    }
    RSVD_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = h->stream;
    rsvd::TablePart pj{jobs, sizeof(rsvd_block_job) * njobs}, pt{terms, sizeof(rsvd_block_term) * nterms},
        ps{start.data(), sizeof(int64_t) * (njobs + 1)};
    rsvd::upload_tables(h, st, pj, pt, ps);
    rsvd::launch_combine_blocks(complex_ != 0, reinterpret_cast<const rsvd_block_job*>(pj.dev),
                                reinterpret_cast<const rsvd_block_term*>(pt.dev),
                                reinterpret_cast<const int64_t*>(ps.dev), njobs, start[njobs], st);
  });
}

int rsvd_grouped_gemm(rsvd_handle h, int complex_, int64_t njobs, const rsvd_gemm_job* jobs) {
  return rsvd::guarded(h, [&] {
    if (njobs < 0) throw rsvd::InvalidArgument("grouped_gemm: negative table size");
    if (njobs == 0) return;
    if (!jobs) throw rsvd::InvalidArgument("grouped_gemm: null table");
    std::vector<int4> tiles;
    for (int64_t j = 0; j < njobs; ++j) {
      const rsvd_gemm_job& jb = jobs[j];
      if (jb.M < 0 || jb.N < 0 || jb.K < 0) throw rsvd::InvalidArgument("grouped_gemm: negative size");
      if (jb.M == 0 || jb.N == 0) continue;
      if (!jb.C || (jb.K > 0 && (!jb.A || !jb.B))) throw rsvd::InvalidArgument("grouped_gemm: null operand");
      const int64_t tm = rsvd::grouped_gemm_tile(jb.M), tn = rsvd::grouped_gemm_tile(jb.N);
      for (int64_t a = 0; a < tm; ++a)
        for (int64_t b = 0; b < tn; ++b)
          tiles.push_back(make_int4(static_cast<int>(j), static_cast<int>(a), static_cast<int>(b), 0));
    }
    if (tiles.empty()) return;
    RSVD_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = h->stream;
    rsvd::TablePart pj{jobs, sizeof(rsvd_gemm_job) * njobs}, pt{tiles.data(), sizeof(int4) * tiles.size()};
    rsvd::upload_tables(h, st, pj, pt);
    rsvd::launch_grouped_gemm(complex_ != 0, reinterpret_cast<const rsvd_gemm_job*>(pj.dev),
                              reinterpret_cast<const int4*>(pt.dev), static_cast<int64_t>(tiles.size()), st);
  });
}

int rsvd_block_sqnorms(rsvd_handle h, int complex_, int64_t nslots, const int64_t* slot_begin,
                       const rsvd_block_job* blocks, double* out) {
  return rsvd::guarded(h, [&] {
    if (nslots < 0) throw rsvd::InvalidArgument("block_sqnorms: negative slot count");
    if (nslots == 0) return;
    if (!slot_begin || !out) throw rsvd::InvalidArgument("block_sqnorms: null argument");
    const int64_t nb = slot_begin[nslots];
    if (slot_begin[0] != 0 || nb < 0 || (nb > 0 && !blocks))
      throw rsvd::InvalidArgument("block_sqnorms: malformed slot table");
    for (int64_t s2 = 0; s2 < nslots; ++s2)
      if (slot_begin[s2 + 1] < slot_begin[s2]) throw rsvd::InvalidArgument("block_sqnorms: malformed slot table");
    RSVD_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = h->stream;
    rsvd::TablePart pb{blocks, sizeof(rsvd_block_job) * nb},
        ps{slot_begin, sizeof(int64_t) * (nslots + 1)};
    rsvd::upload_tables(h, st, pb, ps);
    rsvd::launch_block_sqnorms(complex_ != 0, reinterpret_cast<const rsvd_block_job*>(pb.dev),
                               reinterpret_cast<const int64_t*>(ps.dev), nslots, out, st);
  });
}

}  // extern "C"
#pragma GCC visibility pop
