// Kernel parameter blocks and launch entry points shared by the library's .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace rsfde {

// Kernel attributes (dynamic shared memory opt-in) and the SM count are per device: run `init`
// once per (call site, device).  `Tag` makes every call site (template instantiation) its own cache.
constexpr int kMaxDevices = 64;
template <class Tag, class F>
inline int per_device_once(F init) {
  static std::once_flag flags[kMaxDevices];
  static int result[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
  std::call_once(flags[dev], [&] { result[dev] = init(dev); });
  return result[dev];
}

// SM count of the current device (B200: 148) and the block count of the streaming kernels
// (8 resident 256-thread blocks per SM)
inline int device_sm_count() {
  struct Tag {};
  const int n = per_device_once<Tag>([](int dev) -> int {
    int v = 0;
    return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0 ? v : 148;
  });
  return n > 0 ? n : 148;
}
inline int stream_blocks() { return 8 * device_sm_count(); }

// Grid geometry of the internal layout: C order [x1][x2][x3] (x_d fastest), the last
// dimension padded to P = n_d + 1 with a zero pad element (private layout).
struct Geom {
  int d;
  int n[3];      // interior sizes (unused axes = 1)
  int P;         // padded last dimension
  long long NP;  // total padded length = prod_{i<d-1} n_i * P
};

// e(x, t_{m+1/2}) evaluated on the fly
struct ECoef {
  int kind;                  // 0: none (X = 0), 1: separable, 2: dense device grid
  double a, b;               // a(t_{m+1/2}), b(t_{m+1/2})
  const double* g[3];        // device, length n_i, or null (= 1)
  const double* k[3];        // device, length n_i, or null (= 0)
  const double* grid;        // kind 2: dense layout [x1][x2][x3], N values
  const double* ab;          // device {a, b} overriding a, b when non-null (graph-captured steps: the
                             // time level is written there before each replay)
};
__device__ __forceinline__ double2 e_ab(const ECoef& e) {
  return e.ab ? make_double2(__ldg(e.ab), __ldg(e.ab + 1)) : make_double2(e.a, e.b);
}

// the last-axis pass divides by Lambda(k):
//   PHAT: Lambda_P Lambda_H      PALPHA: Lambda_P        PALPHA_SQRT: Lambda_P^{1/2}
//   HINV: Lambda_H               PALPHA_RSQRT: Lambda_P^{-1/2} (i.e. multiplies by Lambda_P^{1/2})
//   HP_SQRT: Lambda_H Lambda_P^{1/2} (P_alpha^{-1/2} H^{-1}, the two-sided left factor)
enum SpecKind { SPEC_PHAT = 0, SPEC_PALPHA = 1, SPEC_PALPHA_SQRT = 2, SPEC_HINV = 3, SPEC_PALPHA_RSQRT = 4,
                SPEC_HP_SQRT = 5 };

// spectrum tables for the preconditioner scaling on the last axis
struct Spec {
  int kind;
  double ebar;
  double eta[3];
  const double* q[3];     // tau eigenvalues q_i(k), k = 1..n_i (device)
  const double* lamH[3];  // H eigenvalues (device)
  const double* tq[3];    // eta_i q_i(k) / lambda^H_i(k) (device)
};

// first-axis source of the "X" channel of an operator pass
enum XMode { X_INPUT = 0, X_E_TIMES_R = 1, X_ZERO = 2 };

// on-chip 1-D march (onchip_1d.cu): every CN step and GMRES solve in one CTA
struct OnchipParams {
  int n, restart, max_iters, m_begin, m_count;
  double tol, alpha, eta, tau, ebar;
  const double *s, *lamH, *q;          // FCD generator s_k, lambda^H_k, tau eigenvalues q_k (device, n)
  const double *a_half, *b_half;       // e = a(t) + b(t) g(x) + k(x) at the half levels (device, M)
  const double *g, *kk;                // axis factors (device, n) or null
  const double* F;                     // device, m_count vectors of n (F_stride = n) or one (F_stride = 0); may be null
  long long F_stride;
  double* X;                           // u^(m_begin) in, u^(m_begin+m_count) out (device, n)
  int* iters;                          // per-step outputs (device, m_count)
  double* relres;
  unsigned char* conv;
};
size_t onchip_smem_bytes(int n, int restart);
cudaError_t launch_onchip_1d(const OnchipParams& p, cudaStream_t s);
// one CTA per system: d_params = device array of count parameter blocks; smem = max over the systems
cudaError_t launch_onchip_1d_batch(const OnchipParams* d_params, int count, size_t smem, cudaStream_t s);

struct PassParams {
  Geom geo;
  int axis;              // 0-based
  int n, N, L;           // axis length, N = n+1, L = 2N
  long long stride;      // element stride along the axis
  long long inner;       // strided axes: pencils per outer index (= stride)
  long long npairs;      // number of pencil pairs
  int contiguous;        // axis == d-1
  // vectors
  const double* X;
  const double* R;
  const double* B;       // additive vector (physical last pass)
  double* Y;
  double* C;
  const double* rscale;  // device scalar multiplying R (lazy basis normalisation) or null
  int xmode;
  // coefficients
  double hc0, hc1;       // H stencil: 1 - alpha/12, alpha/24
  double eta;            // T coefficient (eta_i times sign / factor)
  double ycoef, bcoef;   // physical last pass: Y = ycoef*y + bcoef*B
  double dst_scale;      // sqrt(2/N)
  ECoef e;
  Spec spec;
  // per-axis tables (device)
  const double* chat;    // circulant spectrum / L, length L
  const double2* tw;     // W_L^k, length L, followed by the seeds W_L^{8k}, length L
  const double* lamH;    // H eigenvalues of this axis (length n)
  // row-layout copies for the L = 4096 three-stage form Lay3<16, 16> (null otherwise): entry r G + t holds
  // chat[k], lamH[k - 1], tq[k - 1] at k = rowk(t, r) (0 where k = 0 or k > n), so that the lanes of a warp
  // read consecutive addresses instead of one 128-byte line each
  const double *chat_rl, *lamH_rl, *tq_rl;
  int flags;             // PASS_FLAG_*
  // global coordinates of this (possibly sharded / transposed) grid: axis i of the local array
  // starts at global index coff[i] of a physical axis with cext[i] interior points; pencils whose
  // global coordinate on a non-pass axis is >= cext are zero pads (never stored)
  // Segmented contiguous axis (slab-sharded teams, rsfde_shard.cu): with seg_lg > 0 the pencils are the
  // all-to-all blocks [r][row][x_l] (x = r 2^seg_lg + x_l, row = pencil): element (pencil, position j) at
  // (x >> seg_lg) seg_stride + pencil 2^seg_lg + (x & (2^seg_lg - 1)), x = j - 1, for every vector of the
  // pass (the last pass reads the receive buffers and writes the send buffer of the next exchange).
  int seg_lg;
  long long seg_stride;
  int coff[3];
  int cext[3];
  // speculative Arnoldi launches: when non-null and skip[0] | skip[1] (the GmresState converged /
  // breakdown flags) is set, the kernel returns at once (see gmres_core in rsfde_host.cu)
  const int* skip;
};
__device__ __forceinline__ bool skip_launch(const int* skip) {
  return skip && ((*(volatile const int*)skip) | (*((volatile const int*)skip + 1)));
}
enum { PASS_FLAG_NO_PIPE = 1 };

// host-side launchers (pass_kernels.cu)
// idx[r G + t] = rowk(t, r) of Lay3<16, 16> (4096 entries): the index map of the row-layout tables
void row_layout_4096(int* idx);
cudaError_t launch_oper_pass(const PassParams& p, bool spectral, bool last, cudaStream_t s);
cudaError_t launch_dst_pass(const PassParams& p, bool last, cudaStream_t s);

// krylov_kernels.cu
struct KrylovDims {
  long long NP;
  int nblk;  // blocks used by the streaming reductions
};
cudaError_t launch_pack(const double* dense, double* padded, const Geom& g, cudaStream_t s);
cudaError_t launch_unpack(const double* padded, double* dense, const Geom& g, cudaStream_t s);
// partial[b*J + i] = sum over block b's elements of (s_i V_i) . z
cudaError_t launch_dots(const double* const* V, const double* vscale, int J, const double* z,
                        double* partial, long long NP, int nblk, cudaStream_t s);
// partial[b*J+i] = sum (s_i V_i) . (z - sum_l c_l s_l V_l), c read from device array coef
cudaError_t launch_dots_after_update(const double* const* V, const double* vscale, int J, const double* z,
                                     const double* coef, double* partial, long long NP, int nblk,
                                     cudaStream_t s);
// out = z - sum_l (c1_l + c2_l) s_l V_l ; partial[b] = ||out||^2 over block b
cudaError_t launch_update_norm(const double* const* V, const double* vscale, int J, const double* z,
                               const double* c1, const double* c2, double* out, double* partial,
                               long long NP, int nblk, cudaStream_t s);
// x += sum_l y_l s_l V_l
cudaError_t launch_axpy_basis(const double* const* V, const double* vscale, int J, const double* y,
                              double* x, long long NP, cudaStream_t s);
// out[i] = sum_b partial[b*J + i] (fixed order), one small block
cudaError_t launch_reduce(const double* partial, int nblk, int J, double* out, cudaStream_t s);
// norm of a vector: partial sums of squares
cudaError_t launch_sumsq(const double* z, double* partial, long long NP, int nblk, cudaStream_t s);
// y = a*x + b*y
cudaError_t launch_axpby(double a, const double* x, double b, double* y, long long NP, cudaStream_t s);
// F = prod_l calH_l f on the closed grid (dense layouts)
cudaError_t launch_compact_source(const double* f_closed, double* F, const Geom& g, const double* alpha,
                                  cudaStream_t s);
// e-hat / e-check reduction over interior grid x M half levels
cudaError_t launch_emaxmin(const ECoef& e, const double* a_half, const double* b_half, int M, int grid_static,
                           const Geom& geo, double* partial, int nblk, cudaStream_t s);

// conditional handle of a graph-captured GMRES cycle (rsfde_host.cu graph_build): h_cont gates the next
// Arnoldi step (its IF node); the kernel that sets it lives in the graph that owns the handle
struct GraphCond {
  unsigned long long h_cont = 0;
  int on = 0;
};

// GMRES control state on the device (one solve)
struct GmresState {
  // small fields first: the host reads back the first 24 bytes after every iteration
  int converged;
  int breakdown;
  double relres;
  double beta0;
  double H[52 * 51];    // rotated Hessenberg R, column-major (ld = 52)
  double cs[51], sn[51];
  double g[52];
  double y[51];
  double hsum[52];      // h1 + h2 of the current column
  // DCGS2 (delayed re-orthogonalisation): the unrotated Hessenberg matrix (column j tentative until
  // the next iteration corrects it), g before the tentative rotation of each column, the update
  // coefficients of the current iteration and the Pythagorean norm nu of the re-orthogonalised vector
  double Hraw[52 * 51];
  double gsave[52];
  double cq[52], cu[52];
  double nu;
  int kcols;            // columns usable by the y solve (j+1, or j after a breakdown in the correction)
  int steps;            // graph-captured cycle: Arnoldi steps executed (set by gmres_init / dcgs_finish_b)
};
// number of blocks (= partial sums) every streaming reduction uses for a vector of length NP
int reduction_blocks(long long NP, int nblk);
// reduce the norm partials, fill Hessenberg column j with h1 + h2, rotate, test convergence.
cudaError_t launch_arnoldi_finish(GmresState* st, const double* h1, const double* h2,
                                  const double* partial_nrm, int nblk, int j, double tol,
                                  double* vscale_next, cudaStream_t s);
// beta = ||r0||: st->g = [beta,0..], beta0, vscale[0] = 1/beta
cudaError_t launch_gmres_init(GmresState* st, const double* partial_nrm, int nblk, double* vscale0,
                              int first_cycle, cudaStream_t s, GraphCond gc = GraphCond());
// y = R^{-1} g for k columns
cudaError_t launch_gmres_solve_y(GmresState* st, int k, cudaStream_t s);

// ---- DCGS2 Arnoldi (one dots pass + one update pass per iteration, krylov_kernels.cu)
// Iteration j: u = s_j V_j is the once-orthogonalised (lazily normalised) new vector, w = K u.
// dots: partial[b*NT + t], NT = 2j+2: t < j: V_i.V_j, j <= t < 2j: V_i.w, 2j: V_j.V_j, 2j+1: V_j.w
cudaError_t launch_dcgs_dots(const double* const* V, int j, const double* w, double* partial, long long NP,
                             int nblk, const int* skip, cudaStream_t s);
// reduce the dots, re-orthogonalise V_j (Pythagorean norm), correct and re-rotate Hessenberg column
// j-1, form the tentative column j and the update coefficients (st->cq, st->cu)
cudaError_t launch_dcgs_finish_a(GmresState* st, const double* partial, int nblk, int j, double* vscale,
                                 const int* skip, cudaStream_t s);
// V_j <- q_j = sum_i cq_i V_i (j > 0, in place), V_{j+1} <- w + sum_i cu_i V_i, ||V_{j+1}||^2 partials
cudaError_t launch_dcgs_update(const double* const* V, int j, const GmresState* st, const double* w,
                               double* partial_nrm, long long NP, int nblk, const int* skip, cudaStream_t s);
// tentative subdiagonal h_{j+1,j}, rotation of column j, convergence flag, vscale[j+1]
cudaError_t launch_dcgs_finish_b(GmresState* st, const double* partial_nrm, int nblk, int j, double tol,
                                 double* vscale, const int* skip, cudaStream_t s, GraphCond gc = GraphCond());
// SWITCH handle <- st->kcols (the y solve / x update variant of a captured cycle)
cudaError_t launch_graph_set_k(const GmresState* st, unsigned long long hk, cudaStream_t s);
// device {a, b} slot of a graph-captured step (ECoef::ab)
cudaError_t launch_set_ab(double* ab, double a, double b, cudaStream_t s);

}  // namespace rsfde
