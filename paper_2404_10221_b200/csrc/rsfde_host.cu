// Host side of the rsfde C ABI (include/rsfde.h): setup tables, operator chains built from
// the per-axis pencil passes, the GMRES driver and the CN time march.  Every step of the
// numerical path runs in the kernels of pass_kernels.cu / krylov_kernels.cu; this file only
// sequences launches and keeps device memory.
#include <cuda_runtime.h>

#include <chrono>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ctx_internal.h"

using namespace rsfde;

namespace {
thread_local std::string g_setup_error;
const char* kProfNames[RSFDE_NPROF] = {"oper_pass_spectral", "oper_pass_physical", "dst_pass", "cgs_dots",
                                       "cgs_dots2", "cgs_update_norm", "x_update", "small"};
}  // namespace

// ------------------------------------------------------------------------------ helpers
static rsfde_status cuda_fail(rsfde_ctx* c, cudaError_t e, const char* what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  if (c) c->err = buf; else g_setup_error = buf;
  return e == cudaErrorMemoryAllocation ? RSFDE_E_NOMEM : RSFDE_E_CUDA;
}
#define CK(expr, what)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(c, _e, what); \
  } while (0)
static cudaEvent_t prof_event(rsfde_ctx* c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// resolve completed launch timings (call after the stream was synchronised)
static void prof_collect(rsfde_ctx* c) {
  for (auto& p : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) c->prof_ms[p.cls] += ms;
    c->free_events.push_back(p.a);
    c->free_events.push_back(p.b);
  }
  c->pending.clear();
  cudaGetLastError();
}

// every kernel launch goes through LAUNCH(class, algorithmic bytes, expr, what)
#define LAUNCH(cls, bytes, expr, what)                                   \
  do {                                                                   \
    c->launches++;                                                       \
    cudaEvent_t _a = nullptr, _b = nullptr;                              \
    if (c->profiling) {                                                  \
      _a = prof_event(c);                                                \
      _b = prof_event(c);                                                \
      cudaEventRecord(_a, s);                                            \
    }                                                                    \
    cudaError_t _e = (expr);                                             \
    if (_e != cudaSuccess) return cuda_fail(c, _e, what);                \
    if (c->profiling) {                                                  \
      cudaEventRecord(_b, s);                                            \
      c->pending.push_back({(cls), _a, _b});                             \
      c->prof_launches[(cls)]++;                                         \
      c->prof_bytes[(cls)] += (double)(bytes);                           \
    }                                                                    \
  } while (0)
#define CKL(expr, what) LAUNCH(7, 0, expr, what)
enum { PC_OPER_SPEC = 0, PC_OPER_PHYS = 1, PC_DST = 2, PC_DOTS = 3, PC_DOTS2 = 4, PC_UPD = 5, PC_XUPD = 6 };
#define TRY(expr)                       \
  do {                                  \
    rsfde_status _s = (expr);           \
    if (_s != RSFDE_OK) return _s;      \
  } while (0)

// zero-initialised device allocation.  Without a stream the memset runs on the legacy default stream
// (setup synchronises the device before returning); lazy allocations inside a call pass the call's
// stream so that the zeroing is ordered before the kernels that read the buffer.
static rsfde_status dalloc(rsfde_ctx* c, void** p, size_t bytes, cudaStream_t s = nullptr, bool on_stream = false) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc");
  c->allocs.push_back(*p);
  c->bytes += (long long)bytes;
  e = on_stream ? cudaMemsetAsync(*p, 0, bytes, s) : cudaMemset(*p, 0, bytes);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemset");
  return RSFDE_OK;
}

template <class T>
static rsfde_status upload(rsfde_ctx* c, T** dst, const T* src, size_t count) {
  TRY(dalloc(c, (void**)dst, count * sizeof(T)));
  cudaError_t e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(c, e, "upload");
  return RSFDE_OK;
}

static bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------------------ setup tables
// FCD generator: s_0 = Gamma(a+1)/Gamma(a/2+1)^2, s_k = (1 - (a+1)/(a/2+k)) s_{k-1}
static void fcd_generator(double a, int n, std::vector<long double>& s) {
  s.assign(n, 0.0L);
  const long double al = a;
  s[0] = tgammal(al + 1.0L) / (tgammal(al / 2.0L + 1.0L) * tgammal(al / 2.0L + 1.0L));
  for (int k = 1; k < n; ++k) s[k] = (1.0L - (al + 1.0L) / (al / 2.0L + (long double)k)) * s[k - 1];
}

// sum_{j=0}^{n-1} w_j s_j cos(pi j k / N), w_0 = 1, w_j = 2: the tau eigenvalue q at index k
// (k = 1..n, Eq.(q) P:158 with divisor N = n+1) and the circulant spectrum c^_k of the order
// L = 2N embedding (c = [s_0..s_{n-1}, 0, 0, 0, s_{n-1}..s_1]) for k = 0..N.
static long double cos_sum(const std::vector<long double>& s, int N, int k) {
  const long double pi = 3.141592653589793238462643383279502884L;
  long double acc = s[0];
  const int n = (int)s.size();
  for (int j = 1; j < n; ++j) {
    const long long r = ((long long)j * k) % (2LL * N);
    acc += 2.0L * s[j] * cosl(pi * (long double)r / (long double)N);
  }
  return acc;
}

static rsfde_status build_axis_tables(rsfde_ctx* c, int i) {
  const int n = c->n[i], N = n + 1, L = 2 * N;
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<long double> s;
  fcd_generator(c->alpha[i], n, s);
  c->s_tab[i].resize(n);
  for (int k = 0; k < n; ++k) c->s_tab[i][k] = (double)s[k];
  // circulant spectrum for k = 0..N (real, even: c^_{L-k} = c^_k); q_k = c^_k for k = 1..n
  std::vector<double> chat(L), chatL(L);
  c->chat_tab[i].resize(L);
  c->q_tab[i].resize(n);
  for (int k = 0; k <= N; ++k) {
    const long double v = cos_sum(s, N, k);
    c->chat_tab[i][k] = (double)v;
    chatL[k] = (double)(v / (long double)L);
    if (k > 0 && k < N) {
      c->chat_tab[i][L - k] = (double)v;
      chatL[L - k] = (double)(v / (long double)L);
    }
    if (k >= 1 && k <= n) c->q_tab[i][k - 1] = (double)v;
  }
  // lambda_k(H_alpha) = 1 - (alpha/6) sin^2(k pi/(2N))
  c->lamH_tab[i].resize(n);
  for (int k = 1; k <= n; ++k) {
    const long double sn = sinl((long double)k * pi / (2.0L * N));
    c->lamH_tab[i][k - 1] = (double)(1.0L - (long double)c->alpha[i] / 6.0L * sn * sn);
  }
  // twiddles W_L^k = exp(-2 pi i k / L)
  // (second half: the seeds W_L^{8k} in the order of k, read by twiddle_col_x with consecutive lanes)
  std::vector<double2> tw(2 * L);
  for (int k = 0; k < L; ++k) {
    const long double ang = 2.0L * pi * (long double)k / (long double)L;
    tw[k] = make_double2((double)cosl(ang), (double)(-sinl(ang)));
  }
  for (int k = 0; k < L; ++k) tw[L + k] = tw[(8 * k) & (L - 1)];
  // eta_i = kappa_i tau / (2 h_i^alpha_i), h_i = 1/(n_i+1)
  const long double h = 1.0L / (long double)N;
  c->eta[i] = (double)((long double)c->kappa[i] * (long double)c->tau / (2.0L * powl(h, (long double)c->alpha[i])));
  TRY(upload(c, &c->d_chat[i], chatL.data(), L));
  TRY(upload(c, &c->d_tw[i], tw.data(), 2 * L));
  TRY(upload(c, &c->d_lamH[i], c->lamH_tab[i].data(), n));
  TRY(upload(c, &c->d_q[i], c->q_tab[i].data(), n));
  std::vector<double> tq(n);
  for (int k = 0; k < n; ++k) tq[k] = c->eta[i] * c->q_tab[i][k] / c->lamH_tab[i][k];
  TRY(upload(c, &c->d_tq[i], tq.data(), n));
  if (L == 4096) {
    std::vector<int> idx(L);
    row_layout_4096(idx.data());
    std::vector<double> a(L), b(L), d(L);
    for (int e = 0; e < L; ++e) {
      const int k = idx[e];
      a[e] = chatL[k];
      b[e] = (k >= 1 && k <= n) ? c->lamH_tab[i][k - 1] : 0.0;
      d[e] = (k >= 1 && k <= n) ? tq[k - 1] : 0.0;
    }
    TRY(upload(c, &c->d_chat_rl[i], a.data(), L));
    TRY(upload(c, &c->d_lamH_rl[i], b.data(), L));
    TRY(upload(c, &c->d_tq_rl[i], d.data(), L));
  }
  return RSFDE_OK;
}

// ------------------------------------------------------------------------------ passes
PassParams rsfde_axis_params(const rsfde_ctx* c, int axis) {
  PassParams p;
  memset(&p, 0, sizeof p);
  p.geo = c->geo;
  p.axis = axis;
  p.n = c->n[axis];
  p.N = p.n + 1;
  p.L = 2 * p.N;
  p.contiguous = axis == c->d - 1;
  long long stride = 1;
  if (!p.contiguous) {
    stride = c->geo.P;
    for (int i = axis + 1; i < c->d - 1; ++i) stride *= c->n[i];
  }
  p.stride = stride;
  p.inner = stride;
  if (p.contiguous) {
    const long long rows = c->geo.NP / c->geo.P;
    p.npairs = (rows + 1) / 2;
  } else {
    p.npairs = c->geo.NP / p.n / 2;
  }
  p.hc0 = 1.0 - c->alpha[axis] / 12.0;
  p.hc1 = c->alpha[axis] / 24.0;
  p.dst_scale = std::sqrt(2.0 / (double)p.N);
  p.ycoef = 1.0;
  p.flags = c->pass_flags;
  p.skip = c->skip;
  p.chat = c->d_chat[axis];
  p.tw = c->d_tw[axis];
  p.lamH = c->d_lamH[axis];
  p.chat_rl = c->d_chat_rl[axis];
  p.lamH_rl = c->d_lamH_rl[axis];
  p.tq_rl = c->d_tq_rl[axis];
  for (int i = 0; i < 3; ++i) {
    p.coff[i] = 0;
    p.cext[i] = c->n[i];
  }
  p.spec.ebar = c->ebar;
  for (int i = 0; i < 3; ++i) {
    p.spec.eta[i] = c->eta[i];
    p.spec.q[i] = c->d_q[i];
    p.spec.lamH[i] = c->d_lamH[i];
    p.spec.tq[i] = c->d_tq[i];
  }
  return p;
}

ECoef rsfde_ecoef_at(const rsfde_ctx* c, int m) {
  ECoef e;
  memset(&e, 0, sizeof e);
  if (c->ab_dev) e.ab = c->d_ab;
  if (c->ekind == RSFDE_COEF_GRID) {
    e.kind = 2;
    e.grid = c->grid + (c->grid_static ? 0 : (long long)m * c->n[0] * c->n[1] * c->n[2]);
  } else {
    e.kind = 1;
    e.a = c->a_half[m];
    e.b = c->b_half[m];
    for (int i = 0; i < 3; ++i) {
      e.g[i] = c->d_g[i];
      e.k[i] = c->d_k[i];
    }
  }
  return e;
}

struct ChainArgs {
  int xmode = X_E_TIMES_R;
  const double* Xin = nullptr;  // X_INPUT source (first pass)
  const double* R = nullptr;
  const double* rscale = nullptr;
  double etafac = 1.0;
  bool spectral = false;
  int spec = SPEC_PHAT;
  double ycoef = 1.0;           // physical last pass: out = ycoef*y + bcoef*B
  const double* B = nullptr;
  double bcoef = 0.0;
  int m = 0;
};

// chain of operator passes over the axes (see pass_kernels.cu header); out must not alias inputs
static rsfde_status oper_chain(rsfde_ctx* c, const ChainArgs& a, double* out, cudaStream_t s) {
  const int d = c->d;
  const double* Xcur = a.Xin;
  const double* Rcur = a.R;
  int buf = 0;
  // axis order of the chain (the per-axis operators commute, Eq.(Salpha)).  In 3D the chain runs
  // x_3 (contiguous) first and puts the spectral last pass on x_1, so that one of the two inverse DST
  // passes is along the contiguous axis (measured 1.4 % faster K chain at 511^3 than x_1 first);
  // RSFDE_AXIS_ORDER=fwd restores x_1 first.
  static const bool fwd = getenv("RSFDE_AXIS_ORDER") && !strcmp(getenv("RSFDE_AXIS_ORDER"), "fwd");
  const bool rev = d == 3 && !fwd;
  int ord[3] = {0, 1, 2};
  if (rev)
    for (int i = 0; i < d; ++i) ord[i] = d - 1 - i;
  for (int k = 0; k < d; ++k) {
    const int ax = ord[k];
    const bool last = k == d - 1;
    PassParams p = rsfde_axis_params(c, ax);
    p.xmode = k == 0 ? a.xmode : X_INPUT;
    p.X = Xcur;
    p.R = Rcur;
    p.rscale = k == 0 ? a.rscale : nullptr;
    p.eta = a.etafac * c->eta[ax];
    if (k == 0 && a.xmode == X_E_TIMES_R) p.e = rsfde_ecoef_at(c, a.m);
    p.spec.kind = a.spec;
    if (last) {
      p.Y = (a.spectral && d > 1) ? c->W[buf] : out;
      p.ycoef = a.ycoef;
      p.B = a.B;
      p.bcoef = a.bcoef;
    } else {
      p.Y = c->W[buf];
      p.C = c->W[buf + 1];
    }
    {
      const double vb = 8.0 * (double)c->geo.NP;
      const double nbytes = vb * (1.0 + (p.xmode == X_INPUT ? 1.0 : 0.0) + (last && p.B ? 1.0 : 0.0) +
                                  (last ? 1.0 : 2.0));
      LAUNCH(a.spectral ? PC_OPER_SPEC : PC_OPER_PHYS, nbytes, launch_oper_pass(p, a.spectral, last, s), "oper pass");
    }
    if (!last) {
      Xcur = c->W[buf];
      Rcur = c->W[buf + 1];
      buf = (buf + 2) % 4;
    }
  }
  if (a.spectral && d > 1) {
    // inverse DSTs along the other axes (chain order reversed)
    const double* in = c->W[buf];
    for (int k = d - 2; k >= 0; --k) {
      const int ax = ord[k];
      PassParams p = rsfde_axis_params(c, ax);
      p.X = in;
      double* o = k == 0 ? out : c->W[(buf + 1) % 4];
      p.Y = o;
      LAUNCH(PC_DST, 16.0 * (double)c->geo.NP, launch_dst_pass(p, false, s), "dst pass");
      in = o;
      buf = (buf + 1) % 4;
    }
  }
  return RSFDE_OK;
}

// y = S Lambda^{-1} S x for the spectrum kind (DSTs along every axis, scaling on the last)
static rsfde_status precond_chain(rsfde_ctx* c, int kind, const double* x, double* out, cudaStream_t s,
                                  const double* xscale = nullptr) {
  const int d = c->d;
  const double* in = x;
  int buf = 0;
  for (int ax = 0; ax < d; ++ax) {
    PassParams p = rsfde_axis_params(c, ax);
    const bool last = ax == d - 1;
    p.X = in;
    p.spec.kind = kind;
    if (ax == 0) p.rscale = xscale;
    double* o = (last && d == 1) ? out : c->W[buf];
    p.Y = o;
    LAUNCH(PC_DST, 16.0 * (double)c->geo.NP, launch_dst_pass(p, last, s), "dst pass");
    in = o;
    buf = (buf + 1) % 4;
  }
  for (int ax = d - 2; ax >= 0; --ax) {
    PassParams p = rsfde_axis_params(c, ax);
    p.X = in;
    double* o = ax == 0 ? out : c->W[buf];
    p.Y = o;
    LAUNCH(PC_DST, 16.0 * (double)c->geo.NP, launch_dst_pass(p, false, s), "dst pass");
    in = o;
    buf = (buf + 1) % 4;
  }
  return RSFDE_OK;
}

// ------------------------------------------------------------------------------ GMRES
static rsfde_status ensure_basis(rsfde_ctx* c, int restart, cudaStream_t s) {
  while ((int)c->V.size() < restart + 1) {
    double* v = nullptr;
    TRY(dalloc(c, (void**)&v, c->geo.NP * sizeof(double), s, true));
    c->V.push_back(v);
  }
  return RSFDE_OK;
}

// b^{(m)} = H E u0 - S_alpha u0 + tau F  (Eq.(tls)) into BUF (u0 = U0, F = FP)
static rsfde_status compute_b(rsfde_ctx* c, int m, cudaStream_t s) {
  ChainArgs a;
  a.xmode = X_E_TIMES_R;
  a.R = c->U0;
  a.etafac = -1.0;
  a.m = m;
  a.B = c->FP;
  a.bcoef = c->tau;
  return oper_chain(c, a, c->BUF, s);
}

// z = K v (v = s*V): A form P_hat^{-1} A v; A~ form P_alpha^{-1} H^{-1} A v
static rsfde_status apply_K(rsfde_ctx* c, int form, int m, const double* v, const double* vscale, double* z,
                            cudaStream_t s) {
  ChainArgs a;
  a.xmode = X_E_TIMES_R;
  a.R = v;
  a.rscale = vscale;
  a.m = m;
  if (form == RSFDE_FORM_A) {
    a.spectral = true;
    a.spec = SPEC_PHAT;
    return oper_chain(c, a, z, s);
  }
  if (form == RSFDE_FORM_TWO_SIDED) {
    // P_alpha^{-1/2} H^{-1} A P_alpha^{-1/2} v  (Eq.(Pls): A~ = H^{-1} A)
    TRY(precond_chain(c, SPEC_PALPHA_SQRT, v, c->TMP2, s, vscale));
    a.R = c->TMP2;
    a.rscale = nullptr;
    TRY(oper_chain(c, a, c->TMP, s));
    return precond_chain(c, SPEC_HP_SQRT, c->TMP, z, s);
  }
  TRY(oper_chain(c, a, c->TMP, s));
  TRY(precond_chain(c, SPEC_HINV, c->TMP, c->TMP2, s));
  return precond_chain(c, SPEC_PALPHA, c->TMP2, z, s);
}

// r = K-preconditioned residual of (b - A x) into out
static rsfde_status precond_residual(rsfde_ctx* c, int form, int m, const double* b, const double* x, double* out,
                                     cudaStream_t s) {
  ChainArgs a;
  a.xmode = X_E_TIMES_R;
  a.R = x;
  a.m = m;
  a.ycoef = -1.0;
  a.B = b;
  a.bcoef = 1.0;
  TRY(oper_chain(c, a, c->TMP, s));
  if (form == RSFDE_FORM_A) return precond_chain(c, SPEC_PHAT, c->TMP, out, s);
  if (form == RSFDE_FORM_TWO_SIDED) return precond_chain(c, SPEC_HP_SQRT, c->TMP, out, s);
  TRY(precond_chain(c, SPEC_HINV, c->TMP, c->TMP2, s));
  return precond_chain(c, SPEC_PALPHA, c->TMP2, out, s);
}

struct Flags {
  int converged;
  int breakdown;
  double relres;
};

static rsfde_status read_flags(rsfde_ctx* c, Flags* f, cudaStream_t s) {
  CK(cudaMemcpyAsync(c->h_flags, c->d_state, sizeof(Flags), cudaMemcpyDeviceToHost, s), "flags copy");
  CK(cudaStreamSynchronize(s), "stream sync");
  memcpy(f, c->h_flags, sizeof(Flags));
  if (c->profiling) prof_collect(c);
  return RSFDE_OK;
}

// One GMRES cycle of DCGS2 Arnoldi steps (krylov_kernels.cu) after gmres_init.  The host runs one
// iteration ahead of the flags: iteration j+1 is enqueued before the convergence flag of iteration j is
// read (an async copy into pinned memory + an event), and every kernel of a step returns at once when
// the device flags say the previous step converged (PassParams::skip), so the GPU never idles on the
// host round trip.  Returns the number of Arnoldi steps done in *k and the last flags in *fl.
static rsfde_status dcgs_cycle(rsfde_ctx* c, int form, int m, int restart, int max_iters, int fixed, double tol,
                               int total, cudaStream_t s, int* k, Flags* fl) {
  const long long NP = c->geo.NP;
  const int nb = reduction_blocks(NP, c->nblk);
  const double vb = 8.0 * (double)NP;
  const int* skip = reinterpret_cast<const int*>(c->d_state);  // converged, breakdown
  const bool no_spec = getenv("RSFDE_NO_SPEC") != nullptr;  // (read per call: tests toggle it)
  const int lag = (c->profiling || no_spec) ? 0 : 1;
  for (int i = 0; i < 2; ++i)
    if (!c->flag_ev[i]) CK(cudaEventCreateWithFlags(&c->flag_ev[i], cudaEventDisableTiming), "event");
  Flags* slots = reinterpret_cast<Flags*>(c->h_flags);
  int jl = 0, jr = 0;
  while (true) {
    const bool can_launch = jl < restart && total + jl < max_iters && !(fixed > 0 && total + jl >= fixed);
    if (can_launch) {
      const int j = jl;
      const double* const* Vp = (const double* const*)c->V.data();
      c->skip = j > 0 ? skip : nullptr;
      const rsfde_status st = apply_K(c, form, m, c->V[j], c->d_vscale + j, c->Z, s);
      c->skip = nullptr;
      TRY(st);
      const int* sk = j > 0 ? skip : nullptr;
      // one dots pass (j+2 vectors) + one update pass (j+2 read, 2 written)
      LAUNCH(PC_DOTS, vb * (j + 2), launch_dcgs_dots(Vp, j, c->Z, c->d_part, NP, c->nblk, sk, s), "dcgs dots");
      CKL(launch_dcgs_finish_a(c->d_state, c->d_part, nb, j, c->d_vscale, sk, s), "dcgs finish a");
      LAUNCH(PC_UPD, vb * (j + 2 + (j > 0 ? 2 : 1)),
             launch_dcgs_update(Vp, j, c->d_state, c->Z, c->d_nrm, NP, c->nblk, sk, s), "dcgs update");
      CKL(launch_dcgs_finish_b(c->d_state, c->d_nrm, nb, j, tol, c->d_vscale, sk, s), "dcgs finish b");
      CK(cudaMemcpyAsync(&slots[j & 1], c->d_state, sizeof(Flags), cudaMemcpyDeviceToHost, s), "flags copy");
      CK(cudaEventRecord(c->flag_ev[j & 1], s), "flags event");
      ++jl;
    }
    if (jr < jl - (can_launch ? lag : 0)) {
      CK(cudaEventSynchronize(c->flag_ev[jr & 1]), "flags wait");
      memcpy(fl, &slots[jr & 1], sizeof(Flags));
      if (c->profiling) {
        CK(cudaStreamSynchronize(s), "stream sync");
        prof_collect(c);
      }
      ++jr;
      const bool stop = fixed > 0 ? total + jr >= fixed : fl->converged != 0;
      if (stop || fl->breakdown || total + jr >= max_iters || jr == restart) break;
    } else if (!can_launch) {
      break;
    }
  }
  *k = jr;
  return RSFDE_OK;
}

// ------------------------------------------------------------------------------ graph-captured cycle
// The first GMRES cycle of a CN step (A form, first-cycle residual shortcut) as ONE CUDA graph: the r0
// chain, ||r0||, then Arnoldi step j as the body of a conditional IF node nested in step j-1's body (the
// node's handle is cleared on the device by dcgs_finish_b on convergence or breakdown, so nothing after
// the last step is launched or evaluated), then a SWITCH on the final column count k running the y
// solve and x += V y for that k.  The host reads the flags once per cycle instead of once per Arnoldi
// step (stopping rule P:513).  RSFDE_NO_GRAPH=1 selects the stream path.  (A handle
// gates exactly one conditional node and is set from the graph that owns it, hence one handle per body.)
static bool graph_eligible(const rsfde_ctx* c, int form, bool mode_fast) {
  if (c->profiling || getenv("RSFDE_NO_GRAPH")) return false;  // (read per call: tests toggle it)
  if (c->ortho != ORTHO_DCGS2 || form != RSFDE_FORM_A || !mode_fast) return false;
  return c->ekind != RSFDE_COEF_GRID || c->grid_static;
}

static void graph_destroy(rsfde_ctx* c) {
  for (cudaStream_t cs : c->cap_s) {  // (a capture abandoned by an error)
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cs && cudaStreamIsCapturing(cs, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk = nullptr;
      if (cudaStreamEndCapture(cs, &junk) == cudaSuccess && junk) cudaGraphDestroy(junk);
    }
  }
  cudaGetLastError();
  if (c->sg.exec) cudaGraphExecDestroy(c->sg.exec);
  if (c->sg.graph) cudaGraphDestroy(c->sg.graph);
  c->sg = rsfde_ctx::StepGraph();
}

// conditional node after the capture frontier of cs; it becomes the new frontier
static cudaError_t add_cond(cudaStream_t cs, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                            unsigned size, cudaGraph_t* bodies) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(cs, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  if (st != cudaStreamCaptureStatusActive) return cudaErrorStreamCaptureInvalidated;
  cudaGraphNodeParams np = {cudaGraphNodeTypeConditional};
  np.conditional.handle = h;
  np.conditional.type = type;
  np.conditional.size = size;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, deps, nd, &np);
  if (e != cudaSuccess) return e;
  for (unsigned i = 0; i < size; ++i) bodies[i] = np.conditional.phGraph_out[i];
  return cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies);
}

// kernels of Arnoldi step j (as in dcgs_cycle; every step of a body starts unconverged)
static rsfde_status capture_arnoldi_step(rsfde_ctx* c, int j, double tol, const GraphCond& gc, cudaStream_t s) {
  const long long NP = c->geo.NP;
  const int nb = reduction_blocks(NP, c->nblk);
  const double vb = 8.0 * (double)NP;
  const int* skip = reinterpret_cast<const int*>(c->d_state);  // breakdown inside the step (finish_a)
  const double* const* Vp = (const double* const*)c->V.data();
  c->skip = nullptr;
  TRY(apply_K(c, RSFDE_FORM_A, 0, c->V[j], c->d_vscale + j, c->Z, s));
  LAUNCH(PC_DOTS, vb * (j + 2), launch_dcgs_dots(Vp, j, c->Z, c->d_part, NP, c->nblk, nullptr, s), "dcgs dots");
  CKL(launch_dcgs_finish_a(c->d_state, c->d_part, nb, j, c->d_vscale, nullptr, s), "dcgs finish a");
  LAUNCH(PC_UPD, vb * (j + 2 + (j > 0 ? 2 : 1)), launch_dcgs_update(Vp, j, c->d_state, c->Z, c->d_nrm, NP, c->nblk, skip, s),
         "dcgs update");
  CKL(launch_dcgs_finish_b(c->d_state, c->d_nrm, nb, j, tol, c->d_vscale, skip, s, gc), "dcgs finish b");
  return RSFDE_OK;
}

static rsfde_status graph_build(rsfde_ctx* c, int restart, int max_iters, int fixed, double tol) {
  graph_destroy(c);
  for (int i = 0; i < 2; ++i)
    if (!c->cap_s[i]) CK(cudaStreamCreateWithFlags(&c->cap_s[i], cudaStreamNonBlocking), "capture stream");
  if (!c->d_ab) TRY(dalloc(c, (void**)&c->d_ab, 2 * sizeof(double)));
  int nsteps = restart < max_iters ? restart : max_iters;
  if (fixed > 0 && fixed < nsteps) nsteps = fixed;
  auto& G = c->sg;
  CK(cudaGraphCreate(&G.graph, 0), "graph create");
  cudaGraphConditionalHandle hc, hk;
  CK(cudaGraphConditionalHandleCreate(&hc, G.graph, 0, cudaGraphCondAssignDefault), "cond handle");
  CK(cudaGraphConditionalHandleCreate(&hk, G.graph, 0, cudaGraphCondAssignDefault), "cond handle");
  GraphCond gc;
  gc.h_cont = hc;
  gc.on = 1;
  const long long NP = c->geo.NP;
  const int nb = reduction_blocks(NP, c->nblk);
  const long long l0 = c->launches;
  const bool prof = c->profiling;
  c->profiling = 0;
  c->ab_dev = true;
  rsfde_status st = RSFDE_OK;
  cudaGraph_t ifb = nullptr;
  std::vector<cudaGraph_t> sw(nsteps + 1, nullptr);
  auto end_capture = [&](cudaStream_t cs) -> rsfde_status {
    cudaGraph_t out = nullptr;
    CK(cudaStreamEndCapture(cs, &out), "end capture");
    return RSFDE_OK;
  };
  auto body = [&]() -> rsfde_status {
    // top level: r0 = P_hat^{-1}(H FH - 2 S_alpha x0), ||r0||, IF step 0 [, IF step 1 ...], SWITCH k
    cudaStream_t cs = c->cap_s[0];
    CK(cudaStreamBeginCaptureToGraph(cs, G.graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed), "begin capture");
    {
      ChainArgs a;
      a.xmode = X_INPUT;
      a.Xin = c->FH;
      a.R = c->X;
      a.etafac = -2.0;
      a.m = 0;
      a.spectral = true;
      a.spec = SPEC_PHAT;
      const cudaStream_t s = cs;
      rsfde_status r = oper_chain(c, a, c->V[0], s);
      if (r == RSFDE_OK) {
        LAUNCH(7, 0, launch_sumsq(c->V[0], c->d_nrm, NP, c->nblk, s), "sumsq");
        LAUNCH(7, 0, launch_gmres_init(c->d_state, c->d_nrm, nb, c->d_vscale, 1, s, gc), "gmres init");
      }
      if (r != RSFDE_OK) {
        cudaGraph_t junk;
        cudaStreamEndCapture(cs, &junk);
        return r;
      }
    }
    G.launches_pre = c->launches - l0;
    CK(add_cond(cs, hc, cudaGraphCondTypeIf, 1, &ifb), "if node");
    CK(launch_graph_set_k(c->d_state, hk, cs), "set k");
    G.launches_pre += 1;
    CK(add_cond(cs, hk, cudaGraphCondTypeSwitch, (unsigned)(nsteps + 1), sw.data()), "switch node");
    TRY(end_capture(cs));
    // Arnoldi steps
    cudaStream_t bs = c->cap_s[1];
    cudaGraph_t cur = ifb;
    for (int j = 0; j < nsteps; ++j) {
      const long long lj = c->launches;
      // the IF node of step j+1 sits in step j's body with a handle owned by that body graph, set by
      // step j's dcgs_finish_b (0 for the last step: nothing to gate)
      GraphCond gj = gc;
      cudaGraphConditionalHandle hn = 0;
      if (j + 1 < nsteps) CK(cudaGraphConditionalHandleCreate(&hn, cur, 0, cudaGraphCondAssignDefault), "cond handle");
      gj.h_cont = hn;
      CK(cudaStreamBeginCaptureToGraph(bs, cur, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed), "begin capture");
      rsfde_status r = capture_arnoldi_step(c, j, tol, gj, bs);
      if (r != RSFDE_OK) {
        cudaGraph_t junk;
        cudaStreamEndCapture(bs, &junk);
        return r;
      }
      cudaGraph_t next = nullptr;
      if (j + 1 < nsteps) CK(add_cond(bs, hn, cudaGraphCondTypeIf, 1, &next), "nested if node");
      TRY(end_capture(bs));
      G.launches_step.push_back(c->launches - lj);
      cur = next;
    }
    // y solve and x update for each final column count k (k = 0: r0 == 0, nothing to do)
    G.launches_end.push_back(0);
    {
      cudaGraphNode_t en;  // (k = 0 body: no work)
      CK(cudaGraphAddEmptyNode(&en, sw[0], nullptr, 0), "empty node");
    }
    for (int k = 1; k <= nsteps; ++k) {
      const long long lk = c->launches;
      CK(cudaStreamBeginCaptureToGraph(bs, sw[k], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed), "begin capture");
      const double* const* Vp = (const double* const*)c->V.data();
      const double* d_y =
          reinterpret_cast<const double*>(reinterpret_cast<const char*>(c->d_state) + offsetof(GmresState, y));
      const cudaStream_t s = bs;
      LAUNCH(7, 0, launch_gmres_solve_y(c->d_state, k, s), "solve y");
      LAUNCH(PC_XUPD, 8.0 * (double)NP * (k + 2), launch_axpy_basis(Vp, c->d_vscale, k, d_y, c->X, NP, s), "x update");
      TRY(end_capture(bs));
      G.launches_end.push_back(c->launches - lk);
    }
    return RSFDE_OK;
  };
  st = body();
  c->ab_dev = false;
  c->profiling = prof;
  c->launches = l0;
  if (st != RSFDE_OK) {
    graph_destroy(c);
    return st;
  }
  CK(cudaGraphInstantiate(&G.exec, G.graph, 0), "graph instantiate");
  G.restart = restart;
  G.max_iters = max_iters;
  G.fixed = fixed;
  G.tol = tol;
  G.nsteps = nsteps;
  return RSFDE_OK;
}

// run the captured first cycle of step m; *steps = Arnoldi steps executed, *fl = final flags
static rsfde_status gmres_graph_cycle(rsfde_ctx* c, int m, int restart, int max_iters, int fixed, double tol,
                                      cudaStream_t s, int* steps, Flags* fl) {
  auto& G = c->sg;
  if (!G.exec || G.restart != restart || G.max_iters != max_iters || G.fixed != fixed || G.tol != tol)
    TRY(graph_build(c, restart, max_iters, fixed, tol));
  if (c->ekind != RSFDE_COEF_GRID) CKL(launch_set_ab(c->d_ab, c->a_half[m], c->b_half[m], s), "set ab");
  CK(cudaGraphLaunch(G.exec, s), "graph launch");
  c->graph_replays++;
  char* h = reinterpret_cast<char*>(c->h_flags);
  CK(cudaMemcpyAsync(h, c->d_state, sizeof(Flags), cudaMemcpyDeviceToHost, s), "flags copy");
  CK(cudaMemcpyAsync(h + 48, reinterpret_cast<const char*>(c->d_state) + offsetof(GmresState, kcols), 2 * sizeof(int),
                     cudaMemcpyDeviceToHost, s),
     "flags copy");
  CK(cudaStreamSynchronize(s), "stream sync");
  memcpy(fl, h, sizeof(Flags));
  int kk[2];
  memcpy(kk, h + 48, sizeof kk);
  const int kcols = kk[0] < 0 ? 0 : kk[0];
  *steps = kk[1];
  // kernels the replay launched (the captured launches of the executed bodies)
  long long n = G.launches_pre;
  for (int j = 0; j < *steps && j < (int)G.launches_step.size(); ++j) n += G.launches_step[j];
  if (kcols < (int)G.launches_end.size()) n += G.launches_end[kcols];
  c->launches += n;
  return RSFDE_OK;
}

// GMRES on K x = P^{-1} b with x = c->X on entry (x0) and exit.
// mode_fast: first-cycle r0 = P_hat^{-1}(H FH - 2 S_alpha x0) with FH = H^{-1} tau F (valid iff
// x0 = u^{(m)}: b - A u = tau F - 2 S_alpha u, Eq.(tls)); later cycles use b (computed on demand).
static rsfde_status gmres_core(rsfde_ctx* c, int m, bool mode_fast, bool have_b, const rsfde_gmres_cfg& cfg,
                               cudaStream_t s, int* iters_out, double* relres_out, int* conv_out) {
  const int restart = cfg.restart;
  const int max_iters = cfg.max_iters > 0 ? cfg.max_iters : 10 * restart;
  const int fixed = cfg.fixed_iters;
  const double tol = fixed > 0 ? -1.0 : cfg.tol;
  const int form = cfg.form;
  TRY(ensure_basis(c, restart, s));
  const long long NP = c->geo.NP;
  const int nb = reduction_blocks(NP, c->nblk);
  int total = 0;
  bool first = true;
  Flags fl{0, 0, 1.0};
  bool converged = false;
  while (true) {
    if (first && c->ortho == ORTHO_DCGS2 && graph_eligible(c, form, mode_fast)) {
      int k = 0;
      TRY(gmres_graph_cycle(c, m, restart, max_iters, fixed, tol, s, &k, &fl));
      total += k;
      converged = fixed > 0 ? (total >= fixed || fl.breakdown != 0) : (fl.converged != 0 || fl.breakdown != 0);
      if (converged || total >= max_iters) break;
      first = false;
      continue;
    }
    if (form == RSFDE_FORM_TWO_SIDED) {
      // residual of the physical iterate u = P^{-1/2} u~ (X holds u on the first cycle, u~ later)
      if (!have_b) {
        TRY(compute_b(c, m, s));
        have_b = true;
      }
      if (first) {
        TRY(precond_residual(c, form, m, c->BUF, c->X, c->V[0], s));
        // X <- u~_0 = P^{1/2} u_0 (Thm 3.9)
        TRY(precond_chain(c, SPEC_PALPHA_RSQRT, c->X, c->Z, s));
        CK(cudaMemcpyAsync(c->X, c->Z, (size_t)NP * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
      } else {
        TRY(precond_chain(c, SPEC_PALPHA_SQRT, c->X, c->Z, s));
        TRY(precond_residual(c, form, m, c->BUF, c->Z, c->V[0], s));
      }
    } else if (first && mode_fast && form == RSFDE_FORM_A) {
      ChainArgs a;
      a.xmode = X_INPUT;
      a.Xin = c->FH;
      a.R = c->X;
      a.etafac = -2.0;
      a.m = m;
      a.spectral = true;
      a.spec = SPEC_PHAT;
      TRY(oper_chain(c, a, c->V[0], s));
    } else {
      if (!have_b) {
        TRY(compute_b(c, m, s));
        have_b = true;
      }
      TRY(precond_residual(c, form, m, c->BUF, c->X, c->V[0], s));
    }
    CKL(launch_sumsq(c->V[0], c->d_nrm, NP, c->nblk, s), "sumsq");
    CKL(launch_gmres_init(c->d_state, c->d_nrm, nb, c->d_vscale, first ? 1 : 0, s), "gmres init");
    TRY(read_flags(c, &fl, s));
    if (fl.converged) {  // r0 == 0: x0 is the solution
      converged = true;
      break;
    }
    int k = 0;
    if (c->ortho == ORTHO_DCGS2) {
      TRY(dcgs_cycle(c, form, m, restart, max_iters, fixed, tol, total, s, &k, &fl));
      total += k;
    }
    for (int j = 0; j < restart && c->ortho != ORTHO_DCGS2; ++j) {
      const int J = j + 1;
      TRY(apply_K(c, form, m, c->V[j], c->d_vscale + j, c->Z, s));
      const double* const* Vp = (const double* const*)c->V.data();
      const double vb = 8.0 * (double)NP;
      LAUNCH(PC_DOTS, vb * (J + 1), launch_dots(Vp, c->d_vscale, J, c->Z, c->d_part, NP, c->nblk, s), "dots");
      CKL(launch_reduce(c->d_part, nb, J, c->d_h1, s), "reduce h1");
      LAUNCH(PC_DOTS2, vb * (J + 1), launch_dots_after_update(Vp, c->d_vscale, J, c->Z, c->d_h1, c->d_part, NP, c->nblk, s),
             "dots2");
      CKL(launch_reduce(c->d_part, nb, J, c->d_h2, s), "reduce h2");
      LAUNCH(PC_UPD, vb * (J + 2),
             launch_update_norm(Vp, c->d_vscale, J, c->Z, c->d_h1, c->d_h2, c->V[j + 1], c->d_nrm, NP, c->nblk, s),
             "update");
      CKL(launch_arnoldi_finish(c->d_state, c->d_h1, c->d_h2, c->d_nrm, nb, j, tol, c->d_vscale + j + 1, s),
          "finish");
      ++total;
      k = j + 1;
      TRY(read_flags(c, &fl, s));
      const bool stop = fixed > 0 ? total >= fixed : fl.converged != 0;
      if (stop || fl.breakdown || total >= max_iters) break;
    }
    CKL(launch_gmres_solve_y(c->d_state, k, s), "solve y");
    const double* const* Vp = (const double* const*)c->V.data();
    const double* d_y = reinterpret_cast<const double*>(reinterpret_cast<const char*>(c->d_state) + offsetof(GmresState, y));
    LAUNCH(PC_XUPD, 8.0 * (double)NP * (k + 2), launch_axpy_basis(Vp, c->d_vscale, k, d_y, c->X, NP, s), "x update");
    // replay mode (fixed_iters > 0) keeps restarting until exactly `fixed` Arnoldi steps ran
    converged = fixed > 0 ? (total >= fixed || fl.breakdown != 0) : (fl.converged != 0 || fl.breakdown != 0);
    if (converged || total >= max_iters) break;
    first = false;
  }
  if (form == RSFDE_FORM_TWO_SIDED) {  // u = P^{-1/2} u~
    TRY(precond_chain(c, SPEC_PALPHA_SQRT, c->X, c->Z, s));
    CK(cudaMemcpyAsync(c->X, c->Z, (size_t)NP * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
  }
  if (iters_out) *iters_out = total;
  if (relres_out) *relres_out = fl.relres;
  if (conv_out) *conv_out = converged ? 1 : 0;
  return RSFDE_OK;
}

// ------------------------------------------------------------------------------ on-chip 1-D march
static bool onchip_eligible(const rsfde_ctx* c, const rsfde_gmres_cfg* cfg) {
  const char* off = getenv("RSFDE_NO_ONCHIP");
  if (off && *off && strcmp(off, "0")) return false;
  if (c->d != 1 || c->ekind != RSFDE_COEF_SEPARABLE) return false;
  if (cfg->form != RSFDE_FORM_A || cfg->x0_policy != RSFDE_X0_PREV || cfg->fixed_iters > 0) return false;
  if (cfg->restart < 1 || cfg->restart > 50) return false;
  return onchip_smem_bytes(c->n[0], cfg->restart) <= 200 * 1024;
}

// parameters of one on-chip march (tables, F staged to the device when it is host memory)
static rsfde_status onchip_prepare(rsfde_ctx* c, int m_begin, int m_count, const double* F, int F_static, bool f_host,
                                   const rsfde_gmres_cfg& cfg, cudaStream_t s, OnchipParams* out) {
  const int n = c->n[0];
  if (!c->d_s0) {
    CK(cudaMalloc(&c->d_s0, n * sizeof(double)), "alloc");
    c->allocs.push_back(c->d_s0);
    CK(cudaMemcpy(c->d_s0, c->s_tab[0].data(), n * sizeof(double), cudaMemcpyHostToDevice), "upload s");
    CK(cudaMalloc(&c->d_on_iters, c->M * sizeof(int)), "alloc");
    CK(cudaMalloc(&c->d_on_relres, c->M * sizeof(double)), "alloc");
    CK(cudaMalloc(&c->d_on_conv, c->M), "alloc");
    c->allocs.push_back(c->d_on_iters);
    c->allocs.push_back(c->d_on_relres);
    c->allocs.push_back(c->d_on_conv);
  }
  const double* Fd = F;
  const long long nF = F ? (F_static ? 1 : m_count) : 0;
  if (F && f_host) {
    if (c->on_F_cap < nF * n) {
      if (c->d_on_F) cudaFree(c->d_on_F);
      CK(cudaMalloc(&c->d_on_F, nF * n * sizeof(double)), "alloc F");
      c->on_F_cap = nF * n;
    }
    CK(cudaMemcpyAsync(c->d_on_F, F, nF * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D F");
    Fd = c->d_on_F;
  }
  OnchipParams& p = *out;
  p.n = n;
  p.restart = cfg.restart;
  p.max_iters = cfg.max_iters > 0 ? cfg.max_iters : 10 * cfg.restart;
  p.m_begin = m_begin;
  p.m_count = m_count;
  p.tol = cfg.tol;
  p.alpha = c->alpha[0];
  p.eta = c->eta[0];
  p.tau = c->tau;
  p.ebar = c->ebar;
  p.s = c->d_s0;
  p.lamH = c->d_lamH[0];
  p.q = c->d_q[0];
  p.a_half = c->d_ahalf;
  p.b_half = c->d_bhalf;
  p.g = c->d_g[0];
  p.kk = c->d_k[0];
  p.F = Fd;
  p.F_stride = F_static ? 0 : n;
  p.X = c->X;
  p.iters = c->d_on_iters;
  p.relres = c->d_on_relres;
  p.conv = c->d_on_conv;
  return RSFDE_OK;
}

// per-step results of an on-chip march into the report (after the stream was synchronised)
static rsfde_status onchip_collect(rsfde_ctx* c, int m_count, rsfde_report* rep, long long* total) {
  std::vector<int> its(m_count);
  std::vector<double> rr(m_count);
  std::vector<unsigned char> cv(m_count);
  CK(cudaMemcpy(its.data(), c->d_on_iters, m_count * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
  CK(cudaMemcpy(rr.data(), c->d_on_relres, m_count * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  CK(cudaMemcpy(cv.data(), c->d_on_conv, m_count, cudaMemcpyDeviceToHost), "D2H");
  *total = 0;
  for (int k = 0; k < m_count; ++k) {
    if (its[k] > 0) *total += its[k];
    if (rep) {
      if (rep->iters) rep->iters[k] = its[k];
      if (rep->final_relres) rep->final_relres[k] = rr[k];
      if (rep->converged) rep->converged[k] = cv[k];
    }
  }
  return RSFDE_OK;
}

static rsfde_status onchip_march(rsfde_ctx* c, int m_begin, int m_count, const double* F, int F_static, bool f_host,
                                 const rsfde_gmres_cfg& cfg, cudaStream_t s, rsfde_report* rep, long long* total) {
  OnchipParams p;
  TRY(onchip_prepare(c, m_begin, m_count, F, F_static, f_host, cfg, s, &p));
  LAUNCH(PC_OPER_SPEC, 0.0, launch_onchip_1d(p, s), "on-chip march");
  CK(cudaStreamSynchronize(s), "stream sync");
  return onchip_collect(c, m_count, rep, total);
}

// ------------------------------------------------------------------------------ ABI
extern "C" {

const char* rsfde_version(void) { return "rsfde-b200 0.1 (sm_100a, FP64)"; }

const char* rsfde_last_error(const rsfde_ctx* c) { return c ? c->err.c_str() : g_setup_error.c_str(); }

long long rsfde_device_bytes(const rsfde_ctx* c) { return c ? c->bytes : 0; }

long long rsfde_launch_count(const rsfde_ctx* c, int reset) {
  if (!c) return 0;
  const long long v = c->launches;
  if (reset) const_cast<rsfde_ctx*>(c)->launches = 0;
  return v;
}

long long rsfde_graph_replays(const rsfde_ctx* c) { return c ? c->graph_replays : 0; }

int rsfde_profile(rsfde_ctx* c, int enable) {
  if (!c) return -1;
  cudaDeviceSynchronize();
  prof_collect(c);
  c->profiling = enable ? 1 : 0;
  for (int i = 0; i < RSFDE_NPROF; ++i) {
    c->prof_launches[i] = 0;
    c->prof_ms[i] = 0;
    c->prof_bytes[i] = 0;
  }
  return RSFDE_NPROF;
}

int rsfde_profile_read(rsfde_ctx* c, int cls, long long* launches, double* ms, double* bytes, const char** name) {
  if (!c || cls < 0 || cls >= RSFDE_NPROF) return -1;
  cudaDeviceSynchronize();
  prof_collect(c);
  if (launches) *launches = c->prof_launches[cls];
  if (ms) *ms = c->prof_ms[cls];
  if (bytes) *bytes = c->prof_bytes[cls];
  if (name) *name = kProfNames[cls];
  return 0;
}

void rsfde_destroy(rsfde_ctx* c) {
  if (!c) return;
  cudaDeviceSynchronize();
  graph_destroy(c);
  for (cudaStream_t cs : c->cap_s)
    if (cs) cudaStreamDestroy(cs);
  for (void* p : c->allocs) cudaFree(p);
  if (c->d_on_F) cudaFree(c->d_on_F);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  prof_collect(c);
  for (cudaEvent_t e : c->free_events) cudaEventDestroy(e);
  for (cudaEvent_t e : c->flag_ev)
    if (e) cudaEventDestroy(e);
  delete c;
}

static rsfde_status setup_fail(rsfde_ctx* c, rsfde_status st, const char* msg) {
  if (msg) g_setup_error = msg;
  else if (c) g_setup_error = c->err;
  rsfde_destroy(c);
  return st;
}

rsfde_status rsfde_setup_internal(rsfde_ctx** out, const rsfde_problem* p, void* stream, bool alloc_work) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!out) return RSFDE_E_CONFIG;
  *out = nullptr;
  if (!p) { g_setup_error = "problem is NULL"; return RSFDE_E_CONFIG; }
  if (p->d < 1 || p->d > 3) { g_setup_error = "d must be 1, 2 or 3"; return RSFDE_E_DIM; }
  for (int i = 0; i < p->d; ++i) {
    if (p->n[i] < 1 || !pow2(p->n[i] + 1) || p->n[i] + 1 > 2048) {
      g_setup_error = "n_i + 1 must be a power of two in [2, 2048]";
      return RSFDE_E_DIM;
    }
    if (!(p->alpha[i] > 1.0 && p->alpha[i] <= 2.0)) { g_setup_error = "alpha_i must lie in (1, 2]"; return RSFDE_E_DOMAIN; }
    if (!(p->kappa[i] > 0.0)) { g_setup_error = "kappa_i must be > 0"; return RSFDE_E_DOMAIN; }
  }
  if (!(p->tau_t > 0.0) || p->M < 1) { g_setup_error = "tau_t must be > 0 and M >= 1"; return RSFDE_E_DOMAIN; }
  if (p->e.kind == RSFDE_COEF_SEPARABLE) {
    if (!p->e.a_half || !p->e.b_half) { g_setup_error = "separable e needs a_half and b_half"; return RSFDE_E_CONFIG; }
  } else if (p->e.kind == RSFDE_COEF_GRID) {
    if (!p->e.grid) { g_setup_error = "grid e needs a device grid"; return RSFDE_E_CONFIG; }
  } else {
    g_setup_error = "unknown coefficient kind";
    return RSFDE_E_CONFIG;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    g_setup_error = "no CUDA device: the rsfde library has no CPU fallback";
    return RSFDE_E_CUDA;
  }
  rsfde_ctx* c = new rsfde_ctx();
  cudaGetDevice(&c->device);
  c->nblk = rsfde::stream_blocks();
  c->d = p->d;
  for (int i = 0; i < 3; ++i) {
    c->n[i] = i < p->d ? p->n[i] : 1;
    c->alpha[i] = i < p->d ? p->alpha[i] : 2.0;
    c->kappa[i] = i < p->d ? p->kappa[i] : 0.0;
  }
  c->tau = p->tau_t;
  c->M = p->M;
  if (getenv("RSFDE_NO_PIPE")) c->pass_flags |= PASS_FLAG_NO_PIPE;
  {
    // Arnoldi orthogonalisation: DCGS2 (default) or the three-pass CGS2 (RSFDE_ORTHO=cgs2)
    const char* o = getenv("RSFDE_ORTHO");
    c->ortho = (o && !strcmp(o, "cgs2")) ? ORTHO_CGS2 : ORTHO_DCGS2;
  }
  c->geo.d = c->d;
  for (int i = 0; i < 3; ++i) c->geo.n[i] = c->n[i];
  c->geo.P = c->n[c->d - 1] + 1;
  long long rows = 1;
  for (int i = 0; i < c->d - 1; ++i) rows *= c->n[i];
  c->geo.NP = rows * c->geo.P;
  rsfde_status st;
  for (int i = 0; i < c->d; ++i)
    if ((st = build_axis_tables(c, i)) != RSFDE_OK) return setup_fail(c, st, nullptr);
  // coefficient
  c->ekind = p->e.kind;
  const cudaStream_t s = S(stream);
  const Geom& G = c->geo;
  if (c->ekind == RSFDE_COEF_SEPARABLE) {
    c->a_half.assign(p->e.a_half, p->e.a_half + c->M);
    c->b_half.assign(p->e.b_half, p->e.b_half + c->M);
    for (int i = 0; i < c->d; ++i) {
      if (p->e.g[i] && (st = upload(c, &c->d_g[i], p->e.g[i], c->n[i])) != RSFDE_OK) return setup_fail(c, st, nullptr);
      if (p->e.k[i] && (st = upload(c, &c->d_k[i], p->e.k[i], c->n[i])) != RSFDE_OK) return setup_fail(c, st, nullptr);
    }
    if ((st = upload(c, &c->d_ahalf, c->a_half.data(), c->M)) != RSFDE_OK) return setup_fail(c, st, nullptr);
    if ((st = upload(c, &c->d_bhalf, c->b_half.data(), c->M)) != RSFDE_OK) return setup_fail(c, st, nullptr);
  } else {
    c->grid = p->e.grid;
    c->grid_static = p->e.grid_static;
  }
  // e-hat / e-check on the device
  {
    ECoef e = rsfde_ecoef_at(c, 0);
    if (c->ekind == RSFDE_COEF_GRID) e.grid = c->grid;
    double* part = nullptr;
    const int nblk = 4 * rsfde::device_sm_count();
    if ((st = dalloc(c, (void**)&part, 2 * nblk * sizeof(double))) != RSFDE_OK) return setup_fail(c, st, nullptr);
    const int Meff = (c->ekind == RSFDE_COEF_GRID && c->grid_static) ? 1 : c->M;
    cudaError_t ce = launch_emaxmin(e, c->d_ahalf, c->d_bhalf, Meff, c->grid_static, G, part, nblk, s);
    if (ce != cudaSuccess) return setup_fail(c, cuda_fail(c, ce, "emaxmin"), nullptr);
    std::vector<double> hp(2 * nblk);
    ce = cudaMemcpyAsync(hp.data(), part, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return setup_fail(c, cuda_fail(c, ce, "emaxmin copy"), nullptr);
    double mx = -INFINITY, mn = INFINITY;
    for (int b = 0; b < nblk; ++b) {
      mx = std::fmax(mx, hp[2 * b]);
      mn = std::fmin(mn, hp[2 * b + 1]);
    }
    c->ehat = mx;
    c->echeck = mn;
    c->ebar = 0.5 * (mx + mn);
    if (!(mn > 0.0)) return setup_fail(c, RSFDE_E_COEFF, "e-check <= 0: e must be positive (P:33)");
  }
  if (!alloc_work) {
    c->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = c;
    return RSFDE_OK;
  }
  // work memory
  const size_t vb = (size_t)G.NP * sizeof(double);
  double** bufs[] = {&c->W[0], &c->W[1], &c->W[2], &c->W[3], &c->Z, &c->X, &c->BUF, &c->U0, &c->FP, &c->FH, &c->TMP, &c->TMP2};
  for (double** b : bufs)
    if ((st = dalloc(c, (void**)b, vb)) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if ((st = dalloc(c, (void**)&c->d_vscale, 64 * sizeof(double))) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if ((st = dalloc(c, (void**)&c->d_h1, 64 * sizeof(double))) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if ((st = dalloc(c, (void**)&c->d_h2, 64 * sizeof(double))) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if ((st = dalloc(c, (void**)&c->d_part, (size_t)c->nblk * 128 * sizeof(double))) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if ((st = dalloc(c, (void**)&c->d_nrm, (size_t)c->nblk * sizeof(double))) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if ((st = dalloc(c, (void**)&c->d_state, sizeof(GmresState))) != RSFDE_OK) return setup_fail(c, st, nullptr);
  if (cudaMallocHost(&c->h_flags, 64) != cudaSuccess) return setup_fail(c, RSFDE_E_NOMEM, "cudaMallocHost");
  // the zeroing memsets ran on the legacy default stream: complete them before any caller stream
  if (cudaDeviceSynchronize() != cudaSuccess) return setup_fail(c, RSFDE_E_CUDA, "setup synchronisation");
  c->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = c;
  return RSFDE_OK;
}

rsfde_status rsfde_setup(rsfde_ctx** out, const rsfde_problem* p, void* stream) {
  return rsfde_setup_internal(out, p, stream, true);
}

rsfde_status rsfde_ebar(const rsfde_ctx* c, double* ebar, double* ehat, double* echeck) {
  if (!c) return RSFDE_E_CONFIG;
  if (ebar) *ebar = c->ebar;
  if (ehat) *ehat = c->ehat;
  if (echeck) *echeck = c->echeck;
  return RSFDE_OK;
}

rsfde_status rsfde_table(const rsfde_ctx* c, int axis, int which, double* out) {
  if (!c || !out) return RSFDE_E_CONFIG;
  if (axis < 0 || axis >= c->d) return RSFDE_E_DIM;
  const std::vector<double>* t = nullptr;
  switch (which) {
    case 0: t = &c->s_tab[axis]; break;
    case 1: t = &c->q_tab[axis]; break;
    case 2: t = &c->lamH_tab[axis]; break;
    case 3: t = &c->chat_tab[axis]; break;
    case 4: out[0] = c->eta[axis]; return RSFDE_OK;
    default: return RSFDE_E_CONFIG;
  }
  memcpy(out, t->data(), t->size() * sizeof(double));
  return RSFDE_OK;
}

rsfde_status rsfde_matvec(rsfde_ctx* c, int op, int m, const double* x, double* y, void* stream) {
  if (!c) return RSFDE_E_CONFIG;
  if (!x || !y || x == y) return RSFDE_E_DIM;
  if (m < 0 || m >= c->M) return RSFDE_E_DOMAIN;
  const cudaStream_t s = S(stream);
  CKL(launch_pack(x, c->BUF, c->geo, s), "pack");
  ChainArgs a;
  a.R = c->BUF;
  a.m = m;
  double* res = c->Z;
  switch (op) {
    case RSFDE_OP_A: TRY(oper_chain(c, a, c->Z, s)); break;
    case RSFDE_OP_ATILDE:
      TRY(oper_chain(c, a, c->TMP2, s));
      TRY(precond_chain(c, SPEC_HINV, c->TMP2, c->Z, s));
      break;
    case RSFDE_OP_S_ALPHA: a.xmode = X_ZERO; TRY(oper_chain(c, a, c->Z, s)); break;
    case RSFDE_OP_H_ALPHA:
      a.xmode = X_INPUT;
      a.Xin = c->BUF;
      a.etafac = 0.0;
      TRY(oper_chain(c, a, c->Z, s));
      break;
    case RSFDE_OP_H_ALPHA_INV: TRY(precond_chain(c, SPEC_HINV, c->BUF, c->Z, s)); break;
    case RSFDE_OP_K:
      a.spectral = true;
      a.spec = SPEC_PHAT;
      TRY(oper_chain(c, a, c->Z, s));
      break;
    default: c->err = "unknown operator"; return RSFDE_E_CONFIG;
  }
  CKL(launch_unpack(res, y, c->geo, s), "unpack");
  return RSFDE_OK;
}

rsfde_status rsfde_precond_apply(rsfde_ctx* c, int kind, const double* x, double* y, void* stream) {
  if (!c) return RSFDE_E_CONFIG;
  if (!x || !y || x == y) return RSFDE_E_DIM;
  int sk;
  switch (kind) {
    case RSFDE_PHAT_INV: sk = SPEC_PHAT; break;
    case RSFDE_PALPHA_INV: sk = SPEC_PALPHA; break;
    case RSFDE_PALPHA_INV_SQRT: sk = SPEC_PALPHA_SQRT; break;
    default: c->err = "unknown preconditioner"; return RSFDE_E_CONFIG;
  }
  const cudaStream_t s = S(stream);
  CKL(launch_pack(x, c->BUF, c->geo, s), "pack");
  TRY(precond_chain(c, sk, c->BUF, c->Z, s));
  CKL(launch_unpack(c->Z, y, c->geo, s), "unpack");
  return RSFDE_OK;
}

rsfde_status rsfde_compact_source(rsfde_ctx* c, const double* f_closed, double* F, void* stream) {
  if (!c) return RSFDE_E_CONFIG;
  if (!f_closed || !F) return RSFDE_E_DIM;
  const cudaStream_t s = S(stream);
  CKL(launch_compact_source(f_closed, F, c->geo, c->alpha, s), "compact source");
  return RSFDE_OK;
}

static rsfde_status check_cfg(rsfde_ctx* c, const rsfde_gmres_cfg* cfg) {
  if (!cfg || cfg->restart < 1 || cfg->restart > 50 || (cfg->fixed_iters <= 0 && !(cfg->tol >= 0.0)) ||
      (cfg->form != RSFDE_FORM_A && cfg->form != RSFDE_FORM_ATILDE && cfg->form != RSFDE_FORM_TWO_SIDED) ||
      (cfg->x0_policy != RSFDE_X0_PREV && cfg->x0_policy != RSFDE_X0_ZERO)) {
    c->err = "bad GMRES configuration (restart in 1..50, tol >= 0, form, x0_policy)";
    return RSFDE_E_CONFIG;
  }
  return RSFDE_OK;
}

rsfde_status rsfde_gmres_step(rsfde_ctx* c, int m, const double* b, double* x, const rsfde_gmres_cfg* cfg, int* iters,
                              double* relres, int* converged, void* stream) {
  if (!c) return RSFDE_E_CONFIG;
  if (!b || !x) return RSFDE_E_DIM;
  if (m < 0 || m >= c->M) return RSFDE_E_DOMAIN;
  TRY(check_cfg(c, cfg));
  const cudaStream_t s = S(stream);
  CKL(launch_pack(b, c->BUF, c->geo, s), "pack b");
  if (cfg->x0_policy == RSFDE_X0_ZERO) CK(cudaMemsetAsync(c->X, 0, c->geo.NP * sizeof(double), s), "memset");
  else CKL(launch_pack(x, c->X, c->geo, s), "pack x");
  TRY(gmres_core(c, m, false, true, *cfg, s, iters, relres, converged));
  CKL(launch_unpack(c->X, x, c->geo, s), "unpack");
  return RSFDE_OK;
}

static bool is_host_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

// dense vector (device or host) -> padded device vector dst, staging host data through Z
static rsfde_status load_dense(rsfde_ctx* c, const double* src, bool host, double* dst, cudaStream_t s) {
  const long long N = (long long)c->n[0] * c->n[1] * c->n[2];
  const double* dsrc = src;
  if (host) {
    CK(cudaMemcpyAsync(c->Z, src, N * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    dsrc = c->Z;
  }
  CKL(launch_pack(dsrc, dst, c->geo, s), "pack");
  return RSFDE_OK;
}

rsfde_status rsfde_solve_steps(rsfde_ctx* c, int m_begin, int m_count, double* u, const double* F, int F_static,
                               const rsfde_gmres_cfg* cfg, rsfde_report* rep, void* stream) {
  if (!c) return RSFDE_E_CONFIG;
  if (!u) return RSFDE_E_DIM;
  if (m_begin < 0 || m_count < 0 || m_begin + m_count > c->M) return RSFDE_E_DOMAIN;
  TRY(check_cfg(c, cfg));
  const cudaStream_t s = S(stream);
  const long long N = (long long)c->n[0] * c->n[1] * c->n[2];
  const size_t vb = (size_t)c->geo.NP * sizeof(double);
  const bool u_host = is_host_ptr(u);
  const bool f_host = F ? is_host_ptr(F) : false;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0), "event");
  CK(cudaEventCreate(&e1), "event");
  CK(cudaEventRecord(e0, s), "event record");
  TRY(load_dense(c, u, u_host, c->X, s));
  // FP = F, FH = tau H^{-1} F (first-cycle residual shortcut)
  auto prepare_F = [&](const double* Fm) -> rsfde_status {
    if (!Fm) {
      CK(cudaMemsetAsync(c->FP, 0, vb, s), "memset");
      CK(cudaMemsetAsync(c->FH, 0, vb, s), "memset");
      return RSFDE_OK;
    }
    TRY(load_dense(c, Fm, f_host, c->FP, s));
    TRY(precond_chain(c, SPEC_HINV, c->FP, c->FH, s));
    CKL(launch_axpby(0.0, c->FH, c->tau, c->FH, c->geo.NP, s), "scale");
    return RSFDE_OK;
  };
  long long total = 0;
  bool stopped = false;
  // small 1-D problems: the whole march in one on-chip kernel (no host round trip per iteration)
  const bool onchip = onchip_eligible(c, cfg) && m_count > 0;
  if (onchip) {
    TRY(onchip_march(c, m_begin, m_count, F, F_static, f_host, *cfg, s, rep, &total));
    m_count = 0;  // skip the generic loop below
  } else if (!F || F_static) {
    TRY(prepare_F(F));
  }
  for (int k = 0; k < m_count; ++k) {
    const int m = m_begin + k;
    if (stopped) {
      if (rep && rep->iters) rep->iters[k] = -1;
      continue;
    }
    if (F && !F_static) TRY(prepare_F(F + (long long)k * N));
    CK(cudaMemcpyAsync(c->U0, c->X, vb, cudaMemcpyDeviceToDevice, s), "copy u0");
    int its = 0, conv = 0;
    double rr = 0;
    if (cfg->x0_policy == RSFDE_X0_ZERO) {
      TRY(compute_b(c, m, s));
      CK(cudaMemsetAsync(c->X, 0, vb, s), "memset x");
      TRY(gmres_core(c, m, false, true, *cfg, s, &its, &rr, &conv));
    } else {
      TRY(gmres_core(c, m, cfg->form != RSFDE_FORM_TWO_SIDED, false, *cfg, s, &its, &rr, &conv));
    }
    total += its;
    if (rep) {
      if (rep->iters) rep->iters[k] = its;
      if (rep->final_relres) rep->final_relres[k] = rr;
      if (rep->converged) rep->converged[k] = (unsigned char)conv;
    }
    if (!conv) stopped = true;
  }
  if (u_host) {
    CKL(launch_unpack(c->X, c->Z, c->geo, s), "unpack");
    CK(cudaMemcpyAsync(u, c->Z, N * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
  } else {
    CKL(launch_unpack(c->X, u, c->geo, s), "unpack");
  }
  CK(cudaEventRecord(e1, s), "event record");
  CK(cudaEventSynchronize(e1), "event sync");
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->loop_seconds = ms * 1e-3;
    rep->setup_seconds = c->setup_seconds;
    rep->total_iters = total;
  }
  return RSFDE_OK;
}

// NEXT-4 batched kernel: every system of the batch marches in its own CTA of ONE launch (all 1-D,
// on-chip eligible, one device); u / F may be host or device memory per system
static rsfde_status onchip_batch(int count, rsfde_ctx* const* ctxs, const int* m_begin, const int* m_count,
                                 double* const* u, const double* const* F, const int* F_static,
                                 const rsfde_gmres_cfg* cfgs, rsfde_report* reps) {
  rsfde_ctx* c = ctxs[0];  // error reporting + LAUNCH accounting of the shared launch
  CK(cudaSetDevice(c->device), "set device");
  cudaStream_t s = nullptr;
  cudaEvent_t ready = nullptr, e0 = nullptr, e1 = nullptr;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
  CK(cudaEventRecord(ready, cudaStreamLegacy), "event");
  CK(cudaStreamWaitEvent(s, ready, 0), "wait");
  CK(cudaEventCreate(&e0), "event");
  CK(cudaEventCreate(&e1), "event");
  CK(cudaEventRecord(e0, s), "event");
  std::vector<OnchipParams> ps(count);
  std::vector<bool> uh(count);
  size_t smem = 0;
  for (int i = 0; i < count; ++i) {
    rsfde_ctx* ci = ctxs[i];
    uh[i] = is_host_ptr(u[i]);
    const double* Fi = F ? F[i] : nullptr;
    const int Fs = F_static ? F_static[i] : 1;
    {
      rsfde_ctx* c = ci;  // (the macros report into the system's context)
      TRY(load_dense(c, u[i], uh[i], c->X, s));
      TRY(onchip_prepare(c, m_begin[i], m_count[i], Fi, Fs, Fi ? is_host_ptr(Fi) : false, cfgs[i], s, &ps[i]));
    }
    const size_t b = onchip_smem_bytes(ci->n[0], cfgs[i].restart);
    smem = b > smem ? b : smem;
  }
  OnchipParams* d_ps = nullptr;
  CK(cudaMallocAsync((void**)&d_ps, count * sizeof(OnchipParams), s), "alloc params");
  CK(cudaMemcpyAsync(d_ps, ps.data(), count * sizeof(OnchipParams), cudaMemcpyHostToDevice, s), "params");
  LAUNCH(PC_OPER_SPEC, 0.0, launch_onchip_1d_batch(d_ps, count, smem, s), "batched on-chip march");
  for (int i = 0; i < count; ++i) {
    rsfde_ctx* c = ctxs[i];
    const long long N = c->n[0];
    if (uh[i]) {
      CKL(launch_unpack(c->X, c->Z, c->geo, s), "unpack");
      CK(cudaMemcpyAsync(u[i], c->Z, N * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    } else {
      CKL(launch_unpack(c->X, u[i], c->geo, s), "unpack");
    }
  }
  CK(cudaEventRecord(e1, s), "event");
  CK(cudaFreeAsync(d_ps, s), "free params");
  CK(cudaStreamSynchronize(s), "sync");
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  for (int i = 0; i < count; ++i) {
    long long total = 0;
    rsfde_report* rep = reps ? &reps[i] : nullptr;
    TRY(onchip_collect(ctxs[i], m_count[i], rep, &total));
    if (rep) {
      rep->loop_seconds = ms * 1e-3;  // the whole batch (one launch)
      rep->setup_seconds = ctxs[i]->setup_seconds;
      rep->total_iters = total;
    }
  }
  cudaEventDestroy(ready);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  return RSFDE_OK;
}

rsfde_status rsfde_solve_steps_batch(int count, rsfde_ctx* const* ctxs, const int* m_begin, const int* m_count,
                                     double* const* u, const double* const* F, const int* F_static,
                                     const rsfde_gmres_cfg* cfgs, rsfde_report* reps, void* const* streams) {
  if (count < 0 || (count > 0 && (!ctxs || !m_begin || !m_count || !u || !cfgs))) return RSFDE_E_CONFIG;
  for (int i = 0; i < count; ++i)
    for (int k = 0; k < i; ++k)
      if (ctxs[i] == ctxs[k]) {
        if (ctxs[i]) ctxs[i]->err = "rsfde_solve_steps_batch: a context appears twice in the batch";
        return RSFDE_E_CONFIG;
      }
  // all systems 1-D and on-chip eligible on one device (and no caller streams): one launch, one CTA
  // per system (RSFDE_NO_BATCH_KERNEL=1 selects the stream-per-system path below)
  {
    const bool no_kernel = getenv("RSFDE_NO_BATCH_KERNEL") != nullptr;
    bool all = count >= 1 && !no_kernel;
    for (int i = 0; all && i < count; ++i) {
      const rsfde_ctx* c = ctxs[i];
      all = c && (!streams || !streams[i]) && c->device == ctxs[0]->device && m_begin[i] >= 0 && m_count[i] > 0 &&
            m_begin[i] + m_count[i] <= c->M && check_cfg(const_cast<rsfde_ctx*>(c), &cfgs[i]) == RSFDE_OK &&
            onchip_eligible(c, &cfgs[i]);
    }
    if (all) return onchip_batch(count, ctxs, m_begin, m_count, u, F, F_static, cfgs, reps);
  }
  std::vector<rsfde_status> st(count, RSFDE_OK);
  std::vector<cudaStream_t> own(count, nullptr);
  // Streams the library creates are ordered after the work already queued on the legacy default
  // stream (an event recorded there is waited on); callers that produced u / F on other streams
  // synchronise those first (the Python binding synchronises torch's current stream).
  std::vector<cudaEvent_t> ready(count, nullptr);
  for (int i = 0; i < count; ++i) {
    if (streams && streams[i]) continue;
    if (!ctxs[i] || cudaSetDevice(ctxs[i]->device) != cudaSuccess ||
        cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ready[i], cudaStreamLegacy) != cudaSuccess)
      return RSFDE_E_CUDA;
  }
  // one host worker and one stream per system: the independent marches overlap on the device (small
  // grids leave most SMs idle) and their per-iteration host syncs overlap on the host
  auto work = [&](int i) {
    rsfde_ctx* c = ctxs[i];
    if (!c) { st[i] = RSFDE_E_CONFIG; return; }
    if (cudaSetDevice(c->device) != cudaSuccess) { st[i] = RSFDE_E_CUDA; return; }
    void* s = streams ? streams[i] : nullptr;
    if (!s) {
      if (cudaStreamCreateWithFlags(&own[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamWaitEvent(own[i], ready[i], 0) != cudaSuccess) { st[i] = RSFDE_E_CUDA; return; }
      s = own[i];
    }
    st[i] = rsfde_solve_steps(c, m_begin[i], m_count[i], u[i], F ? F[i] : nullptr, F_static ? F_static[i] : 1,
                              &cfgs[i], reps ? &reps[i] : nullptr, s);
    if (own[i]) cudaStreamSynchronize(own[i]);
  };
  std::vector<std::thread> th;
  th.reserve(count > 0 ? count - 1 : 0);
  for (int i = 1; i < count; ++i) th.emplace_back(work, i);
  if (count > 0) work(0);
  for (auto& t : th) t.join();
  for (int i = 0; i < count; ++i) {
    if (own[i]) cudaStreamDestroy(own[i]);
    if (ready[i]) cudaEventDestroy(ready[i]);
  }
  for (int i = 0; i < count; ++i)
    if (st[i] != RSFDE_OK) return st[i];
  return RSFDE_OK;
}

}  // extern "C"
