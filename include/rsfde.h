/*
 * rsfde.h -- C ABI of the B200 (sm_100a) tau-preconditioned GMRES solver for the
 * Crank-Nicolson / quasi-compact discretisation of the d-dimensional Riesz space
 * fractional diffusion equation of arXiv 2404.10221 (PAPER.md, cited as P:<line>).
 *
 *   e(x,t) d_t u = sum_i kappa_i d^{alpha_i} u + f  on (0,1)^d,  u = 0 on the boundary
 *
 * Per CN step m the library solves Eq.(tls)
 *     A^{(m)} u^{(m+1)} = (H_alpha E^{(m+1/2)} + S_alpha) u^{(m+1)}
 *                       = (H_alpha E^{(m+1/2)} - S_alpha) u^{(m)} + tau F^{(m+1/2)} = b^{(m)}
 * with GMRES preconditioned on the left by the sine-transform (tau) preconditioner.  The
 * paper's one-sided system P_alpha^{-1} A~ u = P_alpha^{-1} b~ (Eq.(one-sided), P:217-221,
 * A~ = E + H^{-1} S_alpha, b~ = H^{-1} b) is the same Krylov process as
 * P_hat^{-1} A u = P_hat^{-1} b with P_hat = H_alpha P_alpha = ebar H_alpha + tau(S_alpha),
 * because tau matrices commute; the default "A form" runs the latter.
 *
 * Conventions
 *  - All compute runs in hand-written FP64 CUDA kernels on the stream passed in (a
 *    cudaStream_t given as void*; NULL = legacy default stream).  There is no CPU fallback:
 *    without a usable CUDA device every call returns RSFDE_E_CUDA.
 *  - Grid vectors are FP64 values at the interior nodes x_J = (j_1 h_1, ..., j_d h_d),
 *    h_i = 1/(n_i+1), j_i = 1..n_i, stored densely in C order [x_1][x_2][x_3]
 *    (x_d fastest), N = prod n_i values.  (The paper's vector orders x_1 fastest, P:104;
 *    the values are the same grid function.)
 *  - Unless stated otherwise vector arguments are caller-owned DEVICE pointers.  The ctx
 *    owns its tables, Krylov basis and work buffers (padded private layout).
 *  - A ctx is used by one host thread at a time.  Calls are stream-ordered; only GMRES
 *    calls synchronise the stream to read the convergence flags: once per GMRES cycle of a CN
 *    step when the cycle runs as a captured CUDA graph (the default of rsfde_solve_steps, see
 *    rsfde_graph_replays), once per Arnoldi step otherwise (one step ahead: the kernels of step
 *    j+1 are already queued when the flags of step j are read).
 *  - Restriction: every n_i + 1 must be a power of two with 2 <= n_i + 1 <= 2048 (FFT lengths
 *    L = 2(n_i+1) <= 4096 are built); otherwise RSFDE_E_DIM.  The paper's grids (N+1 = 2^k,
 *    P:532-633) and all five BASELINE configs (n = 255, 255^2, 2047^2, 255^3, 511^3) satisfy it.
 */
#ifndef RSFDE_H
#define RSFDE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rsfde_ctx rsfde_ctx; /* opaque */

typedef enum {
  RSFDE_OK = 0,
  RSFDE_E_DIM = 1,    /* d not in {1,2,3}, n_i < 1, n_i+1 not a power of two or too large, NULL vector */
  RSFDE_E_DOMAIN = 2, /* alpha_i not in (1,2] (alpha = 2 kept as the classical limit), kappa_i <= 0,
                         tau_t <= 0, M < 1, m out of [0, M) */
  RSFDE_E_COEFF = 3,  /* e-check <= 0: e must be positive with a positive minimum */
  RSFDE_E_CONFIG = 4, /* missing coefficient tables, bad GMRES configuration */
  RSFDE_E_CUDA = 5,   /* CUDA error (message in rsfde_last_error) */
  RSFDE_E_NCCL = 6,   /* NCCL missing (libnccl.so.2 is dlopen'ed) or an NCCL call of the rsfde_team_* API failed */
  RSFDE_E_NOMEM = 7   /* device allocation failed */
} rsfde_status;

/* coefficient e(x,t) at the half levels t_{m+1/2} = (m+1/2) tau (Eq.(tls)) */
enum { RSFDE_COEF_SEPARABLE = 0, RSFDE_COEF_GRID = 1 };

typedef struct {
  int kind;
  /* SEPARABLE: e(x, t_{m+1/2}) = a_half[m] + b_half[m] * prod_i g_i(x_i) + sum_i k_i(x_i)
     (all five BASELINE configs and the paper's Examples 1-3 have this form).
     Host arrays, copied at setup: a_half, b_half of length M; g[i], k[i] of length n_i
     sampled at the interior nodes of axis i; NULL g[i] means 1, NULL k[i] means 0. */
  const double *a_half, *b_half;
  const double *g[3], *k[3];
  /* GRID: device pointer to e at the interior nodes in the dense layout, M*N values
     (step m at offset m*N) or N values if grid_static != 0.  Not copied: must stay valid. */
  const double *grid;
  int grid_static;
} rsfde_coeff;

typedef struct {
  int d;             /* 1, 2 or 3 */
  int n[3];          /* interior points per axis (n_i = N in the paper) */
  double alpha[3];   /* fractional orders, 1 < alpha_i <= 2 */
  double kappa[3];   /* diffusion coefficients > 0 */
  double tau_t;      /* time step tau = T/M */
  int M;             /* number of CN steps (defines the half levels for e-bar) */
  rsfde_coeff e;
} rsfde_problem;

/* operators for rsfde_matvec (x -> y, time level m for E^{(m+1/2)}) */
enum {
  RSFDE_OP_A = 0,           /* A^{(m)} = H_alpha E + S_alpha                       (Eq.(tls)) */
  RSFDE_OP_ATILDE = 1,      /* A~ = E + H_alpha^{-1} S_alpha                        (Eq.(equi)) */
  RSFDE_OP_S_ALPHA = 2,     /* S_alpha, Eq.(Salpha)                                          */
  RSFDE_OP_H_ALPHA = 3,     /* H_alpha = H_{alpha_d} (x) ... (x) H_{alpha_1}       */
  RSFDE_OP_H_ALPHA_INV = 4, /* H_alpha^{-1} (H is a tau matrix)                                */
  RSFDE_OP_K = 5            /* the preconditioned operator P_hat^{-1} A = P_alpha^{-1} A~     */
};

/* preconditioners for rsfde_precond_apply */
enum {
  RSFDE_PHAT_INV = 0,        /* (ebar H_alpha + tau(S_alpha))^{-1} = S Lambda_hat^{-1} S              */
  RSFDE_PALPHA_INV = 1,      /* P_alpha^{-1} = S Lambda_P^{-1} S, P_alpha of Eq.(Pa)          */
  RSFDE_PALPHA_INV_SQRT = 2  /* P_alpha^{-1/2} = S Lambda_P^{-1/2} S (Eq.(Pls))                */
};

enum { RSFDE_X0_PREV = 0, RSFDE_X0_ZERO = 1 };
/* FORM_A: P_hat^{-1} A u = P_hat^{-1} b (== the paper's one-sided system, default);
   FORM_ATILDE: the literal P_alpha^{-1} A~ u = P_alpha^{-1} b~ chain;
   FORM_TWO_SIDED: the two-sided system P_alpha^{-1/2} A~ P_alpha^{-1/2} u~ = P_alpha^{-1/2} b~,
   u = P_alpha^{-1/2} u~ (Eq.(Pls)), started from u~_0 = P_alpha^{1/2} x_0 (Thm 3.9). */
enum { RSFDE_FORM_A = 0, RSFDE_FORM_ATILDE = 1, RSFDE_FORM_TWO_SIDED = 2 };

typedef struct {
  int restart;      /* GMRES(m) restart length, 1..50 */
  int max_iters;    /* cap on Arnoldi steps per solve (<= 0: 10*restart) */
  double tol;       /* stop when |g_{j+1}| <= tol * ||r_0|| (preconditioned residual) */
  int x0_policy;    /* RSFDE_X0_PREV: x_0 = u^{(m)} (default); RSFDE_X0_ZERO */
  int form;         /* RSFDE_FORM_A (default), RSFDE_FORM_ATILDE or RSFDE_FORM_TWO_SIDED */
  int fixed_iters;  /* > 0: replay mode for parity: ignore tol and run exactly this many
                       Arnoldi steps, restarting every `restart` steps as needed (a lucky breakdown
                       still ends the solve early); the step is then reported converged */
} rsfde_gmres_cfg;

typedef struct {
  int *iters;               /* caller arrays of length m_count, may be NULL */
  double *final_relres;     /* |g_{k+1}| / ||r_0|| at the last step of each solve */
  unsigned char *converged;
  double loop_seconds;      /* device time of the step loop (CUDA events) */
  double setup_seconds;     /* host time of rsfde_setup */
  long long total_iters;
} rsfde_report;

/* Set up: validate, build the 1-D tables on the host in long double (FCD generator P:124-127
   with the alpha/2+k reading, tau eigenvalues q_i (P:158 with divisor N+1), circulant
   spectra, twiddles, lambda^H), upload them, reduce e-hat/e-check on the device
   (P:188-194).  *out receives a new context or NULL on error. */
rsfde_status rsfde_setup(rsfde_ctx **out, const rsfde_problem *p, void *stream);

/* y = op x (device pointers, dense layout, must not alias). */
rsfde_status rsfde_matvec(rsfde_ctx *ctx, int op, int m, const double *x, double *y, void *stream);

/* y = P^{-1} x for the preconditioner kind (device pointers, dense layout, may not alias). */
rsfde_status rsfde_precond_apply(rsfde_ctx *ctx, int kind, const double *x, double *y, void *stream);

/* One GMRES solve of A^{(m)} x = b (device pointers, dense layout): x holds x_0 on entry and
   the solution on exit.  iters/relres/converged are host outputs (may be NULL). */
rsfde_status rsfde_gmres_step(rsfde_ctx *ctx, int m, const double *b, double *x, const rsfde_gmres_cfg *cfg,
                              int *iters, double *relres, int *converged, void *stream);

/* March m_count CN steps from level m_begin: u holds u^{(m_begin)} on entry and
   u^{(m_begin+m_count)} on exit.  F holds F^{(m+1/2)} (the compact-stencil source of the
   Appendix) per step (m_count*N values, step k at offset k*N) or one static
   vector (F_static != 0); F == NULL means F = 0.  u and F may be DEVICE or HOST pointers
   (host pointers are staged through device memory inside the call; the copies are timed
   in loop_seconds).  Returns RSFDE_OK also when a step did not converge: the report flags
   it and the march stops at that step (rep->iters of later steps = -1).
   Small 1-D problems (d = 1, A form, separable e, x0 = u^(m), no replay, restart <= 50 and the
   basis within ~200 KB of shared memory) run the whole march in one on-chip kernel (one CTA:
   no host synchronisation per GMRES iteration); the environment variable RSFDE_NO_ONCHIP=1
   selects the generic path.  Both follow the same algorithm (results agree to rounding). */
rsfde_status rsfde_solve_steps(rsfde_ctx *ctx, int m_begin, int m_count, double *u, const double *F, int F_static,
                               const rsfde_gmres_cfg *cfg, rsfde_report *rep, void *stream);

/* Batched march (the alpha / N sweeps of Tables 1-3, as many
   independent systems at once).  Runs rsfde_solve_steps(ctxs[i], m_begin[i], m_count[i], u[i],
   F[i], F_static[i], &cfgs[i], &reps[i], streams[i]) for i < count.  When every system is 1-D and
   eligible for the on-chip march (see rsfde_solve_steps), all contexts live on one device and no
   streams are given, the whole batch is ONE kernel launch with one CTA per system (each CTA marches
   its system with its own n, alpha, restart, tolerance, source and time levels; loop_seconds is then
   the time of the whole batch; RSFDE_NO_BATCH_KERNEL=1 disables this).  Otherwise: one host worker
   and one CUDA stream per system (streams may be NULL or hold NULL entries: the library then creates
   a non-blocking stream for that system, orders it after the work already queued on the legacy
   default stream, and synchronizes and destroys it before returning; inputs produced on other
   streams must be synchronized by the caller first).  The
   systems must be distinct contexts (RSFDE_E_CONFIG otherwise); each system's results are exactly
   those of its own rsfde_solve_steps call (same kernels, deterministic reductions).  F and F_static
   may be NULL (no source / static).  Returns the first failing system's status (the per-system
   error text is in rsfde_last_error(ctxs[i])); the other systems still run to completion. */
rsfde_status rsfde_solve_steps_batch(int count, rsfde_ctx *const *ctxs, const int *m_begin, const int *m_count,
                                     double *const *u, const double *const *F, const int *F_static,
                                     const rsfde_gmres_cfg *cfgs, rsfde_report *reps, void *const *streams);

/* F^{(m+1/2)} from f(., t_{m+1/2}) sampled on the CLOSED grid (n_i + 2 points per axis, dense C
   layout, boundary samples included): F = (prod_l calH_{alpha_l} f) restricted to the interior,
   calH_l g_j = (1 - alpha_l/12) g_j + alpha_l/24 (g_{j-1} + g_{j+1}) (Eq.(2.2)).  This
   equals the Appendix vectors for d = 1, 2 and is the reading of the garbled d = 3
   Appendix.  Device pointers; N outputs. */
rsfde_status rsfde_compact_source(rsfde_ctx *ctx, const double *f_closed, double *F, void *stream);

/* e-bar = (e-hat + e-check)/2 (Eq.(bard)) and the extremes (host outputs). */
rsfde_status rsfde_ebar(const rsfde_ctx *ctx, double *ebar, double *ehat, double *echeck);

/* Copy a 1-D setup table of axis i (0-based) to host memory `out` (n_i values unless
   stated): which = 0 FCD generator s_k (k=0..n-1), 1 tau eigenvalues q, 2 lambda^H,
   3 circulant spectrum c^ (L = 2(n_i+1) values, NOT divided by L), 4 eta_i (1 value). */
rsfde_status rsfde_table(const rsfde_ctx *ctx, int axis, int which, double *out);

/* Bytes of device memory the context holds (tables, work vectors, basis). */
long long rsfde_device_bytes(const rsfde_ctx *ctx);

/* Kernel launches issued since setup (or the last reset) -- evidence for bench.py. */
long long rsfde_launch_count(const rsfde_ctx *ctx, int reset);

/* Replays of the graph-captured first GMRES cycle since setup.  By default (A form, first-cycle
   residual shortcut, DCGS2) the first cycle of every CN step of rsfde_solve_steps runs as ONE CUDA
   graph whose Arnoldi steps are conditional nodes gated on the device-side convergence flag (stopping
   rule P:513), so the host reads the flags once per cycle; RSFDE_NO_GRAPH=1 in the environment selects
   the stream path (one flags read per Arnoldi step).  Results are bit-identical either way. */
long long rsfde_graph_replays(const rsfde_ctx *ctx);

/* Optional per-kernel timing: with enable != 0 every kernel launch is bracketed by CUDA events
   on its stream and attributed to one of the classes returned by rsfde_profile_read (0 ..
   count-1: spectral operator passes, physical operator passes, DST passes, CGS2 dots, CGS2
   dots after update, CGS2 update+norm, solution update, small kernels).  Resets the counters
   and returns the number of classes.  bytes = algorithmic HBM bytes (reads + writes of FP64
   vectors) of the launches in the class. */
int rsfde_profile(rsfde_ctx *ctx, int enable);
int rsfde_profile_read(rsfde_ctx *ctx, int cls, long long *launches, double *ms, double *bytes, const char **name);

/* ------------------------------------------------------------------------------------------
 * Slab-sharded 3D solver.  The grid is split along x_1 over nranks ranks (x_1 padded
 * to n_1+1, so nranks must divide n_1+1 and n_2+1; the pad plane is the DST-I zero).  Operator
 * passes along x_3 and x_2 run on the x_1-slabs; the fused DST . Lambda^{-1} . DST pass along x_1
 * runs after an all-to-all transpose to x_2-slabs (x_1 contiguous); CGS2 dots are allreduced.
 * nccl_id != NULL (nlocal must be 1): one rank per process, transport = NCCL (id from
 *             rsfde_nccl_unique_id on rank 0, broadcast by the caller; nranks = 1 is allowed and
 *             exercises the NCCL path on one GPU); vectors are the rank's slab x_1 in [x1_lo, x1_lo+count)
 *             (rsfde_team_slab), dense C layout [x_1 local][x_2][x_3].
 * nccl_id == NULL, nlocal = nranks: all ranks emulated in this process on one device (transport =
 *             device copies);
 *             vectors are the whole dense grid.  Used by the single-GPU parity tests.
 * Same conventions as above otherwise (device pointers, stream-ordered, A form only).  The
 * coefficient must be RSFDE_COEF_SEPARABLE (a dense grid e is not sliced per rank): RSFDE_E_CONFIG.
 * Streams: with nranks >= 2 the exchanges run piece by piece (sub-slabs of the x_1 slab,
 * RSFDE_TEAM_CHUNKS, default 4) on an internal exchange stream that is event-ordered with `stream`
 * in both directions: every call is still complete in `stream` order when it returns / when work
 * enqueued on `stream` after it runs.  All ranks must issue the same calls in the same order (one
 * NCCL communicator). */
typedef struct rsfde_team rsfde_team;
rsfde_status rsfde_nccl_unique_id(void *out128);
rsfde_status rsfde_team_setup(rsfde_team **out, const rsfde_problem *p, int nranks, int rank, int nlocal,
                              const void *nccl_id, void *stream);
rsfde_status rsfde_team_slab(const rsfde_team *t, int local, int *x1_lo, int *x1_count);
/* Host-only slab bookkeeping (no device needed): for rank of nranks on the grid n[3], out[0..5] =
   {x1_lo, x1_count (layout A slab; the last rank's count excludes the x1 pad plane), x2_lo, x2_count
   (layout T slab), s = (n1+1)/nranks, s2 = (n2+1)/nranks}; *block_elems = s2*n3*s, the doubles a rank
   sends to each peer per transposed vector, laid out [x2 local < s2][x3 < n3][x1 local < s].
   RSFDE_E_DIM unless nranks divides n1+1 and n2+1; RSFDE_E_CONFIG for bad rank / nranks (1..8). */
rsfde_status rsfde_team_partition(const int n[3], int nranks, int rank, int out[6], long long *block_elems);
/* Host-only piece bookkeeping of the chunked exchanges (no device needed): for nranks >= 2 the slab's
   s = (n1+1)/nranks planes are cut into out[0] = nchunk sub-slabs of out[1] = sc = s/nchunk planes --
   `requested` (<= 0: the RSFDE_TEAM_CHUNKS environment value, default 4) reduced until sc >= 2 divides s
   and nranks*nchunk <= 256 -- and every all-to-all block is laid out [chunk][x2 local < s2][x3 < n3]
   [x1 local < sc]: *piece_elems = s2*n3*sc doubles per (peer, chunk) piece, piece c of the block for
   peer r at offset r*block + c*piece.  The x_1 pencil (x2l, x3) of the receiving rank is the sequence of
   segments (r'', c), r'' = 0..nranks-1, c = 0..nchunk-1, of sc planes each.  nranks = 1: nchunk = 1.
   Errors as rsfde_team_partition. */
rsfde_status rsfde_team_chunking(const int n[3], int nranks, int requested, int out[2], long long *piece_elems);
/* op: RSFDE_OP_K (P_hat^{-1} A) or RSFDE_OP_A */
rsfde_status rsfde_team_matvec(rsfde_team *t, int op, int m, const double *x, double *y, void *stream);
rsfde_status rsfde_team_precond_apply(rsfde_team *t, int kind, const double *x, double *y, void *stream);
rsfde_status rsfde_team_solve_steps(rsfde_team *t, int m_begin, int m_count, double *u, const double *F,
                                    int F_static, const rsfde_gmres_cfg *cfg, rsfde_report *rep, void *stream);
/* F on the local slab of local rank `local` from f on the closed slab x_1 in [x1_lo-1, x1_lo+count],
   x_2, x_3 closed (count+2, n_2+2, n_3+2 values, dense) -- the compact stencil of
   rsfde_compact_source restricted to the slab. */
rsfde_status rsfde_team_compact_source(rsfde_team *t, int local, const double *f_closed_slab, double *F_slab,
                                       void *stream);
long long rsfde_team_launch_count(const rsfde_team *t, int reset);
const char *rsfde_team_last_error(const rsfde_team *t);
void rsfde_team_destroy(rsfde_team *t);

/* Last error message of ctx (or of the last failed setup if ctx == NULL). */
const char *rsfde_last_error(const rsfde_ctx *ctx);

void rsfde_destroy(rsfde_ctx *ctx);

/* library version string */
const char *rsfde_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RSFDE_H */
