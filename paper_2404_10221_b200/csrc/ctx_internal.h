// Internal (not part of the ABI): the context structure shared by the single-GPU host code
// (rsfde_host.cu) and the slab-sharded module (rsfde_shard.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/rsfde.h"
#include "kernels.cuh"

#define RSFDE_NPROF 8
enum { ORTHO_DCGS2 = 0, ORTHO_CGS2 = 1 };

using rsfde::Geom;
using rsfde::GmresState;

struct rsfde_ctx {
  int device = 0;  // CUDA device the context lives on (set by setup)
  int nblk = 0;    // blocks (= partial sums) of the streaming reductions: 8 per SM of that device
  int ortho = 0;   // ORTHO_DCGS2 | ORTHO_CGS2
  const int* skip = nullptr;             // device flags of the speculative Arnoldi launches (PassParams::skip)
  // graph-captured first GMRES cycle of a CN step (rsfde_host.cu gmres_graph): r0, the Arnoldi steps as
  // nested conditional IF nodes and the y solve / x update as a SWITCH on the column count.  The time
  // level reaches the captured kernels through the device slot d_ab = {a(t), b(t)} (ECoef::ab).
  struct StepGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int restart = 0, max_iters = 0, fixed = 0, nsteps = 0;
    double tol = 0;
    long long launches_pre = 0;
    std::vector<long long> launches_step, launches_end;  // per Arnoldi step j / per final column count k
  } sg;
  long long graph_replays = 0;
  double* d_ab = nullptr;
  bool ab_dev = false;  // rsfde_ecoef_at points ECoef::ab at d_ab (set while capturing)
  cudaStream_t cap_s[2] = {nullptr, nullptr};
  cudaEvent_t flag_ev[2] = {nullptr, nullptr};  // flags copies of the last two Arnoldi steps
  // on-chip 1-D march (lazily allocated): generator table, per-step outputs, device copy of host F
  double* d_s0 = nullptr;
  int* d_on_iters = nullptr;
  double* d_on_relres = nullptr;
  unsigned char* d_on_conv = nullptr;
  double* d_on_F = nullptr;
  long long on_F_cap = 0;
  int d = 0;
  int n[3] = {1, 1, 1};
  double alpha[3] = {2, 2, 2}, kappa[3] = {0, 0, 0};
  double tau = 0;
  int M = 0;
  Geom geo{};
  double eta[3] = {0, 0, 0};
  // host copies of the 1-D tables (long double computed, FP64 stored)
  std::vector<double> s_tab[3], q_tab[3], lamH_tab[3], chat_tab[3];
  // device tables
  double* d_chat[3] = {nullptr, nullptr, nullptr};
  double2* d_tw[3] = {nullptr, nullptr, nullptr};
  double* d_lamH[3] = {nullptr, nullptr, nullptr};
  double* d_q[3] = {nullptr, nullptr, nullptr};
  double* d_tq[3] = {nullptr, nullptr, nullptr};
  // row-layout copies (PassParams::chat_rl ...), axes with L = 4096 only
  double* d_chat_rl[3] = {nullptr, nullptr, nullptr};
  double* d_lamH_rl[3] = {nullptr, nullptr, nullptr};
  double* d_tq_rl[3] = {nullptr, nullptr, nullptr};
  // coefficient e
  int ekind = RSFDE_COEF_SEPARABLE;
  std::vector<double> a_half, b_half;
  double* d_g[3] = {nullptr, nullptr, nullptr};
  double* d_k[3] = {nullptr, nullptr, nullptr};
  double *d_ahalf = nullptr, *d_bhalf = nullptr;
  const double* grid = nullptr;
  int grid_static = 0;
  double ebar = 0, ehat = 0, echeck = 0;
  // work vectors (padded layout, zero pads)
  double* W[4] = {nullptr, nullptr, nullptr, nullptr};
  double *Z = nullptr, *X = nullptr, *BUF = nullptr, *U0 = nullptr, *FP = nullptr, *FH = nullptr;
  double *TMP = nullptr, *TMP2 = nullptr;
  std::vector<double*> V;
  double* d_vscale = nullptr;
  double *d_h1 = nullptr, *d_h2 = nullptr, *d_part = nullptr, *d_nrm = nullptr;
  GmresState* d_state = nullptr;
  void* h_flags = nullptr;  // pinned 16 bytes: converged, breakdown, relres
  long long bytes = 0;
  long long launches = 0;
  double setup_seconds = 0;
  std::string err;
  std::vector<void*> allocs;
  // optional per-launch event timing (rsfde_profile): class -> launches, ms, algorithmic bytes
  int pass_flags = 0;  // PASS_FLAG_* (RSFDE_NO_PIPE=1 disables the cp.async-pipelined passes)
  int profiling = 0;
  cudaStream_t prof_stream = nullptr;
  struct Pending {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_events;
  long long prof_launches[RSFDE_NPROF] = {0};
  double prof_ms[RSFDE_NPROF] = {0};
  double prof_bytes[RSFDE_NPROF] = {0};
};


// setup without the work vectors / basis (tables, e-bar only)
extern "C" rsfde_status rsfde_setup_internal(rsfde_ctx** out, const rsfde_problem* p, void* stream, bool alloc_work);
// pass parameters of one axis of the context's (unsharded) grid
rsfde::PassParams rsfde_axis_params(const rsfde_ctx* c, int axis);
rsfde::ECoef rsfde_ecoef_at(const rsfde_ctx* c, int m);
