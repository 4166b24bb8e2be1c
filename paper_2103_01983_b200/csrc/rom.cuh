// rom.cuh — device-side PTROM structures (reduction.hpp:18-302, rom.hpp:17-41).
#pragma once

#include <cuda_runtime.h>

namespace ptrom {

// PODBasis (reduction.hpp:18-26): phi is 2n x m column-major.
struct DBasis {
  long long n = 0;  // particles
  int m = 0;
  double* phi = nullptr;
  double* x_ref = nullptr;
  double* sv = nullptr;
  // Row-major copy for member gathers: particle p owns rm[p·2(m+1) ...]:
  // x row (Φ(p, 0..m-1), x_ref[p]) then y row (Φ(p+n, ·), x_ref[p+n]).
  double* rm = nullptr;
};

// GnatOperator (reduction.hpp:173-180) + the solver's gathered rows
// (rom.hpp:274-289). A is padded to 32 rows, phi_bar to mp columns
// (multiples of 8 for the DMMA tiles; padding is zero).
struct DGnat {
  long long n_s = 0;  // sampled particles (n_t)
  int m_r = 0, m = 0, mp = 0;
  long long* ids = nullptr;
  double* A = nullptr;        // 32 x 2n_s, column-major
  double* phi_bar = nullptr;  // 2n_s x mp, column-major
  double* x0_bar = nullptr;   // 2n_s
};

// SurrogateSourceBasis (reduction.hpp:280-302) in CSR form.
struct DSurrogate {
  int m = 0;
  long long n_c = 0, u = 0, n_t = 0;
  double* phi_tilde = nullptr;  // 2n_c x m, column-major
  double* x0_tilde = nullptr;   // 2n_c
  double* gamma_tilde = nullptr;
  unsigned char* zero_gamma = nullptr;
  long long* mem_off = nullptr;  // n_c + 1
  long long* mem_ids = nullptr;  // ascending particle ids per cluster
  long long max_members = 0;     // largest cluster (host-side; picks the reassign path)
  long long* target_ids = nullptr;
  int* t_order = nullptr;  // processing order of the targets (spatial; null = identity)
  long long* cl_off = nullptr;  // n_t + 1
  int* cl_list = nullptr;       // cluster indices
  long long* d_off = nullptr;   // n_t + 1
  int* d_list = nullptr;        // local direct indices
  long long* direct_ids = nullptr;
  double* direct_phi = nullptr;  // 2u x m, column-major
  double* direct_x0 = nullptr;
  double* direct_gamma = nullptr;
};

// Affine member sums for Γ(μ) = Γa + μ Γb (batched instances).
struct AffineTables {
  double *pa = nullptr, *pb = nullptr;  // 2n_c x m
  double *xa = nullptr, *xb = nullptr;  // 2n_c
  double *ga = nullptr, *gb = nullptr;  // n_c
  double *dga = nullptr, *dgb = nullptr;  // u (direct circulations)
};

// Engine-private row-major copies (tile-friendly operand layouts):
//   ct  [n_c][Q][mp]  cluster rows (Q = 4 affine: S_A x, S_A y, S_B x, S_B y;
//                     Q = 2 exact: Φ̃ x, Φ̃ y), zero-padded to mp modes
//   dt  [u][2][mp]    direct rows Φ_d x, Φ_d y
//   pbr [2 n_t][mp]   Φ̄ rows (x rows then y rows)
struct EngineTables {
  double* ct = nullptr;
  double* dt = nullptr;
  double* pbr = nullptr;
  int q = 2;
  // Γ/2π tables for hyperpair: exact Γ̃/2π, Γ_d/2π; affine (G_A, G_B)/2π, (Γa_d, Γb_d)/2π
  double* hgc = nullptr;
  double2* hgab = nullptr;
  double* hgd = nullptr;
  double2* hgdab = nullptr;
  int* hself = nullptr;  // [n_t] each target's slot in direct_ids or -1
};

// Per-instance Gauss–Newton state.
struct GnState {
  double* ac = nullptr;  // [B][32 x mp]
  double* ar = nullptr;  // [B][32]
  double* g0 = nullptr;
  int* evals = nullptr;
  unsigned char* active = nullptr;
  unsigned char* converged = nullptr;
  int* n_active = nullptr;
  double tol = 0;
  int max_iters = 0;
};

// Source positions per instance ([source][b]) and the pair counter.
struct RomScratch {
  // source positions, (x, y) interleaved: [cluster][instance], [direct][instance]
  double2 *cxy = nullptr, *dxy = nullptr;
  unsigned long long* pairs = nullptr;
  int* sm_ctr = nullptr;  // per-SM work counters of the per-SM hyperpair mapping
  static constexpr int kSmCtr = 1024;
  size_t cap_c = 0, cap_d = 0;
  void ensure(const DSurrogate& s, long long nt, int B);
  void release();
};

}  // namespace ptrom
