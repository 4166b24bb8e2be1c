// ops.cuh — internal (C++) entry points between translation units.
#pragma once
#include "common.cuh"

#include <vector>

namespace ptrom {

double effective_delta(double delta, int form);
// kernel.hpp:84-103 finiteness / δ checks on the device copies of host-API
// inputs (null arrays skipped); raises the reference's config errors in order.
template <class S>
void validate_uploaded(ptrom_ctx* ctx, long long n, const S* dx, const S* dg, S delta, const S* di, const char* who);
void dev_velocity_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta, int form,
                      const double* inflow, long long t_begin, long long t_end, double* f, long long ld);
// Full self-evaluation (every target, every source) over unordered pairs
// (allpairs_sym.cu); applies for n ≥ 16,384 unless PTROM_ALLPAIRS_SYM=0.
bool sym_velocity_applies(ptrom_ctx* ctx, long long n);
void dev_velocity_sym_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta, int form,
                          const double* inflow, double* f);
// The same split over a communicator (n divisible by the world size): rank r
// gets rows [r·n/G, (r+1)·n/G) of f (ld n/G), bit-identical to the single-GPU
// evaluation (allpairs_sym.cu).
bool sym_sharded_applies(ptrom_ctx* ctx, long long n, int world);
void dev_velocity_sym_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, long long n, const double* x_full,
                                  const double* gamma, double delta, int form, const double* inflow, double* f_local);
// The Newton blocks of this rank's rows over unordered pairs, sharded like
// dev_velocity_sym_sharded_f64 (n divisible by the world size).
void dev_jacobian_sym_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, long long n, const double* x_full,
                                  const double* gamma, double delta, int form, double dt_for_inverse,
                                  double* inv_local);
// The Jacobian's (A, B, C) partials over unordered pairs, [nb][3][n] in the
// context scratch (allpairs_sym.cu); every target of a full set.
void dev_jacobian_sym_part(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double dp,
                           double** part_out, int* nb_out, bool size_only);
// (A, B, C) partials [chunks][3][t_count] → the Jacobian rows or, with inv,
// the Newton blocks (I − dt/2·J)⁻¹ (allpairs.cu's fixed-order reduction).
void dev_jacobian_reduce_f64(ptrom_ctx* ctx, const double* part, int chunks, long long t_begin, long long t_count,
                             double dp, double dt_for_inverse, double* jxx, double* jxy, double* jyx, double* jyy,
                             double* inv);
void dev_velocity_sym_f32(ptrom_ctx* ctx, long long n, const float* x, const float* gamma, float delta, int form,
                          const float* inflow, float* f);
void dev_velocity_f32(ptrom_ctx* ctx, long long n, const float* x, const float* gamma, float delta, int form,
                      const float* inflow, long long t_begin, long long t_end, float* f, long long ld);
// jxx..jyy (may be null when inv is given) or the Newton-block inverse of
// (I - dt/2 J) into inv (4 per row) when inv != nullptr.
// Sizes the context's scratch for dev_jacobian_f64 over t_count targets
// without launching (before a graph capture).
void dev_jacobian_reserve_f64(ptrom_ctx* ctx, long long n, long long t_count);
void dev_jacobian_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta, int form,
                      long long t_begin, long long t_end, double* jxx, double* jxy, double* jyx, double* jyy,
                      double dt_for_inverse, double* inv);
void dev_velocity_peers_f64(ptrom_ctx* ctx, long long n, int n_peers, const double* const* peer_base,
                            const long long* peer_off, const double* gamma, double delta, int form,
                            const double* inflow, long long t_begin, long long t_end, const double* tx,
                            const double* ty, double* f, long long ld);
void dev_hamiltonian_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double* out);
void dev_velocity_field_grid_f64(ptrom_ctx* ctx, long long n, const double* x, const double* gamma, double delta,
                                 int form, double x_min, double x_max, long long nx, double y_min, double y_max,
                                 long long ny, double scale, double* grid);
void dev_residual_f64(ptrom_ctx* ctx, long long m, long long ld, const double* xi, const double* fxi,
                      const double* xp, const double* fp, double dt, double* r, double* norm2, double* block_part);
void dev_newton_update_f64(ptrom_ctx* ctx, long long m, long long ld, const double* inv, const double* r, double* x);
size_t residual_block_part_count();

struct FomResult {
  long long velocity_evals = 0;
  long long jacobian_evals = 0;
};
// Small systems (n ≤ 16,384, cooperative launch available, unless
// PTROM_FOM_PERSISTENT=0): the whole trajectory as one persistent kernel
// (fom_persistent.cu).
bool fom_persistent_applies(ptrom_ctx* ctx, long long n);
FomResult fom_simulate_persistent(ptrom_ctx* ctx, long long n, const double* d_x0, const double* d_gamma,
                                  double delta, int form, const double* d_inflow, double dt, long long n_steps,
                                  double tol, int max_iters, int refresh, double* snapshots_out, int* iters,
                                  unsigned char* conv, double* rel_out);
FomResult fom_simulate_device(ptrom_ctx* ctx, long long n, const double* d_x0, const double* d_gamma, double delta,
                              int form, const double* d_inflow, double dt, long long n_steps, double tol,
                              int max_iters, int refresh, double* h_snapshots, int* iters, unsigned char* conv,
                              double* rel_out);

struct Tree;
void tree_build(ptrom_ctx* ctx, Tree& t, long long n, const double* d_px, const double* d_py, const double* d_g,
                long long leaf_cap, int seq_max);
int tree_resolve_uncertain(ptrom_ctx* ctx, Tree& t, const int* d_flag_count);
// Targets are the tree slots [k_begin, k_end) (k_end < 0: all n). With
// f_slots != nullptr the velocities go there in slot order, x then y
// (2·(k_end − k_begin)), instead of d_f in particle order.
unsigned long long tree_eval(ptrom_ctx* ctx, Tree& t, const double* d_x, const double* d_gamma, double delta,
                             int form, int crit_kind, double crit_value, const double* d_inflow, double* d_f,
                             double* jxx, double* jxy, double* jyx, double* jyy, long long k_begin = 0,
                             long long k_end = -1, double* f_slots = nullptr);

}  // namespace ptrom
