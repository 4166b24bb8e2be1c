/* ptrom_b200.h — C ABI of the B200 (sm_100a) hot path for the PTROM
 * reference (/root/reference/proj/include/ptrom). Plain pointers and sizes,
 * no torch or Eigen types. Every entry point names the reference function it
 * replaces (file:line under /root/reference/proj).
 *
 * Conventions:
 *  - State/velocity layout is the reference's SoA [chi_1..chi_N, psi_1..psi_N]
 *    (types.hpp:34-51): particle i owns rows i and i+N.
 *  - Status codes: 0 ok; 2 config_error (types.hpp:23-26, CLI exit 2);
 *    3 numerical_error (types.hpp:28-32, CLI exit 3); 4 CUDA failure.
 *    ptrom_last_error() returns the message (same wording as the reference
 *    where the reference throws).
 *  - ptrom_* functions take HOST buffers, copy in/out on the context stream and
 *    synchronize (drop-in for the reference's by-value returns).
 *    ptrom_dev_* functions take DEVICE buffers, are stream-ordered on the
 *    context stream and do not synchronize; a numerical failure they detect is
 *    latched on the device and reported by ptrom_synchronize().
 *  - n_pair_evals (nullable) receives the number of kernel_pair evaluations
 *    the reference would have made, so an adapter can bump
 *    detail::kernel_eval_counter (kernel.hpp:18-25).
 *  - One context per device per host thread; not reentrant.
 */
#ifndef PTROM_B200_H
#define PTROM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PTROM_OK = 0,
  PTROM_CONFIG_ERROR = 2,
  PTROM_NUMERICAL_ERROR = 3,
  PTROM_CUDA_ERROR = 4
};

/* kernel.hpp:16 KernelForm */
enum { PTROM_FORM_STANDARD = 0, PTROM_FORM_DENOMINATOR_SCALED = 1 };

/* quadtree.hpp:189-203 ClusterCriterion::Kind */
enum { PTROM_CRIT_BARNES_HUT = 0, PTROM_CRIT_NEIGHBOR = 1 };

typedef struct ptrom_ctx ptrom_ctx;

/* ------------------------------------------------------------ lifecycle -- */
int ptrom_create(int device, void* cuda_stream /* nullable: legacy default */, ptrom_ctx** out);
void ptrom_destroy(ptrom_ctx* ctx);
const char* ptrom_last_error(const ptrom_ctx* ctx);
int ptrom_set_stream(ptrom_ctx* ctx, void* cuda_stream);
/* Synchronizes the context stream; returns and clears any latched device
 * status (3 with the reference's message when a kernel saw a singularity). */
int ptrom_synchronize(ptrom_ctx* ctx);
/* Engine tuning knobs (no reference counterpart; results do not depend on
 * them). Keys: "reassign_big_members" (clusters above this size take the
 * one-CTA-per-cluster reassign path, default 4096, min 32), "tree_seq_max"
 * (tree nodes up to this size get bit-exact sequential sums in the subtree
 * CTAs, default 2048), "tree_build_mode" (0 Morton, 1 level build),
 * "allpairs_variant" (tile shape), "hyperpair_variant" (PTROM batched-march
 * hyperpair kernel: 0 default, 1 generic kernel, 2 four-entry rounds at 32
 * warps per SM, 3 per-SM target ranges).
 * Unknown keys are status 2. */
int ptrom_set_tuning(ptrom_ctx* ctx, const char* key, int64_t value);
/* Library/kernel identification for provenance checks. */
const char* ptrom_build_info(void);

/* ----------------------------------------------- all-pairs (host buffers) -- */
/* kernel.hpp:107-129 pairwise_velocity<double> */
int ptrom_pairwise_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma,
                                double delta, int form, const double* inflow /* 2n or NULL */,
                                double* f /* 2n */, uint64_t* n_pair_evals);
/* kernel.hpp:107-129 pairwise_velocity<float> */
int ptrom_pairwise_velocity_f32(ptrom_ctx* ctx, int64_t n, const float* x, const float* gamma,
                                float delta, int form, const float* inflow, float* f,
                                uint64_t* n_pair_evals);
/* kernel.hpp:154-170 inexact_kernel_jacobian<double> (BlockDiagonalJacobian
 * kernel.hpp:134-152 as four n-vectors) */
int ptrom_inexact_kernel_jacobian_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma,
                                      double delta, int form, double* dfx_dx, double* dfx_dy,
                                      double* dfy_dx, double* dfy_dy, uint64_t* n_pair_evals);
/* integrators.hpp:243-272 fom_simulate<double, PairwiseModel<double>> with
 * FomStepper integrators.hpp:117-201 and NewtonConfig integrators.hpp:55-66.
 * snapshots: column-major 2n x n_steps; per-step iterations/converged/
 * relative_residual as StepResult (integrators.hpp:104-111). */
int ptrom_fom_simulate_f64(ptrom_ctx* ctx, int64_t n, const double* x0, const double* gamma, double delta,
                           int form, const double* inflow, double dt, int64_t n_steps, double tol,
                           int max_iters, int jacobian_refresh_period, double* snapshots, int* iterations,
                           uint8_t* converged, double* relative_residual, uint64_t* n_pair_evals);
/* ptrom_fom_simulate_f64 on DEVICE buffers (x0 2n, gamma n, inflow 2n or
 * NULL, snapshots 2n x n_steps column-major or NULL); iterations / converged /
 * relative_residual are HOST arrays of n_steps. Synchronizes. Reports the
 * number of velocity and Jacobian (Newton-block refresh) evaluations, each
 * N(N-1) pairs. */
int ptrom_dev_fom_simulate_f64(ptrom_ctx* ctx, int64_t n, const double* d_x0, const double* d_gamma, double delta,
                               int form, const double* d_inflow, double dt, int64_t n_steps, double tol, int max_iters,
                               int jacobian_refresh_period, double* d_snapshots, int* iterations, uint8_t* converged,
                               double* relative_residual, uint64_t* n_velocity_evals, uint64_t* n_jacobian_evals);
/* kernel.hpp:174-191 hamiltonian<double>: Σ_{i<j} Γi Γj log|x_i - x_j| / 2π.
 * A coincident pair is status 3 "hamiltonian: coincident particles i and j"
 * (the lexicographically first pair, as the reference's loop order). */
int ptrom_hamiltonian_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double* out);
/* kernel.hpp:213-238 velocity_field_grid<double> with LatticeSpec
 * kernel.hpp:194-208 passed as (x_min, x_max, nx, y_min, y_max, ny): grid is
 * ny x nx column-major, grid[j + i*ny] = |f(x_i, y_j)| * c_g * l / gamma_bar.
 * n_pair_evals = nx*ny*n (the reference's kernel_pair counter). */
int ptrom_velocity_field_grid_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma,
                                  double delta, int form, double x_min, double x_max, int64_t nx,
                                  double y_min, double y_max, int64_t ny, double c_g, double l,
                                  double gamma_bar, double* grid, uint64_t* n_pair_evals);

/* --------------------------------------------- all-pairs (device buffers) -- */
/* Velocity of targets [t_begin, t_end) against all n sources (j != i):
 * f[(i-t_begin)] and f[(i-t_begin) + ld_f]. x is the full 2n SoA state,
 * inflow the full 2n vector or NULL. kernel.hpp:107-129 restricted to rows. */
int ptrom_dev_pairwise_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                    double delta, int form, const double* d_inflow, int64_t t_begin,
                                    int64_t t_end, double* d_f, int64_t ld_f);
int ptrom_dev_pairwise_velocity_f32(ptrom_ctx* ctx, int64_t n, const float* d_x, const float* d_gamma,
                                    float delta, int form, const float* d_inflow, int64_t t_begin,
                                    int64_t t_end, float* d_f, int64_t ld_f);
/* Target-sharded velocity with the sources read in place from every rank's
 * HBM (the per-evaluation position exchange fused into the
 * tile loads over NVLink instead of an all-gather). Rank r's block of
 * particles [peer_offsets[r], peer_offsets[r+1]) is SoA (x then y) at device
 * pointer d_peer_blocks[r] (own block or a CUDA-IPC mapping of a peer's,
 * see ptrom_ipc_*); d_peer_blocks / peer_offsets are host arrays. Targets are
 * this rank's rows [t_begin, t_end), SoA at d_local. Γ and the inflow are the
 * full replicated n- and 2n-vectors. Output as ptrom_dev_pairwise_velocity_f64.
 * kernel.hpp:107-129 restricted to rows. n_peers <= 8. */
int ptrom_dev_pairwise_velocity_peers_f64(ptrom_ctx* ctx, int64_t n, int32_t n_peers,
                                          const double* const* d_peer_blocks, const int64_t* peer_offsets,
                                          const double* d_gamma, double delta, int form, const double* d_inflow,
                                          int64_t t_begin, int64_t t_end, const double* d_local, double* d_f,
                                          int64_t ld_f);
/* CUDA IPC helpers for the peer exchange: an IPC-shareable device buffer,
 * its 64-byte handle, mapping a peer's handle into this process, and a
 * stream-ordered device copy (cudaMemcpyDefault: local or peer memory). */
int ptrom_ipc_alloc(ptrom_ctx* ctx, uint64_t bytes, void** d_ptr);
int ptrom_ipc_free(ptrom_ctx* ctx, void* d_ptr);
int ptrom_ipc_get_handle(ptrom_ctx* ctx, void* d_ptr, uint8_t* handle64);
int ptrom_ipc_open_handle(ptrom_ctx* ctx, const uint8_t* handle64, void** d_ptr);
int ptrom_ipc_close_handle(ptrom_ctx* ctx, void* d_ptr);
int ptrom_dev_memcpy(ptrom_ctx* ctx, void* d_dst, const void* d_src, uint64_t bytes);
/* kernel.hpp:154-170 restricted to rows [t_begin, t_end); four vectors of
 * length t_end - t_begin. */
int ptrom_dev_inexact_kernel_jacobian_f64(ptrom_ctx* ctx, int64_t n, const double* d_x,
                                          const double* d_gamma, double delta, int form, int64_t t_begin,
                                          int64_t t_end, double* d_jxx, double* d_jxy, double* d_jyx,
                                          double* d_jyy);
/* Device-buffer hamiltonian: d_out is one double (stream-ordered). */
int ptrom_dev_hamiltonian_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                              double* d_out);
/* Device-buffer velocity_field_grid: d_grid is ny*nx doubles. */
int ptrom_dev_velocity_field_grid_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                      double delta, int form, double x_min, double x_max, int64_t nx,
                                      double y_min, double y_max, int64_t ny, double c_g, double l,
                                      double gamma_bar, double* d_grid);
/* Newton-block refactor fused with the Jacobian (integrators.hpp:181-194):
 * inv = (I - dt/2 J_i)^{-1} for rows [t_begin,t_end), row-major 4 per particle.
 * A singular block latches status 3 "singular Newton block for particle i". */
int ptrom_dev_newton_blocks_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                double delta, int form, double dt, int64_t t_begin, int64_t t_end,
                                double* d_inv /* 4*(t_end-t_begin) */);
/* integrators.hpp:47-53 residual on m rows of a shard (local layout: rows k
 * and k+ld), plus its squared 2-norm summed in a fixed order into
 * *d_norm2 (one double, device). */
int ptrom_dev_residual_f64(ptrom_ctx* ctx, int64_t m, int64_t ld, const double* d_xi, const double* d_fxi,
                           const double* d_xprev, const double* d_fprev, double dt, double* d_r,
                           double* d_norm2);
/* integrators.hpp:161-167: x[k] += inv_k * (-r) for m local rows. */
int ptrom_dev_newton_update_f64(ptrom_ctx* ctx, int64_t m, int64_t ld, const double* d_inv, const double* d_r,
                                double* d_x);

/* ------------------------------------------------------------------ tree -- */
/* quadtree.hpp:34-47 QuadTree, device-resident; owned by the caller, bound to
 * the context that built it. Node ids are the reference's preorder ids. */
typedef struct ptrom_tree ptrom_tree;
/* quadtree.hpp:124-162 build_tree<double>(points N x 2, gamma, leaf_capacity);
 * points given as the two columns px, py. */
int ptrom_tree_build_f64(ptrom_ctx* ctx, int64_t n, const double* px, const double* py, const double* gamma,
                         int64_t leaf_capacity, ptrom_tree** out);
int ptrom_dev_tree_build_f64(ptrom_ctx* ctx, int64_t n, const double* d_px, const double* d_py,
                             const double* d_gamma, int64_t leaf_capacity, ptrom_tree** out);
void ptrom_tree_free(ptrom_tree* tree);
int64_t ptrom_tree_num_nodes(const ptrom_tree* tree);
/* TreeNode fields (quadtree.hpp:15-30) in structure-of-arrays form plus perm,
 * slot, leaf_node (quadtree.hpp:37-39). Any pointer may be NULL. */
int ptrom_tree_export(ptrom_ctx* ctx, const ptrom_tree* tree, double* bounds /* 4/node */, double* width,
                      double* centroid /* 2/node */, double* gamma_sum, int32_t* children /* 4/node */,
                      int64_t* begin, int64_t* end, int32_t* depth, uint8_t* centroid_fallback, int64_t* perm,
                      int64_t* slot, int32_t* leaf_node);
/* quadtree.hpp:213-252 collect_clusters for n_targets target ids, CSR output:
 * cluster node ids (preorder) and direct ids (ascending). Two-call protocol:
 * offsets (n_targets+1 each) are always filled; the lists are written when
 * the capacities suffice. */
int ptrom_collect_clusters(ptrom_ctx* ctx, ptrom_tree* tree, int crit_kind, double crit_value, int64_t n_targets,
                           const int64_t* targets, int64_t* cluster_offsets, int32_t* clusters,
                           int64_t clusters_cap, int64_t* direct_offsets, int64_t* direct, int64_t direct_cap);
/* quadtree.hpp:257-281 bh_velocity<double>(tree, state, sys, criterion). */
int ptrom_bh_velocity_f64(ptrom_ctx* ctx, ptrom_tree* tree, int64_t n, const double* x, const double* gamma,
                          double delta, int form, int crit_kind, double crit_value, const double* inflow,
                          double* f, uint64_t* n_pair_evals);
/* quadtree.hpp:285-308 bh_jacobian<double>. */
int ptrom_bh_jacobian_f64(ptrom_ctx* ctx, ptrom_tree* tree, int64_t n, const double* x, const double* gamma,
                          double delta, int form, int crit_kind, double crit_value, double* dfx_dx,
                          double* dfx_dy, double* dfy_dx, double* dfy_dy);
/* integrators.hpp:96-98 BarnesHutModel::velocity: rebuild the tree from the
 * state (leaf_capacity) and evaluate; host and device-buffer forms. */
int ptrom_barnes_hut_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* x, const double* gamma, double delta,
                                  int form, int crit_kind, double crit_value, int64_t leaf_capacity,
                                  const double* inflow, double* f, uint64_t* n_pair_evals);
int ptrom_dev_barnes_hut_velocity_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                      double delta, int form, int crit_kind, double crit_value,
                                      int64_t leaf_capacity, const double* d_inflow, double* d_f,
                                      uint64_t* n_pair_evals);
/* Target-sharded form (replicated build, far field split by
 * target): builds the same tree as ptrom_dev_barnes_hut_velocity_f64 and
 * evaluates only the targets in tree slots [k_begin, k_end) (slot k holds
 * particle perm[k]; slots are spatially contiguous). Velocities go to
 * d_f_slots in slot order, x then y (2·(k_end − k_begin) doubles); the
 * permutation is written to d_perm (n int32, may be null) so ranks can
 * scatter the gathered shards back to particle order. */
int ptrom_dev_barnes_hut_velocity_slots_f64(ptrom_ctx* ctx, int64_t n, const double* d_x, const double* d_gamma,
                                            double delta, int form, int crit_kind, double crit_value,
                                            int64_t leaf_capacity, const double* d_inflow, int64_t k_begin,
                                            int64_t k_end, double* d_f_slots, int32_t* d_perm,
                                            uint64_t* n_pair_evals);

/* Statistics of the last tree build / evaluation on this context: device
 * time of the build (T1+T2) and of the final traversal pass (T3), kernel
 * interactions and prune tests of that pass, node count, and how many targets
 * hit an uncertain (certified-then-resolved) prune test. */
int ptrom_tree_stats(ptrom_ctx* ctx, double* build_ms, double* eval_ms, uint64_t* interactions,
                     uint64_t* prune_tests, uint64_t* nodes, uint64_t* resolved_targets);
/* Which build produced the last tree on this context: *morton = 1 for the
 * Morton-key sort build, 0 for the level-by-level partition (chosen when the
 * tree needs more than 32 levels, leaf_capacity > 256, or PTROM_TREE_BUILD=levels);
 * *levels = tree levels walked by the Morton build. Same tree either way. */
int ptrom_tree_build_info(ptrom_ctx* ctx, int* morton, int* levels);

/* ----------------------------------------------------------- PTROM online -- */
/* PODBasis (reduction.hpp:18-26): phi is n_dofs x modes column-major. */
typedef struct ptrom_basis ptrom_basis;
int ptrom_basis_create(ptrom_ctx* ctx, int64_t n_dofs, int64_t modes, const double* phi,
                       const double* singular_values /* nullable */, const double* x_ref, ptrom_basis** out);
void ptrom_basis_free(ptrom_basis* basis);
/* rom.hpp:45-58 reconstruct_output: out (n_dofs x n_steps, column-major) row k
 * = x_ref[dofs[k]] + phi.row(dofs[k]) * x_hat; dofs == NULL gives
 * reconstruct_full (rom.hpp:60-64, all 2n rows). x_hat is modes x n_steps
 * column-major (RomTrajectory::x_hat). modes <= 32. */
int ptrom_reconstruct_output_f64(ptrom_ctx* ctx, const ptrom_basis* basis, int64_t n_steps, const double* x_hat,
                                 int64_t n_dofs, const int64_t* dofs /* nullable */, double* out);
int ptrom_dev_reconstruct_output_f64(ptrom_ctx* ctx, const ptrom_basis* basis, int64_t n_steps,
                                     const double* d_xhat, int64_t n_dofs, const int64_t* d_dofs,
                                     double* d_out);
/* GnatOperator (reduction.hpp:173-180): sorted sample ids and A = pinv(P Φ_r)
 * (m_r x 2 n_samples, column-major); gathers Φ̄, x̄⁰ like GnatSolver's
 * constructor (rom.hpp:264-290). m_r <= 32, modes <= 32. */
typedef struct ptrom_gnat_op ptrom_gnat_op;
int ptrom_gnat_op_create(ptrom_ctx* ctx, const ptrom_basis* basis, int64_t n_samples, const int64_t* sample_ids,
                         int64_t m_r, const double* A, ptrom_gnat_op** out);
void ptrom_gnat_op_free(ptrom_gnat_op* op);
/* SurrogateSourceBasis (reduction.hpp:280-302) in CSR form: cluster tables
 * (phi_tilde 2N_c x M column-major, gamma_tilde, x0_tilde, zero_gamma,
 * membership CSR of ascending ids), per-target cluster list CSR, near-field
 * union (direct_ids, direct_phi 2U x M, direct_x0, direct_gamma) and the
 * per-target local direct list CSR. */
typedef struct ptrom_surrogate ptrom_surrogate;
int ptrom_surrogate_create(ptrom_ctx* ctx, int64_t modes, int64_t n_clusters, const double* phi_tilde,
                           const double* gamma_tilde, const double* x0_tilde, const uint8_t* zero_gamma,
                           const int64_t* membership_offsets, const int64_t* membership_ids, int64_t n_targets,
                           const int64_t* target_ids, const int64_t* cluster_offsets, const int64_t* cluster_list,
                           int64_t n_direct, const int64_t* direct_ids, const double* direct_phi,
                           const double* direct_x0, const double* direct_gamma, const int64_t* direct_offsets,
                           const int64_t* direct_list, ptrom_surrogate** out);
void ptrom_surrogate_free(ptrom_surrogate* sur);
int ptrom_surrogate_export(ptrom_ctx* ctx, const ptrom_surrogate* sur, double* phi_tilde, double* gamma_tilde,
                           double* x0_tilde, uint8_t* zero_gamma, double* direct_gamma);
/* reduction.hpp:400-431 reassign_cluster_circulation (in place). */
int ptrom_reassign_cluster_circulation_f64(ptrom_ctx* ctx, ptrom_surrogate* sur, int64_t n, const double* gamma,
                                           const ptrom_basis* basis);
/* rom.hpp:101-155 hyperpair: f (2 n_t), jac (4 x n_t rows dfx_dx, dfx_dy,
 * dfy_dx, dfy_dy), cluster / direct positions (nullable). inflow is the full
 * 2n vector (added at the target ids) or NULL. */
int ptrom_hyperpair_f64(ptrom_ctx* ctx, const ptrom_surrogate* sur, const double* target_positions,
                        const double* x_hat, double delta, int form, int64_t n, const double* inflow, double* f,
                        double* jac, double* cluster_positions, double* direct_positions, uint64_t* n_pair_evals);
/* rom.hpp:404-412 ptrom_simulate: reassigns the surrogate to gamma (in
 * place, like the reference) and runs GnatSolver::simulate on the device.
 * x_hat is M x n_steps column-major; iterations / converged per step. */
int ptrom_ptrom_simulate_f64(ptrom_ctx* ctx, const ptrom_basis* basis, const ptrom_gnat_op* op, ptrom_surrogate* sur,
                             int64_t n, const double* gamma, double delta, int form, const double* inflow, double dt,
                             int64_t n_steps, double tol, int max_iters, double step_length, double* x_hat,
                             int* iterations, uint8_t* converged, uint64_t* n_pair_evals);
/* Batched online queries: n_inst instances of an affine
 * circulation Γ(μ) = gamma_a + μ gamma_b (the surrogate is not modified),
 * processed `batch` instances at a time (0 = default). x_hat is
 * [n_inst][n_steps][M], iterations / converged [n_inst][n_steps]. */
int ptrom_ptrom_simulate_batch_f64(ptrom_ctx* ctx, const ptrom_basis* basis, const ptrom_gnat_op* op,
                                   const ptrom_surrogate* sur, int64_t n, const double* gamma_a,
                                   const double* gamma_b, int64_t n_inst, const double* mu, int64_t batch,
                                   double delta, int form, const double* inflow, double dt, int64_t n_steps,
                                   double tol, int max_iters, double step_length, double* x_hat, int* iterations,
                                   uint8_t* converged, uint64_t* n_pair_evals);

/* ------------------------------------------------- PTROM offline producers -- */
/* reduction.hpp:93-168 greedy_sample (device scoring/selection). phi_r is
 * n_dofs x n_r column-major; out_ids receives n_target sorted ids. */
int ptrom_greedy_sample_f64(ptrom_ctx* ctx, int64_t n_dofs, int64_t n_r, const double* phi_r, int64_t n_target,
                            int64_t n_preseed, const int64_t* preseed, int64_t* out_ids);
/* reduction.hpp:182-220 build_gnat_operator: A (m_r x 2 n_s, column-major). */
int ptrom_build_gnat_operator_f64(ptrom_ctx* ctx, int64_t n_dofs, int64_t m_r, const double* phi_r, int64_t n_s,
                                  const int64_t* ids, double* A);
/* reduction.hpp:236-274 + 304-385: weighted POD tree and cluster_pod on the
 * device (the basis must carry singular values). */
int ptrom_cluster_pod_f64(ptrom_ctx* ctx, const ptrom_basis* basis, const double* gamma, int64_t leaf_capacity,
                          int crit_kind, double crit_value, int64_t n_targets, const int64_t* targets,
                          ptrom_surrogate** out);
/* sizes: n_clusters, n_direct, n_targets, membership entries, cluster-list
 * entries, direct-list entries. */
int ptrom_surrogate_sizes(const ptrom_surrogate* sur, int64_t* sizes);
int ptrom_surrogate_export_lists(ptrom_ctx* ctx, const ptrom_surrogate* sur, int32_t* cluster_node_ids,
                                 int64_t* mem_off, int64_t* mem_ids, int64_t* cl_off, int64_t* cl_list,
                                 int64_t* direct_ids, int64_t* d_off, int64_t* d_list, double* direct_phi,
                                 double* direct_x0);

/* --------------------------------------- PTMX / OfflineBundle I/O (§8f-4) -- */
/* Host I/O in the reference's on-disk layout; no GPU needed except for
 * ptrom_bundle_to_device. ctx may be NULL: the message is then available from
 * ptrom_io_last_error() (thread-local). I/O and format errors are status 2
 * (the reference throws config_error) with the reference's messages. */
typedef struct ptrom_bundle ptrom_bundle;
const char* ptrom_io_last_error(void);
/* io.hpp:53-75 read_matrix: rows, cols, dt, t0 (each nullable); data = NULL
 * reads the header only, else rows*cols column-major doubles (capacity in
 * doubles). */
int ptrom_ptmx_read(ptrom_ctx* ctx, const char* path, uint64_t* rows, uint64_t* cols, double* dt, double* t0,
                    double* data, uint64_t capacity);
/* io.hpp:35-51 write_matrix (a time series when dt/t0 are set, e.g. an x_hat
 * trajectory M x n_steps). */
int ptrom_ptmx_write(ptrom_ctx* ctx, const char* path, uint64_t rows, uint64_t cols, double dt, double t0,
                     const double* data);
/* bundle.cpp:96-141 OfflineBundle::load: index.json + the twelve PTMX files. */
int ptrom_bundle_open(ptrom_ctx* ctx, const char* dir, ptrom_bundle** out);
void ptrom_bundle_free(ptrom_bundle* bundle);
/* sizes[11]: n_dofs, modes, residual modes, n_samples, GNAT rows, n_clusters,
 * n_direct, n_targets, membership entries, cluster-list entries, direct-list
 * entries. */
int ptrom_bundle_sizes(const ptrom_bundle* bundle, int64_t* sizes);
/* The ExperimentConfig object verbatim (JSON text); returns its length. */
int64_t ptrom_bundle_config_json(const ptrom_bundle* bundle, char* buf, int64_t cap);
/* Host copies of every array (NULL skips), column-major matrices, CSR lists. */
int ptrom_bundle_export(const ptrom_bundle* bundle, double* basis_phi, double* basis_sv, double* basis_xref,
                        double* residual_phi, double* residual_sv, double* gnat_a, int64_t* sample_ids,
                        double* phi_tilde, double* x0_tilde, double* gamma_tilde, int32_t* cluster_node_ids,
                        int64_t* mem_off, int64_t* mem_ids, uint8_t* zero_gamma, int64_t* target_ids,
                        int64_t* cl_off, int64_t* cl_list, int64_t* d_off, int64_t* d_list, int64_t* direct_ids,
                        double* direct_phi, double* direct_x0, double* direct_gamma);
/* → the device basis, GNAT operator and surrogate (rom.hpp:264-290 inputs). */
int ptrom_bundle_to_device(ptrom_ctx* ctx, const ptrom_bundle* bundle, ptrom_basis** basis, ptrom_gnat_op** op,
                           ptrom_surrogate** sur);

/* ---------------------------------------------------- multi-GPU -- */
/* SURVEY.md §8b "Multi-GPU: ptrom_comm_init + *_sharded variants". One
 * process (or host thread) per GPU, one ptrom_ctx and one ptrom_comm per rank.
 * Collectives run on the context's stream.
 *
 * NCCL transport: rank 0 calls ptrom_comm_unique_id, the host distributes the
 * 128 bytes to every rank by its own means (MPI_Bcast, a file, a TCP store),
 * and every rank calls ptrom_comm_init. libnccl.so.2 is loaded at run time.
 *
 * Host transport: the caller supplies the two collectives on HOST buffers
 * (an MPI / gloo / shared-memory host already has them); device data is
 * staged through the host and each collective synchronizes. Callbacks return
 * 0 on success. all_gather receives `bytes` from every rank into
 * recv[r * bytes ...] in rank order. */
typedef struct ptrom_comm ptrom_comm;
typedef struct {
  int (*all_gather)(void* user, const void* send, void* recv, uint64_t bytes);
  int (*broadcast)(void* user, void* buf, uint64_t bytes, int root);
} ptrom_host_collectives;
int ptrom_comm_unique_id(uint8_t id_out[128]);
int ptrom_comm_init(ptrom_ctx* ctx, int rank, int world, const uint8_t id[128], ptrom_comm** out);
int ptrom_comm_init_host(ptrom_ctx* ctx, int rank, int world, const ptrom_host_collectives* ops, void* user,
                         ptrom_comm** out);
void ptrom_comm_destroy(ptrom_comm* comm);
/* 1 for the NCCL transport, 0 for host callbacks. */
int ptrom_comm_transport(const ptrom_comm* comm);

/* Target-sharded velocity (kernel.hpp:107-129 for this rank's rows): rank r
 * owns particles [r*n/G, (r+1)*n/G) (m of them). d_x_local is its 2m SoA rows
 * [x..., y...]; the positions of all ranks are exchanged into d_x_full (2n,
 * workspace) and d_f_local (2m) receives this rank's velocities (+ inflow,
 * d_inflow 2n or NULL). NCCL: stream-ordered; host transport: synchronous. */
int ptrom_dev_pairwise_velocity_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int64_t n, const double* d_x_local,
                                            double* d_x_full, const double* d_gamma, double delta, int form,
                                            const double* d_inflow, double* d_f_local);
/* integrators.hpp:243-272 fom_simulate with the targets split across the
 * communicator. Every rank passes the full x0 (2n),
 * gamma (n) and inflow (2n or NULL) as the reference's fom_simulate does and
 * receives its own rows: snapshots_local is 2m x n_steps column-major
 * (column s = [x_lo..x_hi-1, y_lo..y_hi-1] after step s); iterations /
 * converged / relative_residual are identical on every rank. Per Newton
 * iteration: the partial |r|^2 of every rank are all-gathered and summed in
 * rank order (the same decision on every rank, independent of NCCL's
 * reduction order), the Newton update runs on the local rows (the 2x2
 * self-blocks are local) and the updated rows are all-gathered before the
 * velocity of the local targets. n_pair_evals: this rank's share,
 * velocity evaluations x m x (n-1). */
int ptrom_fom_simulate_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int64_t n, const double* x0,
                                   const double* gamma, double delta, int form, const double* inflow, double dt,
                                   int64_t n_steps, double tol, int max_iters, int jacobian_refresh_period,
                                   double* snapshots_local, int* iterations, uint8_t* converged,
                                   double* relative_residual, uint64_t* n_pair_evals);
/* ptrom_ptrom_simulate_batch_f64 with the n_inst instances split evenly
 * across the communicator. The tables are needed on
 * `root` only: basis, op, sur, gamma_a, gamma_b, mu and inflow may be NULL on
 * the other ranks. One grouped broadcast replicates the shared tables (row-
 * major basis, GNAT operator and gathered rows, the surrogate's CSR lists and
 * per-cluster tables) and the parameters; every rank then marches its
 * instances with no communication, and x_hat / iterations / converged are
 * all-gathered in instance order on every rank that passes non-NULL outputs.
 * n_pair_evals: this rank's share. */
int ptrom_ptrom_simulate_batch_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int root, const ptrom_basis* basis,
                                           const ptrom_gnat_op* op, const ptrom_surrogate* sur, int64_t n,
                                           const double* gamma_a, const double* gamma_b, int64_t n_inst,
                                           const double* mu, int64_t batch, double delta, int form,
                                           const double* inflow, double dt, int64_t n_steps, double tol,
                                           int max_iters, double step_length, double* x_hat, int* iterations,
                                           uint8_t* converged, uint64_t* n_pair_evals);

/* Sharded Barnes–Hut velocity (bh_velocity over integrators.hpp:83-102's
 * BarnesHutModel: replicated build, far field split by
 * target). Every rank passes the full state and gets the full f (2n) back,
 * bit-identical to ptrom_barnes_hut_velocity_f64: each rank builds the same
 * tree, evaluates tree slots [r·n/G, (r+1)·n/G), and the slot blocks are
 * all-gathered and scattered to particle order. n_pair_evals sums the ranks. */
int ptrom_barnes_hut_velocity_sharded_f64(ptrom_ctx* ctx, ptrom_comm* comm, int64_t n, const double* x,
                                          const double* gamma, double delta, int form, int crit_kind,
                                          double crit_value, int64_t leaf_capacity, const double* inflow, double* f,
                                          uint64_t* n_pair_evals);

/* --------------------------------------------------------- instrumentation -- */
/* bench.py support: while enabled, the context records CUDA events on its own
 * stream around every launch of the dominant kernel of each call (the
 * all-pairs tile kernel, the tree traversal kernel, the hyperpair kernel).
 * ptrom_profile_end synchronizes and returns the summed duration and the
 * number of launches, then disables recording. */
int ptrom_profile_begin(ptrom_ctx* ctx);
int ptrom_profile_end(ptrom_ctx* ctx, double* total_ms, int64_t* launches);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PTROM_B200_H */
