/*
 * ttdvm_cuda.h -- C ABI of the B200-native TT-DVM explicit step.
 *
 * Drop-in boundary for the hot path of arXiv 1912.04582's C++ reference
 * (proj/include/ttdvm/*.hpp).  The reference has no step symbol and no
 * caller (proj/tools/main.cpp:1); SPEC.md:391 declares
 *     explicit_step(state, mesh, grid, gas, problem, config) -> state
 * and SURVEY.md §8(b) fixes the C ABI below.  Each entry point names the
 * reference interface it replaces.  Plain pointers and sizes only; every
 * function returns a ttdvm_status and never throws.  A context owns all
 * device memory; host buffers are caller-owned and only touched during the
 * call.  Calls are stream-ordered and synchronous at return.  A context is
 * not re-entrant (one per device / rank).
 *
 * TT packing (ttdvm_tt_batch), per tensor, in doubles, mirroring the
 * reference's Eigen col-major cores (proj/include/ttdvm/tt_tensor.hpp:74-76):
 *   [first  n1 x r1, (i,a) at i + n1*a]
 *   [middle n2 slices r1 x r2, slice j (a,b) at j*r1*r2 + a + r1*b]
 *   [last   r2 x n3, (b,k) at b + r2*k]
 */
#ifndef TTDVM_CUDA_H_
#define TTDVM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TTDVM_OK = 0,
  TTDVM_EINVAL = 1,   /* -> std::invalid_argument in the C++ wrapper  */
  TTDVM_EDOMAIN = 2,  /* -> std::runtime_error (cell / face id in message) */
  TTDVM_ENOMEM = 3,
  TTDVM_ECUDA = 4,
  TTDVM_ENCCL = 5,
} ttdvm_status;

typedef struct ttdvm_ctx ttdvm_ctx;

typedef struct {
  int32_t count, n1, n2, n3;
  const int32_t* ranks;   /* [2*count]: r1, r2 per tensor            */
  const int64_t* offsets; /* [count+1]: first double of each tensor   */
  const double* cores;    /* [offsets[count]]                          */
} ttdvm_tt_batch;

/* Boundary condition per mesh group (proj/include/ttdvm/boundary.hpp:13-41).
 * kind: 0 wall, 1 sym-x, 2 sym-y, 3 sym-z, 4 in, 5 out. */
typedef struct {
  int32_t kind;
  double wall_temperature;
  double free_n, free_t, free_u[3];
} ttdvm_bc;

/* Context lifetime.  device = CUDA ordinal.  One context per GPU / rank. */
int ttdvm_cuda_create(int device, ttdvm_ctx** out);
int ttdvm_cuda_destroy(ttdvm_ctx* ctx);
const char* ttdvm_cuda_last_error(const ttdvm_ctx* ctx);

/* VelocityGrid(n, bound) -- proj/src/velocity_grid.cpp:11-19. */
int ttdvm_cuda_set_grid(ttdvm_ctx* ctx, int n, double bound);
/* GasParameters -- proj/include/ttdvm/physics.hpp:11-18:
 * gas = {molecule_mass, gas_constant, prandtl, mu_ref, t_ref, omega}. */
int ttdvm_cuda_set_gas(ttdvm_ctx* ctx, const double gas[6]);

/* UnstructuredMesh arrays consumed by the step
 * (proj/include/ttdvm/mesh.hpp:15-41): normals unit, out of left; right =
 * -1 on boundary faces; group -1 on interior (and periodic) faces; per cell
 * the (face, sign) list, sign +1 iff the normal points out of the cell. */
int ttdvm_cuda_set_mesh(ttdvm_ctx* ctx, int32_t ncell, int32_t nface, const int32_t* left,
                        const int32_t* right, const int32_t* group, const double* area,
                        const double* normal, const double* volume,
                        const int64_t* cell_face_off, const int32_t* cell_face_id,
                        const int8_t* cell_face_sign);

/* Boundary conditions per group (replaces BoundaryCondition::wall/
 * freestream_in/freestream_out/symmetry, proj/src/boundary.cpp:45-82). */
int ttdvm_cuda_set_bcs(ttdvm_ctx* ctx, int32_t ngroup, const ttdvm_bc* bcs);

/* State upload / download (per-cell f, resident across steps). */
int ttdvm_cuda_upload_state(ttdvm_ctx* ctx, const ttdvm_tt_batch* f);
/* Query ranks[2*count] and offsets[count+1] of the resident state. */
int ttdvm_cuda_state_layout(ttdvm_ctx* ctx, int32_t* ranks, int64_t* offsets);
/* Copy the packed state cores (capacity in doubles). */
int ttdvm_cuda_download_state(ttdvm_ctx* ctx, double* cores, int64_t capacity);

/* The explicit step S1, nsteps times: face fluxes
 * Phi = round(xp o f_L + xm o f_R), collision J = compute_collision(f)
 * (proj/src/physics.cpp:112-119), residual R = round(J - sum s A/V Phi),
 * update f = round(f + dt R); all roundings TtTensor::rounded(eps, cap)
 * (proj/src/tt_tensor.cpp:139-193; cap 0 = none, collision uncapped as in
 * the reference). */
int ttdvm_cuda_step(ttdvm_ctx* ctx, double dt, double eps, int32_t cap, int32_t nsteps);

/* One LU-SGS implicit iteration, `niter` times (SPEC.md:399-407 lusgs_step;
 * SURVEY.md §8(f) N4): the explicit residual of ttdvm_cuda_step, then forward
 * and backward Gauss-Seidel sweeps over the cells in index order with the
 * first-order upwind Jacobian splitting; the diagonal is the constant rank-1
 * over-estimate d_i = 1/dt + nu_i + (1/2)(1/V_i) sum_j A_j sqrt(3) xi_box_max,
 * divided out exactly (TtTensor::divided_by_rank_one,
 * proj/src/tt_tensor.cpp:247-261); every bracket and the update are rounded
 * at (eps, cap).  The sweeps run level by level (a cell's level = its longest
 * chain of lower- / higher-indexed neighbours), each level one batched
 * rounding launch, which reproduces the natural-order sweep.  Unpartitioned
 * meshes only. */
int ttdvm_cuda_lusgs_step(ttdvm_ctx* ctx, double dt, double eps, int32_t cap, int32_t niter);
/* Levels (= batched launches) of the forward and backward sweeps. */
int ttdvm_cuda_lusgs_levels(ttdvm_ctx* ctx, int32_t* forward_levels, int32_t* backward_levels);

/* Bounded-memory step: the face fluxes, residuals and updates of a step are
 * formed in `nblocks` contiguous ranges of the owned cells (the fluxes of
 * faces between two blocks are rounded in both), so the flux and residual
 * arenas hold one block at a time.  Same sums, same results as one block.
 * nblocks = 0 (default): one block, multiplied by 4 whenever a step runs out
 * of device memory.  No reference counterpart (the reference holds every
 * intermediate in host memory). */
int ttdvm_cuda_set_blocks(ttdvm_ctx* ctx, int32_t nblocks);

/* ---- Multi-GPU spatial partition (no reference
 * counterpart: the reference is single-process, PAPER.md:478 lists multi-GPU
 * as future work).  One process and one context per GPU; cells [0, nowned)
 * of the context's (local) mesh are stepped, the rest are ghosts behind cut
 * faces.
 *
 * In-library exchange over NCCL: rank 0 makes a unique id
 * (ttdvm_cuda_nccl_unique_id), shares its 128 bytes out of band, every rank
 * joins with ttdvm_cuda_comm_init (or hands over an existing ncclComm_t with
 * ttdvm_cuda_set_comm) and installs its halo plan with
 * ttdvm_cuda_set_partition.  Every ttdvm_cuda_step then begins by exchanging
 * the ghost cells of the state it starts from -- the (r1, r2) pairs, then the
 * packed cores, grouped ncclSend/ncclRecv on a communication stream --
 * overlapped with the moments, f_S and collision roundings of the owned
 * cells; the face fluxes wait for the halo.  A failure on any rank
 * (nonpositive density, out of memory, ...) reaches every rank through an
 * ncclAllReduce(max) of the status code at the end of the step.  libnccl is
 * bound at run time (dlopen of libnccl.so.2; TTDVM_NCCL_LIB overrides):
 * TTDVM_ENCCL when it is missing or a call fails. */
int ttdvm_cuda_nccl_unique_id(char* id128);
int ttdvm_cuda_comm_init(ttdvm_ctx* ctx, int32_t nranks, int32_t rank, const char* id128);
/* nccl_comm: an ncclComm_t the caller owns (NULL detaches). */
int ttdvm_cuda_set_comm(ttdvm_ctx* ctx, void* nccl_comm, int32_t nranks, int32_t rank);
/* Halo plan: per peer q (rank peer_rank[q]) the owned local cells to send,
 * send_ids[send_off[q] .. send_off[q+1]), and the ghost local cells to fill,
 * recv_ids[recv_off[q] .. recv_off[q+1]); both sides list a pair's cells in
 * the same order (ascending global id).  Also sets nowned. */
int ttdvm_cuda_set_partition(ttdvm_ctx* ctx, int32_t nowned, int32_t npeers,
                             const int32_t* peer_rank, const int64_t* send_off,
                             const int32_t* send_ids, const int64_t* recv_off,
                             const int32_t* recv_ids);
/* [0] exchanges, [1] bytes sent, [2] bytes received, [3] host ms spent in
 * the exchange (issue + waits), since the context was created. */
int ttdvm_cuda_halo_stats(ttdvm_ctx* ctx, double* out4);

/* Caller-driven alternative (no communicator set): the caller refreshes
 * the ghosts after every step with the calls below (packed in the
 * ttdvm_tt_batch layout into / out of caller-provided DEVICE buffers that it
 * exchanges itself).  Ghosts carry over unchanged otherwise. */
int ttdvm_cuda_set_owned(ttdvm_ctx* ctx, int32_t nowned);
/* Pack the current states of cells ids[0..count) into dev_dst; fills
 * ranks_out[2*count] and offsets_out[count+1] (doubles).  ENOMEM with
 * offsets_out[count] = required size if capacity is too small. */
int ttdvm_cuda_halo_pack(ttdvm_ctx* ctx, int32_t count, const int32_t* ids, int32_t* ranks_out,
                         int64_t* offsets_out, double* dev_dst, int64_t capacity);
/* Install received ghost states (ranks / offsets as produced by pack). */
int ttdvm_cuda_halo_unpack(ttdvm_ctx* ctx, int32_t count, const int32_t* ids,
                           const int32_t* ranks, const int64_t* offsets, const double* dev_src);

/* Macroparameters of the state the last step started from
 * (compute_macro, proj/src/physics.cpp:17-67), 11 doubles per owned cell:
 * n, u0, u1, u2, T, rho, p, S0, S1, S2, nu (= p / mu(T)). */
int ttdvm_cuda_macros(ttdvm_ctx* ctx, double* out);

/* Intermediates of the last step for lock-step parity (set: 0 = Phi per
 * face, 1 = J rounded before the nu scale, 2 = R per cell, 3 = f_S per
 * cell).  Same two-call protocol as the state. */
int ttdvm_cuda_stage_layout(ttdvm_ctx* ctx, int32_t set, int32_t* count, int32_t* ranks,
                            int64_t* offsets);
int ttdvm_cuda_stage_download(ttdvm_ctx* ctx, int32_t set, double* cores, int64_t capacity);

/* Batched TtTensor::rounded (proj/src/tt_tensor.cpp:139-193) of sums:
 * output o = round(sum_{t in [group_off[o], group_off[o+1])} scale[t] * in[t]).
 * group_off == NULL means one input per output.  The result stays on the
 * device; fetch it with ttdvm_cuda_result_layout / _download.  margins
 * (optional, 2 per output) receives each cut's relative decision margin
 * min |tail + s^2 - budget| / budget over the kept/dropped boundary. */
int ttdvm_cuda_round_batch(ttdvm_ctx* ctx, const ttdvm_tt_batch* in, int32_t nout,
                           const int64_t* group_off, const double* scale, double eps,
                           int32_t cap, double* margins);
/* Re-round the input batch and sums of the last ttdvm_cuda_round_batch call,
 * already resident on the device (config-3 microbench: inputs in HBM),
 * `repeats` times; *ms = device time of all repeats (CUDA events on the
 * library stream).  Same kernels and result as ttdvm_cuda_round_batch. */
int ttdvm_cuda_round_resident(ttdvm_ctx* ctx, double eps, int32_t cap, int32_t repeats,
                              double* ms);
int ttdvm_cuda_result_layout(ttdvm_ctx* ctx, int32_t* ranks, int64_t* offsets);
int ttdvm_cuda_result_download(ttdvm_ctx* ctx, double* cores, int64_t capacity);

/* Batched compute_macro (proj/src/physics.cpp:17-67): 11 doubles per
 * tensor as in ttdvm_cuda_macros (nu needs the gas). */
int ttdvm_cuda_macro_batch(ttdvm_ctx* ctx, const ttdvm_tt_batch* in, double* out);

/* Batched compute_collision (proj/src/physics.cpp:112-125): the result
 * batch holds round(f_S - f, eps) per tensor, i.e. J before its final
 * scaled(nu) (physics.cpp:118); nu = macros[11*t + 10].  macros optional. */
int ttdvm_cuda_collision_batch(ttdvm_ctx* ctx, const ttdvm_tt_batch* in, double eps,
                               double* macros);

/* Face factors of oblique normals (replaces VelocityGrid::abs_xi_estimate /
 * xi_normal_positive / xi_normal_negative, proj/src/velocity_grid.cpp:61-146):
 * mode 0 = abs_xi_estimate(normal, cap), 1 = xi_normal_positive(normal,
 * cap - 2) (i.e. from_full(max(xi_n,0), 1e-12, cap)), 2 = the negative part.
 * normals [3*count] must be unit vectors.  Results go to the result batch
 * (ttdvm_cuda_result_layout / _download).  diag (optional, 4 per normal):
 * chosen candidate's squared Frobenius error, the runner-up's, the choice
 * (2 * h index + strategy) and the smallest kept sigma^2 / sigma_max^2. */
int ttdvm_cuda_face_factors(ttdvm_ctx* ctx, int32_t count, const double* normals, int32_t cap,
                            int32_t mode, double* diag);

/* Diffuse-wall ghost densities n_w of the last step (wall_ghost,
 * proj/src/boundary.cpp:84-101), one per wall face in face order. */
int ttdvm_cuda_wall_densities(ttdvm_ctx* ctx, double* out);

/* Set-up facts of the last step's mesh: [0] distinct oblique normals,
 * [1] of them with a kept singular value below 1e-14 sigma_max (the FP64
 * operand's own noise), [2] wall faces, [3] face-factor build time (us),
 * [4] cell blocks of the step (ttdvm_cuda_set_blocks). */
int ttdvm_cuda_setup_info(ttdvm_ctx* ctx, int64_t* info5);

/* Device time (ms) of the kernels of the last call, by phase:
 * [0] moments, [1] shakhov build, [2] round f_S, [3] round collision,
 * [4] round fluxes, [5] round residual, [6] round update, [7] bookkeeping. */
int ttdvm_cuda_phase_times(ttdvm_ctx* ctx, double* ms8);
/* Canonical work of the last call by phase: FLOPs
 * of the reference rounding algorithm on the actual ranks, compulsory HBM
 * bytes (inputs read once + outputs written once), and rounding launches. */
int ttdvm_cuda_phase_work(ttdvm_ctx* ctx, double* flops8, double* bytes8, int32_t* launches8);
/* Both of the above for the first nphase <= 9 phases; phase [8] is the
 * wall-density kernel (wall_ghost, proj/src/boundary.cpp:84-101).  Phases
 * 0, 1 and 8 report the algorithmic work of the moments (16 convolutions,
 * cores read twice), the rank-4 f_S build (24 n doubles written per cell)
 * and the wall inner products.  Any pointer may be NULL. */
int ttdvm_cuda_phase_report(ttdvm_ctx* ctx, int32_t nphase, double* ms, double* flops,
                            double* bytes, int32_t* launches);
/* ttdvm_cuda_step timed with CUDA events on the library's stream (ms). */
int ttdvm_cuda_timed_step(ttdvm_ctx* ctx, double dt, double eps, int32_t cap, int32_t nsteps,
                          double* ms);
/* Measured FP64 FMA peak of this device (TFLOP/s), the roofline
 * denominator of the FP64-bound rounding kernels. */
int ttdvm_cuda_fp64_peak(ttdvm_ctx* ctx, double* tflops);
/* Diagnostics: per-phase SM cycles (thread 0 of every CTA, summed) of the
 * rounding kernel since the previous call; on != 0 keeps collecting. */
int ttdvm_cuda_round_profile(ttdvm_ctx* ctx, int on, uint64_t* cycles16);
/* Number of kernel launches issued by the last call. */
int64_t ttdvm_cuda_launch_count(const ttdvm_ctx* ctx);
/* Enable/disable per-phase CUDA-event timing (costs one sync per phase). */
int ttdvm_cuda_set_profiling(ttdvm_ctx* ctx, int on);

#ifdef __cplusplus
}
#endif

#endif /* TTDVM_CUDA_H_ */
