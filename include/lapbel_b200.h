/*
 * lapbel_b200.h — C ABI of libb200lb.so, the B200 (sm_100a) implementation of
 * the Laplace-Beltrami GMRES operator-apply hot path of the reference package
 * `lapbel` (/root/reference/pkg/src/lapbel).
 *
 * Conventions (all entry points):
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); work is
 *     enqueued, never synchronised, unless the function says otherwise;
 *   - arrays use the reference's C-contiguous layouts: positions (M,3),
 *     charges (nd,M), dipoles (nd,M,3), pot (nd,Nt), grad (nd,Nt,3),
 *     hess (nd,Nt,3,3) full symmetric (fmm.py:106-113, _pointsum.py:95-108);
 *   - the kernel is sum_j c_j/|x-s_j| - v_j . grad_x 1/|x-s_j| with NO 1/(4 pi)
 *     (fmm.py:3-9); coincident pairs (r == 0) contribute nothing
 *     (fmm.py:136-141, _pointsum.py:41-42);
 *   - return value is an lb_status; lb_last_error_string() describes the last
 *     failure on the calling thread.
 */
#ifndef LAPBEL_B200_H
#define LAPBEL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LB_ABI_VERSION 1

/* Status codes; the Python shim maps them onto the reference's exception
 * types: SHAPE/ARG -> ValueError (fmm.py:60-81,116-123), EPS -> ValueError
 * (fmm.py:1001-1002), CAPACITY -> FmmCapacityError (fmm.py:606-609),
 * KEY -> KeyError (operators.py:119-123), BREAKDOWN -> GmresBreakdown
 * (solver.py:88-89). */
typedef enum {
  LB_OK = 0,
  LB_ERR_SHAPE = 1,
  LB_ERR_EPS = 2,
  LB_ERR_CAPACITY = 3,
  LB_ERR_CUDA = 4,
  LB_ERR_NCCL = 5,
  LB_ERR_ARG = 6,
  LB_ERR_KEY = 7,
  LB_ERR_BREAKDOWN = 8,
  LB_ERR_DEPTH = 9,
  LB_ERR_NEARCAP = 10
} lb_status;

int lb_abi_version(void);
const char* lb_last_error_string(void);
/* Host-side query: SM count and compute capability of the current device. */
int lb_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* Kernel nodes (and all nodes) of a captured CUDA graph (a cudaGraph_t):
 * how many kernels one captured step launches (bench.py gpu_launches). */
int lb_graph_kernel_nodes(void* graph, int64_t* nkernels, int64_t* nnodes);

/* ------------------------------------------------------------------------
 * Direct pairwise sums.
 *
 * lb_p2p replaces evaluate_direct (fmm.py:215-222; blocked numpy
 * _direct_block/_direct_into, fmm.py:130-203).  level: 0 = pot, 1 = pot+grad,
 * 2 = pot+grad+hess.  cmask/dmask: bit l set = density l has active
 * charges/dipoles (FmmSources.charge_active/dipole_active, fmm.py:93-103);
 * charges/dipoles may be NULL when their mask is 0.  grad/hess may be NULL
 * when level excludes them.  accumulate=0 overwrites the outputs,
 * accumulate=1 adds into them.  nd <= 32.
 */
int lb_p2p(const double* tgt, int64_t nt, const double* src, int64_t ns,
           const double* charges, const double* dipoles, int nd,
           uint32_t cmask, uint32_t dmask, int level, double* pot,
           double* grad, double* hess, int accumulate, void* stream);

/* lb_p2p_grouped replaces run_grouped_direct/grouped_direct
 * (_pointsum.py:19-114): group g owns targets t_off[g]:t_off[g+1] (output row
 * t_out[i] of pot/grad/hess, which have ntargets rows) and sources
 * s_off[g]:s_off[g+1].  Outputs are ADDED into (the reference allocates zeros
 * and adds).  Rows must be disjoint across groups, as in the reference's
 * prange.  s_c (nd,nsf), s_v (nd,nsf,3); either may be NULL when its mask is
 * 0.  The Hessian is written full-symmetric. */
int lb_p2p_grouped(const double* t_xyz, const int64_t* t_out,
                   const int64_t* t_off, int64_t ngroups, int64_t ntf,
                   const double* s_xyz, const double* s_c, const double* s_v,
                   const int64_t* s_off, int64_t nsf, int nd, uint32_t cmask,
                   uint32_t dmask, int level, int64_t ntargets, double* pot,
                   double* grad, double* hess, void* stream);

/* ------------------------------------------------------------------------
 * Operator set: the device-resident LayerOperatorSet (operators.py:70-273).
 *
 * Kernel-kind codes follow quadrature.py:47-55 (_KIND_CODES). */
enum {
  LB_KIND_S = 0,
  LB_KIND_D = 1,
  LB_KIND_SPRIME = 2,
  LB_KIND_GRAD_S1 = 3,
  LB_KIND_GRAD_S2 = 4,
  LB_KIND_GRAD_S3 = 5,
  LB_KIND_SPP_PLUS_DPRIME = 6,
  LB_NKINDS = 7
};

/* Everything the apply consumes, as DEVICE pointers that must outlive the
 * handle (they are not copied).  Geometry is SurfaceDiscretization's
 * (surface.py:77-106): nodes/normals (n,3), weights/curvature (n),
 * tangents_u/v (n,3) and inv_metric (n,2,2) (A1 only, may be NULL),
 * over_nodes/over_normals (n_over,3), over_weights (n_over); over_interp is
 * ReferenceElement.over_interp (nbo, nb) row-major (simplex.py:383); the
 * corrections are the scipy CSR arrays of NearCorrections.matrix
 * (quadrature.py:693-700) with ONE shared pattern (indptr int64 (n+1),
 * indices int32 (nnz)) and one value array per kind, NULL for kinds not
 * built.  weight_sum is the host value sum(weights).  phi0 = S[1]
 * (operators.py:99-100) is needed by A1 only and may be set later. */
typedef struct {
  int64_t n, n_over, npatches;
  int nb, nbo;
  const double *nodes, *normals, *weights, *curvature;
  const double *tangents_u, *tangents_v, *inv_metric;
  const double *over_nodes, *over_normals, *over_weights, *over_interp;
  int64_t nnz;
  const int64_t* indptr;
  const int32_t* indices;
  const double* corr[LB_NKINDS];
  double weight_sum;
  const double* phi0;
  /* owned target rows [row0, row0 + nrows) for a sharded apply (nrows < 0:
   * all rows; nrows = 0 is rejected with LB_ERR_SHAPE).  Densities stay full
   * length; only owned rows are written. */
  int64_t row0, nrows;
} lb_opset_desc;

typedef struct lb_opset lb_opset;

/* Allocates the handle's scratch (packed far-field sources, partials, work
 * vectors) once; synchronises the device once. */
int lb_opset_create(const lb_opset_desc* desc, lb_opset** out);
int lb_opset_destroy(lb_opset* h);
int lb_opset_set_phi0(lb_opset* h, const double* phi0);
/* Phi = S^T w (device, n doubles, global rows; NULL detaches): the exact S
 * operator's transpose applied to the node weights, so that the A3 W-average
 * <w, S mu2> / sum(w) (operators.py:261) equals <Phi, mu2> / sum(w) with
 * mu2 = S tau known after the first pass.  With it attached (and no FMM plan)
 * apply_a3's second far sweep accumulates sp_mu1 - sppdp_mu2 - 2H sp_mu2 as
 * ONE sum (no S[mu2] far sum, no S-kind read in the second SpMV pass) and the
 * scalar all-reduce of a sharded apply moves from phase 1 to phase 0
 * (lb_opset_phase_exchange reports it).  The pointer must outlive its use. */
int lb_opset_set_eta_weights(lb_opset* h, const double* phi);
/* FMM far field only: run apply_a3's second far call on two FMM densities
 * (charge c0 with dipole -c1 n, and charge c1; default, 1) or on the
 * reference's three (0: charges c0, c1 and dipole c1 n, operators.py:247-250).
 * Both give the same operator; two densities cut M2L and leaf work by 1/3. */
int lb_opset_set_fmm_a3(lb_opset* h, int two_densities);
/* Route every far-field call of the handle through an FMM plan built on
 * (over_nodes, nodes) (the reference's use_fmm=True path, operators.py:104-112)
 * instead of the exact all-pairs sweeps; NULL restores the sweeps.  The plan
 * must outlive the handle's use of it. */
struct lb_fmm_plan;
int lb_opset_set_fmm(lb_opset* h, struct lb_fmm_plan* plan);
/* out = A_f tau for formulation f in {1,2,3} (apply_a1/a2/a3,
 * operators.py:161-266).  tau/out: device (n), must not alias.  Enqueued on
 * `stream`; no host synchronisation; capturable in a CUDA graph.  Missing
 * correction kind -> LB_ERR_KEY (operators.py:119-123). */
int lb_opset_apply(lb_opset* h, int formulation, const double* tau,
                   double* out, void* stream);
/* Sharded apply: the formulation runs as phases (A3: 3, A2/A1:
 * 2) on the handle's rows; after phase p the caller all-gathers the work
 * vectors lb_opset_phase_exchange lists (rows [row0, row0+nrows) of each
 * rank -> full vectors, see lb_opset_buffers) and, when reduce_scalar is set,
 * sum-all-reduces the handle's scalar.  The result's owned rows are valid
 * after the last phase.  vecs must hold 3 ints. */
int lb_opset_apply_phase(lb_opset* h, int formulation, int phase,
                         const double* tau, double* out, void* stream);
int lb_opset_phase_exchange(const lb_opset* h, int formulation, int phase,
                            int* nvec, int* vecs, int* reduce_scalar);
/* device pointers: work vectors (k * n doubles each, k < 8) and the scalar */
int lb_opset_buffers(const lb_opset* h, double** work, double** scalar,
                     int64_t* row0, int64_t* nrows);

/* out = corrected layer operator of `kind` applied to tau
 * (apply_layer, operators.py:126-155). */
int lb_opset_apply_layer(lb_opset* h, int kind, const double* tau,
                         double* out, void* stream);
/* Per-stage device timing of lb_opset_apply (events between stages; off by
 * default): ms[0..] = consecutive stage durations (far 1, SpMV pass 1, far 2,
 * SpMV pass 2 + glue ...), ms[7] = total (HOST double[8]). */
int lb_opset_set_timing(lb_opset* h, int on);
int lb_opset_stage_times(lb_opset* h, double* ms);
/* Copies the last W-average (eta / ws) the handle computed to dev_out. */
int lb_opset_last_scalar(const lb_opset* h, double* dev_out);

/* Profiling helper: average duration (seconds, written to a HOST double) of
 * `reps` back-to-back launches of one far sweep on the handle's current
 * packed sources: which = 0 S, 1 A3 call 1, 2 A3 call 2, 3 A2 call 1,
 * 4 A2 call 2, 5 A1 call 1, 6 A1 call 2, 7 D.  Synchronises. */
int lb_opset_time_far(lb_opset* h, int which, int reps, double* seconds_host,
                      void* stream);

/* y_j (+)= A_j x_j for njobs <= 4 CSR matrices sharing one pattern
 * (`corr(kind) @ v`, operators.py:119-123).  vals/xs/ys are HOST arrays of
 * njobs DEVICE pointers. */
int lb_csr_spmv(const int64_t* indptr, const int32_t* indices, int64_t nrows,
                int njobs, const double* const* vals, const double* const* xs,
                double* const* ys, int accumulate, void* stream);

/* ------------------------------------------------------------------------
 * GMRES vector kernels (solver.py:48-103).  Deterministic reductions: the
 * scalars land in DEVICE memory, no host synchronisation.
 *
 * lb_arnoldi_mgs: modified Gram-Schmidt of v against rows 0..k of Q
 * (row stride ldq):  for j = 0..k: h[j] = Q_j . v ; v -= h[j] Q_j
 * (solver.py:75-77); then h[k+1] = ||v|| (solver.py:78) and, when
 * h[k+1] > 0, Q_{k+1} = v / h[k+1] (solver.py:80-81).  h: device (k+2). */
int lb_arnoldi_mgs(double* Q, int64_t ldq, int k, int64_t n, double* v,
                   double* h, void* stream);
/* x = sum_j y[j] Q_j, j < k (solver.py:102); y: device (k). */
int lb_combine_rows(const double* Q, int64_t ldq, int k, int64_t n,
                    const double* y, double* x, void* stream);
/* out[0] = x . y  /  out[0] = ||x|| (device scalar) */
int lb_dot(const double* x, const double* y, int64_t n, double* out,
           void* stream);
int lb_nrm2(const double* x, int64_t n, double* out, void* stream);
/* y = x * (1 / s[0]) with s a device scalar (s == 0 leaves y unchanged) */
int lb_scale_inv(const double* x, const double* s, int64_t n, double* y,
                 void* stream);

/* ------------------------------------------------------------------------
 * FMM plan: FmmPlan (fmm.py:722-990) on the device.
 *
 * lb_fmm_plan_create builds the adaptive octree over vstack([spos, tpos]) and
 * the colleague/V/U/W/X lists, bit-exact with _build_tree/_build_lists
 * (fmm.py:559-715): same Morton keys, stable order, DFS-LIFO box ids, list
 * order.  spos/tpos are HOST pointers (plan-time).  flags: LB_FMM_DEVICE_SORT
 * computes the keys and radix-sorts them on the GPU (otherwise host).
 * Capacity overflow -> LB_ERR_CAPACITY (FmmCapacityError, fmm.py:606-609). */
typedef struct lb_fmm_plan lb_fmm_plan;
#define LB_FMM_DEVICE_SORT 1

enum {
  LB_TREE_LEVEL = 0, LB_TREE_IJK, LB_TREE_PARENT, LB_TREE_IS_LEAF, LB_TREE_NSRC,
  LB_TREE_CHILDREN_OFF, LB_TREE_CHILDREN, LB_TREE_SRC_SORTED, LB_TREE_TGT_SORTED,
  LB_TREE_SRC_LO, LB_TREE_SRC_HI, LB_TREE_TGT_LO, LB_TREE_TGT_HI,
  LB_TREE_COLLEAGUES_OFF, LB_TREE_COLLEAGUES, LB_TREE_V_OFF, LB_TREE_V,
  LB_TREE_U_OFF, LB_TREE_U, LB_TREE_W_OFF, LB_TREE_W, LB_TREE_X_OFF, LB_TREE_X
};

int lb_fmm_plan_create(const double* spos, int64_t ns, const double* tpos,
                       int64_t nt, int ncrit, int buffer, int flags,
                       lb_fmm_plan** out);
int lb_fmm_plan_destroy(lb_fmm_plan* plan);
/* sizes[10] = {nbox, nlevels, ns, nt, |children|, |colleagues|, |V|, |U|,
 * |W|, |X|}; geom[4] = {center x y z, half} (HOST arrays, either may be NULL) */
int lb_fmm_plan_info(const lb_fmm_plan* plan, int64_t* sizes, double* geom);
/* copy one int64 tree/list array (LB_TREE_*) into a HOST buffer sized from
 * lb_fmm_plan_info (per-box arrays: nbox; *_OFF: nbox+1; IJK: 3*nbox) */
int lb_fmm_plan_export(const lb_fmm_plan* plan, int what, int64_t* dst);

/* Unit-box translation operators (HOST arrays), as _unit_operators
 * (fmm.py:287-354, rep = 0 "surface": pts = expansion_grid(m) (nrep,3),
 * pinv_up/pinv_dn (nrep,nrep), m2m/l2l 8 x (nrep,nrep) in octant order
 * 4*ox+2*oy+oz) or _unit_operators_grid (fmm.py:431-481, rep = 1 "grid":
 * pts = Chebyshev tensor grid (n^3,3), m2m = m2m_1d 2 x (n,n), vinv (n,n),
 * pinv_up/pinv_dn/l2l unused).  canon: ncanon canonical M2L matrices
 * (nrep,nrep); per lattice offset d (noff of them, off_vec (noff,3)):
 * off_key = its canonical matrix, off_perm (nrep) with
 * K_d[i,j] = canon[off_key][perm[i], perm[j]]. */
typedef struct {
  int rep, m, nrep;
  const double *pts, *pinv_up, *pinv_dn, *m2m, *l2l;
  int ncanon;
  const double* canon;
  int noff;
  const int32_t *off_vec, *off_key, *off_perm;
  const double* vinv;
} lb_fmm_ops;
int lb_fmm_plan_set_operators(lb_fmm_plan* plan, const lb_fmm_ops* ops);
/* FmmPlan.apply (fmm.py:784-990): charges (nd,ns) / dipoles (nd,ns,3) in the
 * plan's source order (DEVICE; NULL when the mask is 0), outputs pot (nd,nt),
 * grad (nd,nt,3), hess (nd,nt,3,3) in target order (DEVICE, overwritten).
 * level 0/1/2 as lb_p2p.  nd <= 32 (processed in chunks of 4). */
int lb_fmm_apply(lb_fmm_plan* plan, const double* charges,
                 const double* dipoles, int nd, uint32_t cmask, uint32_t dmask,
                 int level, double* pot, double* grad, double* hess,
                 void* stream);
/* M2L arithmetic (no reference counterpart: the reference multiplies in
 * fp64).  slices = 0: fp64 DGEMM.  slices = S in [3, 8]: the M2L products run
 * on the tcgen05 tensor cores as int8 GEMMs of S-slice (7 bits each) Ozaki
 * splittings of the canonical matrices and the gathered multipoles, exact
 * int32 accumulation, fp64 recombination; relative error of each M2L product
 * about 1e3 * 2^(-7S) of max|K| max|x| (S = 8: fp64 roundoff).  Needs
 * nrep <= 2048. */
int lb_fmm_plan_set_m2l(lb_fmm_plan* plan, int slices);
/* X / W list evaluation (no reference counterpart; the lists themselves stay
 * the reference's, fmm.py:650-715).  direct = 0: every X and W entry as the
 * reference evaluates it (fmm.py:888-911, 966-988).  direct = 1: an X entry
 * (target box b, source leaf x) whose b is a leaf with 2.5 nt(b) <= nrep, and
 * a W entry (target leaf b, box w) whose w is a leaf with at most nrep
 * sources, are evaluated as direct sums of the leaf's sources at b's targets
 * (they join b's U list): exact where the reference approximates, and fewer
 * pair evaluations.  Results then differ from direct = 0 within the plan's
 * eps.  Rebuilds the device lists on the next apply. */
int lb_fmm_plan_set_xw(lb_fmm_plan* plan, int direct);
/* Owned targets [t0, t1) in the caller's target order (t1 < 0: all, the
 * default).  The tree and lists stay the reference's; M2L, X list, L2L and the
 * leaf stage then run only for boxes with owned targets below them, and only
 * the owned targets' outputs are defined.  A sharded apply gives every rank
 * the same plan with its own row range; the outputs at owned
 * targets equal the unsharded plan's. */
int lb_fmm_plan_set_target_range(lb_fmm_plan* plan, int64_t t0, int64_t t1);
/* Owned sources [s0, s1) (plan source order; s1 < 0: all) of a sharded
 * apply: the upward pass (P2M + M2M) covers only these, so each rank's
 * expansions are partial sums; the upward hook, called on the apply's
 * stream between the M2M and the M2L with the (nbox x nd x nrep) expansion
 * array, must sum them over the ranks in place (an all-reduce). */
typedef void (*lb_fmm_upward_hook)(void* user, double* up, int64_t count, int nd, void* stream);
int lb_fmm_plan_set_source_range(lb_fmm_plan* plan, int64_t s0, int64_t s1);
int lb_fmm_plan_set_upward_hook(lb_fmm_plan* plan, lb_fmm_upward_hook hook, void* user);
/* Low-rank M2L (slices = -1 above): per canonical key k the factors of the
 * truncated SVD  canon_k ~= A_k B_k, A_k (nrep, r_k), B_k (r_k, nrep), both
 * row-major and concatenated over k in key order.  The product then costs
 * 2 nrep r_k instead of nrep^2 per column (fp64 cuBLAS).  A B200 design
 * option with no reference counterpart: the truncation tolerance is the
 * caller's (fmm_plan.py ties it to eps / 100). */
int lb_fmm_plan_set_m2l_factors(lb_fmm_plan* plan, const int32_t* ranks, const double* a,
                                const double* b);
/* device time of each stage of the last apply, ms (HOST double[9]):
 * gather+P2M, M2M, M2L, X, L2L, L2T (grid), leaf (U+DE+W), scatter, total.  Recorded
 * only when timing was enabled with lb_fmm_plan_set_timing(plan, 1). */
int lb_fmm_plan_set_timing(lb_fmm_plan* plan, int on);
int lb_fmm_stage_times(const lb_fmm_plan* plan, double* ms);
/* host wall-clock ms of the plan's setup (HOST double[5]): Morton keys +
 * sort (with LB_FMM_DEVICE_SORT: the whole device tree build), tree (host
 * build: box numbering and ranges; 0 on the device path), interaction lists,
 * device state (built on the first apply; 0 before it), total. */
int lb_fmm_setup_times(const lb_fmm_plan* plan, double* ms);

/* ------------------------------------------------------------------------
 * Near-correction build (quadrature.py, no device
 * counterpart in the reference).
 *
 * Near map (build_near_map, quadrature.py:76-104): target t is near patch p
 * when |x_t - center_p|^2 <= radii_eta_p^2 with radii_eta = (1 + eta) *
 * patch radius (DEVICE arrays).  lb_near_map_count writes the per-target
 * list length (own patch included); the caller scans it into offsets
 * (n + 1) and checks the cap (NearMapCapError, quadrature.py:94-97);
 * lb_near_map_fill writes the lists: own patch first, then ascending. */
int lb_near_map_count(const double* nodes, int64_t n, const double* centers,
                      const double* radii_eta, int64_t npatches,
                      const int64_t* node_patch, int32_t* counts, void* stream);
int lb_near_map_fill(const double* nodes, int64_t n, const double* centers,
                     const double* radii_eta, int64_t npatches,
                     const int64_t* node_patch, const int64_t* offsets,
                     int32_t* patches, void* stream);

/* compute_corrections (quadrature.py:663-701) for all seven kinds (the
 * gradient kinds add the principal-value constants of grad S over the own
 * patch: adaptive curvature/double-layer terms + boundary line integral,
 * quadrature.py:424-498, 562-590).  One
 * entry per near (target, patch) pair; the adaptive subdivision, leaf rules,
 * tolerance (0.1 eps max(sqrt(area fraction), 1e-3)) and geometric forcing are
 * _adaptive_pairs' (quadrature.py:277-420).  values[k][pair_pos[i] + b] =
 * (acc @ vinv - oversampled smooth rule @ over_interp)[b] for pair i.  All
 * pointers DEVICE; rules (u or a, v or b, w) as the reference builds them
 * (triangle_rule(order + 2); Duffy Gauss (order + 2) x (order + 1)); knorm =
 * Koornwinder normalisation sqrt(2(2k+1)(k+l+1)) in k-major order;
 * coeffs_km (npatches, nb, 9) = [x | dx/du | dx/dv] rows in k-major basis
 * order; kmajor_perm as _kmajor_permutation (quadrature.py:147-156).
 * Depth cap 30 -> LB_ERR_DEPTH (AdaptiveDepthError). */
typedef struct {
  int order, nk;
  int kinds[7];
  double eps;
  const double* coeffs_km;
  const double *nodes, *normals, *node_uv;
  const int64_t* node_patch;
  const int64_t* pair_tgt;
  const int32_t* pair_pat;
  const int64_t* pair_pos;
  int64_t npairs;
  const double* srule;
  int nqs;
  const double* drule;
  int nqd;
  const double* knorm;
  const int32_t* kmajor_perm;
  const double* vinv;
  const double* over_interp;
  int nbo;
  const double *over_nodes, *over_normals, *over_weights;
  double* values[7];
  int64_t* stats;  /* optional DEVICE int64[2], accumulated: refinement steps, leaves evaluated */
  /* gradient kinds only (principal-value constants, quadrature.py:562-590):
   * n targets, mean-curvature coefficients (npatches, nb) k-major
   * (curvature @ vinv.T), Gauss-Legendre panel rule on [0, 1] (ng, 2) */
  int64_t n;
  const double* hcoeff_km;
  const double* gauss;
  int ng;
} lb_corr_build_desc;
int lb_corrections_build(const lb_corr_build_desc* desc, void* stream);

/* ------------------------------------------------------------------------
 * Surface geometry from chart expansions (the lbmesh reader
 * `read_mesh`, meshio.py:35-50, ends in build_from_coefficients,
 * surface.py:176-307).  One CTA per patch evaluates nodes, tangents, normals,
 * metric and its inverse, |X_u x X_v|, mean curvature (spectral second
 * derivatives of the stored tangents), the smooth node weights and the
 * oversampled nodes / normals / weights.  Reference-element tables
 * (simplex.py:359-397, row-major, DEVICE): vand, dmat_u, dmat_v (nb x nb),
 * psi_rule and weight_interp (nq x nb), rule_wts (nq), psi_over (no x nb),
 * psi_child (4 x nq x nb: the basis at the rule mapped into each child
 * triangle) and w_interp_o (nq x no/4).  stats (DEVICE double[6]) receives
 * max |D_u X - X_u| over D_v too, max |X_u|,|X_v|, min |X_u x X_v| at the
 * nodes, the same at the oversampled nodes, and the squared norms of the
 * top-degree and of all coefficients of coeffs_x: the caller raises the
 * reference's consistency / DegeneratePatchError checks from them
 * (surface.py:199-223, 265-267).  Outputs are (npatches * nb) or
 * (npatches * no) rows, patch-major. */
typedef struct lb_geom_desc {
  int order, nb, nq, no;
  int64_t npatches;
  const double *coeffs_x, *coeffs_dxdu, *coeffs_dxdv; /* (npatches, nb, 3) */
  const double *vand, *dmat_u, *dmat_v, *psi_rule, *rule_wts, *weight_interp;
  const double *psi_over, *psi_child, *w_interp_o;
  double *nodes, *tangents_u, *tangents_v, *normals; /* (N, 3) */
  double *metric, *inv_metric;                       /* (N, 2, 2) */
  double *sqrt_det_g, *curvature, *weights;          /* (N) */
  double *over_nodes, *over_normals, *over_weights;  /* (N_over, 3/3/1) */
  double* stats;
} lb_geom_desc;
int lb_geom_build(const lb_geom_desc* desc, void* stream);

/* ------------------------------------------------------------------------
 * FP64 tensor-core GEMM of the FMM translations (DMMA 8x8x4, no library):
 * Y[:, c] (+)= alpha * A @ X[kperm_c(:), cols[c]]  with A (M x K) row-major,
 * X / Y column vectors (strides ldx / ldy); cols (optional) gathers X's
 * columns, kperm + kp[c] * K (optional) permutes each column's K index.
 * The kernel behind P2M / M2M / L2L / M2L in lb_fmm_apply. */
int lb_dgemm_cols(const double* A, int lda, int M, int K, const double* X, int64_t ldx,
                  const int64_t* cols, const int32_t* kperm, const int32_t* kp, int64_t ncols,
                  double* Y, int64_t ldy, double alpha, int add, void* stream);

/* ------------------------------------------------------------------------
 * Hardware probes (no reference counterpart): FP64 FMA-pipe peak
 * (flops = blocks*256*iters*256) and the 1/sqrt seed/refinement, used to state
 * the measured fp64 roofline and the kernel's rsqrt accuracy. */
int lb_probe_dfma(double* scratch, int blocks, int iters, void* stream);
/* FP64 tensor-core peak: DMMA 8x8x4 chains, flops = blocks*8*iters*8*512. */
int lb_probe_dmma(double* scratch, int blocks, int iters, void* stream);
/* The same chains with a different A fragment register per DMMA (mode 1) or
 * different A and B fragment registers (mode 2): what a GEMM inner loop
 * feeds the pipe. */
int lb_probe_dmma_operands(double* scratch, int blocks, int iters, int mode, void* stream);
/* Warps 0..nw_mma-1 of every 8-warp block run DMMA chains (it_mma iterations
 * of 8 DMMAs), the others DFMA chains (it_fma iterations of 128 DFMAs per
 * thread): do the FP64 tensor cores and the FP64 FMA pipe overlap? */
int lb_probe_mixed(double* scratch, int blocks, int it_mma, int it_fma, int nw_mma, void* stream);
/* HBM read ceiling in the correction SpMV's access shape: one warp per row of
 * rowlen doubles in each of two streams (a, b: nrows * rowlen doubles each),
 * 256-byte warp loads, eight in flight per stream; out[row] = the row's sum. */
int lb_probe_read_rows(const double* a, const double* b, int64_t nrows, int64_t rowlen, double* out,
                       void* stream);
int lb_probe_rsqrt(const double* x, double* y, int64_t n, int mode,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LAPBEL_B200_H */
