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
  LB_ERR_BREAKDOWN = 8
} lb_status;

int lb_abi_version(void);
const char* lb_last_error_string(void);
/* Host-side query: SM count and compute capability of the current device. */
int lb_device_info(int* sm_count, int* cc_major, int* cc_minor);

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
 * Hardware probes (no reference counterpart): FP64 FMA-pipe peak
 * (flops = blocks*256*iters*256) and the 1/sqrt seed/refinement, used to state
 * the measured fp64 roofline and the kernel's rsqrt accuracy. */
int lb_probe_dfma(double* scratch, int blocks, int iters, void* stream);
int lb_probe_rsqrt(const double* x, double* y, int64_t n, int mode,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LAPBEL_B200_H */
