/*
 * mg.h -- C ABI of libmg, the B200-native (sm_100a) V-cycle of Roberts'
 * diagonally oriented multigrid for Poisson's equation (arXiv math/9907190,
 * /root/reference/PAPER.md, cited as P:line).
 *
 * Problem: solve  nabla^2 u = f  on the unit square (dim 2) or the
 * unit cube (dim 3), homogeneous Dirichlet data (reading A1 of DESIGN.md),
 * on the uniform grid of n = 2^k + 1 nodes per side, h = 1/(n-1).  Each
 * V-cycle forms the residual r = f - L u on the finest grid (5-/7-point
 * Laplacian, or the compact fourth-order Efos2 / Efos4
 * schemes), restricts it down the paper's diagonal hierarchy
 * (Erest2r/Erest2b P:166-176; Erred, Ermagc, Ermagm, Erblu P:426-519), takes
 * one Jacobi step on the coarsest grid, climbs back with one over-relaxed
 * two-colour Jacobi step per level (Eajacr/Eajacb P:350-359 and "similarly
 * for a green grid" P:360; Emprolm/b, Erprolr/m, Egprolg/r P:556-661) and
 * adds the correction: u <- u + v.  There is no interpolation
 * operator.
 *
 * Conventions for every call:
 *  - Arrays are row-major with x fastest: 2D element (i, j) at
 *    base[j * pitch + i]; 3D element (i, j, k) at
 *    base[(k * n + j) * pitch + i] (single GPU).  `pitch` is in elements,
 *    fixed at mg_create_ex time (cfg.pitch; 0 means n, as mg_create uses).
 *    The V-cycle kernels (TMA tiles) read u and f in a "work layout": rows a
 *    multiple of 16 bytes, base 16-byte aligned.  Caller arrays already in
 *    that layout (a pitch whose byte size is a multiple of 16 and aligned
 *    pointers) are read and updated in place.  Otherwise -- e.g. pitch = n,
 *    since n = 2^k + 1 never gives 16-byte rows -- each mg_vcycle /
 *    mg_profile / mg_convergence_factor call copies u and f into library-owned
 *    work arrays (row pitch n rounded up to 128 bytes; one launch of the
 *    library's re-pitch copy kernel per array, 2 x 2 N element moves per call), runs the same kernels there
 *    and copies u back (2 N more).  mg_vcycle_host copies the host arrays
 *    straight into the work layout.  mg_residual and mg_norm read any pitch.
 *  - u, f, r, x are DEVICE pointers on the solver's device unless the name
 *    says _host.  The caller owns them; the library never frees them.  They
 *    must stay alive until the work queued on the solver's stream completes.
 *  - Element type is double (MG_F64) or float (MG_F32) as configured.  All
 *    arithmetic is done in that type, in the canonical evaluation order of
 *    DESIGN.md, without FMA contraction.
 *  - Boundary entries of u must be 0 and are never written.  Boundary entries
 *    of f are read only by the order-4 f-combination (reading A11).
 *  - Calls are asynchronous on the solver's stream (cfg.stream, or the legacy
 *    default stream when NULL) except where noted "synchronises".
 *  - Every call returns an mg_status (0 = MG_OK); no C++ exception crosses
 *    the ABI.  mg_last_error() describes the last failure of a handle.
 *  - A handle is not thread-safe; distinct handles are independent.
 *
 * Multi-GPU (cfg.nranks > 1, nranks a power of two, (n-1)/nranks >= 4,
 * 16-byte row pitch): one process per GPU over NCCL (cfg.nccl_id from
 * mg_nccl_unique_id on rank 0, broadcast by the caller); the grid is cut into
 * y-slabs (dim 2) or z-slabs (dim 3).  Each rank passes only
 * its slab: rows (2D) / planes (3D) [lo, hi) of the global grid
 * (lo = rank (n-1)/nranks, hi = lo + (n-1)/nranks) stored with `ghost` = 2
 * extra rows / planes below and above, i.e. a (hi - lo + 4) x pitch (2D) or
 * (hi - lo + 4) x n x pitch (3D) array whose row / plane 2 is global lo (see
 * mg_local_extent); the global boundary rows / planes 0 and n-1 lie in rank
 * 0's own rows / the last rank's ghost rows and must be 0.  The library fills the ghost rows itself (halo
 * exchange per level).  Levels with fewer than cfg.agglom_points interior
 * nodes (or fewer than 4 rows per rank) are all-gathered and solved
 * redundantly on every rank; residual norms are max-reduced over ranks.
 * With cfg.flags = MG_FLAG_LOOPBACK the nranks ranks are virtual (one process,
 * one GPU, full arrays in and out): the same schedule, halos copied on the
 * device -- used to test the decomposition bit for bit.
 */
#ifndef MG_H
#define MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mg_solver mg_solver;

typedef enum {
  MG_OK = 0,
  MG_EINVAL = -1,        /* bad argument: n != 2^k+1 (k>=2), dim, order, p, pitch, ncycles, NULL */
  MG_ENOMEM = -2,        /* device or host allocation failed */
  MG_ECUDA = -3,         /* a CUDA runtime call failed (message in mg_last_error) */
  MG_ENCCL = -4,         /* an NCCL call failed */
  MG_EUNSUPPORTED = -5,  /* valid but not supported by this build/config (e.g. ranks not dividing n-1) */
  MG_EDIVERGED = -6,     /* a computed residual norm was not finite */
  MG_ENODEV = -7         /* no usable CUDA device (never falls back to the CPU) */
} mg_status;

enum { MG_F64 = 0, MG_F32 = 1 };
/* mg_config.flags */
enum { MG_FLAG_LOOPBACK = 1 };  /* nranks virtual ranks in this process on one GPU (tests the slab
                                   decomposition; caller passes FULL arrays) */
enum { MG_FLAG_CONVENTIONAL = 2 };  /* the paper's "usual" multigrid instead of the diagonal one (SURVEY
                                       8(f) NEXT-3): V(0,1) on
                                       the factor-2 hierarchy, full weighting (9-/27-point), bi/trilinear
                                       interpolation, one two-colour Jacobi sweep per level (DESIGN.md
                                       reading A18), over-relaxation p = p[0] (2D) / p[3] (3D) on the
                                       residual term.  Single GPU; every call of this header applies
                                       (mg_num_levels / mg_level_points describe the diagonal hierarchy). */
enum { MG_FLAG_SLABS = 4 };  /* run the multi-GPU slab solver also for nranks = 1 (one rank owns every row:
                                 the whole transport -- NCCL with cfg.nccl_id, or loopback -- runs with no
                                 neighbours; used to execute the NCCL path on a one-GPU machine) */
enum { MG_NORM_INF = 0, MG_NORM_L2 = 1 };

typedef struct {
  int dim;                 /* 2 or 3 */
  int64_t n;               /* nodes per side incl. boundary, n = 2^k + 1, k >= 2 */
  int order;               /* 2 (5/7-point) or 4 (Efos2 / Efos4) */
  int dtype;               /* MG_F64 or MG_F32 */
  double p[4];             /* 2D: p[0] = p.  3D: p_m, p_r1, p_r2, p_g.
                              Each in (0, 3]. */
  int64_t pitch;           /* elements per row of caller arrays; 0 = n */
  void *stream;            /* cudaStream_t the calls are ordered on; NULL = legacy default stream */
  int device;              /* CUDA device ordinal; -1 = current device */
  int nranks, rank;        /* 1 / 0 for a single GPU */
  const void *nccl_id;     /* 128-byte ncclUniqueId (same on every rank) when nranks > 1 */
  int64_t agglom_points;   /* agglomerate levels with fewer interior nodes; 0 = 1<<18 */
  int flags;               /* MG_FLAG_* (0 for normal use) */
  int sweeps;              /* two-colour Jacobi steps per level on the ascent (0 or 1: the paper's V-cycle).
                              > 1 (2D, single GPU, diagonal scheme; at most 8): the paper's open question of
                              "extra Jacobi iterations at each level" (DESIGN.md
                              reading A19) -- every level, the finest included, repeats its step with its own
                              values in place of the coarser level's.  Runs the plain (non-TMA) kernels. */
} mg_config;

/* Defaults: fp64, pitch = n, NULL stream, current device, 1 rank, p[*] = omega.
 * Errors: MG_EINVAL (n, dim, order, omega), MG_ENODEV, MG_ENOMEM, MG_ECUDA. */
int mg_create(int dim, int64_t n, int order, double omega, mg_solver **out);

/* Full configuration (copied; the caller may free cfg afterwards). */
int mg_create_ex(const mg_config *cfg, mg_solver **out);

/* Frees every library-owned buffer, graph, stream and communicator. NULL ok. */
int mg_destroy(mg_solver *s);

/* Rows (2D) / planes (3D) [lo, hi) of the global grid owned by this rank, and
 * the ghost rows/planes the caller's slab carries on each side.  Single GPU:
 * lo = 0, hi = n, ghost = 0. */
int mg_local_extent(const mg_solver *s, int64_t *lo, int64_t *hi, int64_t *ghost);

/* r = f - L u at every interior node (order as configured; Evpois P:62-67,
 * Efos2, Efos4), r = 0 on the boundary.  r has the layout of u. */
int mg_residual(mg_solver *s, const void *u, const void *f, void *r);

/* ncycles V-cycles in place on u (ncycles = 0: no-op).  res_hist: NULL, or
 * room for ncycles+1 doubles that receive ||f - L u||_inf before every cycle
 * and after the last; a non-NULL res_hist synchronises the stream, needs
 * ncycles < 4096 (MG_EINVAL otherwise; run longer histories in several
 * calls) and returns MG_EDIVERGED if any entry is not finite. */
int mg_vcycle(mg_solver *s, void *u, const void *f, int ncycles, double *res_hist);

/* mg_vcycle with both residual histories of SURVEY 8(a) a16:
 * res_inf as mg_vcycle's res_hist (required when res_l2 is set), and res_l2
 * (NULL, or ncycles+1 doubles) = ||f - L u||_{2,h} = (h^d sum r^2)^(1/2) over
 * the interior nodes before every cycle and after the last.  Both are fused
 * into the passes that form the finest residual (no extra pass over u, f);
 * the L2 sums are accumulated in double, in an order that depends on the
 * launch geometry (equal to a serial sum to rounding).  Synchronises when
 * res_inf is set; errors as mg_vcycle. */
int mg_vcycle_norms(mg_solver *s, void *u, const void *f, int ncycles, double *res_inf, double *res_l2);

/* Same as mg_vcycle on HOST arrays (pitch as configured): copies u and f to
 * the device, runs the cycles, copies u back.  Synchronises.  Pinned host
 * memory makes the copies asynchronous DMA. */
int mg_vcycle_host(mg_solver *s, void *u_host, const void *f_host, int ncycles, double *res_hist);

/* A solve from u = 0 (the V-cycle of P:57-92 iterated from a zero initial
 * approximation, as in every BASELINE config: "V-cycles from u=0") on HOST
 * arrays: f is copied to the device, u
 * starts at 0 there (no upload), `ncycles` V-cycles run, u is copied back
 * into u_host (output only; its previous contents are ignored).  Otherwise as
 * mg_vcycle_host: res_hist (NULL or ncycles+1 doubles) as in mg_vcycle,
 * synchronises, MG_EINVAL on NULL arrays or ncycles < 0. */
int mg_solve_host(mg_solver *s, void *u_host, const void *f_host, int ncycles, double *res_hist);

/* `count` independent solves from u = 0, as mg_solve_host, of the HOST right-
 * hand sides f_hosts[i] into u_hosts[i] (caller layout, pitch as configured).
 * Problem i's upload, its cycles and its download run on three streams over
 * two device staging slots, so on a full-duplex link the download of problem
 * i-1 and the upload of problem i+1 overlap the cycles of problem i; the
 * results equal count calls of mg_solve_host.  Pinned host memory makes the
 * copies asynchronous DMA; entries may alias (the downloads run in problem
 * order, the last one wins).  Synchronises.  MG_EINVAL on count < 0,
 * ncycles < 0 or a NULL array.  Slab (multi-GPU) solvers run the problems one
 * by one. */
int mg_solve_host_batch(mg_solver *s, void *const *u_hosts, const void *const *f_hosts, int count, int ncycles);

/* Global norm of x over the interior nodes: MG_NORM_INF = max |x|,
 * MG_NORM_L2 = (h^d sum x^2)^(1/2).  Reduced over ranks.  Synchronises. */
int mg_norm(mg_solver *s, const void *x, int kind, double *out);

/* Number of interior nodes of level `lev` (0 = finest) and the level count;
 * introspection for tests and the roofline model. */
int mg_num_levels(const mg_solver *s);
int64_t mg_level_points(const mg_solver *s, int lev);

/* Kernel launches queued by one V-cycle on this handle (for the bench's
 * gpu_launches count); with the 2D cross-cycle fusion, a steady-state cycle
 * of a multi-cycle call (the first cycle of a call queues one more). */
int mg_launches_per_cycle(const mg_solver *s);

/* Per-step timing of the V-cycle, for the roofline report.  Runs `ncycles`
 * cycles on (u, f) exactly like mg_vcycle but launched step by step (no CUDA
 * graph) with a CUDA event between steps on the solver's stream; fills up to
 * `cap` entries (one per step of one cycle, finest first) with the step's
 * name, level, kernel launches, mean duration over the cycles and its
 * algorithmic bytes (every array the step must read or write,
 * once, interior nodes only).  Returns the number of steps (> cap: truncated)
 * or a negative mg_status.  Synchronises. */
typedef struct {
  char name[40];
  int level;          /* finer level the step works on (0 = finest) */
  int launches;       /* kernel launches in the step */
  double ms;          /* mean duration per cycle, CUDA events */
  double alg_bytes;   /* algorithmic bytes moved per launch of the step */
} mg_step_stat;
int mg_profile(mg_solver *s, void *u, const void *f, int ncycles, mg_step_stat *out, int cap);

/* Convergence factor of the V-cycle (the paper's rho-bar,
 * "the largest eigenvalue" of the iteration operator, reading A12):
 * power iteration on the error equation.  e is a DEVICE array (layout of u,
 * boundary 0, not all zero) holding the start error; it is normalised, then
 * `iters` times replaced by one V-cycle of it with f = 0, rescaled to unit
 * L2 norm on the device.  ratios (NULL or room for iters doubles) receives
 * ||e_k|| / ||e_{k-1}|| per iteration; *rho = their geometric mean over the
 * second half of the iterations (-> the spectral radius when the dominant
 * eigenvalue is separated; a complex pair still gives its modulus).  On
 * return e holds the normalised last iterate (the slowest error mode).
 * Single GPU (MG_EUNSUPPORTED for nranks > 1); iters >= 2.  Synchronises. */
int mg_convergence_factor(mg_solver *s, void *e, int iters, double *rho, double *ratios);

/* The slab decomposition without a device (host-only planning): rows [lo, hi)
 * owned by `rank`, ghost rows carried on each side, and the first octave
 * whose levels are agglomerated (all-gathered).  nranks = 1: the whole grid.
 * MG_EUNSUPPORTED when the grid cannot be split that way. */
int mg_slab_plan(int dim, int64_t n, int nranks, int rank, int64_t agglom_points, int64_t *lo, int64_t *hi,
                 int64_t *ghost, int *agglom_octave);

/* The multi-GPU schedule the slab solver picks (host-only): *schedule = 1 for
 * the 2D communication-avoiding schedule (one halo exchange of *halo_rows
 * fine rows of u per V-cycle, deep ghost bands computed redundantly;
 * DESIGN.md 8), 0 for the per-level schedule (a halo exchange of 1-2 rows
 * per level; *halo_rows = 2) -- always 0 in 3D and for one rank.
 * MG_EUNSUPPORTED when the grid cannot be split that way. */
int mg_slab_schedule(int dim, int64_t n, int nranks, int64_t agglom_points, int *schedule, int64_t *halo_rows);

/* 128-byte NCCL unique id for cfg.nccl_id (call on one rank, broadcast the
 * bytes to all).  Loads the NCCL library at run time; MG_ENCCL if absent. */
int mg_nccl_unique_id(void *out128);

const char *mg_strerror(int status);
const char *mg_last_error(const mg_solver *s);

#ifdef __cplusplus
}
#endif
#endif /* MG_H */
