/*
 * lbm.h — C ABI of the B200-native MRT lattice Boltzmann stream–collide library
 * (liblbm.so), the hot path of arXiv 2211.02435 (Hennig, Holzer, Rüde, lbmpy 1.1).
 *
 * One call of lbm_step() performs, for every lattice cell of this rank's slab,
 * the fused update of eq:LbUpdateScheme:
 *   pull (or AA in-place) gather of the q populations
 *   -> conserved quantities rho, u                              (eq:DensityAndVelocity[FromDeviation])
 *   -> forward Chimera transform to raw moments                 (eq:RawMomentChimeraTransform)
 *   -> binomial Chimera raw -> central moments             [CENTRAL, CUMULANT]
 *   -> central moments -> cumulants                             (eq:CumulantAndCentralMomentGenFuncs) [CUMULANT]
 *   -> relaxation q* = q + S (q_eq - q)                         (eq:MrtUpdateGeneral / ...DeviationOnly /
 *                                                                ...AbsoluteFromZeroCentered)
 *   -> the inverse transforms and the store of q populations.
 *
 * Conventions
 * -----------
 * Units: lattice units, dx = dt = 1, cs^2 = 1/3, background density rho0 = 1.
 * rho0 is a unit choice (the update is homogeneous of degree one in f; R21): for a
 * background density lambda pass rho / lambda and scale the returned density by lambda.
 *
 * Velocity ordering (the paper leaves it free except xi_0 = 0).  The
 * SLAB AXIS is the last lattice axis (z in 3D, y in 2D).  Order: rest; the velocities with
 * slab component 0; slab component +1; slab component -1 (the negations of the +1 group in
 * the same order).  Inside a group the in-plane part runs (0,0),(1,0),(-1,0),(0,1),(0,-1),
 * (1,1),(-1,-1),(1,-1),(-1,1) (2D: x-part 0, 1, -1), keeping the stencil's members:
 *   D2Q9  (x,y): 0 (0,0) | 1 (1,0) 2 (-1,0) | 3 (0,1) 4 (1,1) 5 (-1,1) | 6 (0,-1) 7 (-1,-1) 8 (1,-1)
 *   D3Q19: 0 | 1-8 in-plane | 9-13 (0,0,1),(1,0,1),(-1,0,1),(0,1,1),(0,-1,1) | 14-18 their negations
 *   D3Q27: 0 | 1-8 in-plane | 9-17 (0,0,1),(1,0,1),(-1,0,1),(0,1,1),(0,-1,1),(1,1,1),(-1,-1,1),
 *          (1,-1,1),(-1,1,1) | 18-26 their negations
 * so opposite(i) pairs (1,2),(3,4),(5,6),(7,8) in-plane and i <-> i + n_up across the slab
 * axis, and the populations crossing a slab face form one contiguous index block.
 *
 * Collision-space bases (one relaxation rate per polynomial, in this order; R2):
 *   D3Q27: 1; x, y, z; xy, xz, yz, x^2-y^2, x^2-z^2 [shear]; x^2+y^2+z^2 [bulk];
 *          xy^2+xz^2, x^2y+yz^2, x^2z+y^2z; xy^2-xz^2, x^2y-yz^2, x^2z-y^2z; xyz;
 *          x^2y^2-2x^2z^2+y^2z^2, x^2y^2+x^2z^2-2y^2z^2; x^2y^2+x^2z^2+y^2z^2;
 *          x^2yz, xy^2z, xyz^2; xy^2z^2, x^2yz^2, x^2y^2z; x^2y^2z^2          (27 rates)
 *   D3Q19: the D3Q27 list without xyz and without the last seven (orders 4 mixed, 5, 6)   (19 rates)
 *   D2Q9 : 1; x, y; xy, x^2-y^2 [shear]; x^2+y^2 [bulk]; x^2y, xy^2; x^2y^2               (9 rates)
 *   POPULATION space (SRT/BGK): a single rate.
 * Rates of the conserved polynomials (orders 0 and 1) are accepted and ignored.
 *
 * Host population arrays: f[i][z][y][x], x fastest, this rank's slab only (2D: f[i][y][x]),
 * in STORED form (delta f = f - f0 when zero_centered), fp64 regardless of storage precision.
 * Host macroscopic arrays: rho[z][y][x]; u[d][z][y][x] (d = 2 for D2Q9, 3 otherwise).
 * For LBM_EQ_SWE the density slot carries the water height h.
 *
 * Errors: every call returns lbm_status; on failure a message is available from
 * lbm_last_error(ctx) (or lbm_last_error(NULL) for a failed lbm_create).  Contexts are
 * thread-compatible, not thread-safe.  All host arrays are borrowed for the duration of the
 * call only; the context owns every device buffer it allocates.
 */
#ifndef LBM_H
#define LBM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lbm_ctx lbm_ctx;

typedef enum {
  LBM_OK = 0,
  LBM_EINVAL = -1,       /* bad argument: null pointer, rate outside [0,2], n_rates != q, extent < 4, ... */
  LBM_EUNSUPPORTED = -2, /* inadmissible combination or not built                     */
  LBM_ENOMEM = -3,       /* device allocation failed                                                     */
  LBM_ECUDA = -4,        /* CUDA runtime error / no device                                               */
  LBM_ENCCL = -5,        /* NCCL unavailable (libnccl.so.2 not loadable) or an NCCL call failed          */
  LBM_ENUMERIC = -6      /* non-finite population detected by lbm_check_finite                          */
} lbm_status;

typedef enum { LBM_D2Q9 = 0, LBM_D3Q19 = 1, LBM_D3Q27 = 2 } lbm_stencil;
typedef enum {
  LBM_SPACE_POPULATION = 0, /* SRT / BGK, T = identity                     */
  LBM_SPACE_RAW = 1,        /* raw moments               */
  LBM_SPACE_CENTRAL = 2,    /* central moments           */
  LBM_SPACE_CUMULANT = 3,   /* cumulants                 */
  /* raw moments in the weighted-orthogonal basis (WO-MRT, Krueger 2017; reading
     R31): the weighted Gram-Schmidt orthogonalisation, <p, r> = sum_i w_i p(xi_i) r(xi_i), of the
     stencil's monomials in graded-lexicographic order (x > y > z): D3Q27 1; x, y, z; x^2, xy, xz,
     y^2, yz, z^2; x^2y, x^2z, xy^2, xyz, xz^2, y^2z, yz^2; x^2y^2, x^2yz, x^2z^2, xy^2z, xyz^2, y^2z^2;
     x^2y^2z, x^2yz^2, xy^2z^2; x^2y^2z^2 (D3Q19: without the xyz-type monomials and orders >= 5;
     D2Q9: 1; x, y; x^2, xy, y^2; x^2y, xy^2; x^2y^2), one rate per orthogonal polynomial in that
     order (the second-order ones, x^2 - 1/3 ..., govern shear AND bulk viscosity).  General rates,
     no body force, continuous equilibrium (absolute, delta, or ABSOLUTE_F0). */
  LBM_SPACE_RAW_WO = 4
} lbm_space;
typedef enum {
  LBM_EQ_ABSOLUTE = 0, /* continuous Maxwellian, absolute form                    */
  LBM_EQ_DELTA = 1,    /* deviation-only delta equilibrium: zero-centered only,
                          not with cumulants                                       */
  LBM_EQ_SWE = 2,      /* shallow water, D2Q9 + absolute storage only; the density slot is the height h:
                          with CENTRAL: Zhou's discrete equilibrium (de Rosis; PAPER.md:998-1021,
                          reading R5); with CUMULANT: the Maxwellian with cs2 = g h / 2 (Venturi;
                          PAPER.md:1023-1026)                                                          */
  LBM_EQ_DISCRETE = 3, /* the equilibrium given as a discrete distribution (
                          reading R29): f_eq_i = w_i rho [1 + 3 xi.u + 9/2 (xi.u)^2 - 3/2 u.u], used
                          in collision space as q_eq = T(f_eq); absolute form.  Equals LBM_EQ_ABSOLUTE
                          for population / raw moments on D2Q9 and D3Q27 (reading R4).  General rates
                          only (no rate specialisation), no body force.                              */
  LBM_EQ_DISCRETE_DELTA = 4, /* its deviation f_eq - f0: zero-centered only, not with cumulants      */
  LBM_EQ_ABSOLUTE_F0 = 5     /* the absolute equilibrium for zero-centered storage with the background
                                added to the POPULATIONS before the transform, q = T(df + f0), and
                                subtracted after the inverse one: eq:MrtUpdateAbsoluteFromZeroCentered
                                written literally (reading R30).  LBM_EQ_ABSOLUTE with
                                zero_centered instead adds the closed-form background moments T(f0) in
                                moment space.  Same values up to rounding; the rounding differs (the
                                Table 3 study).  Zero-centered only; general rates;
                                population, raw (both bases), central-moment and cumulant spaces. */
} lbm_equilibrium;
typedef enum { LBM_FP64 = 0, LBM_FP32 = 1 } lbm_precision;
/* Streaming patterns: two-grid pull; in place: AA (Bailey 2009; several
   ranks with periodic faces, or one rank with periodic and/or no-slip faces), Esoteric Pull (Lehmann 2022; single rank, periodic) and Esoteric
   Twist (Geier & Schoenherr 2017, reading R28: every cell touches only its positive octant
   x + {0,1}^d; single rank, periodic) and Esoteric Push (Lehmann 2022, reading R32: the mirror
   of Esoteric Pull — in each opposite pair the member stored at its streaming destination is
   the second one, opp i > i, so a cell touches its negative half-neighbourhood; single rank,
   periodic).  All four in-place patterns move the same bytes (PAPER.md:861-862 lists them). */
typedef enum {
  LBM_PULL = 0,
  LBM_AA = 1,
  LBM_ESOTERIC_PULL = 2,
  LBM_ESOTERIC_TWIST = 3,
  LBM_ESOTERIC_PUSH = 4
} lbm_streaming;
typedef enum { LBM_BC_PERIODIC = 0, LBM_BC_NOSLIP = 1 } lbm_bc;
typedef enum {
  LBM_REGION_ALL = 0,
  LBM_REGION_BOUNDARY = 1,
  LBM_REGION_INTERIOR = 2,
  /* two fused steps across ranks with an external exchange (multi-rank pull contexts whose
     kernels run two-step sweeps, >= 6 planes per slab, no walls; else LBM_EUNSUPPORTED):
     PAIR_INTERIOR: steps t+1 and t+2 of planes [2, nzl - 2) from the current grid into the
     next (no neighbour data); PAIR_BOUNDARY1: step t+1 of planes {0,1,2} and {nzl-3..nzl-1}
     into 8 scratch planes, then exchange lbm_get_halo(2); PAIR_BOUNDARY2: step t+2 of planes
     {0,1} and {nzl-2,nzl-1} from the scratch into the next grid, then exchange
     lbm_get_halo(1) and lbm_swap once (PAIR_BOUNDARY2 counts the pair's first step). */
  LBM_REGION_PAIR_INTERIOR = 3,
  LBM_REGION_PAIR_BOUNDARY1 = 4,
  LBM_REGION_PAIR_BOUNDARY2 = 5,
  /* three fused steps (2D slabs of >= 10 rows, nx % 256 == 0: lbm_get_halo(3) succeeds): TRIPLE_INTERIOR
     (rows [3, nzl-3), any stream, concurrently with the rest), TRIPLE_BOUNDARY1, exchange
     lbm_get_halo(3) (level-1 scratch rows), TRIPLE_BOUNDARY2, exchange lbm_get_halo(4)
     (level-2 scratch rows), TRIPLE_BOUNDARY3, exchange lbm_get_halo(1), lbm_swap. */
  LBM_REGION_TRIPLE_INTERIOR = 6,
  LBM_REGION_TRIPLE_BOUNDARY1 = 7,
  LBM_REGION_TRIPLE_BOUNDARY2 = 8,
  LBM_REGION_TRIPLE_BOUNDARY3 = 9
} lbm_region;

typedef struct {
  int nx, ny, nz;  /* GLOBAL lattice extents; D2Q9: nz = 1 (the slab axis is then y)        */
  int bc[3][2];    /* [axis][low, high] lbm_bc; periodic must be set on both faces of an axis */
  int precision;   /* lbm_precision (storage and arithmetic precision)                        */
  int streaming;   /* lbm_streaming; Esoteric: one rank, periodic; AA + no-slip: one rank     */
  double swe_g;    /* lattice gravity g (LBM_EQ_SWE only)                                     */
  int device;      /* CUDA device ordinal                                                     */
  void *stream;    /* cudaStream_t to enqueue on, or NULL: the library creates its own        */
  int rank;        /* slab decomposition along the slab axis: this rank ...                  */
  int nranks;      /* ... of nranks (nranks must divide the slab extent; slabs >= 2 planes)   */
  /* In-library NCCL halo exchange: the 128-byte ncclUniqueId that
     rank 0 obtained from lbm_nccl_get_unique_id and every rank received (any host
     transport), or NULL.  Non-NULL: lbm_create joins an NCCL communicator of nranks ranks
     (collective: every rank calls lbm_create; one GPU per rank — NCCL refuses two ranks on
     one device) and lbm_step exchanges the halos with ncclSend / ncclRecv, overlapped with
     the interior planes, whenever the fused peer push (lbm_peer_connect) is not connected.
     With nranks = 1 the single slab exchanges with itself through NCCL (the periodic wrap
     goes through the ghost planes, as on every rank of a decomposition).  The id is read
     during lbm_create only. */
  const void *nccl_id;
  /* Optional device allocator for the population grids (e.g. the torch caching allocator);
     both NULL: cudaMalloc / cudaFree.  dev_alloc returns NULL on failure (LBM_ENOMEM). */
  void *(*dev_alloc)(size_t bytes, void *user);
  void (*dev_free)(void *ptr, void *user);
  void *alloc_user;
} lbm_domain;

/* Device-side halo description of one population grid (nranks > 1).
   send_lo: local slab plane 0, the slab-component -1 population block -> rank-1's recv_hi
   send_hi: local plane n-1, the slab-component +1 block               -> rank+1's recv_lo
   recv_lo/recv_hi: the ghost planes below/above the slab (same population blocks).
   Every block is contiguous, 'bytes' long. */
typedef struct {
  void *send_lo, *send_hi, *recv_lo, *recv_hi;
  size_t bytes;
} lbm_halo;

/* Element layout of one device population grid of a rank's slab (all in ELEMENTS of the
   storage precision): element (zz, i, y, x) at zz*plane + i*pop + y*pitch + x, zz = local
   slab plane + 1 (zz = 0 and zz = planes-1 are the ghost planes).  halo_* are the element
   offsets of the lbm_halo blocks, each halo_elems long. */
typedef struct {
  size_t pitch, pop, plane, planes, elements;
  size_t send_lo, send_hi, recv_lo, recv_hi, halo_elems;  /* pull                              */
  size_t aa_pre_send_lo, aa_pre_send_hi, aa_pre_recv_lo, aa_pre_recv_hi;      /* AA, before odd */
  size_t aa_post_send_lo, aa_post_send_hi, aa_post_recv_lo, aa_post_recv_hi;  /* AA, after odd  */
} lbm_layout;

typedef struct {
  int q, d;                 /* populations per cell, dimensions                          */
  int offset, extent;       /* this rank's slab along the slab axis (global plane index) */
  int nx, ny, nz;           /* global extents                                            */
  size_t pitch;             /* x pitch of the device rows (elements)                      */
  size_t bytes_per_element; /* 8 (fp64) or 4 (fp32)                                       */
  size_t device_bytes;      /* population storage allocated on the device                 */
  long long steps_done;     /* time steps taken since the last init/set                   */
  int rate_specialization;  /* kernel variant chosen from the rates:
                               0 general; 1 fully regularised (every rate but the shear
                               group equals 1, the "R-" methods of PAPER.md:795); 2 higher-
                               order regularised (D3Q27 orders 5-6 equal 1).  Rates equal to
                               one become compile-time constants; set the environment
                               variable LBM_RATE_SPECIALIZATION=0 to force 0.            */
  int temporal_blocking;    /* time steps per sweep of lbm_step: 2 when pairs of steps are
                               fused (pull, single rank, periodic; D3Q19 fp64 with nx % 16 == 0,
                               ny % 8 == 0 (16x8 tiles), or D2Q9 with nx % 256 == 0 (256-cell
                               strips); >= 1184 CTAs = tiles x slab chunks of >= 32 planes;
                               3 for those D2Q9 lattices with >= 8 rows: triples of steps in
                               one sweep (k_pullD_2d), then a pair / single step for the rest
                               of n; LBM_TB_DEPTH=2 (read per call) keeps pairs;
                               the intermediate step stays in shared memory; the same
                               collision code, equal to single steps up to FMA contraction
                               by the compiler, i.e. to rounding), else 1.  Environment
                               LBM_TEMPORAL_BLOCKING: 0 (read at create) forces 1; 1 drops
                               the CTA-count condition.                                    */
  int cuda_graph_steps;     /* time steps per CUDA-graph launch of lbm_step (0: none).  Small
                               single-rank lattices (<= 2^20 cells) are launch-bound: the
                               first lbm_step call captures 32 single steps from each storage
                               parity into two graphs (re-captured after lbm_set_force), and
                               every lbm_step(n) replays floor(n / 32) of them before plain
                               launches of the rest; same kernels, bitwise equal.
                               Environment LBM_CUDA_GRAPHS=0 (read per call) disables it.   */
  int resident_cluster;     /* CTAs of the thread-block cluster that runs ALL n steps of an
                               lbm_step(n) in one launch with the lattice resident in shared
                               memory (2D, pull, single rank; the rows of each CTA plus two
                               ghost rows of both grids must fit its shared memory, <= 512
                               cells per CTA, i.e. lattices up to 8192 cells; halo rows
                               cross via distributed shared memory, one cluster barrier per
                               step; same collision code, bitwise equal); 0: not used.
                               Environment LBM_RESIDENT=0 disables it, LBM_RESIDENT_CLUSTER=k
                               caps the cluster size (both read per call).                 */
  int peer_wait_host;       /* 1 when the fused halo push of this connected context orders its
                               phases on the host (a neighbour shares this GPU; see
                               lbm_peer_connect), 0 for device-side waits or no peer path.  */
} lbm_info;

/* Creates a context: validates admissibility, allocates the population grid(s) (two for
   PULL, one for AA; each with one ghost plane per slab face) and uploads the rates.
   relaxation_rates: n_rates doubles in basis order (1 for POPULATION, q otherwise).
   zero_centered: store delta f = f - f0.  On failure *out = NULL. */
lbm_status lbm_create(lbm_stencil stencil, lbm_space collision_space, lbm_equilibrium equilibrium,
                      const double *relaxation_rates, int n_rates, const lbm_domain *domain,
                      int zero_centered, lbm_ctx **out);
lbm_status lbm_destroy(lbm_ctx *ctx);
const char *lbm_last_error(const lbm_ctx *ctx);
lbm_status lbm_get_info(const lbm_ctx *ctx, lbm_info *info);

/* Writes the post-collision state f*(x, 0) = f_eq(rho, u) of the method's own equilibrium
   (stored form) for this rank's slab.  rho: [cells]; u: [d][cells] (host, fp64).  Resets
   the step counter.  Multi-rank callers must exchange halos of the current grid afterwards. */
lbm_status lbm_init_macroscopic(lbm_ctx *ctx, const double *rho, const double *u);

/* n fused stream–collide time steps, asynchronous on the context stream.
   One rank: the single-rank kernels (two-step sweeps, graph replay or the cluster-resident
   loop where they apply, lbm_info).  Several ranks (or a context created with nccl_id):
   COLLECTIVE, every rank calls it with the same n, ranks stay in lock-step.  It runs the fused
   peer push when the context is connected (lbm_peer_connect; then identical to lbm_step_peer),
   else the in-library NCCL exchange (lbm_domain.nccl_id): per step the two boundary planes,
   then ncclGroupStart / 2 x ncclSend + 2 x ncclRecv (the contiguous halo blocks of lbm_get_halo,
   zero-copy) / ncclGroupEnd on the context stream while the interior planes run on a second
   stream; multi-rank pull contexts with two-step sweeps advance pairs of steps with two
   exchanges per pair (the LBM_REGION_PAIR_* sequence).  The first call after
   lbm_init_macroscopic / lbm_set_populations exchanges the current halo first (lbm_peer_prime
   on the peer path).  LBM_EUNSUPPORTED for a multi-rank context with neither transport (then
   drive lbm_step_region + lbm_get_halo with an external exchange); LBM_ENCCL if NCCL fails. */
lbm_status lbm_step(lbm_ctx *ctx, int n);

/* Writes a fresh 128-byte ncclUniqueId into out128 (rank 0; broadcast it to the other ranks
   and pass it as lbm_domain.nccl_id).  LBM_ENCCL if libnccl.so.2 cannot be loaded (the NCCL
   already loaded into the process, e.g. torch's, is preferred; LBM_NCCL_LIB overrides the
   path) or ncclGetUniqueId fails; the message is in lbm_last_error(NULL). */
lbm_status lbm_nccl_get_unique_id(void *out128);

/* Multi-rank building blocks of one step: run the step's kernel on the given planes on
   'stream' (NULL: context stream), then lbm_swap() once all regions are done and the halos
   were exchanged.  PULL: updates the current grid into the next grid; exchange the next
   grid's halo (lbm_get_halo(1)) before lbm_swap.  AA: the step's kernel is the odd one when
   lbm_info.steps_done is even (state A), else the even one; before an odd step exchange
   lbm_get_halo(0) ("pre": the neighbours' boundary slots the odd step reads), after it
   lbm_get_halo(1) ("post": what the boundary cells wrote into the ghost planes returns to
   the neighbours); even steps touch only their own cells and need no exchange. */
lbm_status lbm_step_region(lbm_ctx *ctx, lbm_region region, void *stream);
lbm_status lbm_swap(lbm_ctx *ctx);
/* PULL: which = 0 the current grid, 1 the next grid, 2 the scratch of the two-step regions
   (LBM_REGION_PAIR_*), 3 / 4 the level-1 / level-2 scratch of the three-step regions
   (LBM_REGION_TRIPLE_*; LBM_EUNSUPPORTED where the context has none).  AA: which = 0 pre-odd,
   1 post-odd. */
lbm_status lbm_get_halo(lbm_ctx *ctx, int which, lbm_halo *out);

lbm_status lbm_sync(lbm_ctx *ctx);

/* Fused halo exchange between slab contexts (nranks > 1) over NVLink peer
   memory (CUDA IPC) or, for contexts of one process, plain device pointers.
   PULL: the kernel of a step's two boundary planes also stores the slab-crossing populations
   (slab component -1 of plane 0, +1 of the last plane) straight into the neighbours' ghost
   planes of the next grid.  AA: the odd step's boundary kernels read and write the
   neighbours' adjacent boundary planes directly (the odd step is race-free on the global
   lattice, so no ghost data moves at all); the even step is local.  Completion is signalled
   through system-scope flags in the neighbours' memory, so no host or NCCL call sits between
   steps.  Canonical reads after an odd AA step first copy the crossing values back into the
   ghost planes (neighbours must not have started their next step).
   Collective protocol: every rank calls lbm_peer_export, the infos are exchanged (any host
   transport), every rank calls lbm_peer_connect with its lower and upper neighbour's info
   (periodic ring along the slab axis), all ranks pass a barrier, then lbm_peer_prime
   (after every lbm_init_macroscopic / lbm_set_populations too; lbm_step does it itself when
   it is due), then lbm_step(n) or lbm_step_peer(n) with the same n on every rank (ranks must
   stay in lock-step; the grids swap identically).
   The interior planes run on a second stream, overlapping the boundary planes and the
   wait for the neighbours.  A wait that exceeds LBM_PEER_TIMEOUT_S seconds (environment,
   default 60) gives up instead of hanging the GPU and is reported by lbm_peer_status.
   Memory ordering: the boundary kernels' stores into peer memory are released per CTA (a CTA
   barrier, then one system-scope fence by thread 0) before the kernel ends, and the one-thread
   signal kernel that follows on the stream fences at system scope before its release store of
   the phase flag; the neighbour's wait kernel acquires it at system scope.  Environment
   LBM_PEER_FENCE (read per call): 1 (default) per CTA, 2 per thread, 0 none (the ordering then
   rests on kernel completion alone). */
typedef struct {
  unsigned char grid_ipc[2][64]; /* cudaIpcMemHandle_t of population grids 0 and 1          */
  unsigned char flags_ipc[64];   /* cudaIpcMemHandle_t of the completion flags              */
  void *grid[2];                 /* device pointers (used for a peer in the same process)    */
  void *flags;
  long long pid;                 /* exporting process id                                      */
  int device, rank, nranks, stencil, precision, nx, ny, nz;
  long long grid_off[2];         /* byte offset of grid k inside the allocation its IPC handle
                                    names (non-zero when lbm_domain.dev_alloc sub-allocates,
                                    e.g. from a caching allocator; CUDA IPC maps whole blocks) */
  unsigned char uuid[16];        /* cudaDeviceProp.uuid of the exporting context's GPU        */
} lbm_peer_info;
lbm_status lbm_peer_export(lbm_ctx *ctx, lbm_peer_info *out);
/* Maps the neighbours' grids and flags; LBM_EINVAL if their lattice, stencil, precision or
   ranks do not match this context's ring; LBM_EUNSUPPORTED for Esoteric Pull / Twist or one rank
   (at export); LBM_ECUDA if the memory cannot be mapped (no peer access; nothing stays mapped).
   Resets the flags.  Waits: when both neighbours run on other GPUs (one process per GPU, the
   deployment case) a one-thread kernel spins on the flags on the device and n >= 32 steps replay
   captured graphs; when a neighbour shares this GPU (uuid), kernels that wait on one another
   must not run as separate launches on one device (nothing co-schedules them; across processes
   a spinning kernel blocks the context switch), so the HOST polls the flags and enqueues each
   phase's kernels only once its neighbours completed the previous one (no graphs; contexts of
   one process must then be stepped from one host thread each).  Environment LBM_PEER_WAIT
   = host | device (read at connect) overrides the choice.  lower = upper = NULL disconnects (unmaps the neighbours; synchronises). */
lbm_status lbm_peer_connect(lbm_ctx *ctx, const lbm_peer_info *lower, const lbm_peer_info *upper);
/* PULL: pushes the current grid's boundary planes into the neighbours' ghost planes; AA:
   only the handshake (orders the neighbours' initialisation before the first step). */
lbm_status lbm_peer_prime(lbm_ctx *ctx);
/* n time steps with the fused halo push (asynchronous on the context stream).  The phase
   counters live on the device, so the loop is a fixed launch sequence: n >= 32 replays
   captured 32-step CUDA graphs (one per grid parity; LBM_CUDA_GRAPHS=0 disables).  PULL
   methods with two-step sweeps (lbm_info.temporal_blocking == 2 on a connected context: >= 6
   planes per slab, no walls) advance pairs of steps: interior planes by the fused sweep, the
   boundary regions by two single steps through 8 scratch planes behind grid 0 with pushes into
   the neighbours' scratch and ghost planes; every rank must call with the same n.
   LBM_PEER_TB=0 (read at create) keeps single steps.  2D slabs of >= 10 rows (nx % 256 == 0)
   advance TRIPLES instead (lbm_info.temporal_blocking == 3: the interior by the depth-3 sweep,
   the boundary regions by three single steps through 22 more scratch planes, three flag phases
   per triple; LBM_TB_DEPTH=2 keeps pairs); captured graphs then hold 36 steps.  Device-side waits: several contexts
   driven from ONE host thread must be stepped in small interleaved chunks (a context's stream
   waits on the GPU for its neighbours, and enqueuing many of its steps first can fill the
   launch queue before the neighbours' work is enqueued).  Host-ordered waits (neighbours on
   this GPU, lbm_info.peer_wait_host): the call returns once its last phase is enqueued, having
   blocked until the neighbours completed each earlier phase, so every context of a process
   needs its own host thread. */
lbm_status lbm_step_peer(lbm_ctx *ctx, int n);
/* *timed_out = 1 if a wait for a neighbour gave up (results invalid); synchronises. */
lbm_status lbm_peer_status(lbm_ctx *ctx, int *timed_out);

/* rho [cells], u [d][cells] of the canonical post-collision state (host, fp64; synchronises). */
lbm_status lbm_get_macroscopic(lbm_ctx *ctx, double *rho, double *u);
/* Canonical post-collision populations f*(x, t) in stored form, independent of the AA parity
   (reading R11), f[i][z][y][x] fp64 (host; synchronises). */
lbm_status lbm_get_populations(lbm_ctx *ctx, double *f);
/* Uniform body force density force[3] (lattice units, physical axes; 2D: force[2] = 0) for the
   following steps: Guo forcing in the paper's source term q^F of eq:MrtUpdateGeneral
   (reading R23): u = (j + F/2) / rho and q^F = (I - S/2) T(F^G) with
   F^G_i = w_i [3 xi.F + 9 (xi.u)(xi.F) - 3 u.F]; the momentum gains F per step (kappa_100 = -F/2
   before, +F/2 after the collision).  Velocities reported for the
   post-collision state are (j - F/2) / rho.  Cumulant methods (reading R26): q^F is F on the
   first-order cumulants and zero on all cumulants of order >= 2 (no T(F^G) exists for the
   nonlinear transform; Guo's source has no second-order central moments).
   LBM_EUNSUPPORTED for the shallow-water methods.  A zero force restores the unforced kernels. */
lbm_status lbm_set_force(lbm_ctx *ctx, const double *force);
/* Force model of the source term (PAPER.md:538-539 names Guo and He):
   LBM_FORCE_GUO (default, reading R23) or LBM_FORCE_HE (reading R27): F^He_i = f_eq_i(rho, u)
   (xi_i - u).F / (rho c_s^2) with the method's own equilibrium at u = (j + F/2)/rho and the same
   q^F = (I - S/2) T(F^He).  For cumulant methods both give the first-order source of R26.
   Takes effect for the current force (re-selects the kernels) and later lbm_set_force calls.
   LBM_EINVAL for an unknown model. */
typedef enum { LBM_FORCE_GUO = 0, LBM_FORCE_HE = 1 } lbm_force_model;
lbm_status lbm_set_force_model(lbm_ctx *ctx, lbm_force_model model);
/* Global sums over this rank's slab of the canonical state, on the device in fp64 with a
   fixed (deterministic) summation order: mass = sum rho, momentum = sum rho u (physical
   x, y, z; 2D: z = 0), kinetic energy = sum rho |u|^2 / 2 (lattice-node form of
   eq:TGA_kin_energy).  Synchronises. */
typedef struct {
  double mass;
  double momentum[3];
  double kinetic_energy;
} lbm_diagnostics;
lbm_status lbm_get_diagnostics(lbm_ctx *ctx, lbm_diagnostics *out);
/* Canonical post-collision populations of selected cells: cells[n] are local linear indices
   x + nx * (y + ny * z) of this rank's slab (2D: x + nx * y); f [n][q] fp64 stored form (host;
   synchronises).  LBM_EINVAL for an index outside the slab. */
lbm_status lbm_get_cells(lbm_ctx *ctx, const long long *cells, long long n, double *f);
/* Sets the canonical state (converted to the storage precision); resets the step counter. */
lbm_status lbm_set_populations(lbm_ctx *ctx, const double *f);
/* Sets lbm_info.steps_done (e.g. to the saved count after a checkpoint restart through
   lbm_set_populations).  Informational only: the canonical state does not depend on it (the
   storage parity of the in-place patterns is tracked separately).  LBM_EINVAL if steps < 0. */
lbm_status lbm_set_steps(lbm_ctx *ctx, long long steps);
/* LBM_ENUMERIC if any stored population of the current state is not finite. */
lbm_status lbm_check_finite(lbm_ctx *ctx);

/* Test hook: the device collision alone (no streaming) on n_cells independent cells,
   host fp64 f_in/f_out [n_cells][q] in stored form, computed in the storage precision. */
lbm_status lbm_test_collide(lbm_ctx *ctx, const double *f_in, double *f_out, long long n_cells);

/* Host-only helpers (no GPU needed). */
/* Stencil of the documented ordering: q, xi [q][3] (2D: xi_z = 0), opposite [q]. */
lbm_status lbm_stencil_info(lbm_stencil stencil, int *q, int *xi, int *opposite);
/* Slab of 'rank' out of 'nranks' along an axis of 'extent' planes. */
lbm_status lbm_slab_extent(int extent, int rank, int nranks, int *offset, int *local_extent);
const char *lbm_version(void);
/* Device grid layout of 'rank' of 'nranks' for a global (nx, ny, nz) lattice (2D: nz = 1). */
lbm_status lbm_grid_layout(lbm_stencil stencil, lbm_precision precision, int nx, int ny, int nz, int nranks,
                           lbm_layout *out);

/* Diagnostics. */
/* Registers per thread and local (spill) bytes of the kernel that dominates this context's
   lbm_step: the cluster-resident loop, the two-step sweep, the odd in-place kernel, or k_pull. */
lbm_status lbm_kernel_attributes(const lbm_ctx *ctx, int *regs, int *local_bytes);
/* Device pointer and size of a population grid (which = 0 current, 1 next; AA: the single grid). */
lbm_status lbm_device_grid(lbm_ctx *ctx, int which, void **ptr, size_t *bytes);
/* The cudaStream_t the context enqueues on. */
void *lbm_stream(lbm_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* LBM_H */
