/*
 * bhcp_b200.h -- C ABI of the B200-native PinT QBVM/MQBVM solver library
 * (libbhcp_b200.so, sm_100a).
 *
 * The reference (pure Python, package `bhcp`) has no FFI; its boundary is the
 * Python signatures exported from pkg/src/bhcp/__init__.py:11-69. Every entry
 * point below replaces the numeric core of one of those functions; the
 * Python package `paper_2107_06381_b200` wraps them with the reference's
 * signatures and error types (see INTEGRATION.md for the ctypes binding).
 *
 *   bhcp_sine_transform     <- space.sine_transform / SpatialSpectrum.transform
 *                              (pkg/src/bhcp/space.py:163-177, 223-231)
 *   bhcp_step_b             <- pint.step_b_parallel + space.shifted_solve
 *                              (pkg/src/bhcp/pint.py:26-66; space.py:234-283)
 *   bhcp_to_eigenspace      <- circulant.to_eigenspace / apply_inverse_basis
 *                              (pkg/src/bhcp/circulant.py:99-106, 156-164)
 *   bhcp_from_eigenspace    <- circulant.from_eigenspace / apply_basis
 *                              (pkg/src/bhcp/circulant.py:108-115, 167-190)
 *   bhcp_pint_solve         <- pint.solve_pint (pkg/src/bhcp/pint.py:69-110),
 *                              fused dataflow
 *   bhcp_pint_solve_unfused <- pint.solve_pint, literal 3-step dataflow
 *   bhcp_pint_modes / bhcp_pint_levels
 *                           <- the two halves of solve_pint used by the slab-
 *                              decomposed multi-GPU driver
 *
 * Conventions
 *   - Plain pointers and sizes only. Device pointers are CUDA device memory
 *     on the plan's device; `stream` is a cudaStream_t passed as void*.
 *   - complex128 data is interleaved (re, im) doubles, i.e. the memory layout
 *     of numpy.complex128 / torch.complex128.
 *   - "level-major" means a C-contiguous (levels, n_space) array, i.e. one
 *     spatial field per time level, matching the trajectory layout of
 *     pint.py:99 (SolveResult.trajectory is (n_levels, n_space)).
 *   - Spatial fields are flattened in C order, first axis outermost
 *     (space.py:64-74); the sine transform runs along axis -1, then -2
 *     (then -3 for the 3D extension), space.py:175-176.
 *   - Functions only enqueue work; results that need a host decision
 *     (singular shift, imaginary residue) are read with bhcp_read_status,
 *     which synchronises the stream.
 *   - Return codes: BHCP_OK, or one of the BHCP_ERR_* below. The message of
 *     the last error on the calling thread is bhcp_last_error().
 */
#ifndef BHCP_B200_H
#define BHCP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BHCP_OK = 0,
  BHCP_ERR_SINGULAR_SHIFT = 1,     /* space.py:234-246 SingularShiftError */
  BHCP_ERR_IMAGINARY_RESIDUE = 2,  /* circulant.py:182-189 ImaginaryResidueError */
  BHCP_ERR_INVALID = 3,            /* ValueError analogues */
  BHCP_ERR_CUDA = 4
};

typedef struct bhcp_space_plan bhcp_space_plan;
typedef struct bhcp_time_plan bhcp_time_plan;

/* Outcome of a solve, filled by bhcp_read_status. */
typedef struct {
  int code;             /* BHCP_OK / BHCP_ERR_SINGULAR_SHIFT / BHCP_ERR_IMAGINARY_RESIDUE */
  int64_t bad_column;   /* first singular column j (pint.py:52-56), -1 if none */
  double residue;       /* ||Im Y||_F  (circulant.py:184) */
  double norm;          /* ||Y||_F     (circulant.py:183) */
} bhcp_status;

/* Size of the small device status block used by the solve / step-b /
 * from-eigenspace entry points (bad column + norm accumulators). */
size_t bhcp_status_bytes(void);

int bhcp_version(void);
const char* bhcp_last_error(void);

/* Space plan: Dirichlet grid with num_cells subdivisions per axis, dim in
 * {1,2,3} (3 is this library's extension; the reference stops at 2,
 * space.py:42-43). mu1_host holds the m = num_cells-1 one-dimensional
 * eigenvalues (4/h^2) sin^2(k pi / 2M) computed by the caller with the
 * reference expression (space.py:209-211), so shifts match bit for bit.
 * 2D mode eigenvalues are mu1[k1] + mu1[k2] (numpy add.outer, space.py:215);
 * 3D ones (no reference) are the sum of the sorted triple,
 * (mu1[lo] + mu1[mid]) + mu1[hi], shared bit for bit by all permutations. */
int bhcp_space_plan_create(int device, int dim, int num_cells,
                           const double* mu1_host, bhcp_space_plan** out);
void bhcp_space_plan_destroy(bhcp_space_plan* plan);

/* Time plan: n_levels = N+1 (circulant.py:50-53). gamma_host and
 * gamma_inv_host are 2*n_levels doubles (diagonal of Gamma and its inverse,
 * circulant.py:148); shifts_host is 2*n_levels doubles, s_j = d_j / tau
 * (pint.py:95). */
int bhcp_time_plan_create(int device, int n_levels, const double* gamma_host,
                          const double* gamma_inv_host, const double* shifts_host,
                          bhcp_time_plan** out);
void bhcp_time_plan_destroy(bhcp_time_plan* plan);

/* Orthonormal DST-I over the spatial axes of `batch` level-major fields.
 * in/out may alias. is_complex selects complex128 vs float64 data. */
int bhcp_sine_transform(const bhcp_space_plan* sp, const void* in, void* out,
                        int is_complex, int64_t batch, void* stream);

/* One axis pass of the orthonormal DST-I over `batch` level-major fields:
 * axis 0 = the contiguous axis (-1), 1 = axis -2, 2 = axis -3. in/out may
 * alias. bhcp_sine_transform is the sequence of passes 0..dim-1. */
int bhcp_sine_axis(const bhcp_space_plan* sp, const void* in, void* out,
                   int is_complex, int64_t batch, int axis, void* stream);

/* Step (b): for each level j < batch solve (shift_j I - lap) x = rhs_j with
 * the spectral method (DST, divide by shift_j + mu_k, DST). in/out are
 * level-major complex128 (batch, n_space) and may alias; shifts_dev holds
 * 2*batch doubles. The first singular column is recorded in status_dev. */
int bhcp_step_b(const bhcp_space_plan* sp, const void* in, void* out,
                const double* shifts_dev, int64_t batch, void* status_dev,
                void* stream);

/* Step (a): out = ifft_ortho(in * gamma) along the time axis for `batch`
 * sequences. Element t of sequence b is at in[b*in_sb + t*in_st] (element
 * units). One of the two strides must be 1. in_is_complex selects
 * float64/complex128 input; output is complex128. */
int bhcp_to_eigenspace(const bhcp_time_plan* tp, const void* in, int in_is_complex,
                       int64_t batch, int64_t in_sb, int64_t in_st, void* out,
                       int64_t out_sb, int64_t out_st, void* stream);

/* Step (c): Y = fft_ortho(in) / gamma along the time axis; writes Re Y
 * (out_is_complex = 0, float64) or Y (complex128); accumulates ||Re Y||^2 and
 * ||Im Y||^2 into status_dev (reset it with bhcp_status_reset first). */
int bhcp_from_eigenspace(const bhcp_time_plan* tp, const void* in, int64_t batch,
                         int64_t in_sb, int64_t in_st, void* out, int out_is_complex,
                         int64_t out_sb, int64_t out_st, void* status_dev,
                         void* stream);

/* Reset a status block (bad column = none, norms = 0, and the pass-A work
 * counter that the kernels of bhcp_pint_modes / _modes_to / _modes_sym_to
 * schedule their warps with -- a status block must be reset once before
 * its first use; those kernels leave the counter at 0 when they finish). */
int bhcp_status_reset(void* status_dev, void* stream);

/* Synchronise `stream`, read the status block and apply the reference's
 * decision rules: singular shift first (pint.py:52-56), then the imaginary
 * residue test ||Im|| > tol * max(||Y||, tiny) (circulant.py:182-189). */
int bhcp_read_status(const void* status_dev, double tol, bhcp_status* st, void* stream);

/* Fused solve: y (n_levels, n_space) float64 from the
 * final data g (n_space float64) and the condition divisor (methods.py:85-96).
 * ws must hold bhcp_pint_workspace_bytes() bytes of device memory; the status
 * block is inside ws (bhcp_pint_status_ptr). Kernels: status reset, the DST of
 * g, pass A, and the level passes -- for 2D m + 1 = 1024 one level-group kernel
 * (bhcp_pint_levels_fused), whose scratch (counters + two level tiles of Z,
 * 134 MB) is part of ws. Capturable in a CUDA graph; the level-group kernel is
 * a cooperative launch. */
size_t bhcp_pint_workspace_bytes(const bhcp_space_plan* sp, const bhcp_time_plan* tp);
void* bhcp_pint_status_ptr(const bhcp_space_plan* sp, const bhcp_time_plan* tp, void* ws);
int bhcp_pint_solve(const bhcp_space_plan* sp, const bhcp_time_plan* tp,
                    const double* g_dev, double divisor, double* y_dev, void* ws,
                    size_t ws_bytes, void* stream);

/* Literal 3-step dataflow of pint.py:89-99 on level-major complex buffers:
 * rhs assembly, step (a) time transform, step (b), step (c). ws must hold
 * bhcp_pint_unfused_workspace_bytes() bytes. */
size_t bhcp_pint_unfused_workspace_bytes(const bhcp_space_plan* sp, const bhcp_time_plan* tp);
void* bhcp_pint_unfused_status_ptr(const bhcp_space_plan* sp, const bhcp_time_plan* tp, void* ws);
int bhcp_pint_solve_unfused(const bhcp_space_plan* sp, const bhcp_time_plan* tp,
                            const double* g_dev, double divisor, double* y_dev,
                            void* ws, size_t ws_bytes, void* stream);

/* Pass A with per-slab destinations: slab s (levels [slab_bounds[s],
 * slab_bounds[s+1])) of this rank's W goes to slab_dst[s] (host array of
 * nslabs device pointers), in the blocked layout of bhcp_pint_modes. A
 * destination may be another GPU's receive buffer mapped into this process
 * (NVLink peer memory), so pass A stores straight into the rank that runs
 * the level passes on that slab and no separate all-to-all runs
 * (distributed.py, transport "peer"). Replaces, with the all-to-all, the
 * reference's space<->time transpose. */
int bhcp_pint_modes_to(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat,
                       int64_t k_begin, int64_t k_end, double* const* slab_dst, int nslabs,
                       const int64_t* slab_bounds, void* status, void* stream);

/* Symmetric pass A for the multi-GPU solve. The modes kernels compute one
 * mode of every mirror pair (k1,k2) / (k2,k1) (2D) or (k1,k2,k3) /
 * (k2,k1,k3) (3D; for n = 257 every permutation of a sorted triple), whose
 * shifted spectra are bit-identical, from a tile list. bhcp_pint_sym_tiles returns the list length for (sp, tp), or 0 when
 * that time length has no symmetric kernel. bhcp_pint_modes_sym_to
 * computes tiles [tile_begin, tile_end) and stores every mode of each class
 * into every level slab s: at slab_dst[s] + slab_koff[s][k1] +
 * ((t - b[s]) / 8 * P1 + r) * 8 + (t - b[s]) % 8, where slab_koff[s] is the
 * device int64 block table (length m) of slab s's receiver, as for
 * bhcp_pint_levels_blocked. P ranks that split the list evenly do half the
 * FFT work of a k1-slab split, and store straight into the receivers (peer
 * memory). */
int64_t bhcp_pint_sym_tiles(const bhcp_space_plan* sp, const bhcp_time_plan* tp);
int bhcp_pint_modes_sym_to(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat,
                           int64_t tile_begin, int64_t tile_end, double* const* slab_dst,
                           const int64_t* const* slab_koff, int nslabs,
                           const int64_t* slab_bounds, void* status, void* stream);

/* The two halves of the fused solve (also used by the slab-decomposed
 * multi-GPU driver).
 * bhcp_pint_ghat: ghat = DST(g) * scale (n_space float64), scale = 1/(divisor*n).
 * bhcp_pint_modes: for spatial modes [k_begin, k_end) write
 *   W(k, t) = ghat[k] * Re(gamma_inv_t * FFT_t(1/(s_j + mu_k)))
 *   and accumulate the residue norms / first singular column into status_dev
 *   (reset with bhcp_status_reset before its first use: the pass-A kernels
 *   also take their work from a counter in it).
 *   Layout of W (K = k_end - k_begin, k local, P1 = m^(dim-1)):
 *     dim 1 (nslabs = 0):  level-major, W[t * K + k]
 *     dim >= 2:            blocked by level slabs s (nslabs = 0: one slab
 *       [0, n); else host int64 bounds b[0..nslabs], b[0] = 0, b[nslabs] = n,
 *       inner bounds multiples of 8; mode range = whole k1 planes):
 *       W[off_s + ((k1 * NT_s + tl / 8) * P1 + r) * 8 + tl % 8]
 *       k = k1 * P1 + r, tl = t - b[s], NT_s = ceil((b[s+1]-b[s]) / 8),
 *       off_s = K * 8 * sum_{s' < s} NT_{s'} -- one contiguous chunk per slab.
 * bhcp_pint_level_pass: pass 0 = inverse DST along the last spatial axis from
 *   W into the level-major y (nlev, n_space): dim 1 level-major W; dim >= 2
 *   blocked W with k1's first block at koff_dev[k1] (device int64 table of
 *   length m) or, when koff_dev is null, the single-slab layout above.
 *   pass p >= 1 = inverse DST along axis -(p+1) in place on y.
 * bhcp_pint_w_pass: inverse DST along spatial axis `axis` (0 .. dim-2) in
 *   place on the blocked W of `nlev` levels (single-slab layout, or a receive
 *   buffer whose k1 blocks sit at the uniform stride NT * m^(dim-1) * 8, which
 *   is what the slab layouts produce). TMA tensor loads/stores; needs dim 2/3
 *   and m + 1 in {256, 512} (bhcp_pint_w_passes_supported), W 16-byte
 *   aligned.
 * bhcp_pint_levels / bhcp_pint_levels_blocked: all spatial passes, W (or the
 *   receive buffer) -> y. levels_blocked needs dim >= 2; its koff_dev is
 *   either NULL -- k1 blocks at the uniform stride NT * P1 * 8, the layout
 *   bhcp_pint_modes / _modes_to / _modes_sym_to write for one level slab --
 *   or a device int64 table of m block offsets, which may be arbitrary.
 *   Uniform input (bhcp_pint_levels, or koff_dev NULL): when
 *   bhcp_pint_w_passes_supported, the strided axes run first in place on the
 *   input (which is therefore overwritten), then the last axis into y, all on
 *   TMA views of the one stride. An explicit table runs the general passes
 *   (pass 0 into y, then the strided axes on y) and leaves the input
 *   untouched. */
int bhcp_pint_ghat(const bhcp_space_plan* sp, const double* g_dev, double scale,
                   double* ghat_dev, void* stream);
int bhcp_pint_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp,
                    const double* ghat_dev, int64_t k_begin, int64_t k_end,
                    double* w_dev, int nslabs, const int64_t* slab_bounds,
                    void* status_dev, void* stream);
int bhcp_pint_level_pass(const bhcp_space_plan* sp, const double* in_dev,
                         const int64_t* koff_dev, double* y_dev, int64_t nlev,
                         int pass, void* stream);
int bhcp_pint_w_pass(const bhcp_space_plan* sp, double* w_dev, int64_t nlev, int axis,
                     void* stream);
int bhcp_pint_w_passes_supported(const bhcp_space_plan* sp);
int bhcp_pint_levels(const bhcp_space_plan* sp, double* in_dev, double* out_dev,
                     int64_t batch, void* stream);
int bhcp_pint_levels_blocked(const bhcp_space_plan* sp, double* in_dev,
                             const int64_t* koff_dev, double* out_dev, int64_t batch,
                             void* stream);
/* bhcp_pint_levels_fused: all spatial passes, blocked W (uniform k1 stride, as
 * bhcp_pint_levels) -> y, as ONE persistent kernel over level groups that stay
 * in L2 where bhcp_pint_levels_sync_bytes(sp, nlev) > 0 (dim 2, m + 1 = 1024:
 * k_dst_lvl4 -- row tasks W -> a scratch Z inside sync_dev, column tasks Z -> y
 * while the level tile is still L2-resident; 16 instead of 32 B/DOF of
 * compulsory HBM traffic). sync_dev: a device buffer of at least that many
 * bytes, used as per-level-tile counters and the two Z level-tile slots (the
 * call zeroes the counters on the stream); it must not be shared by
 * concurrent calls. Where the sync size is 0 this is bhcp_pint_levels (any
 * dim; the input may be overwritten) and sync_dev is ignored. Reference: the per-level
 * DSTs of pint.py:94-96 / space.py:163-177. */
/* bhcp_pint_solve_batch: nb independent fused solves of one g on one space
 * plan (BASELINE config 5: the alpha sweep, 64 alpha x 2 kinds), each with its
 * own time plan tps[i] (its omega) and divisor divisors[i] (host array), all
 * time plans of one length. y_dev holds the nb trajectories one after the
 * other ((nb, n_levels, n_space) float64); status_dev holds nb status blocks
 * (bhcp_status_bytes() each, read with bhcp_read_status). One DST of g serves
 * every pair; for 1D with n = 4097 pass A of up to 32 pairs runs as one launch
 * and the level phase of all pairs as one transpose and one rows DST, so a
 * chunk of the sweep needs no host synchronisation. Each trajectory is bitwise
 * the one bhcp_pint_solve gives for that pair. Reference: solve_pint
 * (pint.py:69-110) per (kind, alpha) as the driver's sweep calls it
 * (bench.py:196-209, 265-271). */
size_t bhcp_pint_batch_workspace_bytes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, int nb);
int bhcp_pint_solve_batch(const bhcp_space_plan* sp, const bhcp_time_plan* const* tps, int nb,
                          const double* g_dev, const double* divisors, double* y_dev, void* status_dev,
                          void* ws, size_t ws_bytes, void* stream);
size_t bhcp_pint_levels_sync_bytes(const bhcp_space_plan* sp, int64_t nlev);
int bhcp_pint_levels_fused(const bhcp_space_plan* sp, const double* in_dev, double* out_dev,
                           int64_t nlev, void* sync_dev, void* stream);

/* Relative residual of a pint-kind trajectory (replaces
 * methods.residual / SolveResult.residual_norm, pkg/src/bhcp/methods.py:239-247,
 * 281-285): result_host[0] = ||rhs - A y||, result_host[1] = ||rhs|| (plain
 * 2-norms; the reference ratio is [0] / [1]). A y uses the backward-Euler
 * rows, the corner 1/divisor and the Dirichlet Laplacian with mesh width h.
 * ws: bhcp_residual_workspace_bytes() bytes of device memory. Synchronises. */
size_t bhcp_residual_workspace_bytes(void);
int bhcp_residual_norm(const bhcp_space_plan* sp, const double* y_dev, int64_t n_levels,
                       double tau, double divisor, double h, const double* g_dev,
                       void* ws, double* result_host, void* stream);

/* Closed-form per-mode solve of any of the four kinds (
 * replaces baseline.solve_spectral_oracle, pkg/src/bhcp/baseline.py:67-112):
 * y (num_steps+1, n_space) = DST(DST(g)/D_k * rho_k^t). kind: 0 qbvm,
 * 1 mqbvm, 2 pint-qbvm, 3 pint-mqbvm. Verification / reference solver only;
 * bhcp_pint_solve never uses it. */
size_t bhcp_spectral_workspace_bytes(const bhcp_space_plan* sp, int64_t n_levels);
int bhcp_spectral_solve(const bhcp_space_plan* sp, int kind, double alpha, double tau,
                        int64_t num_steps, const double* g_dev, double* y_dev, void* ws,
                        size_t ws_bytes, void* stream);

/* Forward model in per-mode form (baseline.march_forward,
 * baseline.py:115-129, equal to the N-step recursion to roundoff):
 * g = DST(rho^N DST(z0)). */
int bhcp_march_forward(const bhcp_space_plan* sp, double tau, int64_t num_steps,
                       const double* z0_dev, double* g_dev, void* stream);

/* Out-of-place transpose of a (rows, cols) matrix of 8- or 16-byte elements. */
int bhcp_transpose(const void* in, void* out, int64_t rows, int64_t cols,
                   int elem_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BHCP_B200_H */
