/*
 * splitfft_b200.h -- C ABI of the B200-native split-format DFT.
 *
 * The reference (`splitfft`, pure Python/NumPy) has no FFI: its boundary is
 * the Python operator API in pkg/src/splitfft/__init__.py:14-55.  Each entry
 * point below replaces one piece of that API so that a ctypes / cffi / cgo
 * binding can drive the GPU path with plain pointers and sizes
 * (INTEGRATION.md shows the bindings).  No torch types cross this boundary.
 *
 * Conventions
 *   - Every call returns an int status: SFFT_OK (0) or an SFFT_E* code.
 *     sfft_last_error() returns a thread-local message for the last failure.
 *     Python maps 1 -> ValueError, 2 -> CapacityError, 3 -> RuntimeError,
 *     mirroring the reference's exception types (transform.py:72-76,
 *     errors.py:4-5).
 *   - Plans are immutable after creation and may be shared by host threads;
 *     exec calls are re-entrant on distinct buffers (transform.py:46-52).
 *   - exec calls are asynchronous and stream-ordered on `stream`
 *     (a cudaStream_t, NULL = legacy default stream); they never allocate
 *     and never synchronise.
 */
#ifndef SPLITFFT_B200_H
#define SPLITFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFFT_ABI_VERSION 1

/* status codes */
#define SFFT_OK 0
#define SFFT_EINVAL 1    /* bad argument            -> ValueError    */
#define SFFT_ECAPACITY 2 /* size above a limit       -> CapacityError */
#define SFFT_ECUDA 3     /* CUDA runtime failure     -> RuntimeError  */

/* dtypes: the arithmetic type of the planes */
#define SFFT_F32 0
#define SFFT_F64 1

/* algorithm, transform.py:41-43 (Algorithm.DIT / Algorithm.DIF) */
#define SFFT_DIT 0
#define SFFT_DIF 1

/* direction: forward kernel exp(-j 2 pi n k / N), unnormalised; inverse by
 * the channel-swap identity with 1/N (transform.py:273-298) */
#define SFFT_FORWARD (-1)
#define SFFT_INVERSE (+1)

/* kernel family of the fused (log2n <= 12) path */
#define SFFT_KERNEL_AUTO 0  /* TMA-fed persistent kernel when the rows allow it, else LDG/STG */
#define SFFT_KERNEL_LDG 1   /* per-thread global loads/stores (any stride/alignment, interleaved) */
#define SFFT_KERNEL_TMA 2   /* require the TMA kernel (planar, 16-byte aligned rows and strides) */
#define SFFT_KERNEL_PASS 3  /* log2n > 12: one launch per stage group (auto's choice except fp64 log2n = 28) */
#define SFFT_KERNEL_PASS2 4 /* 20 <= log2n <= 28: L2-fused group pairs, two launches (auto: fp64 log2n = 28 only) */

/* plan limit, transform.py:32 (MAX_PLAN_M) */
#define SFFT_MAX_LOG2N 30

typedef struct sfft_plan sfft_plan;

/* ABI version of the loaded library (== SFFT_ABI_VERSION). */
int sfft_abi_version(void);

/* Thread-local message describing the last failed call on this thread. */
const char *sfft_last_error(void);

/* Replaces make_plan(m, algorithm, max_m=...) (transform.py:65-85).
 * Validation order and messages follow the reference: log2n < 0 -> EINVAL
 * "stage count m must be >= 0"; log2n > max_log2n -> ECAPACITY "exceeds the
 * plan limit"; unknown algorithm -> EINVAL.  Builds the snapped stage-factor
 * table on the host (twiddle.py:46-57, transform.py:82) and uploads it to
 * `device`.  max_log2n <= SFFT_MAX_LOG2N. */
int sfft_plan_create(int log2n, int dtype, int algorithm, int device,
                     int max_log2n, sfft_plan **out);

/* Same, with an explicit register radix (log2; 0 = tuned default) and
 * kernel family (SFFT_KERNEL_*), optionally OR-ed with SFFT_PRE_OFF /
 * SFFT_PRE_ON (fp32: fetch each pass's base factors before the data; the
 * default follows the tuned table).  Used by the tuner and the tests. */
#define SFFT_PRE_OFF 0x10
#define SFFT_PRE_ON 0x20
int sfft_plan_create_ex(int log2n, int dtype, int algorithm, int device,
                        int max_log2n, int log2_radix, int kernel,
                        sfft_plan **out);

int sfft_plan_destroy(sfft_plan *plan);

/* Plan introspection: log2n, dtype, algorithm, device, number of kernel
 * launches per exec, register radix (log2), kernel family used for aligned
 * planar rows (SFFT_KERNEL_*).  Any pointer may be NULL. */
int sfft_plan_info(const sfft_plan *plan, int *log2n, int *dtype,
                   int *algorithm, int *device, int *launches_per_exec,
                   int *log2_radix, int *kernel);

/* The launch schedule exec uses for `batch` rows (interleaved != 0: the
 * interleaved layout): kernel launches per exec, and HBM sweeps per exec --
 * passes that read and write the whole signal once (one launch per sweep).
 * No reference analogue (introspection, used for the roofline unit). */
int sfft_exec_schedule(const sfft_plan *plan, int64_t batch, int interleaved,
                       int *launches, int *sweeps);

/* The kernel exec launches for `batch` aligned planar rows (interleaved != 0:
 * the interleaved layout): family (SFFT_KERNEL_TMA / _LDG / _PASS), its
 * log2 register radix, and `warp` = 1 when it is the warp-per-signal
 * bulk-copy kernel (fp64 N = 1024 radix 32).  kernel=auto plans switch
 * kernels by batch size.  Introspection for the bench's roofline label. */
int sfft_exec_kernel(const sfft_plan *plan, int64_t batch, int interleaved,
                     int *family, int *log2_radix, int *warp);

/* Bytes of device workspace exec needs for `batch` rows (0 for the fused
 * single-kernel path, log2n <= 12). */
int sfft_workspace_bytes(const sfft_plan *plan, int64_t batch, size_t *bytes);

/* The hot path.  Replaces the split->split composite
 * SplitSignal(re, im) -> interleave -> fft|ifft -> deinterleave
 * (service/app.py:43-52, transform.py:273-298), batched over `batch` rows.
 * Planar SoA: x_re/x_im/y_re/y_im are device pointers to `batch` rows of
 * 2^log2n elements of the plan dtype; row r of a plane starts at
 * ptr + r*stride elements.  In place (y == x) is allowed.
 * direction: SFFT_FORWARD or SFFT_INVERSE.  workspace: device pointer of at
 * least sfft_workspace_bytes() bytes (may be NULL when that is 0). */
int sfft_exec_split(const sfft_plan *plan, const void *x_re, const void *x_im,
                    void *y_re, void *y_im, int64_t batch, int64_t in_stride,
                    int64_t out_stride, int direction, void *workspace,
                    void *stream);

/* Same transform on the reference's interleaved layout
 * (InterleavedBuffer, layout.py:46-86: [re0, im0, re1, im1, ...]).
 * x/y point at `batch` rows of 2^log2n (re, im) pairs; strides count pairs.
 * Replaces fft(plan, buf) / ifft(plan, buf) (transform.py:273-298). */
int sfft_exec_interleaved(const sfft_plan *plan, const void *x, void *y,
                          int64_t batch, int64_t in_stride, int64_t out_stride,
                          int direction, void *workspace, void *stream);

/* The literal per-stage operators on the interleaved layout, in place,
 * batched over `batch` rows of 2^log2n (re, im) pairs (stride in pairs):
 * butterfly_stage W^(i) -- within each block of 2^i pairs, pair q and pair
 * q + 2^(i-1) become their sum and difference (transform.py:88-101) -- and
 * twiddle_stage D^(i) -- pair q >= 1 of each block's second half is
 * multiplied by the plan's stage-i factor w_i[q], the identity column left
 * untouched (transform.py:104-120; stage 1 is the identity).  Composed with
 * the pairwise bit reversal they reproduce fft_dit / fft_dif bit for bit
 * (fp64).  EINVAL "stage index i out of range for m=..." as the reference. */
int sfft_exec_butterfly_stage(int dtype, int log2n, int stage, void *data,
                              int64_t batch, int64_t stride, int device,
                              void *stream);
int sfft_exec_twiddle_stage(const sfft_plan *plan, int stage, void *data,
                            int64_t batch, int64_t stride, void *stream);

/* ---- one transform sharded over nranks GPUs (four-step, one all-to-all) ----
 * N = 2^log2n = N1 * N2 with N1 = 2^floor(log2n/2).  Data distribution
 * (G = nranks, power of two; rank g):
 *   input   x[n], n = N2*n1 + n2, on rank g = n2 / (N2/G), local [n1][n2 % (N2/G)]
 *   output  X[k], k = k1 + N1*k2, on rank h = k1 / (N1/G), local [k2][k1 % (N1/G)]
 * phase 0 runs stages 1..log2 N1 (length-N1 transforms of the local columns)
 * and writes the all-to-all SEND buffer [dest rank][n2 local][k1 local]
 * (G contiguous segments of N/G^2 elements per plane); after an all-to-all of
 * both planes (segment r of rank g -> slot g of rank r's RECV buffer) phase 1
 * runs stages log2 N1 + 1 .. log2n on the RECV buffer and writes the local
 * output.  DIT only; the inverse swaps channels at phase 0 input and phase 1
 * output (transform.py:286-298).  Same arithmetic as the single-GPU plan. */
typedef struct sfft_dist_plan sfft_dist_plan;
int sfft_dist_plan_create(int log2n, int dtype, int nranks, int rank,
                          int device, sfft_dist_plan **out);
int sfft_dist_plan_destroy(sfft_dist_plan *plan);
/* elements per rank (N/G), log2 N1, elements per all-to-all segment (N/G^2) */
int sfft_dist_layout(const sfft_dist_plan *plan, int64_t *local_elems,
                     int *log2n1, int64_t *segment_elems);
int sfft_dist_workspace_bytes(const sfft_dist_plan *plan, size_t *bytes);
/* Pass-kernel launches of phase 0 and phase 1 (each launch reads and writes
 * the rank's N/G elements of both planes once: the HBM sweep count). */
int sfft_dist_schedule(const sfft_dist_plan *plan, int *launches_phase0,
                       int *launches_phase1);
int sfft_dist_exec_phase(const sfft_dist_plan *plan, int phase,
                         const void *x_re, const void *x_im, void *y_re,
                         void *y_im, int direction, void *workspace,
                         void *stream);
/* Phase 0 with the exchange fused into its last launch: instead of writing
 * the send buffer, the kernel stores each destination segment straight into
 * that rank's RECEIVE buffer (slot = this rank) through peer pointers
 * (NVLink/NVSwitch P2P, e.g. torch symmetric memory) -- no separate
 * all-to-all.  peer_re/peer_im: npeers (= nranks <= 8) device pointers of the
 * ranks' receive planes.  The caller orders it with a barrier before (peers
 * done reading) and after (all writes landed) and then runs phase 1. */
int sfft_dist_exec_phase0_p2p(const sfft_dist_plan *plan, const void *x_re,
                              const void *x_im, void *const *peer_re,
                              void *const *peer_im, int npeers, int direction,
                              void *workspace, void *stream);

/* Host-only helpers (no GPU needed). */

/* Stage-m factor table w[q] = cos - j sin of 2 pi q / 2^m, snapped, for
 * q < 2^(log2n-1): wr = real, wi = imaginary part exactly as the reference's
 * FftPlan.stage_factors[m-1] (transform.py:80-84).  Stage i uses
 * w[q << (m-i)]. */
int sfft_twiddle_table(int log2n, double *wr, double *wi);

/* Census of count_flops (transform.py:312-335): out[0..4] = real_mults,
 * real_adds, generic_rotations, quarter_turns, identity_rotations. */
int sfft_count_flops(int log2n, int64_t *out5);

/* Number of kernels this library has launched in this process. */
int64_t sfft_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SPLITFFT_B200_H */
