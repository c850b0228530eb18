/*
 * adaln_b200.h -- C ABI of the B200 (sm_100a) fused LayerNorm-Modulate (AdaLN) operator.
 *
 * This is the drop-in boundary under the reference's Python operator API
 * (`adaptiveload.adaln`, /root/reference/pkg/src/adaptiveload/adaln/__init__.py).
 * The reference selects a backend module exposing
 *     forward(x, scale, shift, eps) -> (y, mu, rstd)                 _kernels_numba.py:37-42
 *     backward_dx(dy, x, scale, mu, rstd) -> dx                       _kernels_numba.py:65-68
 *     backward_naive(dy, x, scale, mu, rstd) -> (dx, dscale, dshift)  _kernels_numba.py:86-91
 *     dtile_reduce(dy, x, mu, rstd, d_tile, n_tile, fp32_accum)       _kernels_numba.py:130-137
 * (chosen once by _select_backend, adaln/__init__.py:38-53).  The entry points below replace
 * that module: al_adaln_forward replaces `forward`; al_adaln_backward replaces
 * `backward_naive` and `dtile_reduce` + `backward_dx` (dx and dscale/dshift in one pass).
 *
 * Conventions
 *  - Plain pointers to DEVICE memory, sizes in elements, no torch types.  The library never
 *    allocates or frees: the caller owns every output and the workspace.
 *  - All work is stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *    default stream).  Calls are asynchronous; nothing synchronises the host.
 *  - Layout: x, y, dy, dx are row-major [batch, seq, dim] (= [N, dim] rows, N = batch*seq).
 *    scale/shift are [batch, dim] with row stride `mod_stride` elements (mod_stride = dim for
 *    per-sample modulation, 0 to broadcast one [dim] vector over every row -- the reference's
 *    2-D case, adaln/__init__.py:88-96).
 *  - dtype codes: AL_F32, AL_BF16, AL_F16 compute in fp32; AL_F64 computes in fp64.
 *    mean/rstd/dscale/dshift are fp32 for the 16/32-bit dtypes and fp64 for AL_F64.
 *  - dscale/dshift are [batch, dim] when mod_stride != 0, else [dim] (summed over all rows).
 *  - `nonfinite` (device int*, may be NULL): set to 1 by the kernels if an input they validate
 *    (x/scale/shift in forward; dy/x/scale in backward) holds NaN/Inf.  This folds the
 *    reference's `_as_f64` isfinite scan (adaln/__init__.py:81-85) into the single HBM pass;
 *    the caller checks it when it wants the reference's NonFiniteInput behaviour.
 *  - Results are deterministic: fixed CTA->row mapping and a fixed stage-2 reduction order
 *    (SPEC.md:462), so repeated calls are bit-identical.
 */
#ifndef ADALN_B200_H_
#define ADALN_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define AL_API __attribute__((visibility("default")))
#else
#define AL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python layer maps them onto the reference exception types (errors.py:72-85) */
#define AL_OK 0
#define AL_ERR_SHAPE 1      /* ShapeMismatch   (adaln/__init__.py:90,93,127,149)        */
#define AL_ERR_TILE 3       /* InvalidTile     (adaln/__init__.py:151-153)              */
#define AL_ERR_VALUE 5      /* ValueError      (eps <= 0, adaln/__init__.py:105-106)    */
#define AL_ERR_DTYPE 6      /* unsupported dtype code                                    */
#define AL_ERR_WORKSPACE 7  /* workspace too small / NULL                                */
#define AL_ERR_CUDA 8       /* CUDA runtime error; al_last_error() has the text         */

/* dtype codes */
#define AL_F32 0
#define AL_BF16 1
#define AL_F16 2
#define AL_F64 3

/* ABI version of this header (bumped on any signature change or addition): 5. */
AL_API int al_abi_version(void);

/* Human-readable message for the last error on the calling thread. */
AL_API const char* al_last_error(void);

/* Optional: load every kernel image and set its shared-memory attribute on `device`, so later
 * calls are safe inside CUDA-graph capture.  Called lazily by the first launch otherwise. */
AL_API int al_device_init(int device);

/*
 * Forward: y = (x - mu) * rstd * (1 + scale) + shift, mu/rstd per row (population variance,
 * eps inside the sqrt), one HBM read of x and one write of y + mean + rstd.
 * Replaces _kernels_numba.forward / _forward_kernel (_kernels_numba.py:18-42) and the
 * per-call validation of adaln_forward (adaln/__init__.py:99-108).
 */
AL_API int al_adaln_forward(const void* x, const void* scale, const void* shift,
                     void* y, void* mean, void* rstd,
                     int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride,
                     int dtype, double eps, int* nonfinite, void* stream);

/*
 * Gated residual + forward, fused: the DiT block's
 *     x_out = x + gate (.) f          gate per sample like scale/shift ([B, D] rows at mod_stride)
 *     y, mean, rstd = AdaLN(x_out, scale, shift)
 * in one pass (reads x, f; writes x_out, y, mean, rstd).  x_out is rounded to the storage dtype
 * once (single fp32/fp64 fma), and the statistics are those of the rounded x_out, so y equals
 * al_adaln_forward(x_out, ...) bit for bit.  The reference has no fused form: its block calls
 * the residual add and `adaln_forward` separately (adaln/__init__.py:99-108 on the residual
 * stream); gradients compose from al_adaln_backward (dx_out += dxn; df = gate * dx_out;
 * dgate = sum_s f * dx_out).  x_out may not alias x or f.
 */
AL_API int al_adaln_gate_residual_forward(const void* x, const void* f, const void* gate,
                     const void* scale, const void* shift,
                     void* x_out, void* y, void* mean, void* rstd,
                     int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride,
                     int dtype, double eps, int* nonfinite, void* stream);

/* Scratch bytes al_gate_residual_backward needs for its per-CTA dgate partials. */
AL_API int64_t al_gate_residual_backward_workspace_bytes(int64_t batch, int64_t seq, int64_t dim,
                                                  int64_t mod_stride, int dtype);

/*
 * Backward of the gated residual of al_adaln_gate_residual_forward: with
 * G = dxn + gxo (dxn = al_adaln_backward's dx at x_out; gxo = the gradient reaching x_out from
 * elsewhere, NULL for none), writes dx = G, df = gate (.) G ([batch, seq, dim]) and
 * dgate = sum over each sample's rows of f (.) G ([batch, dim] at mod_stride, or [dim] when
 * mod_stride = 0; fp32, fp64 for fp64) -- the last in a fixed order (per-CTA partials, then the
 * AdaLN stage-2 kernel).  One pass: 3 reads + 2 writes per element.
 */
AL_API int al_gate_residual_backward(const void* dxn, const void* gxo, const void* f,
                              const void* gate, void* dx, void* df, void* dgate,
                              void* workspace, int64_t workspace_bytes, int64_t batch,
                              int64_t seq, int64_t dim, int64_t mod_stride, int dtype,
                              void* stream);

/*
 * Fused Q/K RMSNorm of a packed QKV projection ("Q-Norm + K-Norm"; the
 * reference names this op only in its design notes, PAPER.md:301 -- there is no reference
 * implementation, so parity is against a float64 restatement in the tests):
 *     q_n = q * rsqrt(mean(q^2) + eps) * wq,   k_n = k * rsqrt(mean(k^2) + eps) * wk
 * over the full width `dim`, q/k/v being the slices [0, dim), [dim, 2 dim), [2 dim, 3 dim) of
 * each `row_stride`-element row of `qkv` (the [N, 3 dim] output of one projection GEMM).
 * Writes q_n, k_n ([n_rows, dim] contiguous), optionally a contiguous copy of v (`vc`, NULL to
 * skip), and rstd [n_rows][2] (fp32; fp64 for fp64).  dim * element size must be a multiple of
 * 16 bytes and at most 4 KB (dim <= 2048 bf16 / 1024 fp32).
 */
AL_API int al_qk_rmsnorm_forward(const void* qkv, int64_t row_stride, const void* wq,
                          const void* wk, void* qn, void* kn, void* vc, void* rstd,
                          int64_t n_rows, int64_t dim, int dtype, double eps, int* nonfinite,
                          void* stream);

/* Scratch bytes al_qk_rmsnorm_backward needs for its per-CTA dwq/dwk partials. */
AL_API int64_t al_qk_rmsnorm_backward_workspace_bytes(int64_t n_rows, int64_t dim, int dtype);

/*
 * Backward of al_qk_rmsnorm_forward: writes the whole gradient row of the projection output,
 * dqkv = [dq | dk | dv] (dv copied from `dv`, the gradient of `vc`; NULL leaves that slice
 * untouched), and dwq, dwk [dim] (fp32; fp64 for fp64) summed over the rows in a fixed order
 * (per-CTA partials, then the AdaLN stage-2 kernel): deterministic run to run.
 */
AL_API int al_qk_rmsnorm_backward(const void* qkv, int64_t row_stride, const void* wq,
                           const void* wk, const void* rstd, const void* dqn, const void* dkn,
                           const void* dv, void* dqkv, void* dwq, void* dwk, void* workspace,
                           int64_t workspace_bytes, int64_t n_rows, int64_t dim, int dtype,
                           int* nonfinite, void* stream);

/* Bytes of scratch al_adaln_backward needs for the stage-1 (per-CTA) dscale/dshift partials. */
AL_API int64_t al_adaln_backward_workspace_bytes(int64_t batch, int64_t seq, int64_t dim,
                                          int64_t mod_stride, int dtype, int64_t n_tile);

/*
 * Backward: dx (_backward_dx_kernel, _kernels_numba.py:45-62) and dscale/dshift
 * (_reduce_naive_kernel :71-83 / _dtile_kernel_* :94-127) in one pass over dy and x.
 * Stage 1: each CTA owns a contiguous row range and every thread owns fixed feature columns
 * (the paper's D-tile mapping); per-column fp32 partials go to `workspace`.  Stage 2 sums the
 * partials over CTAs in ascending CTA order (fp64 accumulator) in a second kernel (or, opt-in,
 * in the same cooperative launch behind a grid barrier).
 * d_tile / n_tile: the reference TileConfig (adaln/__init__.py:70-73), validated with the
 * reference bounds (1 <= d_tile <= dim, 1 <= n_tile <= rows per reduction group); n_tile caps
 * the rows per stage-1 partial; 0/0 selects the default tiling (adaln_backward_naive).
 * flags: AL_BWD_DETERMINISTIC keeps the whole row range statically partitioned, so dscale and
 * dshift are bit-identical run to run.  Without it (and with 0/0 tiling) the last ~30 % of the
 * rows (inside the last group) are handed out dynamically to whichever CTA is free, which
 * balances the SMs' unequal share of HBM bandwidth; dx is unchanged, and the last group's
 * dscale/dshift then vary at fp32 rounding level with the (timing-dependent) assignment.
 */
#define AL_BWD_DETERMINISTIC 1
AL_API int al_adaln_backward(const void* dy, const void* x, const void* scale,
                      const void* mean, const void* rstd,
                      void* dx, void* dscale, void* dshift,
                      void* workspace, int64_t workspace_bytes,
                      int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride,
                      int dtype, int64_t d_tile, int64_t n_tile,
                      int flags, int* nonfinite, void* stream);

/*
 * Tuning overrides for benchmarking sweeps (0 = automatic).  kernel: 0 = forward, 1 = backward.
 * vecs_per_thread in {1,2,4}; rows_per_stage in {1,2,4}; smem_budget in bytes per CTA;
 * force_generic = 1 routes through the generic (any-shape) kernels.  variant: forward -- the rows
 * kernel flavour (0 auto, 1 packed row, 2 compiler-expanded row, 3 packed + L2 prefetch,
 * 4 mixed-precision 16-bit, 5 TMA-staged lookahead, 6 two rows per warp); backward -- 0 separate stage-2 kernel, 2 stage 2 fused into the
 * stage-1 kernel behind a cooperative grid barrier.  Process-global.  For the forward kernel a nonzero
 * vecs_per_thread / rows_per_stage selects the wide (TMA ring) path.
 */
AL_API int al_set_tuning(int kernel, int vecs_per_thread, int rows_per_stage, int smem_budget,
                         int force_generic, int variant);

/* Describe the launch al_adaln_{forward,backward} would use: writes
 * {path (0 generic, 1 TMA ring, 2 rows-in-registers), grid, threads, vecs_per_thread (rows
 * path: 16-byte vectors per lane), rows_per_stage (rows path: the kernel flavour -- 0 expanded,
 * 1 packed, 2 mixed 16-bit, 3 staged, 4 two rows per warp), stages, smem_bytes}. */
AL_API int al_describe_launch(int kernel, int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride,
                       int dtype, int64_t n_tile, int64_t out[7]);

/* Diagnostics: launch one single-thread kernel on `stream` that spins for `spin_ns`
 * nanoseconds of %globaltimer and writes {globaltimer delta (ns), clock64 delta (SM cycles)}
 * to the device buffer out[2] -- the SM clock actually running between two hot kernels
 * (nvidia-smi samples every >= 10 ms and cannot resolve one 0.1 ms launch). */
AL_API int al_debug_clock_probe(unsigned long long* out, unsigned int spin_ns, void* stream);

/* Diagnostics: per-launch device timestamps.  While `buf` is set, every al_adaln_forward and
 * al_adaln_backward launch takes the next pair of buf[capacity][2] (round robin, reset to pair 0
 * by this call) and writes {earliest CTA start, latest CTA end} (%globaltimer ns; the backward's
 * end is its stage-2 kernel's) with atomicMin / atomicMax -- the caller initialises the pairs to
 * {UINT64_MAX, 0}.  Nothing is inserted into the stream, so the kernels' PDL overlap (which an
 * event record between two launches breaks) is measured as it runs.  NULL disables. */
AL_API int al_debug_set_timestamps(unsigned long long* buf, int capacity);

/* Diagnostics: chunks stolen so far by the deterministic work-stealing backward on protocol
 * slot `device_slot` of the current device (cumulative over launches). */
AL_API int al_debug_steal_count(int device_slot, unsigned int* out);

#ifdef __cplusplus
}
#endif

#endif /* ADALN_B200_H_ */
