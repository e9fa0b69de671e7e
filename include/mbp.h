/*
 * mbp.h -- C ABI of the B200-native multi-matrix belief-propagation (MBP)
 * reconciliation decoder (libmbp_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void*, a cudaStream_t or NULL for the legacy
 * stream).  Every entry point returns an mbp_status; mbp_last_error() gives
 * the message of the calling thread's last failure.
 *
 * The entry points replace the reference's native seam:
 *
 *   mbp_ensemble_create      <- DecoderWorkspace.__init__ stacked layout
 *                               (pkg/src/mmrecon/decoder.py:88-111) over a
 *                               MatrixEnsemble (matrix.py:173-212)
 *   mbp_syndrome_batch[_device]
 *                            <- compute_syndrome -> _kernels.syndrome_pass
 *                               (decoder.py:137-144; _kernels.py:220-227),
 *                               once per matrix per frame (bench.py:129,
 *                               session.py:253)
 *   mbp_decode_batch[_device]
 *                            <- decode -> _kernels.decode_loop
 *                               (decoder.py:207-274; _kernels.py:323-379),
 *                               batched over frames (bench.py:159-179,
 *                               session.py:305-319)
 *   mbp_c2v_pass / mbp_v2c_pass / mbp_posterior_pass
 *                            <- c2v_update / v2c_update / soft_decision
 *                               (decoder.py:155-200; _kernels.py:230-301)
 *
 * Bit formats are the reference BitBlock layout (bits.py:1-5): bit i of a
 * block in byte i>>3 at position i&7, one row of ceil(len/8) bytes per
 * frame.  A frame's syndrome row is u segments of ceil(m/8) bytes (matrix 0
 * first), the wire layout of protocol.pack_syndromes (protocol.py:137-143).
 */
#ifndef MBP_H
#define MBP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mbp_status {
    MBP_OK = 0,
    MBP_EINVAL = 1,        /* bad argument or shape (reference: ValueError)   */
    MBP_ECUDA = 2,         /* CUDA runtime failure (RuntimeError)             */
    MBP_EUNSUPPORTED = 3,  /* e.g. a check degree above MBP_MAX_CHECK_DEGREE  */
    MBP_ENOMEM = 4         /* device or pinned-host allocation failed         */
} mbp_status;

#define MBP_MAX_CHECK_DEGREE 64
#define MBP_MAX_MATRICES 16

/* DecoderConfig (decoder.py:53-68) plus the device-only knobs. */
typedef enum { MBP_JOINT_GRAPH = 0, MBP_ISOLATED_PER_MATRIX = 1 } mbp_combining_mode;
typedef enum {
    MBP_FP32_PHI = 0,   /* production: fp32 messages, Eq. 6 evaluated in the
                           phi = -ln tanh(x/2) domain (same rule, exact extrinsic
                           sums)                          */
    MBP_FP64_TANH = 1   /* parity mode: fp64 messages, the reference's literal
                           tanh product in ascending order and 2*atanh          */
} mbp_precision;
enum {
    MBP_RECORD_HISTORY = 1,  /* keep the hard decision after every sweep     */
    MBP_KEEP_STATE = 2,      /* keep posteriors/messages readable after decode */
    MBP_PROFILE_PHASES = 4,  /* record a globaltimer stamp at every phase barrier */
    MBP_NO_COMPACTION = 8,   /* never repack undecided frames into dense groups   */
    MBP_EXPLICIT_MESSAGES = 16 /* fp32 joint undamped runs: use the explicit-message
                                  kernel (every c2v stored) instead of the scatter
                                  kernel; needed to read c2v back                 */
};

typedef struct mbp_decoder_config {
    int32_t max_iterations;  /* >= 1, default 60                    */
    int32_t combining_mode;  /* mbp_combining_mode, default joint   */
    int32_t precision;       /* mbp_precision, default MBP_FP32_PHI */
    int32_t flags;           /* MBP_RECORD_HISTORY | MBP_KEEP_STATE */
    double llr_clamp;        /* > 0, default 30                     */
    double damping;          /* [0, 1], default 0                   */
} mbp_decoder_config;

typedef struct mbp_ensemble mbp_ensemble;    /* device copy of H_1..H_u  */
typedef struct mbp_workspace mbp_workspace;  /* per-batch device buffers */

typedef struct mbp_ensemble_info {
    int32_t n, m, u;
    int64_t edges;
    int32_t max_check_degree, max_var_degree;
    int32_t device;
    int32_t sm_count;
} mbp_ensemble_info;

/* ---- library ----------------------------------------------------------- */
const char *mbp_last_error(void);
const char *mbp_version(void);
int mbp_device_count(int *count);

/* ---- ensemble ------------------------------------------------------------
 * chk_ptr: int64[u*m+1], chk_var: int32[E] -- the vertically stacked graph,
 * edges check-major with matrix 0 first (decoder.py:94-105); each matrix's
 * rows sorted ascending with no parallel edges (matrix.py:96-103).  The
 * variable-side view (ascending edge ids per variable, decoder.py:106-111)
 * is built here.  Matrix l owns checks [l*m, (l+1)*m).                    */
int mbp_ensemble_create(int32_t n, int32_t m, int32_t u, const int64_t *chk_ptr,
                        const int32_t *chk_var, int device, mbp_ensemble **out);
int mbp_ensemble_destroy(mbp_ensemble *ens);
int mbp_ensemble_get_info(const mbp_ensemble *ens, mbp_ensemble_info *info);

/* ---- workspace -------------------------------------------------------------
 * Device buffers for up to max_frames frames decoded with cfg (one CUDA
 * stream per workspace; distinct workspaces may run concurrently).        */
int mbp_workspace_create(mbp_ensemble *ens, int32_t max_frames, const mbp_decoder_config *cfg,
                         mbp_workspace **out);
int mbp_workspace_destroy(mbp_workspace *ws);
/* Change max_iterations / llr_clamp / damping / flags without reallocating
 * when the buffer shape allows (precision and combining mode are fixed). */
int mbp_workspace_configure(mbp_workspace *ws, const mbp_decoder_config *cfg);

/* ---- Alice side: syndromes z^l = H_l x (mod 2), Eq. 1 ---------------------
 * keys: [batch][ceil(n/8)]  ->  syn: [batch][u][ceil(m/8)]                  */
int mbp_syndrome_batch_device(mbp_workspace *ws, const uint8_t *keys, int64_t batch,
                              uint8_t *syn, void *stream);
int mbp_syndrome_batch(mbp_workspace *ws, const uint8_t *keys, int64_t batch, uint8_t *syn);

/* ---- Bob side: batched MBP decode ----------------------------------------
 * noisy: [batch][ceil(n/8)], syn: [batch][u][ceil(m/8)], e: crossover
 * probability per frame (e_stride 1) or one for all (e_stride 0), each in
 * (0, 0.5).  Outputs per frame: corrected [batch][ceil(n/8)] (the last hard
 * decision, also for unconverged frames), converged u8, iterations i32
 * (0 for a zero-error frame, max_iterations on failure), mismatches i32
 * (residual syndrome mismatches over all u*m checks, 0 when converged).
 * _device: all pointers are device memory, work is enqueued on `stream`
 * and the call returns without synchronising.  Host variant: host pointers
 * (pinned -- see mbp_host_alloc -- for full-speed copies), copies in,
 * decodes, copies out and synchronises.                                   */
int mbp_decode_batch_device(mbp_workspace *ws, const uint8_t *noisy, const uint8_t *syn,
                            const double *e, int32_t e_stride, int64_t batch,
                            uint8_t *corrected, uint8_t *converged, int32_t *iterations,
                            int32_t *mismatches, void *stream);
int mbp_decode_batch(mbp_workspace *ws, const uint8_t *noisy, const uint8_t *syn,
                     const double *e, int32_t e_stride, int64_t batch, uint8_t *corrected,
                     uint8_t *converged, int32_t *iterations, int32_t *mismatches);

/* ---- state of the last decode (MBP_KEEP_STATE / MBP_RECORD_HISTORY) -------
 * Frame indices are relative to the last (single-chunk) batch.             */
int mbp_workspace_read_posterior(mbp_workspace *ws, int64_t frame, double *posterior_n);
int mbp_workspace_read_c2v(mbp_workspace *ws, int64_t frame, double *c2v_E);
/* v2c as last formed by the check phase (damping with MBP_KEEP_STATE only):
 * the message the final sweep's C2V consumed, i.e. the previous v2c of the
 * last v2c_pass.                                                           */
int mbp_workspace_read_v2c(mbp_workspace *ws, int64_t frame, double *v2c_E);
/* rows [0, rows) of frame's decision history, packed [rows][ceil(n/8)] */
int mbp_workspace_read_history(mbp_workspace *ws, int64_t frame, int32_t rows, uint8_t *out);

/* globaltimer (ns) stamps of the last decode's chunk (MBP_PROFILE_PHASES):
 * kernel start, then after each grid barrier (3 per executed sweep: check,
 * variable, syndrome phases, plus the final stop test), then kernel end;
 * *count of those are written, followed (cap permitting) by 4 compaction
 * stamps: start, slot maps built, arrays moved, done (0 if none).        */
int mbp_workspace_read_phase_times(mbp_workspace *ws, uint64_t *ns, int32_t cap, int32_t *count);

/* ---- single phases on explicit per-edge messages of ONE frame ------------
 * (decoder.py:155-200).  Host arrays in the reference's float64 layout:
 * v2c/c2v [E], priors/posterior [n]; syn_bits u8[m] of the given matrix.
 * Computed with the device kernels in the given precision, on a stream of
 * the ensemble's own (not the legacy default stream); synchronous.         */
int mbp_c2v_pass(mbp_ensemble *ens, int32_t precision, int32_t matrix_index,
                 const uint8_t *syn_bits, double clamp, const double *v2c, double *c2v);
int mbp_v2c_pass(mbp_ensemble *ens, int32_t precision, int32_t matrix_index, int32_t joint,
                 double damping, double clamp, const double *c2v, const double *priors,
                 double *v2c);
int mbp_posterior_pass(mbp_ensemble *ens, int32_t precision, const double *c2v,
                       const double *priors, double *posterior);

/* ---- matrix construction (host) -----------------------------------------
 * Progressive edge growth with the reference's tie-break stream
 * (_kernels.peg_build, _kernels.py:57-161; matrix.peg_construct,
 * matrix.py:215-234): the same seed gives the same matrix.  col_deg[n]
 * column degrees; output rows chk_ptr[m+1], chk_var[sum(col_deg)] (sorted
 * rows).  MBP_EUNSUPPORTED when no check can be attached.                  */
int mbp_peg_build(int32_t n, int32_t m, const int32_t *col_deg, uint64_t seed, int64_t *chk_ptr,
                  int32_t *chk_var);
/* The same construction with each edge's BFS on GPU `device` (level-
 * synchronous, discovery order kept exact) and the tie-break stream on the
 * calling thread: the matrix mbp_peg_build gives, at n = 2^20 in minutes
 * instead of hours.  Column degrees <= 4, check degrees <= 16.           */
int mbp_peg_build_device(int32_t n, int32_t m, const int32_t *col_deg, uint64_t seed,
                         int64_t *chk_ptr, int32_t *chk_var, int device);
/* The same construction in stages: variables [v_begin, v_end) on top of the
 * graph in vn_adj ([n][4] int32 check ids per variable in edge order, -1 =
 * none; rows < v_begin complete), which receives the new rows; *state is the
 * tie-break stream at v_begin (derived from seed when v_begin == 0) and at
 * v_end on return.  Stages chained over [0, n) give mbp_peg_build_device's
 * matrix (a long build can checkpoint and resume).                        */
int mbp_peg_build_device_range(int32_t n, int32_t m, const int32_t *col_deg, uint64_t seed,
                               uint64_t *state, int32_t v_begin, int32_t v_end, int32_t *vn_adj,
                               int device);

/* ---- synthetic BSC frames (the reference's frame streams) ---------------
 * Rows [batch][ceil(n/8)] of Alice's keys and Bob's noisy keys for frames
 * first .. first+batch-1 of a grid point, bit-identical to the reference's
 * bench._frame_inputs (bench.py:123-130) / channel.rng_stream
 * (channel.py:29-35): frame idx's key is
 *   Philox(SeedSequence((seed, *path, idx, 0))).integers(0, 2, n, uint8)
 * and its flips Philox(SeedSequence((seed, *path, idx, 1))).random(n) < e.
 * prefix: the SeedSequence entropy words of (seed, *path) -- each integer
 * as its little-endian uint32 words, 0 as one zero word (numpy's
 * _coerce_to_uint32_array) -- at most 21 words.  _device: rows in device
 * memory, enqueued on `stream`.  Host variant: the same code on `threads`
 * host threads (no GPU needed).                                             */
int mbp_frames_generate_device(int32_t n, const uint32_t *prefix, int32_t prefix_len, int64_t first,
                               int64_t batch, double e, uint8_t *keys, uint8_t *noisy, void *stream);
int mbp_frames_generate(int32_t n, const uint32_t *prefix, int32_t prefix_len, int64_t first,
                        int64_t batch, double e, uint8_t *keys, uint8_t *noisy, int32_t threads);

/* ---- pinned host memory for the host-buffer entry points ---------------- */
void *mbp_host_alloc(size_t bytes);
void mbp_host_free(void *p);

/* ---- timing of the last decode (CUDA events on the launching stream) -----
 * decode_kernel_ms: the cooperative decode kernel of the last chunk;
 * e2e_ms: the last host-buffer mbp_decode_batch call from its first H2D copy
 * to its last D2H copy (both on the workspace's own stream); sweeps_run:
 * flooding sweeps the last chunk executed (max over its frames).  Any output
 * pointer may be NULL.                                                      */
int mbp_workspace_last_timing(mbp_workspace *ws, float *decode_kernel_ms, float *e2e_ms,
                              int32_t *sweeps_run);
/* sweeps the last chunk executed and the sweep at whose start undecided
 * frames were compacted into dense groups (0: no compaction).             */
int mbp_workspace_last_stats(mbp_workspace *ws, int32_t *sweeps_run, int32_t *compaction_sweep);

#ifdef __cplusplus
}
#endif
#endif /* MBP_H */
