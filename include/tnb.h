/*
 * tnb.h -- C ABI of the B200-native contraction hot path (libtnb.so).
 *
 * Drop-in boundary for the reference's hot path, /root/reference/pkg/src/tntz:
 *   entries   core.py:394-460   (t[idx] via indexing.py:120-130)
 *   full      core.py:337-359   (TnTensor.full, core.py:176-177)
 *   chain_dot core.py:362-384   (arithmetic.dot, arithmetic.py:189-193)
 *   norm      core.py:387-391   (TnTensor.norm, core.py:179-180)
 *   per-node preparation: promote_cp_node core.py:266-296,
 *                         node_tt_core core.py:307-327, apply_factor 330-334
 *
 * The reference is a pure-Python API with no FFI; these entry points are what
 * its ctypes binding would call.  Conventions:
 *   - every pointer to tensor data is a DEVICE pointer (fp32 values, int64
 *     indices), row-major / C order;
 *   - the caller owns every buffer; workspace sizes are queried first;
 *   - every launch is asynchronous on the given stream (a cudaStream_t, passed
 *     as void*; NULL = legacy default stream);
 *   - status codes only, no exceptions cross the ABI; tnb_last_error() gives a
 *     thread-local message for the last non-zero status;
 *   - no global mutable state (except the opt-in kernel timing below): calls
 *     on distinct streams/threads are safe.  The bucketed entries path forks
 *     one thread-local side stream per device (created on first use) to build
 *     its tables concurrently with the index pass, and joins it back into the
 *     caller's stream before the per-entry kernel (TNB_TABLE_STREAM=0: no
 *     fork).  The side stream has the device's highest stream priority
 *     (TNB_TABLE_PRIO=0: default priority).
 */
#ifndef TNB_H_
#define TNB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define TNB_OK 0
#define TNB_EINVAL 1      /* shape / rank / argument contract violated        */
#define TNB_EINDEX 2      /* reserved: index errors are reported via err_mode */
#define TNB_ECUDA 3       /* CUDA launch or runtime error                      */
#define TNB_EWORKSPACE 4  /* workspace smaller than the queried size          */

/* node kinds (core.py:29-30) */
#define TNB_KIND_TT 0
#define TNB_KIND_CP 1

/* repacked slice layouts */
#define TNB_LAYOUT_DENSE 0 /* [B?][J][r_left][r_right] contiguous r_l x r_r tiles */
#define TNB_LAYOUT_DIAG 1  /* [B?][J][R]: interior CP node, diagonal copy-tensor */

/* CP positions (core.py:32-34) */
#define TNB_POS_INTERIOR 0
#define TNB_POS_LEFT 1
#define TNB_POS_RIGHT 2
#define TNB_POS_SINGLE 3 /* one-mode chain: the copy tensor reduces to a sum */

/* entries algorithm selector (0 = automatic) */
#define TNB_ALGO_AUTO 0
#define TNB_ALGO_LAYERED 1  /* one launch per mode over a global state buffer */
#define TNB_ALGO_CHAIN 2    /* one thread per sample, cores via L1/L2          */
#define TNB_ALGO_BUCKETED 3 /* per-CTA counting sort, warp-shared core slices  */
#define TNB_ALGO_GSORT 4    /* one global sort by a merged interior mode, tcgen05 */

/*
 * One node exactly as the reference stores it (ModeNode, core.py:41-99).
 * TT core: [B?][r_left][internal][r_right]; CP core: [B?][internal][rank].
 * factor (Tucker basis, J x I): [B?][phys][internal] or NULL.
 */
typedef struct {
  int32_t kind;     /* TNB_KIND_TT / TNB_KIND_CP                        */
  int32_t internal; /* I = core.shape[-2]                                */
  int32_t phys;     /* J = factor.shape[-2] if factor else I             */
  int32_t r_left;   /* TT: core.shape[-3]; CP: rank R                    */
  int32_t r_right;  /* TT: core.shape[-1]; CP: rank R                    */
  int32_t pad_;
  const float* core;
  const float* factor;
} tnb_node;

/* One repacked mode operator, as the kernels consume it. */
typedef struct {
  int32_t layout;  /* TNB_LAYOUT_DENSE / TNB_LAYOUT_DIAG            */
  int32_t phys;    /* J                                             */
  int32_t r_left;  /* effective chain ranks (CP: 1 outward at ends) */
  int32_t r_right;
  float* slices;   /* see TNB_LAYOUT_*                              */
} tnb_mode;

typedef struct {
  int32_t n_modes;
  int32_t pad_;
  int64_t batch; /* 0 = unbatched, else B: every mode has a leading B axis */
  const tnb_mode* modes; /* HOST array of n_modes descriptors */
} tnb_chain;

/* --- library ------------------------------------------------------------ */
const char* tnb_version(void);
const char* tnb_last_error(void);
/* Returns TNB_OK when a device of compute capability 10.x is current. */
int tnb_device_check(void);

/* --- K0: per-node preparation ------------------------------------------- */
/*
 * Validates the rank chain (core.py:244-263, boundary ranks 1 core.py:131-133)
 * and fills layout/phys/r_left/r_right of modes[0..n) (slices untouched).
 * Replaces the implicit per-call node_tt_core of core.py:307-327.
 */
int tnb_plan_modes(const tnb_node* nodes, int32_t n_modes, tnb_mode* modes);
/* Number of floats mode k's repacked slices occupy (per the plan). */
int64_t tnb_mode_floats(const tnb_mode* mode, int64_t batch);
/*
 * Fills modes[k].slices: promotes CP nodes (core.py:266-296) and absorbs
 * Tucker factors (apply_factor, core.py:330-334) once per tensor.
 */
int tnb_repack_f32(const tnb_node* nodes, int32_t n_modes, int64_t batch,
                   const tnb_mode* modes, void* stream);
/*
 * Dense TT core of mode k in the reference layout [B?][r_l][J][r_r]
 * (node_tt_core with absorb_factor=True, core.py:307-327).
 */
int tnb_tt_core_f32(const tnb_chain* chain, int32_t k, float* out, void* stream);
/*
 * promote_cp_node (core.py:266-296) of one CP node, factor NOT applied:
 * out is [B?][1|R][I][R|1] (TNB_POS_LEFT/INTERIOR/RIGHT) or [B?][1][I][1]
 * (TNB_POS_SINGLE, the sum of core.py:316-320).
 */
int tnb_promote_cp_f32(const tnb_node* node, int32_t position, int64_t batch,
                       float* out, void* stream);

/* --- K1: entry evaluation  (core.py:394-460) ----------------------------- */
/*
 * idx: int64 [m][n_modes] row-major, raw user indices (negatives allowed);
 * out: fp32 [m] (unbatched) or [m][batch].
 * TNB_ALGO_AUTO picks, for fp32: the fused two-table kernel when mode
 * merging reduces the chain to a prefix and a suffix table (any rank), else
 * the global-sort tcgen05 path (TNB_ALGO_GSORT) for unbatched chains with
 * m >= 2^18 whose merged chain is first . dense . [diag] . last with ranks
 * <= 32 that are multiples of 4, else
 * the bucketed kernels for m >= 2^16 and ranks <= 32 -- batched chains too,
 * one element at a time over shared tile records (_step_entries_batched,
 * core.py:447-460) -- else the register chain (rank <= 32) or the layered
 * algorithm.
 * err_mode: device int32; on completion it holds the LOWEST mode that had an
 * index outside [-J, J) (the ContractViolationError "index out of bounds on
 * mode k" of core.py:409-416), or a value >= n_modes when all were valid.
 * When it reports an error the contents of out are unspecified.
 */
int64_t tnb_entries_workspace_bytes(const tnb_chain* chain, int64_t m, int32_t algo);
int tnb_entries_f32(const tnb_chain* chain, const int64_t* idx, int64_t m,
                    float* out, int32_t* err_mode, int32_t algo,
                    void* workspace, int64_t workspace_bytes, void* stream);

/*
 * Index transport codec for HOST index matrices (the end-to-end path of
 * entries: t[idx] with idx in host memory, core.py:394-416).  PCIe is the
 * bound there (80 B per cfg2 sample), and every value of a typical index
 * matrix fits in one byte.
 *
 * tnb_narrow_indices_host: HOST function.  Narrows count int64 values to
 * int8 (width 1) or int16 (width 2) in out, using nthreads host threads
 * (<= 0: all hardware threads).  *fits = 1 when every value lay in the
 * narrow type's range, else 0 (out unspecified; send the int64 matrix).  A
 * pure range check on the raw values: negative wrapping, the per-mode
 * bounds check and the lowest-OOB-mode report stay in tnb_entries_f32, which
 * sees exactly the caller's values after tnb_widen_indices.
 * tnb_widen_indices: device, asynchronous on stream: out[i] = (int64) in[i];
 * both buffers 16-byte aligned.
 * tnb_host_threads: the hardware thread count the codec uses by default.
 */
int tnb_narrow_indices_host(const int64_t* idx, int64_t count, int32_t width, void* out,
                            int32_t nthreads, int32_t* fits);
int tnb_widen_indices(const void* in, int32_t width, int64_t count, int64_t* out, void* stream);
int tnb_host_threads(void);

/* --- K2: dense decompression  (core.py:337-359) -------------------------- */
/*
 * Writes the C-order slab of full(t) whose leading (mode-0) index lies in
 * [lead_lo, lead_hi): (lead_hi-lead_lo) * prod(J_1..J_{N-1}) floats, per batch
 * element (batched: out is [B][slab]).  [0, J_0) is the whole tensor; a slab
 * equals the reference's full(t[lo:hi]) (indexing.py:132-137).
 */
int64_t tnb_full_workspace_bytes(const tnb_chain* chain, int64_t lead_lo, int64_t lead_hi);
int tnb_full_f32(const tnb_chain* chain, int64_t lead_lo, int64_t lead_hi, float* out,
                 void* workspace, int64_t workspace_bytes, void* stream);

/* --- K3: inner products  (core.py:362-391) ------------------------------- */
/*
 * out[e] = <a_e, b_e> for every batch element (one float when unbatched).
 * Kernels: rank-16 TT chains (fp32) on the mma.sync split-TF32 kernel;
 * other dense chains (any rank, fp32 and fp64) on the chunked kernel (slices
 * staged in shared memory, 16-byte loads); chains with interior CP modes on
 * the per-slice kernel.
 * Shapes and batching must agree (ContractViolationError in core.py:368-371).
 */
int tnb_dot_f32(const tnb_chain* a, const tnb_chain* b, float* out, void* stream);
/* out[e] = sqrt(max(<t_e, t_e>, 0))  (core.py:387-391) */
int tnb_norm_f32(const tnb_chain* t, float* out, void* stream);

/* --- float64 instantiation -------------------------- */
/*
 * The reference computes in float64 (core.py:37-38, 54).  These entry points
 * run the same contracts in double on the generic kernels (register chain /
 * layered entries, step kernels + SIMT GEMM for full, per-pair transfer
 * matrices for dot/norm; no tensor cores, no bucketing), so results can be
 * checked against the reference at its own tolerances.  Every pointer in the
 * node / mode structs and every data argument then points to DOUBLE data
 * (element counts from tnb_mode_floats are the same).
 */
int tnb_repack_f64(const tnb_node* nodes, int32_t n_modes, int64_t batch,
                   const tnb_mode* modes, void* stream);
int tnb_tt_core_f64(const tnb_chain* chain, int32_t k, double* out, void* stream);
int tnb_promote_cp_f64(const tnb_node* node, int32_t position, int64_t batch,
                       double* out, void* stream);
int64_t tnb_entries_workspace_bytes_f64(const tnb_chain* chain, int64_t m, int32_t algo);
int tnb_entries_f64(const tnb_chain* chain, const int64_t* idx, int64_t m,
                    double* out, int32_t* err_mode, int32_t algo,
                    void* workspace, int64_t workspace_bytes, void* stream);
int64_t tnb_full_workspace_bytes_f64(const tnb_chain* chain, int64_t lead_lo, int64_t lead_hi);
int tnb_full_f64(const tnb_chain* chain, int64_t lead_lo, int64_t lead_hi, double* out,
                 void* workspace, int64_t workspace_bytes, void* stream);
int tnb_dot_f64(const tnb_chain* a, const tnb_chain* b, double* out, void* stream);
int tnb_norm_f64(const tnb_chain* t, double* out, void* stream);

/* --- plan introspection and kernel timing (bench / profiling) ------------ */
/*
 * What tnb_entries_f32(chain, ., m, ., ., algo, ...) will run: the resolved
 * algorithm, the mode merging of the bucketed path (leading / trailing modes
 * contracted into prefix / suffix tables and runs of interior CP modes into
 * diagonal product tables, once per call, so the per-entry kernel runs a
 * shorter "virtual" chain) and the algorithmic flops of the per-entry kernel
 * and of the table build.  No device work.
 */
typedef struct {
  int32_t algo;          /* TNB_ALGO_LAYERED / CHAIN / BUCKETED               */
  int32_t n_virtual;     /* modes of the chain the per-entry kernel runs       */
  int32_t prefix_modes;  /* original modes in the prefix table (1 = no table)  */
  int32_t suffix_modes;  /* original modes in the suffix table (1 = no table)  */
  int64_t prefix_rows;   /* rows of the prefix table (0 = none)                */
  int64_t suffix_rows;   /* rows of the suffix table (0 = none)                */
  double kernel_flops;   /* per call: 2*r_l*r_r per dense step, R per diagonal */
  double table_flops;    /* per call: building the tables                      */
  int32_t diag_tables;   /* runs of interior CP modes merged into product tables */
  int32_t table_launches;/* kernel launches that build the tables per call     */
  int32_t compute_kernel;/* bucketed: 0 = state kernel, 1 = stream kernel (one
                            sorted mode; no per-sample state in shared memory),
                            2 = two-table kernel (the chain merges into a prefix
                            and a suffix table: one fused gather-dot, any rank) */
  int32_t tile;          /* bucketed: samples per tile                          */
  double tensor_flops;   /* per call: tensor-core (split-TF32 mma.sync) flops
                            the compute kernel issues, 3 MMAs per product      */
} tnb_entries_info;
int tnb_entries_plan(const tnb_chain* chain, int64_t m, int32_t algo, tnb_entries_info* info);

/*
 * Opt-in CUDA-event timing of libtnb's own kernels on their launching
 * streams (the only process-global state; off by default).  Names:
 * "entries_prep", "entries_sort", "entries_compute", "entries_tables",
 * "full_gemm", "dot".
 * enable(0/1) resets every accumulator; read() waits for the recorded events.
 */
int tnb_timing_enable(int32_t on);
int tnb_timing_read(const char* kernel, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* TNB_H_ */
