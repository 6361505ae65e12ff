/*
 * tsgpu.h -- C ABI of libtsgpu.so, the B200 device layer of the tuner.
 *
 * The reference (tunescape, pure Python) has NO device layer: its only
 * executors are the replay backend and the subprocess backend
 * (pkg/src/tunescape/measure.py:170-186, :218-305) dispatched from
 * measure() (:308-324).  This library is the in-process executor that
 * slots in at that seam: one call compiles a configuration (what the
 * command backend's external program did with its compiler), one loads
 * it, one runs warmup+benchmark launches with per-run CUDA-event timing
 * (the program's TUNE_TIME_MS lines, measure.py:189-203), and one
 * verifies the output on the device.  Failures are returned as codes
 * that map 1:1 onto the reference's Status enum (measure.py:38-43):
 *
 *   TSG_OK                 -> Status.OK
 *   TSG_ERR_COMPILE        -> Status.COMPILE_FAILED   (NVRTC error)
 *   TSG_ERR_INVALID        -> Status.INVALID          (launch rejected:
 *                             too many threads/registers/smem)
 *   TSG_ERR_RUNTIME        -> Status.RUNTIME_FAILED   (fault during run;
 *                             the context is poisoned, respawn worker)
 *   TSG_ERR_TIMEOUT        -> Status.TIMEOUT          (watchdog)
 *   TSG_ERR_SETUP / TSG_ERR_ARG -> raised as DeviceError/ProtocolError
 *                             in Python (never a Status).
 *
 * Ownership: the library owns device memory, modules and contexts
 * behind opaque handles; the caller owns host buffers.  Only opaque
 * handles and raw device addresses (uint64) cross the boundary.  All
 * functions return an int status; tsg_last_error() gives the message
 * of the last failure on the calling thread.
 *
 * Threading: tsg_compile is context-free and thread-safe (run it from a
 * host compile pool); everything else takes a context and must not be
 * called concurrently on the same context ("measurement on a single
 * backend is strictly sequential").
 */
#ifndef TSGPU_H
#define TSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TSG_OK = 0,
  TSG_ERR_COMPILE = 1,
  TSG_ERR_INVALID = 2,
  TSG_ERR_RUNTIME = 3,
  TSG_ERR_TIMEOUT = 4,
  TSG_ERR_SETUP = 5,
  TSG_ERR_ARG = 6
};

typedef struct tsg_ctx tsg_ctx;
typedef struct tsg_module tsg_module;
typedef struct tsg_kernel tsg_kernel;

/* One kernel launch of a (possibly multi-launch) timed run.  `args` is
 * the cuLaunchKernel kernelParams array: one pointer per kernel
 * parameter, pointing at the parameter's value.  cluster[] = {0,0,0} or
 * {1,1,1} means no cluster launch.  flags: TSG_LAUNCH_PDL launches with
 * programmatic stream serialization (the kernel may be scheduled while the
 * previous kernel in the stream drains; it must execute
 * griddepcontrol.wait before touching that kernel's results; round 2 --
 * the field moved `args` from offset 48 to 56). */
#define TSG_LAUNCH_PDL 1u
typedef struct {
  tsg_kernel* fn;
  unsigned grid[3];
  unsigned block[3];
  unsigned cluster[3];
  unsigned smem_bytes;
  unsigned flags;
  void** args;
} tsg_launch_t;

/* Device properties reported by tsg_device_info. */
typedef struct {
  char name[256];
  int cc_major, cc_minor;
  int sm_count;
  int max_threads_per_block;
  int max_smem_per_block_optin;
  int max_smem_per_sm;
  int l2_bytes;
  int regs_per_sm;
  int clock_khz;
  int mem_clock_khz;
  int mem_bus_bits;
  size_t total_mem;
} tsg_device_info_t;

/* Version / diagnostics ------------------------------------------------ */
const char* tsg_last_error(void);
const char* tsg_error_string(int code);
int tsg_nvrtc_version(int* major, int* minor);
int tsg_driver_version(int* version);

/* Context (replaces: nothing -- the reference has no device; ref seam is
 * BackendDescriptor, measure.py:114-144) ---------------------------------- */
int tsg_init(int device, tsg_ctx** ctx);
int tsg_destroy(tsg_ctx* ctx);
int tsg_device_info(tsg_ctx* ctx, tsg_device_info_t* info);
/* Kernels launched through this context since tsg_init (evidence that
 * the native path ran). */
uint64_t tsg_launch_count(tsg_ctx* ctx);

/* Compilation: CUDA C++ source -> sm_100a cubin via NVRTC.  Context
 * free, thread safe.  `name_expr` may be NULL (extern "C" kernels) or a
 * template instantiation expression whose lowered (mangled) name is
 * written to `lowered` (size lowered_len).  The cubin is malloc'd and
 * must be released with tsg_free_host.  Replaces the compile step that
 * the reference delegates to the benchmark program behind
 * `command_template` (measure.py:233-245). */
int tsg_compile(const char* source, const char* program_name, const char* name_expr,
                const char* const* options, int n_options, void** image,
                size_t* image_bytes, char* lowered, size_t lowered_len, char* log,
                size_t log_len);
void tsg_free_host(void* p);

/* Modules ---------------------------------------------------------------- */
int tsg_module_load(tsg_ctx* ctx, const void* image, size_t image_bytes, tsg_module** mod);
int tsg_module_unload(tsg_module* mod);
int tsg_get_function(tsg_module* mod, const char* name, tsg_kernel** fn);
/* Kernel Tuner `cmem_args`: copy host bytes into a __constant__ symbol. */
int tsg_set_constant(tsg_module* mod, const char* symbol, const void* host, size_t bytes);
int tsg_func_attrs(tsg_kernel* fn, int* num_regs, int* static_smem, int* max_threads,
                   int* local_bytes);
/* Opt in to >48 KiB dynamic shared memory (hotspot needs up to 64 KiB,
 * ts/spaces/hotspot.spec:25). */
int tsg_set_max_dynamic_smem(tsg_kernel* fn, int bytes);
/* Preferred shared-memory carveout of the unified L1/smem (percent of the
 * maximum, 0..100): kernels that stage tiles in smem ask for 100 so the
 * occupancy is not capped by a small default carveout. */
int tsg_set_smem_carveout(tsg_kernel* fn, int percent);
/* Resident blocks per SM for a launch shape (cuOccupancyMaxActive-
 * BlocksPerMultiprocessor): lets a host size its grid in whole waves
 * (the hotspot stream kernel picks its row-segment count from it). */
int tsg_occupancy(tsg_kernel* fn, int block_threads, int dyn_smem, int* blocks_per_sm);

/* Device memory ------------------------------------------------------------ */
int tsg_alloc(tsg_ctx* ctx, size_t bytes, uint64_t* dptr);
int tsg_free(tsg_ctx* ctx, uint64_t dptr);
int tsg_h2d(tsg_ctx* ctx, uint64_t dst, const void* src, size_t bytes);
int tsg_d2h(tsg_ctx* ctx, void* dst, uint64_t src, size_t bytes);
int tsg_d2d(tsg_ctx* ctx, uint64_t dst, uint64_t src, size_t bytes);
int tsg_memset32(tsg_ctx* ctx, uint64_t dst, uint32_t value, size_t count);
int tsg_host_register(void* p, size_t bytes);
int tsg_host_unregister(void* p);

/* Execution ---------------------------------------------------------------- */
/* Run the launch sequence once, untimed, and synchronise (run_kernel). */
int tsg_run(tsg_ctx* ctx, const tsg_launch_t* seq, int n_launch, double timeout_ms);
/* The measurement protocol (measure.py:59-79): `warmup` unrecorded runs,
 * then `runs` recorded runs, each run = the whole launch sequence
 * bracketed by CUDA events on the context's stream.  With flush_l2 != 0
 * a >L2-sized buffer is overwritten before every run, outside the
 * events.  times_ms[runs] receives per-run device times. */
int tsg_run_timed(tsg_ctx* ctx, const tsg_launch_t* seq, int n_launch, int warmup, int runs,
                  int flush_l2, double timeout_ms, float* times_ms);
/* Per-launch device times of the LAST timed run (n_launch floats), for
 * roofline accounting of the dominant kernel. */
int tsg_last_launch_times(tsg_ctx* ctx, float* times_ms, int n_launch);

/* Pipelined protocol (new; same measurement as tsg_run_timed).  Submit
 * enqueues, into slot 0..TSG_SLOTS-1, the output poison (NaN fill of
 * `poison_out`, n_out floats; 0 = none), the warm-up + timed runs and,
 * when `ref` != 0, the on-device comparison of poison_out against ref --
 * and returns without waiting.  Collect waits (watchdog `timeout_ms`) and
 * returns the per-run times, the last run's per-launch times (n_launch
 * floats, may be NULL) and the comparison.  A slot must be collected
 * before it is submitted again; tsg_slot_reset drops a failed submission.
 * Several slots let the host prepare configuration i+1 while the device
 * runs configurations i, i-1, ... (replaces the per-configuration synchronisations of
 * tsg_memset32 + tsg_run_timed + tsg_compare_f32). */
#define TSG_SLOTS 16
/* The L2 flush before every run: write `write_bytes` of one buffer (0 =
 * the default, 1.25 x L2), then optionally read `read_bytes` of another so
 * that the timed run starts with only CLEAN lines in L2 (default 0: no
 * read phase). */
int tsg_set_flush_bytes(tsg_ctx* ctx, size_t write_bytes, size_t read_bytes);
int tsg_submit_timed(tsg_ctx* ctx, int slot, const tsg_launch_t* seq, int n_launch, int warmup, int runs,
                     int flush_l2, uint64_t poison_out, size_t n_out, uint64_t ref, double rtol,
                     double atol);
int tsg_collect(tsg_ctx* ctx, int slot, double timeout_ms, float* times_ms, float* launch_ms, int n_launch,
                double* max_abs_err, double* max_abs_ref, uint64_t* n_bad, uint64_t* n_nonfinite);
int tsg_slot_reset(tsg_ctx* ctx, int slot);
/* Device timeline of a collected slot (until its next submission): start
 * and end of the whole submission in ms since the context's first
 * submission, and the warm-up run's duration (sweep-efficiency analysis). */
int tsg_slot_timeline(tsg_ctx* ctx, int slot, double* start_ms, double* end_ms, float* warmup_ms);

/* TMA: encode a 2-D fp32 tensor map (CUtensorMap, 128 bytes written to
 * `desc128`) for `cp.async.bulk.tensor` in kernels that take it as a
 * __grid_constant__ parameter.  dim0 is contiguous; stride1_bytes is the
 * byte pitch of dim1; box0 x box1 elements per copy; swizzle_bytes in
 * {0, 32, 64, 128}. */
int tsg_tma_encode_2d_f32(tsg_ctx* ctx, void* desc128, uint64_t gaddr, uint64_t dim0, uint64_t dim1,
                          uint64_t stride1_bytes, uint32_t box0, uint32_t box1, int swizzle_bytes);

/* Stream markers for timing a whole region (e.g. one benchmark step of
 * many configurations) on the context's stream: record event `slot`
 * (0..15), then read the device time between two recorded slots (waits
 * for the later one). */
int tsg_event_record(tsg_ctx* ctx, int slot);
int tsg_event_elapsed(tsg_ctx* ctx, int slot_begin, int slot_end, float* ms);

/* Stream ordering against work enqueued OUTSIDE this library (new; the
 * reference has no device layer).  The context launches on its own
 * non-blocking stream, so it is unordered with any other stream -- e.g.
 * the one torch.distributed's NCCL receive completes on.  A caller that
 * hands buffers between the two MUST order them explicitly:
 *   tsg_stream_wait(ctx, s):   later work on the context stream waits for
 *                              everything enqueued on `s` so far;
 *   tsg_stream_signal(ctx, s): later work on `s` waits for everything
 *                              enqueued on the context stream so far.
 * `s` is a CUstream / cudaStream_t handle value (0 = the legacy default
 * stream).  tsg_stream_handle returns the context stream's own handle.
 * tsg_launch_async enqueues a launch sequence without waiting (tsg_run
 * waits); tsg_copy_async is a device-to-device copy on the context
 * stream; tsg_sync waits for the context stream (watchdog timeout_ms). */
int tsg_stream_handle(tsg_ctx* ctx, uint64_t* stream);
int tsg_stream_wait(tsg_ctx* ctx, uint64_t stream);
int tsg_stream_signal(tsg_ctx* ctx, uint64_t stream);
int tsg_launch_async(tsg_ctx* ctx, const tsg_launch_t* seq, int n_launch);
int tsg_copy_async(tsg_ctx* ctx, uint64_t dst, uint64_t src, size_t bytes);
int tsg_sync(tsg_ctx* ctx, double timeout_ms);

/* On-device verification (Kernel Tuner `answer`/`atol`): compares
 * float32 arrays `out` and `ref` of n elements.  Reports max |out-ref|,
 * max |ref|, number of elements with |out-ref| > atol + rtol*|ref| and
 * number of non-finite outputs. */
int tsg_compare_f32(tsg_ctx* ctx, uint64_t out, uint64_t ref, size_t n, double rtol, double atol,
                    double* max_abs_err, double* max_abs_ref, uint64_t* n_bad,
                    uint64_t* n_nonfinite);

#ifdef __cplusplus
}
#endif
#endif /* TSGPU_H */
