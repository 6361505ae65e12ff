// libtsgpu.so -- the B200 device layer behind include/tsgpu.h.
//
// Driver API for modules/launches/events (so every configuration is an
// independently loadable cubin), NVRTC for sm_100a compilation, and two
// small runtime-API kernels of our own (device-side verification and
// the L2 flush) that run on the same primary context.
#include "../../include/tsgpu.h"

#include <cuda_runtime.h>
#include <nvrtc.h>

#include "driver_table.h"

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

std::string cu_msg(CUresult r) {
  const char* name = nullptr;
  const char* str = nullptr;
  if (tsg_drv().loaded) {
    cuGetErrorName(r, &name);
    cuGetErrorString(r, &str);
  }
  return std::string(name ? name : "CUDA_ERROR_?") + ": " + (str ? str : "");
}

// Launch-time errors that mean "this configuration cannot run here"
// (Status.INVALID) as opposed to a device fault (Status.RUNTIME_FAILED).
bool is_config_error(CUresult r) {
  switch (r) {
    case CUDA_ERROR_INVALID_VALUE:
    case CUDA_ERROR_OUT_OF_MEMORY:
    case CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES:
    case CUDA_ERROR_INVALID_IMAGE:
    case CUDA_ERROR_NO_BINARY_FOR_GPU:
    case CUDA_ERROR_INVALID_CLUSTER_SIZE:
    case CUDA_ERROR_INVALID_HANDLE:
    case CUDA_ERROR_SHARED_OBJECT_INIT_FAILED:
      return true;
    default:
      return false;
  }
}

}  // namespace

struct tsg_ctx {
  int device = 0;
  CUdevice dev = 0;
  CUcontext cu = nullptr;
  CUstream stream = nullptr;
  std::vector<CUevent> events;  // 2 per recorded run + per-launch pairs
  CUdeviceptr flush_buf = 0;
  size_t flush_bytes = 0;
  CUdeviceptr flush_rbuf = 0;  // optional read phase (clean lines); 0 bytes = write-only flush
  size_t flush_rbytes = 0;
  CUdeviceptr scratch = 0;  // compare accumulators
  std::atomic<uint64_t> launches{0};
  bool poisoned = false;
  std::vector<float> last_launch_ms;
  CUevent marks[16] = {};
  bool lmem_to_max = false;  // CU_CTX_LMEM_RESIZE_TO_MAX applied
  CUevent epoch = nullptr;   // device-timeline origin of the submission slots
  // pipelined submission slots (tsg_submit_timed / tsg_collect)
  struct Slot {
    std::vector<CUevent> ev;  // [2*total run brackets][n+1 launch marks][done]
    CUdeviceptr scratch = 0;  // compare accumulators
    unsigned long long* host = nullptr;  // pinned copy of the accumulators
    int warmup = 0, runs = 0, n = 0;
    bool verify = false, active = false;
  } slots[TSG_SLOTS];
  tsg_device_info_t info{};
};

struct tsg_module {
  tsg_ctx* ctx;
  CUmodule mod;
};

struct tsg_kernel {
  tsg_module* mod;
  CUfunction fn;
};

namespace {

int make_current(tsg_ctx* c) {
  if (!c) return fail(TSG_ERR_ARG, "null context");
  if (c->poisoned)
    return fail(TSG_ERR_RUNTIME, "context poisoned by an earlier device fault; restart the worker");
  CUresult r = cuCtxSetCurrent(c->cu);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuCtxSetCurrent: " + cu_msg(r));
  return TSG_OK;
}

int ensure_events(tsg_ctx* c, size_t n) {
  while (c->events.size() < n) {
    CUevent e;
    CUresult r = cuEventCreate(&e, CU_EVENT_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuEventCreate: " + cu_msg(r));
    c->events.push_back(e);
  }
  return TSG_OK;
}

// Wait for the stream with a host-side watchdog.
int wait_stream(tsg_ctx* c, CUevent last, double timeout_ms) {
  auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  for (;;) {
    CUresult r = cuEventQuery(last);
    if (r == CUDA_SUCCESS) return TSG_OK;
    if (r != CUDA_ERROR_NOT_READY) {
      c->poisoned = true;
      return fail(TSG_ERR_RUNTIME, "device fault: " + cu_msg(r));
    }
    double el = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && el > timeout_ms) {
      c->poisoned = true;
      char buf[96];
      snprintf(buf, sizeof buf, "exceeded %g ms", timeout_ms);
      return fail(TSG_ERR_TIMEOUT, buf);
    }
    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

int launch_one(tsg_ctx* c, const tsg_launch_t& L) {
  if (!L.fn) return fail(TSG_ERR_ARG, "launch with null kernel");
  CUresult r;
  bool cluster = L.cluster[0] * L.cluster[1] * L.cluster[2] > 1;
  bool pdl = (L.flags & TSG_LAUNCH_PDL) != 0;
  if (!cluster && !pdl) {
    r = cuLaunchKernel(L.fn->fn, L.grid[0], L.grid[1], L.grid[2], L.block[0], L.block[1],
                       L.block[2], L.smem_bytes, c->stream, L.args, nullptr);
  } else {
    CUlaunchConfig cfg{};
    cfg.gridDimX = L.grid[0];
    cfg.gridDimY = L.grid[1];
    cfg.gridDimZ = L.grid[2];
    cfg.blockDimX = L.block[0];
    cfg.blockDimY = L.block[1];
    cfg.blockDimZ = L.block[2];
    cfg.sharedMemBytes = L.smem_bytes;
    cfg.hStream = c->stream;
    CUlaunchAttribute attr[2] = {};
    unsigned na = 0;
    if (cluster) {
      attr[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
      attr[na].value.clusterDim.x = L.cluster[0];
      attr[na].value.clusterDim.y = L.cluster[1];
      attr[na].value.clusterDim.z = L.cluster[2];
      ++na;
    }
    if (pdl) {  // programmatic dependent launch (sm_90+): overlap this launch's
                // scheduling with the previous kernel's drain
      attr[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      attr[na].value.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    r = cuLaunchKernelEx(&cfg, L.fn->fn, L.args, nullptr);
  }
  if (r != CUDA_SUCCESS) {
    if (is_config_error(r)) return fail(TSG_ERR_INVALID, "launch rejected: " + cu_msg(r));
    c->poisoned = true;
    return fail(TSG_ERR_RUNTIME, "launch failed: " + cu_msg(r));
  }
  c->launches.fetch_add(1, std::memory_order_relaxed);
  return TSG_OK;
}

// ---- utility kernels (runtime API, same primary context) ----------------

__global__ void __launch_bounds__(256) compare_f32_kernel(const float* __restrict__ out,
                                                          const float* __restrict__ ref, size_t n,
                                                          float rtol, float atol,
                                                          unsigned long long* acc) {
  // acc[0] = bits of max |out-ref|, acc[1] = bits of max |ref|,
  // acc[2] = n_bad, acc[3] = n_nonfinite
  float max_err = 0.f, max_ref = 0.f;
  unsigned long long bad = 0, nonfinite = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float o = out[i], r = ref[i];
    if (!isfinite(o)) {
      ++nonfinite;
      ++bad;
      continue;
    }
    float e = fabsf(o - r), a = fabsf(r);
    max_err = fmaxf(max_err, e);
    max_ref = fmaxf(max_ref, a);
    if (e > atol + rtol * a) ++bad;
  }
  for (int off = 16; off > 0; off >>= 1) {
    max_err = fmaxf(max_err, __shfl_xor_sync(0xffffffffu, max_err, off));
    max_ref = fmaxf(max_ref, __shfl_xor_sync(0xffffffffu, max_ref, off));
    bad += __shfl_xor_sync(0xffffffffu, bad, off);
    nonfinite += __shfl_xor_sync(0xffffffffu, nonfinite, off);
  }
  if ((threadIdx.x & 31) == 0) {
    // non-negative floats order like their bit patterns
    atomicMax(&acc[0], (unsigned long long)__float_as_uint(max_err));
    atomicMax(&acc[1], (unsigned long long)__float_as_uint(max_ref));
    if (bad) atomicAdd(&acc[2], bad);
    if (nonfinite) atomicAdd(&acc[3], nonfinite);
  }
}

__global__ void __launch_bounds__(256) flush_kernel(uint4* __restrict__ buf, size_t n16, unsigned salt) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    buf[i] = make_uint4(salt, (unsigned)i, salt ^ 0x9e3779b9u, 0u);
}

// optional second flush phase (tsg_set_flush_bytes, off by default): READ a
// different >= L2-sized buffer, so the dirty lines the write phase left in
// L2 are written back outside the timed events.  Measured on B200
// (tools/flush_probe.py, 96 MiB read): 28.7 us after a write-only flush of
// 1x or 3x L2 (identical: 1x already evicts everything), 24.6 us after
// write + read, 22.5 us after a read-only flush, 14.9 us unflushed.  The
// default stays write-only, the way Kernel Tuner flushes (an L2-sized
// buffer written before each run), so times compare like for like.
__global__ void __launch_bounds__(256) flush_read_kernel(const uint4* __restrict__ buf, size_t n16,
                                                         unsigned* sink) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned x = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = __ldcg(buf + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x9e3779b9u) sink[blockIdx.x & 15] = x;  // practically never; keeps the loads
}

int flush_l2(tsg_ctx* c) {
  if (!c->flush_buf) {
    // 1.25 x L2 written: as effective as 3 x (measured, tools/flush_probe.py)
    // at 40% of the cost
    if (!c->flush_bytes)
      c->flush_bytes = ((size_t)5 * (c->info.l2_bytes > 0 ? c->info.l2_bytes : (128 << 20)) / 4 + 15) & ~(size_t)15;
    CUresult r = cuMemAlloc(&c->flush_buf, c->flush_bytes < 16 ? 16 : c->flush_bytes);
    if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "flush buffer: " + cu_msg(r));
  }
  if (c->flush_rbytes && !c->flush_rbuf) {
    CUresult r = cuMemAlloc(&c->flush_rbuf, c->flush_rbytes);
    if (r == CUDA_SUCCESS) r = cuMemsetD32Async(c->flush_rbuf, 0, c->flush_rbytes / 4, c->stream);
    if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "flush read buffer: " + cu_msg(r));
  }
  static unsigned salt = 1;
  if (c->flush_bytes) {
    c->launches.fetch_add(1, std::memory_order_relaxed);
    flush_kernel<<<c->info.sm_count * 4, 256, 0, (cudaStream_t)c->stream>>>(
        (uint4*)c->flush_buf, c->flush_bytes / 16, salt++);
  }
  if (c->flush_rbytes) {
    c->launches.fetch_add(1, std::memory_order_relaxed);
    flush_read_kernel<<<c->info.sm_count * 4, 256, 0, (cudaStream_t)c->stream>>>(
        (const uint4*)c->flush_rbuf, c->flush_rbytes / 16, (unsigned*)c->scratch + 8);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TSG_ERR_RUNTIME, std::string("flush: ") + cudaGetErrorString(e));
  return TSG_OK;
}

}  // namespace

extern "C" {

const char* tsg_last_error(void) { return g_err.c_str(); }

const char* tsg_error_string(int code) {
  switch (code) {
    case TSG_OK: return "ok";
    case TSG_ERR_COMPILE: return "compile_failed";
    case TSG_ERR_INVALID: return "invalid";
    case TSG_ERR_RUNTIME: return "runtime_failed";
    case TSG_ERR_TIMEOUT: return "timeout";
    case TSG_ERR_SETUP: return "setup_error";
    case TSG_ERR_ARG: return "bad_argument";
    default: return "unknown";
  }
}

int tsg_nvrtc_version(int* major, int* minor) {
  if (nvrtcVersion(major, minor) != NVRTC_SUCCESS) return fail(TSG_ERR_SETUP, "nvrtcVersion failed");
  return TSG_OK;
}

int tsg_driver_version(int* version) {
  if (const char* why = tsg_load_driver()) return fail(TSG_ERR_SETUP, why);
  CUresult r = cuDriverGetVersion(version);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuDriverGetVersion: " + cu_msg(r));
  return TSG_OK;
}

int tsg_init(int device, tsg_ctx** out) {
  if (!out) return fail(TSG_ERR_ARG, "null output");
  if (const char* why = tsg_load_driver()) return fail(TSG_ERR_SETUP, why);
  CUresult r = cuInit(0);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuInit: " + cu_msg(r));
  auto* c = new tsg_ctx();
  c->device = device;
  if ((r = cuDeviceGet(&c->dev, device)) != CUDA_SUCCESS) {
    delete c;
    return fail(TSG_ERR_SETUP, "cuDeviceGet: " + cu_msg(r));
  }
  if ((r = cuDevicePrimaryCtxRetain(&c->cu, c->dev)) != CUDA_SUCCESS) {
    delete c;
    return fail(TSG_ERR_SETUP, "cuDevicePrimaryCtxRetain: " + cu_msg(r));
  }
  cuCtxSetCurrent(c->cu);
  // Keep local memory at its high-water mark: by default the driver shrinks
  // it again after a kernel that needed more, so every launch of a spilling
  // configuration re-grows it (device-wide sync + reallocation, measured as
  // 25-60 ms stalls per such configuration in a sweep).  cuCtxSetFlags is a
  // CUDA 12.1 entry point, looked up optionally; TSG_LMEM_RESIZE_TO_MAX=0
  // keeps the driver default (A/B measurements).
  {
    const char* env = getenv("TSG_LMEM_RESIZE_TO_MAX");
    typedef CUresult (*GetFlagsFn)(unsigned*);
    typedef CUresult (*SetFlagsFn)(unsigned);
    auto getf = (GetFlagsFn)dlsym(RTLD_DEFAULT, "cuCtxGetFlags");
    auto setf = (SetFlagsFn)dlsym(RTLD_DEFAULT, "cuCtxSetFlags");
    unsigned flags = 0;
    if (!(env && env[0] == '0') && getf && setf && getf(&flags) == CUDA_SUCCESS)
      c->lmem_to_max = setf(flags | CU_CTX_LMEM_RESIZE_TO_MAX) == CUDA_SUCCESS;
  }
  cudaSetDevice(device);  // runtime API shares the primary context
  if ((r = cuStreamCreate(&c->stream, CU_STREAM_NON_BLOCKING)) != CUDA_SUCCESS) {
    cuDevicePrimaryCtxRelease(c->dev);
    delete c;
    return fail(TSG_ERR_SETUP, "cuStreamCreate: " + cu_msg(r));
  }
  tsg_device_info_t& I = c->info;
  cuDeviceGetName(I.name, sizeof I.name, c->dev);
  auto attr = [&](CUdevice_attribute a) {
    int v = 0;
    cuDeviceGetAttribute(&v, a, c->dev);
    return v;
  };
  I.cc_major = attr(CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR);
  I.cc_minor = attr(CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR);
  I.sm_count = attr(CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT);
  I.max_threads_per_block = attr(CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_BLOCK);
  I.max_smem_per_block_optin = attr(CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN);
  I.max_smem_per_sm = attr(CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR);
  I.l2_bytes = attr(CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE);
  I.regs_per_sm = attr(CU_DEVICE_ATTRIBUTE_MAX_REGISTERS_PER_MULTIPROCESSOR);
  I.clock_khz = attr(CU_DEVICE_ATTRIBUTE_CLOCK_RATE);
  I.mem_clock_khz = attr(CU_DEVICE_ATTRIBUTE_MEMORY_CLOCK_RATE);
  I.mem_bus_bits = attr(CU_DEVICE_ATTRIBUTE_GLOBAL_MEMORY_BUS_WIDTH);
  cuDeviceTotalMem(&I.total_mem, c->dev);
  if ((r = cuMemAlloc(&c->scratch, 64)) != CUDA_SUCCESS) {
    cuDevicePrimaryCtxRelease(c->dev);
    delete c;
    return fail(TSG_ERR_SETUP, "scratch alloc: " + cu_msg(r));
  }
  *out = c;
  return TSG_OK;
}

int tsg_destroy(tsg_ctx* c) {
  if (!c) return TSG_OK;
  cuCtxSetCurrent(c->cu);
  if (!c->poisoned) {
    cuStreamSynchronize(c->stream);
    for (CUevent e : c->events) cuEventDestroy(e);
    if (c->flush_buf) cuMemFree(c->flush_buf);
    if (c->flush_rbuf) cuMemFree(c->flush_rbuf);
    if (c->scratch) cuMemFree(c->scratch);
    if (c->epoch) cuEventDestroy(c->epoch);
    for (auto& sl : c->slots) {
      for (CUevent e : sl.ev) cuEventDestroy(e);
      if (sl.scratch) cuMemFree(sl.scratch);
      if (sl.host) {
        cuMemHostUnregister(sl.host);
        free(sl.host);
      }
    }
    cuStreamDestroy(c->stream);
  }
  cuDevicePrimaryCtxRelease(c->dev);
  delete c;
  return TSG_OK;
}

int tsg_device_info(tsg_ctx* c, tsg_device_info_t* info) {
  if (!c || !info) return fail(TSG_ERR_ARG, "null argument");
  *info = c->info;
  return TSG_OK;
}

uint64_t tsg_launch_count(tsg_ctx* c) { return c ? c->launches.load() : 0; }

int tsg_compile(const char* source, const char* program_name, const char* name_expr,
                const char* const* options, int n_options, void** image, size_t* image_bytes,
                char* lowered, size_t lowered_len, char* log, size_t log_len) {
  if (!source || !image || !image_bytes) return fail(TSG_ERR_ARG, "null argument");
  *image = nullptr;
  *image_bytes = 0;
  if (log && log_len) log[0] = 0;
  nvrtcProgram prog;
  nvrtcResult nr = nvrtcCreateProgram(&prog, source, program_name ? program_name : "kernel.cu", 0,
                                      nullptr, nullptr);
  if (nr != NVRTC_SUCCESS) return fail(TSG_ERR_COMPILE, nvrtcGetErrorString(nr));
  if (name_expr && *name_expr) nvrtcAddNameExpression(prog, name_expr);
  nr = nvrtcCompileProgram(prog, n_options, options);
  size_t loglen = 0;
  nvrtcGetProgramLogSize(prog, &loglen);
  std::string plog(loglen, '\0');
  if (loglen) nvrtcGetProgramLog(prog, &plog[0]);
  if (log && log_len) {
    size_t k = std::min(log_len - 1, strlen(plog.c_str()));
    memcpy(log, plog.c_str(), k);
    log[k] = 0;
  }
  if (nr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(TSG_ERR_COMPILE, std::string(nvrtcGetErrorString(nr)) + "\n" + plog);
  }
  if (name_expr && *name_expr && lowered && lowered_len) {
    const char* low = nullptr;
    if (nvrtcGetLoweredName(prog, name_expr, &low) == NVRTC_SUCCESS && low) {
      strncpy(lowered, low, lowered_len - 1);
      lowered[lowered_len - 1] = 0;
    }
  }
  size_t n = 0;
  nr = nvrtcGetCUBINSize(prog, &n);
  if (nr != NVRTC_SUCCESS || n == 0) {
    nvrtcDestroyProgram(&prog);
    return fail(TSG_ERR_COMPILE, "no cubin produced (compile for a real sm_XXXa architecture)");
  }
  void* buf = malloc(n);
  nvrtcGetCUBIN(prog, (char*)buf);
  nvrtcDestroyProgram(&prog);
  *image = buf;
  *image_bytes = n;
  return TSG_OK;
}

void tsg_free_host(void* p) { free(p); }

int tsg_module_load(tsg_ctx* c, const void* image, size_t image_bytes, tsg_module** out) {
  (void)image_bytes;
  int s = make_current(c);
  if (s) return s;
  CUmodule m;
  CUresult r = cuModuleLoadData(&m, image);
  if (r != CUDA_SUCCESS) {
    if (is_config_error(r)) return fail(TSG_ERR_INVALID, "cuModuleLoadData: " + cu_msg(r));
    return fail(TSG_ERR_RUNTIME, "cuModuleLoadData: " + cu_msg(r));
  }
  *out = new tsg_module{c, m};
  return TSG_OK;
}

int tsg_module_unload(tsg_module* m) {
  if (!m) return TSG_OK;
  if (!m->ctx->poisoned) {
    cuCtxSetCurrent(m->ctx->cu);
    cuModuleUnload(m->mod);
  }
  delete m;
  return TSG_OK;
}

int tsg_get_function(tsg_module* m, const char* name, tsg_kernel** out) {
  if (!m || !name || !out) return fail(TSG_ERR_ARG, "null argument");
  CUfunction f;
  CUresult r = cuModuleGetFunction(&f, m->mod, name);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_ARG, std::string("no kernel '") + name + "': " + cu_msg(r));
  *out = new tsg_kernel{m, f};
  return TSG_OK;
}

int tsg_set_constant(tsg_module* m, const char* symbol, const void* host, size_t bytes) {
  int s = make_current(m ? m->ctx : nullptr);
  if (s) return s;
  CUdeviceptr p;
  size_t sz = 0;
  CUresult r = cuModuleGetGlobal(&p, &sz, m->mod, symbol);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_ARG, std::string("no symbol '") + symbol + "': " + cu_msg(r));
  if (bytes > sz) return fail(TSG_ERR_ARG, "constant data larger than symbol");
  r = cuMemcpyHtoD(p, host, bytes);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "cmem upload: " + cu_msg(r));
  return TSG_OK;
}

int tsg_func_attrs(tsg_kernel* k, int* regs, int* static_smem, int* max_threads, int* local_bytes) {
  if (!k) return fail(TSG_ERR_ARG, "null kernel");
  if (regs) cuFuncGetAttribute(regs, CU_FUNC_ATTRIBUTE_NUM_REGS, k->fn);
  if (static_smem) cuFuncGetAttribute(static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, k->fn);
  if (max_threads) cuFuncGetAttribute(max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, k->fn);
  if (local_bytes) cuFuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, k->fn);
  return TSG_OK;
}

int tsg_set_max_dynamic_smem(tsg_kernel* k, int bytes) {
  if (!k) return fail(TSG_ERR_ARG, "null kernel");
  CUresult r = cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_INVALID, "dynamic smem opt-in: " + cu_msg(r));
  return TSG_OK;
}

int tsg_set_smem_carveout(tsg_kernel* k, int percent) {
  if (!k) return fail(TSG_ERR_ARG, "null kernel");
  CUresult r = cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, percent);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_INVALID, "carveout: " + cu_msg(r));
  return TSG_OK;
}

int tsg_occupancy(tsg_kernel* k, int block_threads, int dyn_smem, int* blocks_per_sm) {
  if (!k || !blocks_per_sm) return fail(TSG_ERR_ARG, "null kernel/output");
  int s = make_current(k->mod ? k->mod->ctx : nullptr);
  if (s) return s;
  CUresult r = cuOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k->fn, block_threads, (size_t)dyn_smem);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_INVALID, "occupancy query: " + cu_msg(r));
  return TSG_OK;
}

int tsg_alloc(tsg_ctx* c, size_t bytes, uint64_t* dptr) {
  int s = make_current(c);
  if (s) return s;
  CUdeviceptr p;
  CUresult r = cuMemAlloc(&p, bytes ? bytes : 16);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuMemAlloc: " + cu_msg(r));
  *dptr = (uint64_t)p;
  return TSG_OK;
}

int tsg_free(tsg_ctx* c, uint64_t dptr) {
  if (!c || c->poisoned) return TSG_OK;
  cuCtxSetCurrent(c->cu);
  cuMemFree((CUdeviceptr)dptr);
  return TSG_OK;
}

int tsg_h2d(tsg_ctx* c, uint64_t dst, const void* src, size_t bytes) {
  int s = make_current(c);
  if (s) return s;
  CUresult r = cuMemcpyHtoDAsync((CUdeviceptr)dst, src, bytes, c->stream);
  if (r == CUDA_SUCCESS) r = cuStreamSynchronize(c->stream);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "H2D: " + cu_msg(r));
  return TSG_OK;
}

int tsg_d2h(tsg_ctx* c, void* dst, uint64_t src, size_t bytes) {
  int s = make_current(c);
  if (s) return s;
  CUresult r = cuMemcpyDtoHAsync(dst, (CUdeviceptr)src, bytes, c->stream);
  if (r == CUDA_SUCCESS) r = cuStreamSynchronize(c->stream);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "D2H: " + cu_msg(r));
  return TSG_OK;
}

int tsg_d2d(tsg_ctx* c, uint64_t dst, uint64_t src, size_t bytes) {
  int s = make_current(c);
  if (s) return s;
  CUresult r = cuMemcpyDtoDAsync((CUdeviceptr)dst, (CUdeviceptr)src, bytes, c->stream);
  if (r == CUDA_SUCCESS) r = cuStreamSynchronize(c->stream);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "D2D: " + cu_msg(r));
  return TSG_OK;
}

int tsg_memset32(tsg_ctx* c, uint64_t dst, uint32_t value, size_t count) {
  int s = make_current(c);
  if (s) return s;
  CUresult r = cuMemsetD32Async((CUdeviceptr)dst, value, count, c->stream);
  if (r == CUDA_SUCCESS) r = cuStreamSynchronize(c->stream);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "memset: " + cu_msg(r));
  return TSG_OK;
}

int tsg_host_register(void* p, size_t bytes) {
  if (const char* why = tsg_load_driver()) return fail(TSG_ERR_SETUP, why);
  CUresult r = cuMemHostRegister(p, bytes, 0);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuMemHostRegister: " + cu_msg(r));
  return TSG_OK;
}

int tsg_host_unregister(void* p) {
  if (tsg_load_driver()) return TSG_OK;
  cuMemHostUnregister(p);
  return TSG_OK;
}

int tsg_run(tsg_ctx* c, const tsg_launch_t* seq, int n, double timeout_ms) {
  int s = make_current(c);
  if (s) return s;
  if ((s = ensure_events(c, 1))) return s;
  for (int i = 0; i < n; ++i)
    if ((s = launch_one(c, seq[i]))) return s;
  cuEventRecord(c->events[0], c->stream);
  return wait_stream(c, c->events[0], timeout_ms);
}

int tsg_run_timed(tsg_ctx* c, const tsg_launch_t* seq, int n, int warmup, int runs, int flush,
                  double timeout_ms, float* times_ms) {
  int s = make_current(c);
  if (s) return s;
  if (runs < 1 || warmup < 0 || n < 1) return fail(TSG_ERR_ARG, "bad protocol");
  const int total = warmup + runs;
  // events: [2*total run brackets] [n+1 per-launch marks of the last run]
  if ((s = ensure_events(c, 2 * (size_t)total + n + 1))) return s;
  CUevent* ev = c->events.data();
  CUevent* lev = ev + 2 * total;
  for (int r = 0; r < total; ++r) {
    if (flush && (s = flush_l2(c))) return s;
    cuEventRecord(ev[2 * r], c->stream);
    const bool last = (r == total - 1);
    for (int i = 0; i < n; ++i) {
      if (last) cuEventRecord(lev[i], c->stream);
      if ((s = launch_one(c, seq[i]))) {
        cuStreamSynchronize(c->stream);
        return s;
      }
    }
    if (last) cuEventRecord(lev[n], c->stream);
    cuEventRecord(ev[2 * r + 1], c->stream);
  }
  if ((s = wait_stream(c, ev[2 * total - 1], timeout_ms))) return s;
  for (int r = warmup; r < total; ++r) {
    float ms = 0.f;
    cuEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]);
    times_ms[r - warmup] = ms;
  }
  c->last_launch_ms.assign(n, 0.f);
  for (int i = 0; i < n; ++i) cuEventElapsedTime(&c->last_launch_ms[i], lev[i], lev[i + 1]);
  return TSG_OK;
}

// ---- pipelined measurement -------------------------------------------------
// tsg_submit_timed enqueues one configuration's whole protocol -- output
// poison, warm-up + timed runs (flushes, events), on-device comparison and
// the accumulator copy to pinned host memory -- and returns WITHOUT waiting;
// tsg_collect waits for that slot and reads it.  With two slots the host
// prepares and enqueues configuration i+1 while the GPU still runs i, so
// the stream never idles between configurations (module load, constant
// upload, argument packing and the Python bookkeeping all overlap device
// work).  Per-run times are still event pairs around each run on the one
// stream: the measured quantity is unchanged.
int tsg_submit_timed(tsg_ctx* c, int slot, const tsg_launch_t* seq, int n, int warmup, int runs, int flush,
                     uint64_t poison_out, size_t n_out, uint64_t ref, double rtol, double atol) {
  int s = make_current(c);
  if (s) return s;
  if (slot < 0 || slot >= TSG_SLOTS) return fail(TSG_ERR_ARG, "slot out of range");
  if (runs < 1 || warmup < 0 || n < 1) return fail(TSG_ERR_ARG, "bad protocol");
  auto& sl = c->slots[slot];
  if (sl.active) return fail(TSG_ERR_ARG, "slot still in flight (collect it first)");
  const int total = warmup + runs;
  const size_t need = 2 * (size_t)total + n + 3;  // + slot start + done
  while (sl.ev.size() < need) {
    CUevent e;
    CUresult r = cuEventCreate(&e, CU_EVENT_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuEventCreate: " + cu_msg(r));
    sl.ev.push_back(e);
  }
  if (!sl.scratch) {
    CUresult r = cuMemAlloc(&sl.scratch, 64);
    if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "slot scratch: " + cu_msg(r));
    void* h = nullptr;
    if (posix_memalign(&h, 4096, 4096)) return fail(TSG_ERR_SETUP, "slot host buffer");
    memset(h, 0, 4096);
    r = cuMemHostRegister(h, 4096, 0);
    if (r != CUDA_SUCCESS) {
      free(h);
      return fail(TSG_ERR_SETUP, "slot host register: " + cu_msg(r));
    }
    sl.host = static_cast<unsigned long long*>(h);
  }
  CUevent* ev = sl.ev.data();
  CUevent* lev = ev + 2 * total;
  CUresult r;
  if (!c->epoch) {
    if ((r = cuEventCreate(&c->epoch, CU_EVENT_DEFAULT)) != CUDA_SUCCESS)
      return fail(TSG_ERR_SETUP, "cuEventCreate: " + cu_msg(r));
    cuEventRecord(c->epoch, c->stream);
  }
  cuEventRecord(ev[need - 2], c->stream);  // slot start (before the poison)
  if (poison_out && (r = cuMemsetD32Async((CUdeviceptr)poison_out, 0x7FC00000u, n_out, c->stream)) != CUDA_SUCCESS)
    return fail(TSG_ERR_RUNTIME, "poison: " + cu_msg(r));
  for (int k = 0; k < total; ++k) {
    if (flush && (s = flush_l2(c))) return s;
    cuEventRecord(ev[2 * k], c->stream);
    const bool last = (k == total - 1);
    for (int i = 0; i < n; ++i) {
      if (last) cuEventRecord(lev[i], c->stream);
      if ((s = launch_one(c, seq[i]))) return s;  // rejected launch: nothing of this slot waits
    }
    if (last) cuEventRecord(lev[n], c->stream);
    cuEventRecord(ev[2 * k + 1], c->stream);
  }
  if (ref) {
    cuMemsetD32Async(sl.scratch, 0, 8, c->stream);
    compare_f32_kernel<<<c->info.sm_count * 8, 256, 0, (cudaStream_t)c->stream>>>(
        (const float*)poison_out, (const float*)ref, n_out, (float)rtol, (float)atol,
        (unsigned long long*)sl.scratch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TSG_ERR_RUNTIME, std::string("compare: ") + cudaGetErrorString(e));
    c->launches.fetch_add(1, std::memory_order_relaxed);
    if ((r = cuMemcpyDtoHAsync(sl.host, sl.scratch, 32, c->stream)) != CUDA_SUCCESS)
      return fail(TSG_ERR_RUNTIME, "compare copy: " + cu_msg(r));
  }
  cuEventRecord(ev[need - 1], c->stream);
  sl.warmup = warmup;
  sl.runs = runs;
  sl.n = n;
  sl.verify = ref != 0;
  sl.active = true;
  return TSG_OK;
}

int tsg_collect(tsg_ctx* c, int slot, double timeout_ms, float* times_ms, float* launch_ms, int n_launch,
                double* max_abs_err, double* max_abs_ref, uint64_t* n_bad, uint64_t* n_nonfinite) {
  int s = make_current(c);
  if (s) return s;
  if (slot < 0 || slot >= TSG_SLOTS) return fail(TSG_ERR_ARG, "slot out of range");
  auto& sl = c->slots[slot];
  if (!sl.active) return fail(TSG_ERR_ARG, "slot not submitted");
  sl.active = false;
  const int total = sl.warmup + sl.runs;
  CUevent* ev = sl.ev.data();
  if ((s = wait_stream(c, ev[2 * (size_t)total + sl.n + 2], timeout_ms))) return s;
  for (int k = sl.warmup; k < total; ++k) cuEventElapsedTime(&times_ms[k - sl.warmup], ev[2 * k], ev[2 * k + 1]);
  CUevent* lev = ev + 2 * total;
  c->last_launch_ms.assign(sl.n, 0.f);
  for (int i = 0; i < sl.n; ++i) cuEventElapsedTime(&c->last_launch_ms[i], lev[i], lev[i + 1]);
  if (launch_ms)
    for (int i = 0; i < n_launch; ++i) launch_ms[i] = i < sl.n ? c->last_launch_ms[i] : 0.f;
  if (sl.verify) {
    const unsigned long long* acc = sl.host;
    unsigned u0 = (unsigned)acc[0], u1 = (unsigned)acc[1];
    float f0, f1;
    memcpy(&f0, &u0, 4);
    memcpy(&f1, &u1, 4);
    if (max_abs_err) *max_abs_err = f0;
    if (max_abs_ref) *max_abs_ref = f1;
    if (n_bad) *n_bad = acc[2];
    if (n_nonfinite) *n_nonfinite = acc[3];
  }
  return TSG_OK;
}

/* Device timeline of a collected slot (valid until the slot is submitted
 * again): start / end of its whole submission in ms since the first
 * submission on this context, and its warm-up run's duration. */
int tsg_slot_timeline(tsg_ctx* c, int slot, double* start_ms, double* end_ms, float* warmup_ms) {
  if (!c) return fail(TSG_ERR_ARG, "null context");
  if (slot < 0 || slot >= TSG_SLOTS) return fail(TSG_ERR_ARG, "slot out of range");
  auto& sl = c->slots[slot];
  if (sl.active || !c->epoch || sl.ev.empty()) return fail(TSG_ERR_ARG, "slot not collected");
  const size_t total = sl.warmup + sl.runs;
  const size_t start = 2 * total + sl.n + 1, done = start + 1;
  float a = 0.f, b = 0.f, w = 0.f;
  cuEventElapsedTime(&a, c->epoch, sl.ev[start]);
  cuEventElapsedTime(&b, c->epoch, sl.ev[done]);
  if (sl.warmup > 0) cuEventElapsedTime(&w, sl.ev[0], sl.ev[1]);
  if (start_ms) *start_ms = a;
  if (end_ms) *end_ms = b;
  if (warmup_ms) *warmup_ms = w;
  return TSG_OK;
}

/* Drop a slot whose submission failed part-way (after the stream drained). */
int tsg_slot_reset(tsg_ctx* c, int slot) {
  if (!c) return fail(TSG_ERR_ARG, "null context");
  if (slot < 0 || slot >= TSG_SLOTS) return fail(TSG_ERR_ARG, "slot out of range");
  c->slots[slot].active = false;
  return TSG_OK;
}

int tsg_tma_encode_2d_f32(tsg_ctx* c, void* desc128, uint64_t gaddr, uint64_t dim0, uint64_t dim1,
                          uint64_t stride1_bytes, uint32_t box0, uint32_t box1, int swizzle_bytes) {
  int s = make_current(c);
  if (s) return s;
  if (!desc128) return fail(TSG_ERR_ARG, "null descriptor buffer");
  CUtensorMapSwizzle sw;
  switch (swizzle_bytes) {
    case 0: sw = CU_TENSOR_MAP_SWIZZLE_NONE; break;
    case 32: sw = CU_TENSOR_MAP_SWIZZLE_32B; break;
    case 64: sw = CU_TENSOR_MAP_SWIZZLE_64B; break;
    case 128: sw = CU_TENSOR_MAP_SWIZZLE_128B; break;
    default: return fail(TSG_ERR_ARG, "swizzle must be 0/32/64/128");
  }
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {stride1_bytes};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(reinterpret_cast<CUtensorMap*>(desc128), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                      reinterpret_cast<void*>(gaddr), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_INVALID, "cuTensorMapEncodeTiled: " + cu_msg(r));
  return TSG_OK;
}

int tsg_set_flush_bytes(tsg_ctx* c, size_t write_bytes, size_t read_bytes) {
  int s = make_current(c);
  if (s) return s;
  cuStreamSynchronize(c->stream);
  if (c->flush_buf) cuMemFree(c->flush_buf);
  if (c->flush_rbuf) cuMemFree(c->flush_rbuf);
  c->flush_buf = c->flush_rbuf = 0;
  c->flush_bytes = (write_bytes + 15) & ~(size_t)15;
  c->flush_rbytes = (read_bytes + 15) & ~(size_t)15;
  return TSG_OK;
}

int tsg_event_record(tsg_ctx* c, int slot) {
  int s = make_current(c);
  if (s) return s;
  if (slot < 0 || slot >= 16) return fail(TSG_ERR_ARG, "event slot out of range");
  if (!c->marks[slot]) {
    CUresult r = cuEventCreate(&c->marks[slot], CU_EVENT_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuEventCreate: " + cu_msg(r));
  }
  CUresult r = cuEventRecord(c->marks[slot], c->stream);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "cuEventRecord: " + cu_msg(r));
  return TSG_OK;
}

int tsg_event_elapsed(tsg_ctx* c, int a, int b, float* ms) {
  int s = make_current(c);
  if (s) return s;
  if (a < 0 || a >= 16 || b < 0 || b >= 16 || !c->marks[a] || !c->marks[b])
    return fail(TSG_ERR_ARG, "event slot not recorded");
  if ((s = wait_stream(c, c->marks[b], 0))) return s;
  CUresult r = cuEventElapsedTime(ms, c->marks[a], c->marks[b]);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "cuEventElapsedTime: " + cu_msg(r));
  return TSG_OK;
}

// ---- ordering against foreign streams (torch / NCCL) -----------------------
// One event per direction and call: record on the producer stream, wait on
// the consumer.  Events are created with timing disabled (cheapest to
// record) and destroyed right away -- the wait keeps its own reference.
namespace {
int order_streams(tsg_ctx* c, CUstream producer, CUstream consumer) {
  CUevent e;
  CUresult r = cuEventCreate(&e, CU_EVENT_DISABLE_TIMING);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_SETUP, "cuEventCreate: " + cu_msg(r));
  r = cuEventRecord(e, producer);
  if (r == CUDA_SUCCESS) r = cuStreamWaitEvent(consumer, e, 0);
  cuEventDestroy(e);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_ARG, "stream ordering: " + cu_msg(r));
  (void)c;
  return TSG_OK;
}
}  // namespace

int tsg_stream_handle(tsg_ctx* c, uint64_t* stream) {
  if (!c || !stream) return fail(TSG_ERR_ARG, "null argument");
  *stream = (uint64_t)(uintptr_t)c->stream;
  return TSG_OK;
}

int tsg_stream_wait(tsg_ctx* c, uint64_t stream) {
  int s = make_current(c);
  if (s) return s;
  return order_streams(c, (CUstream)(uintptr_t)stream, c->stream);
}

int tsg_stream_signal(tsg_ctx* c, uint64_t stream) {
  int s = make_current(c);
  if (s) return s;
  return order_streams(c, c->stream, (CUstream)(uintptr_t)stream);
}

int tsg_launch_async(tsg_ctx* c, const tsg_launch_t* seq, int n) {
  int s = make_current(c);
  if (s) return s;
  for (int i = 0; i < n; ++i)
    if ((s = launch_one(c, seq[i]))) return s;
  return TSG_OK;
}

int tsg_copy_async(tsg_ctx* c, uint64_t dst, uint64_t src, size_t bytes) {
  int s = make_current(c);
  if (s) return s;
  CUresult r = cuMemcpyDtoDAsync((CUdeviceptr)dst, (CUdeviceptr)src, bytes, c->stream);
  if (r != CUDA_SUCCESS) return fail(TSG_ERR_RUNTIME, "D2D async: " + cu_msg(r));
  return TSG_OK;
}

int tsg_sync(tsg_ctx* c, double timeout_ms) {
  int s = make_current(c);
  if (s) return s;
  if ((s = ensure_events(c, 1))) return s;
  cuEventRecord(c->events[0], c->stream);
  return wait_stream(c, c->events[0], timeout_ms);
}

int tsg_last_launch_times(tsg_ctx* c, float* t, int n) {
  if (!c) return fail(TSG_ERR_ARG, "null context");
  for (int i = 0; i < n; ++i) t[i] = i < (int)c->last_launch_ms.size() ? c->last_launch_ms[i] : 0.f;
  return TSG_OK;
}

int tsg_compare_f32(tsg_ctx* c, uint64_t out, uint64_t ref, size_t n, double rtol, double atol,
                    double* max_abs_err, double* max_abs_ref, uint64_t* n_bad,
                    uint64_t* n_nonfinite) {
  int s = make_current(c);
  if (s) return s;
  cuMemsetD32Async(c->scratch, 0, 8, c->stream);
  int blocks = c->info.sm_count * 8;
  compare_f32_kernel<<<blocks, 256, 0, (cudaStream_t)c->stream>>>(
      (const float*)out, (const float*)ref, n, (float)rtol, (float)atol,
      (unsigned long long*)c->scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TSG_ERR_RUNTIME, std::string("compare: ") + cudaGetErrorString(e));
  c->launches.fetch_add(1, std::memory_order_relaxed);
  unsigned long long acc[4];
  CUresult r = cuMemcpyDtoHAsync(acc, c->scratch, sizeof acc, c->stream);
  if (r == CUDA_SUCCESS) r = cuStreamSynchronize(c->stream);
  if (r != CUDA_SUCCESS) {
    c->poisoned = true;
    return fail(TSG_ERR_RUNTIME, "compare sync: " + cu_msg(r));
  }
  unsigned u0 = (unsigned)acc[0], u1 = (unsigned)acc[1];
  float f0, f1;
  memcpy(&f0, &u0, 4);
  memcpy(&f1, &u1, 4);
  if (max_abs_err) *max_abs_err = f0;
  if (max_abs_ref) *max_abs_ref = f1;
  if (n_bad) *n_bad = acc[2];
  if (n_nonfinite) *n_nonfinite = acc[3];
  return TSG_OK;
}

}  // extern "C"
