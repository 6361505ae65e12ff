// Driver API reached through dlopen("libcuda.so.1") + cuGetProcAddress,
// so libtsgpu.so loads (and NVRTC compiles) on hosts without a GPU
// driver; tsg_init is the first call that needs one.
#pragma once
#include <cuda.h>
#include <dlfcn.h>

#define TSG_DRIVER_FUNCS(X) \
  X(cuCtxSetCurrent) \
  X(cuDeviceGet) \
  X(cuDeviceGetAttribute) \
  X(cuDeviceGetName) \
  X(cuDevicePrimaryCtxRelease) \
  X(cuDevicePrimaryCtxRetain) \
  X(cuDeviceTotalMem) \
  X(cuDriverGetVersion) \
  X(cuEventCreate) \
  X(cuEventDestroy) \
  X(cuEventElapsedTime) \
  X(cuEventQuery) \
  X(cuEventRecord) \
  X(cuFuncGetAttribute) \
  X(cuFuncSetAttribute) \
  X(cuGetErrorName) \
  X(cuGetErrorString) \
  X(cuInit) \
  X(cuLaunchKernel) \
  X(cuLaunchKernelEx) \
  X(cuMemAlloc) \
  X(cuMemFree) \
  X(cuMemHostRegister) \
  X(cuMemHostUnregister) \
  X(cuMemcpyDtoDAsync) \
  X(cuMemcpyDtoHAsync) \
  X(cuMemcpyHtoD) \
  X(cuMemcpyHtoDAsync) \
  X(cuMemsetD32Async) \
  X(cuModuleGetFunction) \
  X(cuModuleGetGlobal) \
  X(cuModuleLoadData) \
  X(cuModuleUnload) \
  X(cuOccupancyMaxActiveBlocksPerMultiprocessor) \
  X(cuStreamCreate) \
  X(cuStreamDestroy) \
  X(cuStreamSynchronize) \
  X(cuStreamWaitEvent) \
  X(cuTensorMapEncodeTiled) \

struct TsgDriver {
#define TSG_DECL(f) decltype(&f) p_##f = nullptr;
  TSG_DRIVER_FUNCS(TSG_DECL)
#undef TSG_DECL
  bool loaded = false;
};

inline TsgDriver& tsg_drv() {
  static TsgDriver d;
  return d;
}

// Returns nullptr on success, else a message.
inline const char* tsg_load_driver() {
  TsgDriver& d = tsg_drv();
  if (d.loaded) return nullptr;
  void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return "libcuda.so.1 not found (no NVIDIA driver on this host)";
  typedef CUresult (*GetProc)(const char*, void**, int, cuuint64_t, CUdriverProcAddressQueryResult*);
  GetProc gp = (GetProc)dlsym(h, "cuGetProcAddress_v2");
  if (!gp) return "driver lacks cuGetProcAddress_v2 (need CUDA 12+ driver)";
  CUdriverProcAddressQueryResult st;
#define TSG_LOAD(f) \
  if (gp(#f, (void**)&d.p_##f, 12000, CU_GET_PROC_ADDRESS_DEFAULT, &st) != CUDA_SUCCESS || !d.p_##f) return "missing driver symbol " #f;
  TSG_DRIVER_FUNCS(TSG_LOAD)
#undef TSG_LOAD
  d.loaded = true;
  return nullptr;
}

#undef cuCtxSetCurrent
#define cuCtxSetCurrent (tsg_drv().p_cuCtxSetCurrent)
#undef cuDeviceGet
#define cuDeviceGet (tsg_drv().p_cuDeviceGet)
#undef cuDeviceGetAttribute
#define cuDeviceGetAttribute (tsg_drv().p_cuDeviceGetAttribute)
#undef cuDeviceGetName
#define cuDeviceGetName (tsg_drv().p_cuDeviceGetName)
#undef cuDevicePrimaryCtxRelease
#define cuDevicePrimaryCtxRelease (tsg_drv().p_cuDevicePrimaryCtxRelease)
#undef cuDevicePrimaryCtxRetain
#define cuDevicePrimaryCtxRetain (tsg_drv().p_cuDevicePrimaryCtxRetain)
#undef cuDeviceTotalMem
#define cuDeviceTotalMem (tsg_drv().p_cuDeviceTotalMem)
#undef cuDriverGetVersion
#define cuDriverGetVersion (tsg_drv().p_cuDriverGetVersion)
#undef cuEventCreate
#define cuEventCreate (tsg_drv().p_cuEventCreate)
#undef cuEventDestroy
#define cuEventDestroy (tsg_drv().p_cuEventDestroy)
#undef cuEventElapsedTime
#define cuEventElapsedTime (tsg_drv().p_cuEventElapsedTime)
#undef cuEventQuery
#define cuEventQuery (tsg_drv().p_cuEventQuery)
#undef cuEventRecord
#define cuEventRecord (tsg_drv().p_cuEventRecord)
#undef cuOccupancyMaxActiveBlocksPerMultiprocessor
#define cuOccupancyMaxActiveBlocksPerMultiprocessor (tsg_drv().p_cuOccupancyMaxActiveBlocksPerMultiprocessor)
#undef cuFuncGetAttribute
#define cuFuncGetAttribute (tsg_drv().p_cuFuncGetAttribute)
#undef cuFuncSetAttribute
#define cuFuncSetAttribute (tsg_drv().p_cuFuncSetAttribute)
#undef cuGetErrorName
#define cuGetErrorName (tsg_drv().p_cuGetErrorName)
#undef cuGetErrorString
#define cuGetErrorString (tsg_drv().p_cuGetErrorString)
#undef cuInit
#define cuInit (tsg_drv().p_cuInit)
#undef cuLaunchKernel
#define cuLaunchKernel (tsg_drv().p_cuLaunchKernel)
#undef cuLaunchKernelEx
#define cuLaunchKernelEx (tsg_drv().p_cuLaunchKernelEx)
#undef cuMemAlloc
#define cuMemAlloc (tsg_drv().p_cuMemAlloc)
#undef cuMemFree
#define cuMemFree (tsg_drv().p_cuMemFree)
#undef cuMemHostRegister
#define cuMemHostRegister (tsg_drv().p_cuMemHostRegister)
#undef cuMemHostUnregister
#define cuMemHostUnregister (tsg_drv().p_cuMemHostUnregister)
#undef cuMemcpyDtoDAsync
#define cuMemcpyDtoDAsync (tsg_drv().p_cuMemcpyDtoDAsync)
#undef cuMemcpyDtoHAsync
#define cuMemcpyDtoHAsync (tsg_drv().p_cuMemcpyDtoHAsync)
#undef cuMemcpyHtoD
#define cuMemcpyHtoD (tsg_drv().p_cuMemcpyHtoD)
#undef cuMemcpyHtoDAsync
#define cuMemcpyHtoDAsync (tsg_drv().p_cuMemcpyHtoDAsync)
#undef cuMemsetD32Async
#define cuMemsetD32Async (tsg_drv().p_cuMemsetD32Async)
#undef cuModuleGetFunction
#define cuModuleGetFunction (tsg_drv().p_cuModuleGetFunction)
#undef cuModuleGetGlobal
#define cuModuleGetGlobal (tsg_drv().p_cuModuleGetGlobal)
#undef cuModuleLoadData
#define cuModuleLoadData (tsg_drv().p_cuModuleLoadData)
#undef cuModuleUnload
#define cuModuleUnload (tsg_drv().p_cuModuleUnload)
#undef cuStreamCreate
#define cuStreamCreate (tsg_drv().p_cuStreamCreate)
#undef cuStreamDestroy
#define cuStreamDestroy (tsg_drv().p_cuStreamDestroy)
#undef cuStreamSynchronize
#define cuStreamSynchronize (tsg_drv().p_cuStreamSynchronize)
#undef cuStreamWaitEvent
#define cuStreamWaitEvent (tsg_drv().p_cuStreamWaitEvent)
#undef cuTensorMapEncodeTiled
#define cuTensorMapEncodeTiled (tsg_drv().p_cuTensorMapEncodeTiled)
