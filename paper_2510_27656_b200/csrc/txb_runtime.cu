// Runtime half of libtxb200: error strings, symmetric allocations, CUDA IPC
// handle export/import and peer enablement.  This is the B200 stand-in for
// the reference's region registry and rkey descriptors (engine.py:314-350,
// wire.py:64-97): a registered region is a cudaMalloc allocation, its
// descriptor is the 64-byte cudaIpcMemHandle, and "posting" to it is a
// kernel store through the mapped peer pointer.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "txb_common.cuh"

namespace txb {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  cudaGetLastError();  // clear a non-sticky error
  return TXB_ERR_CUDA;
}

}  // namespace txb

using namespace txb;

extern "C" {

const char* txb_last_error(void) { return g_err; }

int txb_version(void) { return 1; }

int txb_device_count(int* out) {
  TXB_CUDA(cudaGetDeviceCount(out));
  return TXB_OK;
}

int txb_alloc(int device, uint64_t bytes, void** out_ptr) {
  if (!out_ptr) {
    set_error("txb_alloc: null out pointer");
    return TXB_ERR_REGION;
  }
  TXB_ON_DEVICE(device);
  void* p = nullptr;
  TXB_CUDA(cudaMalloc(&p, bytes ? bytes : 256));
  TXB_CUDA(cudaMemset(p, 0, bytes ? bytes : 256));
  TXB_CUDA(cudaDeviceSynchronize());
  *out_ptr = p;
  return TXB_OK;
}

int txb_free(int device, void* ptr) {
  TXB_ON_DEVICE(device);
  TXB_CUDA(cudaFree(ptr));
  return TXB_OK;
}

int txb_memset(int device, void* ptr, int value, uint64_t bytes, void* stream) {
  TXB_ON_DEVICE(device);
  TXB_CUDA(cudaMemsetAsync(ptr, value, bytes, (cudaStream_t)stream));
  return TXB_OK;
}

int txb_ipc_export(int device, void* ptr, uint8_t* out_handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == TXB_IPC_HANDLE_BYTES, "ipc handle size");
  TXB_ON_DEVICE(device);
  cudaIpcMemHandle_t h;
  TXB_CUDA(cudaIpcGetMemHandle(&h, ptr));
  memcpy(out_handle, &h, sizeof(h));
  return TXB_OK;
}

int txb_ipc_import(int device, const uint8_t* handle, void** out_ptr) {
  TXB_ON_DEVICE(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  TXB_CUDA(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TXB_OK;
}

int txb_ipc_close(int device, void* ptr) {
  TXB_ON_DEVICE(device);
  TXB_CUDA(cudaIpcCloseMemHandle(ptr));
  return TXB_OK;
}

int txb_enable_peer(int device, int peer_device) {
  if (device == peer_device) return TXB_OK;
  TXB_ON_DEVICE(device);
  int ok = 0;
  TXB_CUDA(cudaDeviceCanAccessPeer(&ok, device, peer_device));
  if (!ok) {
    set_error("device %d cannot access peer %d", device, peer_device);
    return TXB_ERR_REGION;
  }
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return TXB_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return TXB_OK;
}

int txb_check_failures(int device, uint32_t* out) {
  if (!out) {
    set_error("txb_check_failures: null output");
    return TXB_ERR_PROTOCOL;
  }
  *out = 0;
#ifdef TXB_CHECKED
  TXB_ON_DEVICE(device);
  TXB_CUDA(cudaDeviceSynchronize());
  *out = (check_failures_engine() | check_failures_moe() | check_failures_codec()) | 0x80000000u;
#else
  (void)device;
#endif
  return TXB_OK;
}

int txb_preload(int device) {
  TXB_ON_DEVICE(device);
  static bool done[64] = {false};
  if (device >= 0 && device < 64 && done[device]) return TXB_OK;
  TXB_CUDA(preload_engine());
  TXB_CUDA(preload_moe());
  TXB_CUDA(preload_codec());
  if (device >= 0 && device < 64) done[device] = true;
  return TXB_OK;
}

int txb_stream_create(int device, void** out_stream) {
  if (!out_stream) {
    set_error("txb_stream_create: null out pointer");
    return TXB_ERR_TRANSFER;
  }
  TXB_ON_DEVICE(device);
  cudaStream_t st = nullptr;
  TXB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *out_stream = (void*)st;
  return TXB_OK;
}

int txb_stream_destroy(int device, void* stream) {
  TXB_ON_DEVICE(device);
  TXB_CUDA(cudaStreamDestroy((cudaStream_t)stream));
  return TXB_OK;
}

int txb_host_device_ptr(void* host_ptr, void** out_device_ptr) {
  cudaPointerAttributes a;
  TXB_CUDA(cudaPointerGetAttributes(&a, host_ptr));
  if (a.type != cudaMemoryTypeHost) {
    set_error("pointer %p is not page-locked host memory", host_ptr);
    return TXB_ERR_REGION;
  }
  TXB_CUDA(cudaHostGetDevicePointer(out_device_ptr, host_ptr, 0));
  return TXB_OK;
}

}  // extern "C"
