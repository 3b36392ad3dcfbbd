// ss_ipc.cu — cross-process device hand-off of client exchange buffers (CUDA IPC).
//
// The paper's co-located mode shares a pre-allocated CUDA exchange tensor between a client
// process and the executor process (share_memory_ / rebuild_cuda_tensor); the
// reference package's process mode otherwise frames every payload through host memory
// (harness.py:243-260, 367-394 -> RemoteChannel, transport.py:104-161). These entry points let
// a client process export its request / reply / y_base buffers ONCE (per grow) and the executor
// process map them; ordering between the two processes' streams uses interprocess events.
// See include/ss_b200.h for the contract; paper_2507_03220_b200/ipc.py is the Python side.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "../../include/ss_b200.h"

namespace {

thread_local std::string g_ipc_err;

int ipc_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_ipc_err = buf;
  return code;
}

int ipc_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SS_OK;
  cudaGetLastError();
  return ipc_fail(SS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

using PFN_getAddressRange_t = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

PFN_getAddressRange_t address_range_fn() {
  static PFN_getAddressRange_t fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess)
      return (PFN_getAddressRange_t) nullptr;
    return reinterpret_cast<PFN_getAddressRange_t>(p);
  }();
  return fn;
}

// One mapping per exported allocation per process (cudaIpcOpenMemHandle must not be called
// twice on one handle in a process): keyed by the handle bytes, reference counted, and every
// opened pointer (base + offset) remembers its mapping.
struct Mapping {
  void* base = nullptr;
  int refs = 0;
};
std::mutex g_mu;
std::map<std::string, Mapping> g_maps;
std::map<void*, std::string> g_opened;   // returned pointer -> handle key (multiset via refs)
std::map<void*, int> g_opened_refs;

}  // namespace

extern "C" {

const char* ss_ipc_last_error(void) { return g_ipc_err.c_str(); }

int ss_ipc_export(const void* dptr, uint64_t bytes, ss_ipc_mem* out) {
  if (!dptr || !out) return ipc_fail(SS_E_ARG, "ss_ipc_export: null argument");
  std::memset(out, 0, sizeof *out);
  cudaPointerAttributes attr;
  if (int rc = ipc_cuda(cudaPointerGetAttributes(&attr, dptr), "cudaPointerGetAttributes")) return rc;
  if (attr.type != cudaMemoryTypeDevice)
    return ipc_fail(SS_E_ARG, "ss_ipc_export: %p is not device memory", dptr);
  PFN_getAddressRange_t range = address_range_fn();
  if (!range) return ipc_fail(SS_E_CUDA, "cuMemGetAddressRange unavailable");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(attr.device);
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = range(&base, &size, (CUdeviceptr)dptr);
  if (r != CUDA_SUCCESS) {
    cudaSetDevice(prev);
    return ipc_fail(SS_E_CUDA, "cuMemGetAddressRange failed (%d)", (int)r);
  }
  const uint64_t offset = (uint64_t)((CUdeviceptr)dptr - base);
  if (offset + bytes > size) {
    cudaSetDevice(prev);
    return ipc_fail(SS_E_ARG, "ss_ipc_export: %llu bytes at offset %llu exceed the allocation (%zu)",
                    (unsigned long long)bytes, (unsigned long long)offset, size);
  }
  cudaIpcMemHandle_t h;
  int rc = ipc_cuda(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle");
  cudaSetDevice(prev);
  if (rc) return rc;
  static_assert(sizeof(h) == sizeof(out->handle), "IPC handle size");
  std::memcpy(out->handle, &h, sizeof h);
  out->offset = offset;
  out->bytes = bytes;
  out->device = attr.device;
  return SS_OK;
}

int ss_ipc_alloc(int device, uint64_t bytes, void** dptr, ss_ipc_mem* out) {
  if (!dptr || !out || bytes == 0) return ipc_fail(SS_E_ARG, "ss_ipc_alloc: bad argument");
  *dptr = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  if (int rc = ipc_cuda(cudaSetDevice(device), "cudaSetDevice")) return rc;
  void* p = nullptr;
  int rc = ipc_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  cudaSetDevice(prev);
  if (rc) return rc == SS_E_CUDA ? SS_E_NOMEM : rc;
  rc = ss_ipc_export(p, bytes, out);
  if (rc) {
    cudaFree(p);
    return rc;
  }
  *dptr = p;
  return SS_OK;
}

int ss_ipc_free(void* dptr) {
  if (!dptr) return SS_OK;
  return ipc_cuda(cudaFree(dptr), "cudaFree");
}

int ss_ipc_open(int device, const ss_ipc_mem* mem, void** dptr) {
  if (!mem || !dptr) return ipc_fail(SS_E_ARG, "ss_ipc_open: null argument");
  *dptr = nullptr;
  const std::string key(reinterpret_cast<const char*>(mem->handle), sizeof mem->handle);
  std::lock_guard<std::mutex> g(g_mu);
  Mapping& m = g_maps[key];
  if (!m.base) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (int rc = ipc_cuda(cudaSetDevice(device), "cudaSetDevice")) {
      g_maps.erase(key);
      return rc;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, mem->handle, sizeof h);
    // a client on another GPU: the mapping is peer memory, reached over NVLink
    int rc = ipc_cuda(cudaIpcOpenMemHandle(&m.base, h, cudaIpcMemLazyEnablePeerAccess),
                      "cudaIpcOpenMemHandle");
    cudaSetDevice(prev);
    if (rc) {
      g_maps.erase(key);
      return rc;
    }
  }
  m.refs++;
  void* p = static_cast<char*>(m.base) + mem->offset;
  g_opened[p] = key;
  g_opened_refs[p]++;
  *dptr = p;
  return SS_OK;
}

int ss_ipc_close(void* dptr) {
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_opened.find(dptr);
  if (it == g_opened.end()) return ipc_fail(SS_E_ARG, "ss_ipc_close: %p was not opened", dptr);
  const std::string key = it->second;
  if (--g_opened_refs[dptr] == 0) {
    g_opened_refs.erase(dptr);
    g_opened.erase(it);
  }
  auto mit = g_maps.find(key);
  if (mit == g_maps.end()) return SS_OK;
  if (--mit->second.refs == 0) {
    int rc = ipc_cuda(cudaIpcCloseMemHandle(mit->second.base), "cudaIpcCloseMemHandle");
    g_maps.erase(mit);
    return rc;
  }
  return SS_OK;
}

int ss_ipc_event_create(int device, void** event, ss_ipc_evt* out) {
  if (!event || !out) return ipc_fail(SS_E_ARG, "ss_ipc_event_create: null argument");
  *event = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  if (int rc = ipc_cuda(cudaSetDevice(device), "cudaSetDevice")) return rc;
  cudaEvent_t e = nullptr;
  int rc = ipc_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess),
                    "cudaEventCreateWithFlags(interprocess)");
  if (!rc) {
    cudaIpcEventHandle_t h;
    rc = ipc_cuda(cudaIpcGetEventHandle(&h, e), "cudaIpcGetEventHandle");
    if (rc) {
      cudaEventDestroy(e);
    } else {
      static_assert(sizeof(h) == sizeof(out->handle), "IPC event handle size");
      std::memcpy(out->handle, &h, sizeof h);
      *event = e;
    }
  }
  cudaSetDevice(prev);
  return rc;
}

int ss_ipc_event_open(int device, const ss_ipc_evt* h, void** event) {
  if (!h || !event) return ipc_fail(SS_E_ARG, "ss_ipc_event_open: null argument");
  *event = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  if (int rc = ipc_cuda(cudaSetDevice(device), "cudaSetDevice")) return rc;
  cudaIpcEventHandle_t eh;
  std::memcpy(&eh, h->handle, sizeof eh);
  cudaEvent_t e = nullptr;
  int rc = ipc_cuda(cudaIpcOpenEventHandle(&e, eh), "cudaIpcOpenEventHandle");
  cudaSetDevice(prev);
  if (!rc) *event = e;
  return rc;
}

int ss_ipc_event_record(void* event, void* stream) {
  if (!event) return ipc_fail(SS_E_ARG, "ss_ipc_event_record: null event");
  return ipc_cuda(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream), "cudaEventRecord");
}

int ss_ipc_event_wait(void* stream, void* event) {
  if (!event) return ipc_fail(SS_E_ARG, "ss_ipc_event_wait: null event");
  return ipc_cuda(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0),
                  "cudaStreamWaitEvent");
}

int ss_ipc_event_sync(void* event) {
  if (!event) return ipc_fail(SS_E_ARG, "ss_ipc_event_sync: null event");
  return ipc_cuda(cudaEventSynchronize((cudaEvent_t)event), "cudaEventSynchronize");
}

int ss_ipc_event_destroy(void* event) {
  if (!event) return SS_OK;
  return ipc_cuda(cudaEventDestroy((cudaEvent_t)event), "cudaEventDestroy");
}

}  // extern "C"
