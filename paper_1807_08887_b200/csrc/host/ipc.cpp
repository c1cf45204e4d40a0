// CUDA IPC plumbing for one-process-per-GPU execution: each rank exports its arena, every peer
// maps it ON ITS OWN DEVICE (the current device set explicitly, peer access enabled explicitly), so the
// MultiFetch / reduce kernels of a rank load the peer's HBM over NVLink through the mapped address.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "common.h"

namespace {
using PFN_getAddressRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_getAddressRange g_range = nullptr;
std::once_flag g_range_once;

PFN_getAddressRange address_range_fn() {
  std::call_once(g_range_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_range = reinterpret_cast<PFN_getAddressRange>(fn);
  });
  return g_range;
}
}  // namespace

extern "C" int tofu_ipc_export(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  return tofu::guard([&]() {
    if (!dev_ptr || !handle_out || !offset_out) throw tofu::Error(TOFU_ERR_ARG, "null argument");
    auto fn = address_range_fn();
    if (!fn) throw tofu::Error(TOFU_ERR_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
      throw tofu::Error(TOFU_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess)
      throw tofu::Error(TOFU_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(cudaGetLastError()));
    std::memcpy(handle_out, &h, sizeof h);
    *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    return TOFU_OK;
  });
}

extern "C" int tofu_ipc_open(const void* handle, int64_t offset, int local_device, int peer_device, void** ptr_out) {
  return tofu::guard([&]() {
    if (!handle || !ptr_out || offset < 0 || local_device < 0) throw tofu::Error(TOFU_ERR_ARG, "bad argument");
    if (cudaSetDevice(local_device) != cudaSuccess) throw tofu::Error(TOFU_ERR_CUDA, "cudaSetDevice");
    if (peer_device >= 0 && peer_device != local_device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, local_device, peer_device);
      if (!can) throw tofu::Error(TOFU_ERR_CUDA, "no peer access between the two GPUs");
      const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        throw tofu::Error(TOFU_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      cudaGetLastError();  // clear "already enabled"
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) throw tofu::Error(TOFU_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    *ptr_out = static_cast<char*>(base) + offset;
    return TOFU_OK;
  });
}

extern "C" int tofu_ipc_close(void* mapped_ptr, int64_t offset) {
  if (!mapped_ptr) return tofu::fail(TOFU_ERR_ARG, "null pointer");
  return cudaIpcCloseMemHandle(static_cast<char*>(mapped_ptr) - offset) == cudaSuccess ? TOFU_OK
                                                                                        : tofu::fail(TOFU_ERR_CUDA, "cudaIpcCloseMemHandle");
}
