// ipc.cu — CUDA IPC export/import of workspaces for the multi-process
// runtime (one process per GPU; peers' landing slots and flags are written
// through NVLink by the producer kernels' fused peer stores).
#include <map>
#include <mutex>

#include "launch.hpp"

namespace kd {
namespace {
typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
GetRangeFn get_range() {
  static GetRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (GetRangeFn)p;
  });
  return fn;
}
std::mutex g_mu;
std::map<void*, void*> g_base_of;  // mapped ptr -> mapped allocation base
}  // namespace
}  // namespace kd

using namespace kd;

extern "C" {

kd_status kd_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return fail(KD_ERR_INVALID_ARG, "kd_ipc_get_handle: NULL argument");
  GetRangeFn fn = get_range();
  if (!fn) return fail(KD_ERR_CUDA, "kd_ipc_get_handle: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return fail(KD_ERR_CUDA, "kd_ipc_get_handle: address range");
  cudaIpcMemHandle_t h;
  KD_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  std::memcpy(handle64, &h, 64);
  *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
  return KD_OK;
}

kd_status kd_ipc_open(const void* handle64, uint64_t offset, void** mapped_ptr) {
  if (!handle64 || !mapped_ptr) return fail(KD_ERR_INVALID_ARG, "kd_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void* base = nullptr;
  KD_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  void* p = (uint8_t*)base + offset;
  std::lock_guard<std::mutex> lk(g_mu);
  g_base_of[p] = base;
  *mapped_ptr = p;
  return KD_OK;
}

kd_status kd_ipc_close(void* mapped_ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_base_of.find(mapped_ptr);
  if (it == g_base_of.end()) return fail(KD_ERR_INVALID_ARG, "kd_ipc_close: pointer was not opened by kd_ipc_open");
  cudaError_t e = cudaIpcCloseMemHandle(it->second);
  g_base_of.erase(it);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcCloseMemHandle");
  return KD_OK;
}

}  // extern "C"
