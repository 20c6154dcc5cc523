// vmm.cu — a growable device arena on CUDA virtual memory management.
//
// The paper's long rows grow their allocation 2x on overflow and, on the APU, profit from
// re-allocatable memory that needs no copy ([P:741-745]: 1.2x on average, up to 1.8x).  The
// discrete-GPU analogue here: one virtual address range is reserved up front
// (cuMemAddressReserve, no physical memory), and physical memory is created and mapped at its
// end on demand (cuMemCreate + cuMemMap + cuMemSetAccess).  Data already written never moves,
// the arena never needs a re-allocation, and a growth step costs only the new pages.
// Driver entry points are fetched at run time (cudaGetDriverEntryPoint), so libspgemm needs
// no link against libcuda.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace sg {

namespace {

struct DriverVmm {
  PFN_cuMemAddressReserve reserve = nullptr;
  PFN_cuMemAddressFree free_va = nullptr;
  PFN_cuMemCreate create = nullptr;
  PFN_cuMemRelease release = nullptr;
  PFN_cuMemMap map = nullptr;
  PFN_cuMemUnmap unmap = nullptr;
  PFN_cuMemSetAccess access = nullptr;
  PFN_cuMemGetAllocationGranularity gran = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const DriverVmm& drv() {
  static DriverVmm d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuMemAddressReserve", &d.reserve) && entry("cuMemAddressFree", &d.free_va) &&
           entry("cuMemCreate", &d.create) && entry("cuMemRelease", &d.release) && entry("cuMemMap", &d.map) &&
           entry("cuMemUnmap", &d.unmap) && entry("cuMemSetAccess", &d.access) &&
           entry("cuMemGetAllocationGranularity", &d.gran);
  });
  return d;
}

struct Impl {
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<std::pair<size_t, size_t>> maps;  // (offset, size) of each mapped block
};

CUmemAllocationProp props(int dev) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  return p;
}

cudaError_t cu_err(CUresult r) {
  if (r == CUDA_SUCCESS) return cudaSuccess;
  if (r == CUDA_ERROR_OUT_OF_MEMORY) return cudaErrorMemoryAllocation;
  return cudaErrorUnknown;
}

}  // namespace

// Released arenas are kept (reservation and mapped pages) for the next multiply on the device,
// like the library's memory pool keeps freed workspace: mapping and unmapping tens of GB of
// physical pages per multiply is host time inside the step.  spgemm_trim_workspace_cache
// releases them (vmm_trim).
static std::mutex g_cache_mu;
static std::vector<VmmArena> g_cache;

static void release_now(VmmArena* a);

cudaError_t vmm_reserve(VmmArena* a, size_t bytes) {
  const DriverVmm& d = drv();
  if (!d.ok) return cudaErrorNotSupported;
  cudaGetDevice(&a->device);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int best = -1;
    for (int i = 0; i < (int)g_cache.size(); ++i)
      if (g_cache[i].device == a->device && g_cache[i].reserved >= bytes &&
          (best < 0 || g_cache[i].reserved < g_cache[best].reserved))
        best = i;
    if (best >= 0) {
      *a = g_cache[best];
      g_cache.erase(g_cache.begin() + best);
      return cudaSuccess;
    }
  }
  vmm_trim();  // no cached arena fits: do not keep pages for ones that will not be reused
  CUmemAllocationProp p = props(a->device);
  size_t g = 0;
  CUresult r = d.gran(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return cu_err(r);
  a->gran = g;
  a->reserved = (bytes + g - 1) / g * g;
  if (a->reserved == 0) a->reserved = g;
  CUdeviceptr base = 0;
  r = d.reserve(&base, a->reserved, 0, 0, 0);
  if (r != CUDA_SUCCESS) return cu_err(r);
  a->base = reinterpret_cast<void*>(base);
  a->mapped = 0;
  a->impl = new Impl();
  return cudaSuccess;
}

// Back [0, bytes) of the arena with physical memory: one new block mapped at the current end
// (earlier blocks and the data in them stay where they are).
cudaError_t vmm_ensure(VmmArena* a, size_t bytes) {
  if (bytes <= a->mapped) return cudaSuccess;
  if (bytes > a->reserved) return cudaErrorMemoryAllocation;
  const DriverVmm& d = drv();
  Impl* im = static_cast<Impl*>(a->impl);
  const size_t want = (bytes + a->gran - 1) / a->gran * a->gran;
  // grow at least 2x the mapped size (fewer, larger blocks), within the reservation
  size_t size = want - a->mapped;
  if (size < a->mapped && a->mapped + a->mapped <= a->reserved) size = a->mapped;
  CUmemAllocationProp p = props(a->device);
  CUmemGenericAllocationHandle h;
  CUresult r = d.create(&h, size, &p, 0);
  if (r == CUDA_ERROR_OUT_OF_MEMORY) {  // pages held by cached arenas: release them, retry
    vmm_trim();
    r = d.create(&h, size, &p, 0);
  }
  if (r != CUDA_SUCCESS) return cu_err(r);
  const CUdeviceptr at = reinterpret_cast<CUdeviceptr>(a->base) + a->mapped;
  r = d.map(at, size, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    d.release(h);
    return cu_err(r);
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = a->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = d.access(at, size, &acc, 1);
  if (r != CUDA_SUCCESS) {
    d.unmap(at, size);
    d.release(h);
    return cu_err(r);
  }
  im->handles.push_back(h);
  im->maps.emplace_back(a->mapped, size);
  a->mapped += size;
  return cudaSuccess;
}

void vmm_release(VmmArena* a) {
  if (!a->base) return;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (g_cache.size() < 4) {
      g_cache.push_back(*a);
      *a = VmmArena{};
      return;
    }
  }
  release_now(a);
}

void vmm_trim() {
  std::vector<VmmArena> all;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    all.swap(g_cache);
  }
  for (auto& a : all) release_now(&a);
}

static void release_now(VmmArena* a) {
  if (!a->base) return;
  const DriverVmm& d = drv();
  Impl* im = static_cast<Impl*>(a->impl);
  const CUdeviceptr base = reinterpret_cast<CUdeviceptr>(a->base);
  if (im) {
    for (auto& m : im->maps) d.unmap(base + m.first, m.second);
    for (auto h : im->handles) d.release(h);
    delete im;
  }
  d.free_va(base, a->reserved);
  *a = VmmArena{};
}

}  // namespace sg
