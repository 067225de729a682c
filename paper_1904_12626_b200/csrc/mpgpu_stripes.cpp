// Striped device regions: one contiguous virtual address range whose physical
// 2 MB chunks live in the HBM of different GPUs (chunk c on rank owners[c]:
// round-robin, or a table balancing the modelled key traffic per GPU),
// built with the CUDA virtual-memory API (cuMemCreate / cuMemMap).
//
// Why: the shared-key join has every rank read its filter thresholds from, and
// RED.MIN its candidates into, one set of key arrays while it computes
// (DESIGN.md §7). With the keys in one GPU's memory, that GPU serves every
// other rank's tile prefetches (~170 GB/s per rank at 2.7e12 cells/s, i.e.
// ~1.2 TB/s at N = 8). Striping the key arrays across all ranks spreads the
// same traffic over every GPU's NVLink ports, and the kernels are unchanged:
// they index one flat array. Reference counterpart: the min-merge of worker
// profiles in stomp (profile.hpp:66-68, 80-83).
//
// Multi-process (one process per GPU): every rank creates its own chunks,
// exports each as a POSIX file descriptor (passed to the other ranks over a
// Unix socket by the caller, SCM_RIGHTS), imports the others' chunks, then maps
// all of them. One process driving several GPUs: mpgpu_stripes_create_local
// creates every chunk itself and grants every device access.
//
// Driver entry points are resolved at run time through cudart
// (cudaGetDriverEntryPointByVersion), so the library does not link libcuda and
// still loads on a machine without a driver.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "mpgpu_internal.h"
#include "mprof_gpu.h"

using mpgpu_internal::set_error;

namespace {

struct Driver {
  bool ok = false;
  std::string why;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
};

template <class F>
bool resolve(const char* name, F& fn, std::string& why) {
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  void* p = nullptr;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p) {
    cudaGetLastError();
    why = std::string("driver entry point ") + name + " unavailable";
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    std::string& w = d.why;
    d.ok = resolve("cuMemCreate", d.create, w) && resolve("cuMemRelease", d.release, w) &&
           resolve("cuMemAddressReserve", d.reserve, w) &&
           resolve("cuMemAddressFree", d.addr_free, w) && resolve("cuMemMap", d.map, w) &&
           resolve("cuMemUnmap", d.unmap, w) && resolve("cuMemSetAccess", d.set_access, w) &&
           resolve("cuMemGetAllocationGranularity", d.granularity, w) &&
           resolve("cuMemExportToShareableHandle", d.export_handle, w) &&
           resolve("cuMemImportFromShareableHandle", d.import_handle, w);
  });
  return d;
}

mpgpu_status cu_fail(CUresult r, const char* what) {
  return set_error(r == CUDA_ERROR_OUT_OF_MEMORY ? MPGPU_ENOMEM : MPGPU_ECUDA,
                   std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
}

CUmemAllocationProp chunk_prop(int device, bool shareable) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes =
      shareable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  return prop;
}

}  // namespace

struct mpgpu_stripes {
  int n_ranks = 1, rank = 0, device = 0;
  size_t chunk = 0;                               // bytes per chunk (VMM granularity)
  std::vector<CUmemGenericAllocationHandle> h;    // per chunk, 0 until created / imported
  std::vector<int> owner;                         // rank (local mode: device slot) of each chunk
  std::vector<int> access_devs;                   // devices granted read/write access
  CUdeviceptr base = 0;
  size_t mapped = 0;                              // chunks mapped so far
};

namespace {
// owners[c] when given (and in range), else round-robin
std::vector<int> owner_table(size_t n_chunks, int n_ranks, const int32_t* owners) {
  std::vector<int> o(n_chunks);
  for (size_t c = 0; c < n_chunks; ++c) {
    const int w = owners ? owners[c] : -1;
    o[c] = (w >= 0 && w < n_ranks) ? w : (int)(c % (size_t)n_ranks);
  }
  return o;
}
}  // namespace

extern "C" {

int64_t mpgpu_stripes_granularity(int32_t device) {
  const Driver& d = drv();
  if (!d.ok) {
    set_error(MPGPU_EUNSUPPORTED, d.why);
    return -1;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    set_error(MPGPU_ECUDA, "cudaSetDevice failed");
    return -1;
  }
  cudaFree(nullptr);
  const CUmemAllocationProp prop = chunk_prop(device, true);
  size_t g = 0;
  if (CUresult r = d.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM); r != CUDA_SUCCESS) {
    cu_fail(r, "cuMemGetAllocationGranularity");
    return -1;
  }
  return (int64_t)g;
}

mpgpu_stripes* mpgpu_stripes_create(int64_t bytes, int32_t n_ranks, int32_t rank, int32_t device,
                                    const int32_t* owners) {
  const Driver& d = drv();
  if (!d.ok) {
    set_error(MPGPU_EUNSUPPORTED, d.why);
    return nullptr;
  }
  if (bytes <= 0 || n_ranks < 1 || rank < 0 || rank >= n_ranks) {
    set_error(MPGPU_EPARAM, "bad striped-region arguments");
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    set_error(MPGPU_ECUDA, "cudaSetDevice failed");
    return nullptr;
  }
  cudaFree(nullptr);  // make sure the primary context exists before driver calls
  const CUmemAllocationProp prop = chunk_prop(device, true);
  size_t g = 0;
  if (CUresult r = d.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM); r != CUDA_SUCCESS) {
    cu_fail(r, "cuMemGetAllocationGranularity");
    return nullptr;
  }
  auto* s = new mpgpu_stripes();
  s->n_ranks = n_ranks;
  s->rank = rank;
  s->device = device;
  s->chunk = g;
  const size_t n_chunks = ((size_t)bytes + g - 1) / g;
  s->h.assign(n_chunks, 0);
  s->owner = owner_table(n_chunks, n_ranks, owners);
  s->access_devs = {device};
  for (size_t c = 0; c < n_chunks; ++c) {
    if (s->owner[c] != rank) continue;
    if (CUresult r = d.create(&s->h[c], g, &prop, 0); r != CUDA_SUCCESS) {
      cu_fail(r, "cuMemCreate");
      mpgpu_stripes_destroy(s);
      return nullptr;
    }
  }
  return s;
}

mpgpu_stripes* mpgpu_stripes_create_local(int64_t bytes, int32_t n_devices, const int32_t* devices,
                                          const int32_t* owners) {
  const Driver& d = drv();
  if (!d.ok) {
    set_error(MPGPU_EUNSUPPORTED, d.why);
    return nullptr;
  }
  if (bytes <= 0 || n_devices < 1 || !devices) {
    set_error(MPGPU_EPARAM, "bad striped-region arguments");
    return nullptr;
  }
  size_t g = 0;
  for (int q = 0; q < n_devices; ++q) {
    if (cudaSetDevice(devices[q]) != cudaSuccess) {
      cudaGetLastError();
      set_error(MPGPU_ECUDA, "cudaSetDevice failed");
      return nullptr;
    }
    cudaFree(nullptr);
    const CUmemAllocationProp prop = chunk_prop(devices[q], false);
    size_t gq = 0;
    if (CUresult r = d.granularity(&gq, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM); r != CUDA_SUCCESS) {
      cu_fail(r, "cuMemGetAllocationGranularity");
      return nullptr;
    }
    g = std::max(g, gq);
  }
  auto* s = new mpgpu_stripes();
  s->n_ranks = n_devices;
  s->rank = -1;  // local: every chunk is created here
  s->device = devices[0];
  s->chunk = g;
  const size_t n_chunks = ((size_t)bytes + g - 1) / g;
  s->h.assign(n_chunks, 0);
  s->owner = owner_table(n_chunks, n_devices, owners);
  for (int q = 0; q < n_devices; ++q) {
    bool seen = false;
    for (int a : s->access_devs) seen |= a == devices[q];
    if (!seen) s->access_devs.push_back(devices[q]);
  }
  for (size_t c = 0; c < n_chunks; ++c) {
    const int dev = devices[s->owner[c]];
    const CUmemAllocationProp prop = chunk_prop(dev, false);
    if (CUresult r = d.create(&s->h[c], g, &prop, 0); r != CUDA_SUCCESS) {
      cu_fail(r, "cuMemCreate");
      mpgpu_stripes_destroy(s);
      return nullptr;
    }
  }
  void* base = nullptr;
  if (mpgpu_stripes_map(s, &base) != MPGPU_OK) {
    mpgpu_stripes_destroy(s);
    return nullptr;
  }
  return s;
}

int64_t mpgpu_stripes_num_chunks(const mpgpu_stripes* s) { return s ? (int64_t)s->h.size() : 0; }

int64_t mpgpu_stripes_chunk_bytes(const mpgpu_stripes* s) { return s ? (int64_t)s->chunk : 0; }

int32_t mpgpu_stripes_owner(const mpgpu_stripes* s, int64_t chunk) {
  if (!s || chunk < 0 || chunk >= (int64_t)s->h.size()) return -1;
  return (int32_t)s->owner[chunk];
}

int32_t mpgpu_stripes_export_fd(mpgpu_stripes* s, int64_t chunk) {
  if (!s || chunk < 0 || chunk >= (int64_t)s->h.size() || s->rank < 0 ||
      s->owner[chunk] != s->rank || !s->h[chunk]) {
    set_error(MPGPU_EPARAM, "chunk not owned by this rank");
    return -1;
  }
  int fd = -1;
  if (CUresult r = drv().export_handle(&fd, s->h[chunk], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
      r != CUDA_SUCCESS) {
    cu_fail(r, "cuMemExportToShareableHandle");
    return -1;
  }
  return fd;
}

mpgpu_status mpgpu_stripes_import_fd(mpgpu_stripes* s, int64_t chunk, int32_t fd) {
  if (!s || chunk < 0 || chunk >= (int64_t)s->h.size() || s->h[chunk] || fd < 0)
    return set_error(MPGPU_EPARAM, "bad chunk import");
  if (cudaSetDevice(s->device) != cudaSuccess) {
    cudaGetLastError();
    return set_error(MPGPU_ECUDA, "cudaSetDevice failed");
  }
  CUresult r = drv().import_handle(&s->h[chunk], (void*)(uintptr_t)fd,
                                   CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    s->h[chunk] = 0;
    return cu_fail(r, "cuMemImportFromShareableHandle");
  }
  return MPGPU_OK;
}

mpgpu_status mpgpu_stripes_map(mpgpu_stripes* s, void** d_base) {
  if (!s || !d_base) return set_error(MPGPU_EPARAM, "null argument");
  const Driver& d = drv();
  if (s->base) {
    *d_base = (void*)s->base;
    return MPGPU_OK;
  }
  for (auto h : s->h)
    if (!h) return set_error(MPGPU_EPARAM, "striped region: a chunk was never imported");
  if (cudaSetDevice(s->device) != cudaSuccess) {
    cudaGetLastError();
    return set_error(MPGPU_ECUDA, "cudaSetDevice failed");
  }
  const size_t total = s->h.size() * s->chunk;
  if (CUresult r = d.reserve(&s->base, total, s->chunk, 0, 0); r != CUDA_SUCCESS) {
    s->base = 0;
    return cu_fail(r, "cuMemAddressReserve");
  }
  for (size_t c = 0; c < s->h.size(); ++c) {
    if (CUresult r = d.map(s->base + c * s->chunk, s->chunk, 0, s->h[c], 0); r != CUDA_SUCCESS) {
      s->mapped = c;
      return cu_fail(r, "cuMemMap");
    }
  }
  s->mapped = s->h.size();
  std::vector<CUmemAccessDesc> acc(s->access_devs.size());
  for (size_t q = 0; q < acc.size(); ++q) {
    acc[q].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[q].location.id = s->access_devs[q];
    acc[q].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  if (CUresult r = d.set_access(s->base, total, acc.data(), acc.size()); r != CUDA_SUCCESS)
    return cu_fail(r, "cuMemSetAccess");
  *d_base = (void*)s->base;
  return MPGPU_OK;
}

void mpgpu_stripes_destroy(mpgpu_stripes* s) {
  if (!s) return;
  const Driver& d = drv();
  if (d.ok) {
    cudaSetDevice(s->device);
    cudaDeviceSynchronize();
    if (s->base) {
      for (size_t c = 0; c < s->mapped; ++c) d.unmap(s->base + c * s->chunk, s->chunk);
      d.addr_free(s->base, s->h.size() * s->chunk);
    }
    for (auto h : s->h)
      if (h) d.release(h);
  }
  cudaGetLastError();
  delete s;
}

int32_t mpgpu_device_pci_bus_id(int32_t device, char* buf, int32_t len) {
  if (!buf || len < 16) return -1;
  if (cudaDeviceGetPCIBusId(buf, len, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return 0;
}

int32_t mpgpu_peer_atomics(int32_t device, const char* peer_pci_bus_id) {
  if (!peer_pci_bus_id) return -1;
  int peer = -1;
  if (cudaDeviceGetByPCIBusId(&peer, peer_pci_bus_id) != cudaSuccess) {
    cudaGetLastError();
    return -1;  // the peer is not visible to this process: cannot be verified
  }
  if (peer == device) return 1;  // same GPU (functional multi-process runs)
  int ok = 0;
  if (cudaDeviceGetP2PAttribute(&ok, cudaDevP2PAttrNativeAtomicSupported, device, peer) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  int access = 0;
  if (cudaDeviceGetP2PAttribute(&access, cudaDevP2PAttrAccessSupported, device, peer) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return ok && access ? 1 : 0;
}

}  // extern "C"
