// okg_cusolver.h -- the dense SPD factorisation used ONCE at setup for a large
// coarsest multigrid level (nc > 2000, e.g. 26^3 = 17,576 at 400^3 / 800^3),
// where the host Cholesky + inverse (okg_tables.cpp, O(nc^3) on one core) would
// take hours.  It replaces the reference's CholeskyFactor construction
// (multigrid.hpp:82-83, dense.hpp:175-195); the per-V-cycle coarse solve stays
// our own kernel (k_coarse_gemv).  cuSOLVER is resolved at run time (dlopen of
// libcusolver.so.11), like NCCL in okg_nccl.h, so libokg.so has no link-time
// dependency on it and small hierarchies never load it.
#pragma once
#include <cusolverDn.h>
#include <dlfcn.h>

#include <string>
#include <type_traits>

namespace okg {

struct CusolverApi {
  bool ok = false;
  cusolverStatus_t (*Create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*Destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*SetStream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*PotrfBufferSize)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*Potrf)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*PotriBufferSize)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*Potri)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*) = nullptr;
};

// nullptr + message when cuSOLVER cannot be loaded
inline const CusolverApi* cusolver_api(std::string* why) {
  static CusolverApi api;
  static std::string err;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = nullptr;
    for (const char* name : {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!h) {
      const char* e = dlerror();
      err = std::string("dlopen(libcusolver.so.11): ") + (e ? e : "not found");
    } else {
      bool all = true;
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        if (!fp) {
          all = false;
          err = std::string("libcusolver lacks ") + name;
        }
      };
      sym(api.Create, "cusolverDnCreate");
      sym(api.Destroy, "cusolverDnDestroy");
      sym(api.SetStream, "cusolverDnSetStream");
      sym(api.PotrfBufferSize, "cusolverDnDpotrf_bufferSize");
      sym(api.Potrf, "cusolverDnDpotrf");
      sym(api.PotriBufferSize, "cusolverDnDpotri_bufferSize");
      sym(api.Potri, "cusolverDnDpotri");
      api.ok = all;
    }
  }
  if (!api.ok && why) *why = err;
  return api.ok ? &api : nullptr;
}

}  // namespace okg
