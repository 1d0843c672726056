// Shared plumbing for the C ABI: error codes, thread-local message, CUDA checks.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "sfeec_b200.h"

namespace sfeec_b200 {

// Mirrors the reference error contract (core.hpp:70-72): InvalidParameter ->
// SFEEC_EINVAL, runtime failures -> the specific code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);

// Boolean environment switch: unset -> dflt, "0" -> false, anything else true.
// Read once when a handle is created, never per launch.
inline bool env_flag(const char* name, bool dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) != 0 : dflt;
}

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(SFEEC_EINVAL, msg);
}

// Runs f(), mapping exceptions to the ABI's integer codes.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return SFEEC_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    return SFEEC_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SFEEC_ECUDA;
  }
}

// Host CSR with int64 row pointers (the device layouts are built from it).
struct HostCSR {
  int64_t rows = 0, cols = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col_idx;
  std::vector<double> val;
  int64_t nnz() const { return (int64_t)col_idx.size(); }
};

HostCSR csr_from_view(const sfeec_csr& v);
void csr_validate(const sfeec_csr& v, const char* name);
HostCSR csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int32_t* r,
                          const int32_t* c, const double* v);
HostCSR csr_symmetric_part(const HostCSR& q);
HostCSR csr_transpose(const HostCSR& a);
void csr_to_owned(HostCSR&& m, sfeec_csr_owned* out);

}  // namespace sfeec_b200
