// NCCL entry points resolved at run time. The process usually already holds
// torch's libnccl.so.2 (torch.distributed plumbing); linking a second copy at
// build time would make the two fight over the SONAME, so the library binds
// to whichever libnccl.so.2 is loaded (dlopen RTLD_NOLOAD), else loads the
// system one. Types come from the NCCL header; no symbol is linked.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "common.hpp"

namespace sfeec_b200 {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;

  static const Nccl& get() {
    static Nccl n = [] {
      Nccl r;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) throw Error(SFEEC_ENCCL, "libnccl.so.2 not found");
#define SFEEC_NCCL_SYM(field, name)                                          \
  r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, #name));            \
  if (!r.field) throw Error(SFEEC_ENCCL, "NCCL symbol " #name " missing");
      SFEEC_NCCL_SYM(get_unique_id, ncclGetUniqueId)
      SFEEC_NCCL_SYM(comm_init_rank, ncclCommInitRank)
      SFEEC_NCCL_SYM(comm_destroy, ncclCommDestroy)
      SFEEC_NCCL_SYM(send, ncclSend)
      SFEEC_NCCL_SYM(recv, ncclRecv)
      SFEEC_NCCL_SYM(all_reduce, ncclAllReduce)
      SFEEC_NCCL_SYM(group_start, ncclGroupStart)
      SFEEC_NCCL_SYM(group_end, ncclGroupEnd)
      SFEEC_NCCL_SYM(error_string, ncclGetErrorString)
#undef SFEEC_NCCL_SYM
      return r;
    }();
    return n;
  }

  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw Error(SFEEC_ENCCL, std::string(what) + ": " + error_string(r));
  }
};

}  // namespace sfeec_b200
