// A group of processes on one node sharing device buffers through CUDA IPC,
// synchronised on the host: a POSIX shared-memory segment holds one fixed-size
// slot per rank (IPC memory handles and the geometry a neighbour needs) and a
// sense-reversing barrier. An exchange built on it is: stream sync, barrier,
// cudaMemcpyAsync pulls from the neighbours' mapped buffers, stream sync,
// barrier. No kernel ever waits on another rank, so the ranks may share one
// GPU (the multi-process tests do; B200_PROFILING.md's Xid 109 hazard is about
// kernels spinning on each other).
#pragma once
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.hpp"

namespace sfeec_b200 {

class IpcGroup {
 public:
  // id128: 16 random bytes shared by the ranks (sfeec_ipc_unique_id); every
  // rank owns `slot_bytes` of the segment
  IpcGroup(const char* prefix, const void* id128, int rank, int nranks, size_t slot_bytes)
      : rank_(rank), nranks_(nranks), slot_(slot_bytes) {
    char hex[40];
    const unsigned char* b = (const unsigned char*)id128;
    for (int i = 0; i < 16; ++i) std::snprintf(hex + 2 * i, 3, "%02x", b[i]);
    name_ = std::string("/") + prefix + "_" + hex;
    bytes_ = sizeof(Head) + slot_ * (size_t)nranks;
    int fd = -1;
    const auto t0 = std::chrono::steady_clock::now();
    auto late = [&] { return std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120); };
    if (rank == 0) {
      fd = shm_open(name_.c_str(), O_CREAT | O_RDWR, 0600);
      require(fd >= 0, "IPC group: shm_open failed");
      require(ftruncate(fd, (off_t)bytes_) == 0, "IPC group: ftruncate failed");
    } else {
      while ((fd = shm_open(name_.c_str(), O_RDWR, 0600)) < 0) {
        require(!late(), "IPC group: rank 0's segment did not appear");
        usleep(1000);
      }
      while (lseek(fd, 0, SEEK_END) < (off_t)bytes_) {
        require(!late(), "IPC group: segment not sized");
        usleep(1000);
      }
    }
    void* m = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    require(m != MAP_FAILED, "IPC group: mmap failed");
    head_ = (Head*)m;
    if (rank == 0) {
      head_->count.store(0);
      head_->gen.store(0);
      head_->magic.store(kMagic, std::memory_order_release);
    } else {
      while (head_->magic.load(std::memory_order_acquire) != kMagic) {
        require(!late(), "IPC group: segment not initialised");
        usleep(1000);
      }
    }
  }
  ~IpcGroup() {
    if (head_) munmap(head_, bytes_);
  }
  IpcGroup(const IpcGroup&) = delete;
  IpcGroup& operator=(const IpcGroup&) = delete;

  void* slot(int q) const { return (char*)head_ + sizeof(Head) + slot_ * (size_t)q; }
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  // call once every rank has mapped the segment (after a barrier)
  void unlink_name() {
    if (rank_ == 0) shm_unlink(name_.c_str());
  }
  void barrier() {
    const int g = head_->gen.load(std::memory_order_acquire);
    if (head_->count.fetch_add(1, std::memory_order_acq_rel) + 1 == nranks_) {
      head_->count.store(0, std::memory_order_relaxed);
      head_->gen.fetch_add(1, std::memory_order_acq_rel);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    while (head_->gen.load(std::memory_order_acquire) == g) {
      require(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(300),
              "IPC group: barrier timed out (a rank died?)");
      sched_yield();
    }
  }

 private:
  static constexpr int kMagic = 0x5feec1;
  struct Head {
    std::atomic<int> magic, count, gen;
    int pad;
  };
  int rank_, nranks_;
  size_t slot_, bytes_ = 0;
  std::string name_;
  Head* head_ = nullptr;
};

}  // namespace sfeec_b200
