// ehmg_comm.cuh -- single-node multi-process communicator for the z-slab
// path: one process per GPU, device buffers shared through CUDA IPC (peer
// pointers; copies between GPUs go over NVLink/NVSwitch), host-side
// synchronisation through a POSIX shared-memory segment:
//   * barrier()        sense-reversing barrier on lock-free atomics;
//   * allreduce(v, k)  small double vectors, summed in rank order on every
//                      rank (deterministic: identical results everywhere);
//   * exchange_blob()  all-gather of small byte blobs (IPC handles, sizes).
// The GPU work of a rank is synchronised with its stream before each barrier,
// so peer copies never race with kernels of another process (no device-side
// spinning across processes).
#pragma once

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cstring>
#include <string>
#include <thread>

constexpr int kCommMaxRanks = 16;
constexpr int kCommRedSlots = 64;
constexpr int kCommBlob = 4096;

struct CommShm {
  std::atomic<int> arrived;
  std::atomic<int> sense;
  std::atomic<int> attached;
  double red[kCommMaxRanks][kCommRedSlots];
  unsigned char blob[kCommMaxRanks][kCommBlob];
};

struct NodeComm {
  int rank = 0, n = 1;
  std::string name;
  CommShm* shm = nullptr;
  int local_sense = 0;

  void open(const std::string& job, int r, int nranks) {
    if (nranks < 1 || nranks > kCommMaxRanks) throw std::runtime_error("comm: 1..16 ranks");
    rank = r;
    n = nranks;
    name = "/ehmg_" + job;
    int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("comm: shm_open failed for " + name);
    if (ftruncate(fd, sizeof(CommShm)) != 0) {
      ::close(fd);
      throw std::runtime_error("comm: ftruncate failed");
    }
    void* p = mmap(nullptr, sizeof(CommShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    if (p == MAP_FAILED) throw std::runtime_error("comm: mmap failed");
    shm = static_cast<CommShm*>(p);
    // a fresh segment is zero-filled: arrived = sense = attached = 0
    shm->attached.fetch_add(1);
    while (shm->attached.load() < n) std::this_thread::yield();
  }
  void close() {
    if (!shm) return;
    barrier();
    const int left = shm->attached.fetch_sub(1) - 1;
    munmap(shm, sizeof(CommShm));
    shm = nullptr;
    if (left == 0) shm_unlink(name.c_str());
  }
  ~NodeComm() {
    if (shm) munmap(shm, sizeof(CommShm));
  }

  void barrier() {
    if (n == 1) return;
    local_sense ^= 1;
    if (shm->arrived.fetch_add(1) + 1 == n) {
      shm->arrived.store(0);
      shm->sense.store(local_sense);
    } else {
      while (shm->sense.load() != local_sense) std::this_thread::yield();
    }
  }
  // v[0..k) <- sum over ranks (rank order), identical on every rank
  void allreduce(double* v, int k) {
    if (n == 1) return;
    if (k > kCommRedSlots) throw std::runtime_error("comm: allreduce too wide");
    std::memcpy(shm->red[rank], v, sizeof(double) * k);
    barrier();
    for (int i = 0; i < k; ++i) {
      double s = 0;
      for (int r = 0; r < n; ++r) s += shm->red[r][i];
      v[i] = s;
    }
    barrier();
  }
  // every rank contributes `bytes` and receives all ranks' blobs
  void exchange_blob(const void* mine, int bytes, void* all) {
    if (bytes > kCommBlob) throw std::runtime_error("comm: blob too large");
    std::memcpy(shm->blob[rank], mine, bytes);
    barrier();
    for (int r = 0; r < n; ++r) std::memcpy(static_cast<char*>(all) + (size_t)r * bytes, shm->blob[r], bytes);
    barrier();
  }
};
