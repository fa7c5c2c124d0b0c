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
#include <chrono>
#include <stdexcept>
#include <cstring>
#include <string>
#include <thread>

constexpr int kCommMaxRanks = 16;
constexpr int kCommRedSlots = 64;
constexpr int kCommBlob = 4096;

constexpr int kCommReady = 0x45484d47;  // "EHMG"

struct CommShm {
  std::atomic<int> ready;     // kCommReady once rank 0 initialised this segment
  std::atomic<int> failed;    // a rank gave up: every barrier throws, close() skips its barrier
  std::atomic<int> arrived;
  std::atomic<int> sense;
  std::atomic<int> attached;
  std::atomic<long long> xseq[kCommMaxRanks];  // halo exchanges whose event record each rank has enqueued
  double red[kCommMaxRanks][kCommRedSlots];
  unsigned char blob[kCommMaxRanks][kCommBlob];
};

struct NodeComm {
  int rank = 0, n = 1;
  std::string name;
  CommShm* shm = nullptr;
  int local_sense = 0;
  double timeout_s = 120.0;

  static CommShm* map_fd(int fd) {
    void* p = mmap(nullptr, sizeof(CommShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    return p == MAP_FAILED ? nullptr : static_cast<CommShm*>(p);
  }
  void deadline_check(const std::chrono::steady_clock::time_point& t0, const char* what) {
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
      throw std::runtime_error(std::string("comm: timed out waiting for ") + what + " (" + name + ")");
  }

  // Rank 0 invalidates any segment a crashed job left under this name
  // (ready = 0, failed = 1), unlinks it and creates a fresh one exclusively;
  // the other ranks attach only to a segment whose ready flag is set and
  // start over if it is invalidated while they wait for the others.
  void open(const std::string& job, int r, int nranks) {
    if (nranks < 1 || nranks > kCommMaxRanks) throw std::runtime_error("comm: 1..16 ranks");
    if (r < 0 || r >= nranks) throw std::runtime_error("comm: rank out of range");
    rank = r;
    n = nranks;
    name = "/ehmg_" + job;
    const auto t0 = std::chrono::steady_clock::now();
    if (rank == 0) {
      int ofd = shm_open(name.c_str(), O_RDWR, 0600);
      if (ofd >= 0) {
        struct stat st;
        if (fstat(ofd, &st) == 0 && st.st_size >= (off_t)sizeof(CommShm)) {
          if (CommShm* old = map_fd(ofd)) {
            old->ready.store(0);
            old->failed.store(1);
            munmap(old, sizeof(CommShm));
          }
        } else {
          ::close(ofd);
        }
        shm_unlink(name.c_str());
      }
      int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) throw std::runtime_error("comm: shm_open failed for " + name);
      if (ftruncate(fd, sizeof(CommShm)) != 0) {
        ::close(fd);
        shm_unlink(name.c_str());
        throw std::runtime_error("comm: ftruncate failed");
      }
      shm = map_fd(fd);
      if (!shm) throw std::runtime_error("comm: mmap failed");
      shm->failed.store(0);
      for (int r = 0; r < kCommMaxRanks; ++r) shm->xseq[r].store(0);
      shm->arrived.store(0);
      shm->sense.store(0);
      shm->attached.store(1);
      shm->ready.store(kCommReady);
      while (shm->attached.load() < n) {
        if (shm->failed.load()) throw std::runtime_error("comm: a peer rank failed during open");
        deadline_check(t0, "ranks to attach");
        std::this_thread::yield();
      }
      return;
    }
    for (;;) {
      deadline_check(t0, "rank 0's segment");
      int fd = shm_open(name.c_str(), O_RDWR, 0600);
      if (fd < 0) {
        std::this_thread::yield();
        continue;
      }
      struct stat st;
      if (fstat(fd, &st) != 0 || st.st_size < (off_t)sizeof(CommShm)) {
        ::close(fd);
        std::this_thread::yield();
        continue;
      }
      CommShm* p = map_fd(fd);
      if (!p) throw std::runtime_error("comm: mmap failed");
      if (p->ready.load() != kCommReady || p->failed.load()) {
        munmap(p, sizeof(CommShm));
        std::this_thread::yield();
        continue;
      }
      p->attached.fetch_add(1);
      bool stale = false;
      while (p->attached.load() < n) {
        if (p->ready.load() != kCommReady) { stale = true; break; }
        if (p->failed.load()) {
          munmap(p, sizeof(CommShm));
          throw std::runtime_error("comm: a peer rank failed during open");
        }
        deadline_check(t0, "ranks to attach");
        std::this_thread::yield();
      }
      if (stale) {  // attached to a segment rank 0 has just replaced
        munmap(p, sizeof(CommShm));
        continue;
      }
      shm = p;
      return;
    }
  }
  // Mark the job failed: peers blocked in a barrier throw instead of pairing
  // this rank's teardown barrier with their exchange barriers.
  void fail() {
    if (shm) shm->failed.store(1);
  }
  void close() {
    if (!shm) return;
    if (!shm->failed.load()) {
      try {
        barrier();
      } catch (...) {
      }
    }
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
      while (shm->sense.load() != local_sense) {
        if (shm->failed.load()) throw std::runtime_error("comm: a peer rank failed");
        std::this_thread::yield();
      }
    }
  }
  // Enqueue-order handshake of the halo exchanges: a rank publishes that it
  // has enqueued the event record of its exchange number `seq`; a neighbour
  // waits for that (host spin, no GPU drain) before it makes its stream wait
  // on the event -- the GPU streams then order the exchange among themselves.
  void publish(long long seq) {
    if (shm) shm->xseq[rank].store(seq, std::memory_order_release);
  }
  void wait_for(int r, long long seq) {
    if (n == 1) return;
    while (shm->xseq[r].load(std::memory_order_acquire) < seq) {
      if (shm->failed.load()) throw std::runtime_error("comm: a peer rank failed");
      std::this_thread::yield();
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
