// Intra-node process group: shared-memory barrier + allgather (see tmgx_node.hpp).
#include "tmgx_node.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "tmg_grid.hpp"

namespace tmgx {

struct NodeGroup::Shm {
  alignas(64) std::atomic<std::uint64_t> count;  // arrivals in the current generation
  alignas(64) std::atomic<std::uint64_t> gen;    // completed barriers
  alignas(64) std::atomic<int> aborted;
  alignas(64) std::atomic<int> detached;
  std::uint64_t len[kMaxProcs];
  char data[kMaxProcs][kSlotBytes];
};

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

NodeGroup::NodeGroup(const std::string& job, int nproc, int proc) : P(nproc), me(proc) {
  if (P < 1 || P > kMaxProcs || me < 0 || me >= P) throw tmg::ConfigError("node group: bad process count / index");
  if (job.empty() || job.size() > 200 || job.find('/') != std::string::npos)
    throw tmg::ConfigError("node group: job token must be a non-empty name without '/'");
  if (const char* e = std::getenv("TMGX_BARRIER_TIMEOUT")) timeout_s_ = std::atof(e);
  name_ = "/tmgx_" + job;
  // every process creates-or-opens the segment; ftruncate to the same size is idempotent and
  // a fresh segment is zero-filled, which is the initial state of the barrier
  const int fd = shm_open(name_.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) throw tmg::CudaError("node group: shm_open " + name_ + " failed");
  if (ftruncate(fd, sizeof(Shm)) != 0) {
    close(fd);
    throw tmg::CudaError("node group: ftruncate failed");
  }
  void* p = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw tmg::CudaError("node group: mmap failed");
  shm_ = static_cast<Shm*>(p);
  barrier();  // everyone attached
}

NodeGroup::~NodeGroup() {
  if (!shm_) return;
  // the last process to leave removes the name (a crashed peer leaves it: tokens are per job)
  if (shm_->detached.fetch_add(1) + 1 == P) shm_unlink(name_.c_str());
  munmap(shm_, sizeof(Shm));
}

void NodeGroup::abort() {
  if (shm_) shm_->aborted.store(1);
  failed_.store(true);
}

// Wait until the generation observed on arrival has completed. Spins briefly, then yields:
// with several processes per GPU (tests) the host cores are shared with the peers' drivers.
bool NodeGroup::wait_gen(double timeout_s) {
  const std::uint64_t g = shm_->gen.load(std::memory_order_acquire);
  if (shm_->count.fetch_add(1, std::memory_order_acq_rel) + 1 == (std::uint64_t)P) {
    shm_->count.store(0, std::memory_order_relaxed);
    shm_->gen.fetch_add(1, std::memory_order_release);
    return true;
  }
  const double t0 = now_s();
  for (long spin = 0; shm_->gen.load(std::memory_order_acquire) == g; ++spin) {
    if (shm_->aborted.load(std::memory_order_relaxed)) return false;
    if (spin < 2000) continue;
    if (spin < 20000) {
      sched_yield();
      continue;
    }
    const timespec ts{0, 20000};
    nanosleep(&ts, nullptr);
    if ((spin & 255) == 0 && now_s() - t0 > timeout_s) {
      shm_->aborted.store(1);
      return false;
    }
  }
  return true;
}

void NodeGroup::barrier(double timeout_s) {
  if (!wait_gen(timeout_s > 0 ? timeout_s : timeout_s_)) {
    failed_.store(true);
    throw tmg::CudaError("node group: barrier timed out or a peer process aborted");
  }
}

std::vector<std::string> NodeGroup::allgather(const std::string& mine) {
  if (mine.size() > kSlotBytes) throw tmg::Error("node group: allgather payload too large");
  barrier();  // previous readers of the board are done
  std::memcpy(shm_->data[me], mine.data(), mine.size());
  shm_->len[me] = mine.size();
  barrier();
  std::vector<std::string> all((size_t)P);
  for (int q = 0; q < P; ++q) all[(size_t)q].assign(shm_->data[q], shm_->len[q]);
  return all;
}

void CUDART_CB NodeGroup::host_barrier(void* self) {
  auto* g = static_cast<NodeGroup*>(self);
  if (g->failed_.load()) return;
  if (!g->wait_gen(g->timeout_s_)) g->failed_.store(true);
}

void NodeGroup::enqueue_barrier(cudaStream_t s) {
  const cudaError_t e = cudaLaunchHostFunc(s, &NodeGroup::host_barrier, this);
  if (e != cudaSuccess) throw tmg::CudaError(std::string("cudaLaunchHostFunc: ") + cudaGetErrorString(e));
}

}  // namespace tmgx
