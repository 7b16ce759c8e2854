// Intra-node process group for the one-process-per-GPU runs (the spawn_world / Comm analog,
// comm.hpp:75-207, for processes instead of rank threads).
//
// A POSIX shared-memory segment named after a job token carries a sense-counting barrier and an
// allgather board. The solver uses it to exchange CUDA IPC handles of its receive mailboxes once
// at setup; afterwards every data movement is a kernel storing straight into a peer's mailbox
// (NVLink / NVSwitch peer memory, or the same HBM when the processes share a GPU), and the only
// synchronisation is a host barrier enqueued in the stream (cudaLaunchHostFunc, so it can be
// captured into a CUDA graph as a host node). No kernel ever waits on another process's kernel.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <string>
#include <vector>

namespace tmgx {

class NodeGroup {
 public:
  static constexpr int kMaxProcs = 64;
  static constexpr size_t kSlotBytes = 1 << 16;

  NodeGroup(const std::string& job, int nproc, int proc);
  ~NodeGroup();
  NodeGroup(const NodeGroup&) = delete;
  NodeGroup& operator=(const NodeGroup&) = delete;

  // host barrier over the group; throws tmg::CudaError on timeout or when a peer aborted
  void barrier(double timeout_s = -1.0);
  // every process contributes `mine` (<= kSlotBytes); returns all contributions by process
  std::vector<std::string> allgather(const std::string& mine);
  // stream-ordered barrier: the stream proceeds once every process's stream reached its barrier
  void enqueue_barrier(cudaStream_t s);
  // set when a stream barrier timed out (host callbacks cannot throw)
  bool failed() const { return failed_.load(); }
  void abort();

  const int P, me;

 private:
  struct Shm;
  Shm* shm_ = nullptr;
  std::string name_;
  std::atomic<bool> failed_{false};
  double timeout_s_ = 600.0;
  bool wait_gen(double timeout_s);
  static void CUDART_CB host_barrier(void* self);
};

}  // namespace tmgx
