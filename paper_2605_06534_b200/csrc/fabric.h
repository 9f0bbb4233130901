// fabric.h -- how the ranks of one sync see each other's device memory.
//
// The P2P exchange needs, per rank, the mailbox and receive regions of every
// other rank (and their serving arenas, for direct dense boxes) mapped into
// its own address space.  Two fabrics provide that:
//   * NcclFabric: one process per GPU (the deployment, bench.py): CUDA IPC
//     handles all-gathered over the NCCL communicator;
//   * GroupFabric: every rank an engine of ONE process (ws_group, e.g. all
//     ranks of a layout on one GPU for parity tests): pointers are shared
//     directly through a host barrier, one host thread per rank.
// Every call is collective over the ranks.
#pragma once

#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "wsync.h"

namespace wsync {

class Fabric {
 public:
  Fabric(int world, int rank) : world_(world), rank_(rank) {}
  virtual ~Fabric() = default;
  int world() const { return world_; }
  int rank() const { return rank_; }
  // Every rank passes a pointer into one of its device allocations (null:
  // nothing to share); (*out)[g] is rank g's pointer as usable here
  // ((*out)[rank] = p).  Fails on every rank if any mapping fails.
  virtual ws_status share(void* p, std::vector<void*>* out) = 0;
  // Releases a pointer share() returned for another rank.
  virtual void release(void* p) = 0;
  // *v = min over ranks of *v (also a barrier).
  virtual ws_status all_min(int* v) = 0;

 protected:
  int world_, rank_;
};

class NcclFabric : public Fabric {
 public:
  NcclFabric(int world, int rank, ncclComm_t comm) : Fabric(world, rank), comm_(comm) {}
  ws_status share(void* p, std::vector<void*>* out) override;
  void release(void* p) override;
  ws_status all_min(int* v) override;

 private:
  ncclComm_t comm_;
};

// State shared by the ranks of one process-local group.
struct GroupShared {
  explicit GroupShared(int world) : world(world), slots(world), ints(world) {}
  void barrier();
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned generation = 0;
  std::vector<void*> slots;
  std::vector<int> ints;
};

class GroupFabric : public Fabric {
 public:
  GroupFabric(int world, int rank, GroupShared* g) : Fabric(world, rank), g_(g) {}
  ws_status share(void* p, std::vector<void*>* out) override;
  void release(void*) override {}
  ws_status all_min(int* v) override;

 private:
  GroupShared* g_;
};

}  // namespace wsync
