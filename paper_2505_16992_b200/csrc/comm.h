// comm.h -- host side of the slab communicator (see comm.cuh).
#pragma once

#include <cstdint>

#include "comm.cuh"

namespace pf {

struct CommHost {
  int rank = 0, world = 1;
  int64_t plane = 0, nxl = 0;
  void *sym = nullptr;           // own symmetric buffer
  int64_t sym_bytes = 0;
  int64_t spec_off = 0, spec_bytes = 0;
  CommDev *dev = nullptr;        // device copy of `host`
  CommDev host{};
  bool ipc_opened[kMaxRanks] = {};
  void *pinned = nullptr;        // staging for CommDev reads
};

}  // namespace pf
