// NCCL communicator handle (one rank per GPU): C1 model averaging
// (gnn.cu) and the sharded feature-store refresh (features.cu).
#pragma once

#include <nccl.h>

#include "common.hpp"

struct catgnn_comm_s {
  ncclComm_t comm = nullptr;
  catgnn_ctx ctx = nullptr;
  int nranks = 1, rank = 0;
};
