// Collectives of the sharded path (nsp_comm.cu).
#pragma once
#include "nsp_internal.h"

namespace nspi {
nsp_status comm_init(nsp_ctx* c);                                 // after the local setup; collective
nsp_status comm_allreduce(nsp_ctx* c, double* buf, size_t count);  // in-place sum on c->stream
void comm_free(nsp_ctx* c);
}  // namespace nspi
