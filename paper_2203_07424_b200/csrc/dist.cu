// dist.cu — NCCL bootstrap for the sharded modes.  One process per GPU;
// the ncclUniqueId is created by rank 0 (rec_nccl_get_unique_id) and broadcast by the
// caller (torch.distributed is only the bootstrap plumbing).
#include <nccl.h>

#include "model.h"

namespace rec {

rec_status dist_init(rec_model_s* m, const void* nccl_id) {
  if (!nccl_id) {
    set_error("nccl_id must be non-null when world > 1 and shard != REPLICA");
    return REC_E_INVALID_ARG;
  }
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, m->world, id, m->rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank failed: %s", ncclGetErrorString(r));
    return REC_E_NCCL;
  }
  m->nccl_comm = comm;
  return REC_OK;
}

void dist_destroy(rec_model_s* m) {
  if (m && m->nccl_comm) {
    ncclCommDestroy(static_cast<ncclComm_t>(m->nccl_comm));
    m->nccl_comm = nullptr;
  }
}

}  // namespace rec

extern "C" {

int32_t rec_nccl_unique_id_size(void) { return static_cast<int32_t>(sizeof(ncclUniqueId)); }

rec_status rec_nccl_get_unique_id(void* out) {
  if (!out) {
    rec::set_error("out must be non-null");
    return REC_E_INVALID_ARG;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    rec::set_error("ncclGetUniqueId failed: %s", ncclGetErrorString(r));
    return REC_E_NCCL;
  }
  memcpy(out, &id, sizeof(id));
  return REC_OK;
}

}  // extern "C"
