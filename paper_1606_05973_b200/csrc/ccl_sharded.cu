// ccl_sharded.cu -- NCCL bootstrap helpers for ccl_label_sharded (ccl_bands.cu).
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include "ccl.h"
#include "ccl_internal.cuh"

extern "C" {

ccl_status ccl_nccl_get_unique_id(uint8_t id_out[128]) {
    if (!id_out) return CCL_INVALID_ARGUMENT;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return CCL_NCCL_ERROR;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id_out, &id, sizeof(id));
    return CCL_OK;
}

ccl_status ccl_nccl_comm_create(const uint8_t id[128], int nranks, int rank,
                                ccl_nccl_comm_t *comm_out) {
    if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return CCL_INVALID_ARGUMENT;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c;
    if (ncclCommInitRank(&c, nranks, uid, rank) != ncclSuccess) return CCL_NCCL_ERROR;
    *comm_out = reinterpret_cast<ccl_nccl_comm_t>(c);
    return CCL_OK;
}

ccl_status ccl_nccl_comm_destroy(ccl_nccl_comm_t comm) {
    if (!comm) return CCL_INVALID_ARGUMENT;
    return ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)) == ncclSuccess ? CCL_OK
                                                                              : CCL_NCCL_ERROR;
}

}  // extern "C"
