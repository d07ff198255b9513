// comm.cu -- communicator and fused collectives (filled in next).
#include "uzip_internal.h"

extern "C" {
uzip_status_t uzip_comm_init(uzip_comm_t *, int, int, int, uzip_allgather_fn, void *, const uzip_config_t *) {
  return UZIP_ERR_NOT_IMPLEMENTED;
}
uzip_status_t uzip_comm_init_all(uzip_comm_t *, int, const int *, const uzip_config_t *) {
  return UZIP_ERR_NOT_IMPLEMENTED;
}
uzip_status_t uzip_comm_destroy(uzip_comm_t) { return UZIP_ERR_NOT_IMPLEMENTED; }
uzip_status_t uzip_send(const void *, size_t, uzip_dtype_t, int, uzip_comm_t, void *) {
  return UZIP_ERR_NOT_IMPLEMENTED;
}
uzip_status_t uzip_recv(void *, size_t, uzip_dtype_t, int, uzip_comm_t, void *) { return UZIP_ERR_NOT_IMPLEMENTED; }
uzip_status_t uzip_allgather(const void *, void *, size_t, uzip_dtype_t, uzip_comm_t, void *) {
  return UZIP_ERR_NOT_IMPLEMENTED;
}
uzip_status_t uzip_reduce_scatter(const void *, void *, size_t, uzip_dtype_t, uzip_op_t, uzip_comm_t, void *) {
  return UZIP_ERR_NOT_IMPLEMENTED;
}
uzip_status_t uzip_allreduce(const void *, void *, size_t, uzip_dtype_t, uzip_op_t, uzip_comm_t, void *) {
  return UZIP_ERR_NOT_IMPLEMENTED;
}
uzip_status_t uzip_comm_get_async_error(uzip_comm_t, uzip_status_t *) { return UZIP_ERR_NOT_IMPLEMENTED; }
uzip_status_t uzip_get_stats(uzip_comm_t, uzip_stats_t *) { return UZIP_ERR_NOT_IMPLEMENTED; }
}
