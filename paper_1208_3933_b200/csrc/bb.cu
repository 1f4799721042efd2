// bb.cu — device-resident B&B (placeholder until the expand/prune kernels land).
#include "fsp_internal.h"

extern "C" int fsp_bb_solve(const fsp_instance *, int32_t, int64_t, double, int32_t *, int32_t *,
                            fsp_bb_stats *)
{
    return fsp_fail(FSP_EINVAL, "not implemented");
}
extern "C" int fsp_bb_init(const fsp_instance *, int32_t, int32_t, int32_t, void **) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_step(void *, int32_t, void *) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_ub_ptr(void *, int64_t **) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_ub_sync(void *, void *) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_pool_size(void *, int64_t *) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int64_t fsp_bb_node_bytes(void *) { return 0; }
extern "C" int fsp_bb_export(void *, int64_t, void *, int64_t *) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_import(void *, const void *, int64_t) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_result(void *, int32_t *, int32_t *) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" int fsp_bb_get_stats(void *, fsp_bb_stats *) { return fsp_fail(FSP_EINVAL, "not implemented"); }
extern "C" void fsp_bb_free(void *) {}
