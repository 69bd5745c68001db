// Temporary: kernels not yet implemented report SK_ERR_UNSUPPORTED.
#include "sk_internal.h"
namespace sk {
namespace {
int unsup(sk_run*) { set_error("kernel not implemented yet"); return SK_ERR_UNSUPPORTED; }
int unsup_l(sk_run*, const LoopCtl&, cudaStream_t) { return SK_ERR_UNSUPPORTED; }
void noop(sk_run*) {}
const KernelOps kU = {unsup, unsup_l, noop};
}
const KernelOps* life_ops() { return &kU; }
const KernelOps* restore_ops() { return &kU; }
const KernelOps* map_ops() { return &kU; }
}
extern "C" int sk_sobel_frames(const uint8_t*, int64_t, int64_t, uint8_t*, int64_t, int64_t, int32_t, int64_t, int64_t, int64_t*, void*) { return SK_ERR_UNSUPPORTED; }
extern "C" int sk_amf_frames(const uint8_t*, int64_t, int64_t, uint8_t*, int64_t, int64_t, int32_t, int64_t, int64_t, int32_t, int64_t*, void*) { return SK_ERR_UNSUPPORTED; }
