// Kernel-id dispatch for the map/life kernels behind the run API.
#include "sk_internal.h"

namespace sk {

const KernelOps* u8_ops();
const KernelOps* amf_ops();

const KernelOps* life_ops() { return u8_ops(); }

}  // namespace sk
