// hash_tiled.cu -- WMH_ALGO_TILED (placeholder until the tiled kernel lands).
#include "common.cuh"

namespace wmh {

wmh_status launch_hash_tiled(const HashArgs &a, bool *handled) {
    (void)a;
    *handled = false;
    return WMH_OK;
}

}  // namespace wmh
