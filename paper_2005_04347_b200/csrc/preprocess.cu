// preprocess.cu -- device preprocessing (compute_required, segment, flatten).
#include "engine.hpp"

using namespace asnn_b200;

extern "C" {

int asnn_dev_compute_required(asnn_dev* dev, const asnn_network_desc*, uint8_t*) {
    return fail(dev, ASNN_E_UNAVAILABLE, "device preprocessing not built yet");
}

int asnn_dev_segment(asnn_dev* dev, const asnn_network_desc*, const uint8_t*, uint32_t*, uint32_t*) {
    return fail(dev, ASNN_E_UNAVAILABLE, "device preprocessing not built yet");
}

int asnn_dev_build_layout(asnn_dev* dev, const asnn_network_desc*, asnn_dev_layout**) {
    return fail(dev, ASNN_E_UNAVAILABLE, "device preprocessing not built yet");
}

int asnn_dev_build_population(asnn_dev* dev, uint32_t, const asnn_network_desc*, asnn_dev_layout**) {
    return fail(dev, ASNN_E_UNAVAILABLE, "device preprocessing not built yet");
}

}  // extern "C"
