// corpus.hpp -- the host-side network a corpus handle owns (asnn_dev.h
// asnn_corpus): generators (netgen.cpp) and the device parser (parse.cu).
#pragma once

#include <cstdint>
#include <vector>

struct asnn_corpus {
    std::vector<std::uint32_t> nodes, inputs, outputs, src, dst;
    std::vector<float> w;
};
