// corpus.hpp -- the host-side network a corpus handle owns (asnn_dev.h
// asnn_corpus): generators (netgen.cpp) and the device parser (parse.cu).
#pragma once

#include <cstdint>
#include <vector>

struct asnn_corpus {
    std::vector<std::uint32_t> nodes, inputs, outputs, src, dst;
    std::vector<float> w;
};

// Config 4's band boundaries and Pareto scale (netgen.cpp; shared with gen.cu).
double powerlaw_xm(uint32_t n_nodes, uint32_t n_in, uint32_t n_out, uint64_t target_edges, double alpha);
std::vector<std::uint32_t> powerlaw_band_starts(uint32_t n_nodes, uint32_t bands, uint32_t n_in, uint32_t n_out);
