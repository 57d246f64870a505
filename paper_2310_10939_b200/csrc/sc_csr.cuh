// sc_csr.cuh -- a CSR generated and kept on one GPU (sc_generate*.cu), the input of
// sc_graph_create_from_csr without a host round trip of the column / weight arrays.
#pragma once

#include <stdint.h>

struct sc_csr {
    int device = 0;
    int64_t n = 0;              // vertices kept
    int64_t n_gen = 0;          // vertices generated
    int64_t nnz = 0;
    int64_t *d_rp = nullptr;
    int32_t *d_col = nullptr;
    double *d_deg = nullptr;
    double *d_val = nullptr;    // nullptr: unit weights
    int32_t *d_orig = nullptr;  // original (generated) id of every kept vertex
};
