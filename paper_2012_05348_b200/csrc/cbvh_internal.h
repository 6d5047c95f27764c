// cbvh_internal.h — shared between builder.cpp and cbvh_device.cu (product
// code only; the oracle never includes this).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/cbvh.h"

namespace cbvh {

// Records `msg` as the calling thread's last error and returns `code`.
int set_error(int code, const char* msg);

int build_blob(const cbvh_mesh* mesh, int branching, int bits, const cbvh_build_opts* opts,
               std::vector<uint8_t>& out);

// Parse + validate the fixed 256-byte blob header.
int parse_header(const uint8_t* p, size_t bytes, cbvh_header* h);

// Blob topology word:
//   leaf:     bit 31 = 1, bits 29..30 = ntri - 1, bits 0..28 = first triangle
//   internal: bit 31 = 0, bits 28..30 = nchild - 1, bits 0..27 = first child
constexpr uint32_t kLeafBit = 0x80000000u;
// topology word of a padding slot of an aligned treelet (never referenced)
constexpr uint32_t kPadTopo = 0x7FFFFFFFu;

}  // namespace cbvh
