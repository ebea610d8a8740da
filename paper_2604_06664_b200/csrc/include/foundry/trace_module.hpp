// Real sm_100a device binaries for cataloged kernels (SAVE/pack side).
//
// The reference catalogs simulated FNDB images whose hidden pointer offsets
// only its simulated driver knows (kernel_image.hpp:23-26). On B200 every
// cataloged binary becomes a real cubin with one .entry per entrypoint — exact
// reference name, exact argument-buffer size — whose body (trace_body.cu) is
// the on-device replay check. LOAD restores them with cuLibraryLoadData
// (SURVEY §8(a) A3), mirroring restore_binaries (binary_catalog.cpp:200-227).
#pragma once

#include <cstdint>
#include <filesystem>
#include <string>
#include <vector>

#include "foundry/archive.hpp"

namespace foundry {

// PTX text of the module for one cataloged binary.
std::string trace_module_ptx(const KernelImage& image, uint32_t binary_ordinal,
                             bool needs_device_init);
// ptxas -arch=sm_100a of PTX text -> cubin bytes.
std::vector<uint8_t> compile_ptx_to_cubin(const std::string& ptx);
// Writes binaries/<hash>.sm_100a.cubin for every cataloged binary and records
// their digests in the manifest.
void write_trace_cubins(const std::filesystem::path& archive, unsigned threads = 0);

// The embedded device body (generated at build time from kernels/trace_body.cu).
const char* trace_body_ptx();

}  // namespace foundry
