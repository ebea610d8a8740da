// SAVE-side archive writer for tier-R synthetic workloads (offline tooling;
// SURVEY §8(f3)). It emits the reference archive layout byte for byte
// (reference pipeline.cpp:249-405 + workload_gen.cpp:354-531 +
// rank_forge.cpp:97-130 + binary_catalog.cpp:108-183), so archives written
// here and by the reference build are interchangeable, and then (optionally)
// adds the B200 artefacts: templates.fdt (packed template store) and one
// sm_100a cubin per cataloged binary.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <optional>
#include <string>

#include "foundry/archive.hpp"
#include "foundry/workload.hpp"

namespace foundry {

// Expected per-node replay record (reference TraceRecord, sim_driver.hpp:62-73).
struct TraceRecord {
    uint32_t node_id = 0;
    NodeType type = NodeType::Empty;
    std::string kernel_name;
    Dim3 grid, block;
    uint32_t shared_mem_bytes = 0;
    uint64_t arg_digest = 0;
    std::vector<uint64_t> addresses;
    bool operator==(const TraceRecord&) const = default;
};

struct LaunchTrace {
    std::vector<TraceRecord> records;
    bool operator==(const LaunchTrace&) const = default;
    std::string to_text() const;  // reference sim_driver.cpp:21-38 format
};

std::string traces_to_text(const std::map<uint32_t, LaunchTrace>& traces);

struct SaveOptions {
    std::optional<uint64_t> base_address;
    bool b200_artifacts = true;  // templates.fdt + cubins (+ manifest digests)
    unsigned threads = 0;
};

struct SaveResult {
    std::filesystem::path archive_dir;
    Manifest manifest;
    std::map<uint32_t, LaunchTrace> traces;  // expected replay per batch (capture-time state)
    std::vector<AllocationRecord> allocation_records;
};

SaveResult save(const WorkloadSpec& spec, const std::filesystem::path& out,
                const SaveOptions& options = {});

// Adds the B200 artefacts to an existing (reference-written) archive:
// templates.fdt and binaries/<hash>.sm_100a.cubin, with manifest digests.
void pack_archive(const std::filesystem::path& archive, unsigned threads = 0);

}  // namespace foundry
