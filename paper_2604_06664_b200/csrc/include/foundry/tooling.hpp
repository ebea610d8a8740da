// Offline tooling surface re-exported by the Python package:
// inspect / JSON graph documents / archive diff / bench. Output formats follow
// the reference (pipeline.cpp:586-744, graph_model.cpp:315-572, :847-929).
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <string>
#include <utility>

#include "foundry/graph_model.hpp"
#include "foundry/workload.hpp"

namespace foundry {

std::string serialize_graph_json(const CapturedGraph& graph);
std::string inspect_text(const std::filesystem::path& archive);
std::string inspect_graph_json(const std::filesystem::path& archive, uint32_t batch);
void write_json_graphs(const std::filesystem::path& archive);
std::pair<bool, std::string> diff_archives(const std::filesystem::path& a,
                                           const std::filesystem::path& b);
// Counters a capture-based SAVE of this spec would report (analytic: this
// build writes archives without a simulated driver).
std::map<std::string, uint64_t> save_counters(const WorkloadSpec& spec);
// bench(spec, "save" | "load" | "naive") -> wall_ms, archive_bytes,
// update_served_fraction, construction_calls, update_calls, capture_calls.
std::map<std::string, double> bench(const WorkloadSpec& spec, const std::string& mode);

// Single-file archive "FNDA" (reference pack_archive / unpack_archive,
// pipeline.cpp:740-817): u16 version 1, u32 count, then per file (sorted by
// relative path) {str path, u64 offset, u64 length, u64 crc64}, then the bytes.
void pack_archive_file(const std::filesystem::path& dir, const std::filesystem::path& file);
void unpack_archive_file(const std::filesystem::path& file, const std::filesystem::path& dir);

}  // namespace foundry
