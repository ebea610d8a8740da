// Synthetic decode workloads (SAVE-side input generator, tier R).
//
// The spec vocabulary, canonical text, presets and closed-form expectations
// are the reference's (workload_gen.hpp:16-205, workload_gen.cpp:87-352) so a
// spec file means the same graph set in both builds; LOAD uses
// WorkloadSpec::parse_text + build_init_plan to replay the deterministic
// allocation sequence (pipeline.cpp:465-467,531).
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

namespace foundry {

struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    uint64_t next() {
        uint64_t z = (state += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t bound) { return bound ? next() % bound : 0; }
};

inline uint64_t mix_seed(uint64_t a, uint64_t b) {
    return SplitMix64(a ^ (b * 0x9E3779B97F4A7C15ull)).next();
}

enum class CommMode : uint8_t { none = 0, spmd = 1 };

struct WorkloadSpec {
    uint64_t seed = 1;
    uint32_t batch_max = 8;
    uint32_t layers = 2;
    uint32_t kernels_per_layer = 3;
    std::vector<uint32_t> thresholds;
    double hidden_offset_density = 1.0;
    CommMode comm = CommMode::none;
    uint32_t collectives_per_layer = 0;
    uint64_t kv_cache_bytes = 1ull << 20;
    uint64_t weights_bytes_per_layer = 128ull << 10;
    uint64_t io_bytes = 64ull << 10;
    uint64_t scratch_bytes_per_batch = 16ull << 10;
    bool batch1_special = false;
    bool spmd_uniform = true;
    bool emit_raw_collective = false;

    void validate() const;
    std::string canonical_text() const;
    uint64_t digest() const;
    static WorkloadSpec parse_text(const std::string& text);
    uint32_t variant_for_batch(uint32_t batch) const;
    std::vector<uint32_t> effective_thresholds() const;
    bool operator==(const WorkloadSpec&) const = default;
};

std::vector<std::string> preset_names();
WorkloadSpec preset(const std::string& name);
WorkloadSpec resolve_workload(const std::string& name_or_path);

struct CollectiveKind {
    std::string_view kind, stub_name, real_name;
};
const std::vector<CollectiveKind>& collective_kinds();

struct ExpectedOutcome {
    uint32_t group_count = 0;
    std::vector<uint32_t> group_sizes;
    uint64_t final_offset = 0;
    uint32_t nodes_per_graph = 0;
    bool operator==(const ExpectedOutcome&) const = default;
};
ExpectedOutcome expected_outcome(const WorkloadSpec& spec);

struct InitStep {
    enum class Kind : uint8_t { alloc, release };
    Kind kind = Kind::alloc;
    uint32_t slot = 0;
    std::string tag;
    uint64_t size = 0;
    bool operator==(const InitStep&) const = default;
};
std::vector<InitStep> build_init_plan(const WorkloadSpec& spec);

}  // namespace foundry
