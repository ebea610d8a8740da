// WorkloadSpec parsing / validation / presets / closed-form expectations
// (semantics: reference workload_gen.cpp:87-352).
#include "foundry/workload.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>

#include "foundry/bytes.hpp"
#include "foundry/errors.hpp"
#include "foundry/hash.hpp"

namespace foundry {

namespace {
constexpr uint64_t kProbeBytes = 64ull << 10;
constexpr uint64_t kGranule = 64ull << 10;
uint64_t round_up(uint64_t v, uint64_t g) { return (v + g - 1) / g * g; }
}  // namespace

std::vector<uint32_t> WorkloadSpec::effective_thresholds() const {
    std::vector<uint32_t> t = thresholds;
    if (batch1_special && batch_max >= 2) t.push_back(2);
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    return t;
}

uint32_t WorkloadSpec::variant_for_batch(uint32_t batch) const {
    uint32_t v = 0;
    for (uint32_t t : effective_thresholds()) v += batch >= t ? 1 : 0;
    return v;
}

void WorkloadSpec::validate() const {
    auto check = [](bool ok, const char* msg) { require(ok, Errc::spec_violation, msg); };
    check(batch_max >= 1, "batch_max must be >= 1");
    check(layers >= 1, "layers must be >= 1");
    check(kernels_per_layer >= 1 && kernels_per_layer <= 8, "kernels_per_layer must be in [1, 8]");
    for (size_t i = 0; i < thresholds.size(); ++i) {
        check(thresholds[i] >= 2 && thresholds[i] <= batch_max, "thresholds must lie in [2, batch_max]");
        check(i == 0 || thresholds[i] > thresholds[i - 1], "thresholds must be strictly increasing");
    }
    check(hidden_offset_density > 0.0 && hidden_offset_density <= 1.0,
          "hidden_offset_density must be in (0, 1]");
    if (comm == CommMode::spmd) {
        check(collectives_per_layer >= 1, "spmd comm requires collectives_per_layer >= 1");
        check(io_bytes >= 256ull * layers * collectives_per_layer,
              "comm staging buffer too small for the collective offsets");
        check(spmd_uniform, "single-rank capture requires rank-uniform execution (spmd_uniform)");
    } else {
        check(collectives_per_layer == 0, "collectives_per_layer requires comm = spmd");
        check(!emit_raw_collective, "emit_raw_collective requires comm = spmd");
    }
    check(io_bytes >= 64ull * batch_max, "io_bytes must cover 64 bytes per batch element");
    check(kv_cache_bytes >= 4096ull * kernels_per_layer,
          "kv_cache_bytes too small for per-slot interior pointers");
    check(scratch_bytes_per_batch >= 64, "scratch_bytes_per_batch must be >= 64");
}

std::string WorkloadSpec::canonical_text() const {
    std::ostringstream o;
    o << "seed = " << seed << "\n";
    o << "batch_max = " << batch_max << "\n";
    o << "layers = " << layers << "\n";
    o << "kernels_per_layer = " << kernels_per_layer << "\n";
    o << "thresholds = ";
    for (size_t i = 0; i < thresholds.size(); ++i) o << (i ? "," : "") << thresholds[i];
    o << "\n";
    char d[32];
    std::snprintf(d, sizeof d, "%.6f", hidden_offset_density);
    o << "hidden_offset_density = " << d << "\n";
    o << "comm = " << (comm == CommMode::spmd ? "spmd" : "none") << "\n";
    o << "collectives_per_layer = " << collectives_per_layer << "\n";
    o << "kv_cache_bytes = " << kv_cache_bytes << "\n";
    o << "weights_bytes_per_layer = " << weights_bytes_per_layer << "\n";
    o << "io_bytes = " << io_bytes << "\n";
    o << "scratch_bytes_per_batch = " << scratch_bytes_per_batch << "\n";
    o << "batch1_special = " << (batch1_special ? 1 : 0) << "\n";
    o << "spmd_uniform = " << (spmd_uniform ? 1 : 0) << "\n";
    o << "emit_raw_collective = " << (emit_raw_collective ? 1 : 0) << "\n";
    return o.str();
}

uint64_t WorkloadSpec::digest() const {
    const std::string t = canonical_text();
    return crc64(t.data(), t.size());
}

namespace {
std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return {};
    const auto e = s.find_last_not_of(" \t\r");
    return s.substr(b, e - b + 1);
}
}  // namespace

WorkloadSpec WorkloadSpec::parse_text(const std::string& text) {
    WorkloadSpec s;
    s.thresholds.clear();
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        if (const auto hash = line.find('#'); hash != std::string::npos) line.resize(hash);
        const auto eq = line.find('=');
        if (eq == std::string::npos) {
            require(trim(line).empty(), Errc::spec_violation, "bad spec line: " + line);
            continue;
        }
        const std::string key = trim(line.substr(0, eq));
        const std::string val = trim(line.substr(eq + 1));
        try {
            auto u32 = [&] { return static_cast<uint32_t>(std::stoul(val)); };
            auto u64 = [&] { return static_cast<uint64_t>(std::stoull(val)); };
            if (key == "seed") s.seed = u64();
            else if (key == "batch_max") s.batch_max = u32();
            else if (key == "layers") s.layers = u32();
            else if (key == "kernels_per_layer") s.kernels_per_layer = u32();
            else if (key == "thresholds") {
                s.thresholds.clear();
                std::istringstream items(val);
                std::string item;
                while (std::getline(items, item, ','))
                    if (!item.empty()) s.thresholds.push_back(static_cast<uint32_t>(std::stoul(item)));
            } else if (key == "hidden_offset_density") s.hidden_offset_density = std::stod(val);
            else if (key == "comm") {
                if (val == "none") s.comm = CommMode::none;
                else if (val == "spmd") s.comm = CommMode::spmd;
                else raise(Errc::spec_violation, "comm must be none or spmd");
            } else if (key == "collectives_per_layer") s.collectives_per_layer = u32();
            else if (key == "kv_cache_bytes") s.kv_cache_bytes = u64();
            else if (key == "weights_bytes_per_layer") s.weights_bytes_per_layer = u64();
            else if (key == "io_bytes") s.io_bytes = u64();
            else if (key == "scratch_bytes_per_batch") s.scratch_bytes_per_batch = u64();
            else if (key == "batch1_special") s.batch1_special = std::stoul(val) != 0;
            else if (key == "spmd_uniform") s.spmd_uniform = std::stoul(val) != 0;
            else if (key == "emit_raw_collective") s.emit_raw_collective = std::stoul(val) != 0;
            else raise(Errc::spec_violation, "unknown spec key '" + key + "'");
        } catch (const std::invalid_argument&) {
            raise(Errc::spec_violation, "bad value for '" + key + "': " + val);
        } catch (const std::out_of_range&) {
            raise(Errc::spec_violation, "value out of range for '" + key + "'");
        }
    }
    s.validate();
    return s;
}

std::vector<std::string> preset_names() { return {"micro", "dense-small", "moe-spmd"}; }

WorkloadSpec preset(const std::string& name) {
    WorkloadSpec s;
    if (name == "micro") {
        s.seed = 7;
        s.batch_max = 8;
        s.layers = 2;
        s.kernels_per_layer = 3;
        s.thresholds = {3, 5};
        s.hidden_offset_density = 1.0;
        s.kv_cache_bytes = 1ull << 20;
        s.weights_bytes_per_layer = 128ull << 10;
        s.io_bytes = 64ull << 10;
        s.scratch_bytes_per_batch = 16ull << 10;
    } else if (name == "dense-small") {
        s.seed = 11;
        s.batch_max = 512;
        s.layers = 25;
        s.kernels_per_layer = 4;
        s.thresholds = {8, 16, 24, 32, 48, 64, 80, 96, 112, 128,
                        160, 192, 224, 256, 288, 320, 384, 448, 480};
        s.hidden_offset_density = 0.6;
        s.kv_cache_bytes = 16ull << 20;
        s.weights_bytes_per_layer = 256ull << 10;
        s.io_bytes = 64ull << 10;
        s.scratch_bytes_per_batch = 4096;
    } else if (name == "moe-spmd") {
        s.seed = 13;
        s.batch_max = 512;
        s.layers = 12;
        s.kernels_per_layer = 8;
        s.thresholds = {16, 32, 48, 64, 96, 128, 160, 192, 224, 256, 320, 384, 448, 496};
        s.hidden_offset_density = 0.5;
        s.comm = CommMode::spmd;
        s.collectives_per_layer = 2;
        s.kv_cache_bytes = 16ull << 20;
        s.weights_bytes_per_layer = 256ull << 10;
        s.io_bytes = 64ull << 10;
        s.scratch_bytes_per_batch = 8192;
    } else {
        raise(Errc::invalid_argument, "unknown preset '" + name + "'");
    }
    s.validate();
    return s;
}

WorkloadSpec resolve_workload(const std::string& name_or_path) {
    for (const auto& n : preset_names())
        if (n == name_or_path) return preset(n);
    const auto bytes = slurp(name_or_path);
    return WorkloadSpec::parse_text(std::string(bytes.begin(), bytes.end()));
}

const std::vector<CollectiveKind>& collective_kinds() {
    static const std::vector<CollectiveKind> kinds = {
        {"allreduce", "stub_allreduce", "nccl_ring_allreduce"},
        {"alltoall", "stub_alltoall", "nvshmem_alltoall_ll"},
    };
    return kinds;
}

ExpectedOutcome expected_outcome(const WorkloadSpec& spec) {
    spec.validate();
    ExpectedOutcome out;
    std::vector<uint32_t> b = spec.effective_thresholds();
    b.insert(b.begin(), 1);
    b.push_back(spec.batch_max + 1);
    for (size_t i = 0; i + 1 < b.size(); ++i) out.group_sizes.push_back(b[i + 1] - b[i]);
    out.group_count = static_cast<uint32_t>(out.group_sizes.size());
    out.nodes_per_graph = 2 + spec.layers * (spec.kernels_per_layer + spec.collectives_per_layer);
    uint64_t off = spec.layers * round_up(spec.weights_bytes_per_layer, kGranule);
    off += round_up(spec.kv_cache_bytes, kGranule);
    off += round_up(spec.io_bytes, kGranule);
    if (spec.comm == CommMode::spmd) off += round_up(spec.io_bytes, kGranule);
    off += round_up(kProbeBytes, kGranule);
    for (uint32_t batch = 1; batch <= spec.batch_max; ++batch)
        off += round_up(spec.scratch_bytes_per_batch * batch, kGranule);
    out.final_offset = off;
    return out;
}

std::vector<InitStep> build_init_plan(const WorkloadSpec& spec) {
    std::vector<InitStep> plan;
    uint32_t slot = 0;
    for (uint32_t l = 0; l < spec.layers; ++l)
        plan.push_back({InitStep::Kind::alloc, slot++, "weights_l" + std::to_string(l),
                        spec.weights_bytes_per_layer});
    plan.push_back({InitStep::Kind::alloc, slot++, "kv_pool", spec.kv_cache_bytes});
    plan.push_back({InitStep::Kind::alloc, slot++, "io", spec.io_bytes});
    if (spec.comm == CommMode::spmd)
        plan.push_back({InitStep::Kind::alloc, slot++, "comm_staging", spec.io_bytes});
    const uint32_t probe = slot;
    plan.push_back({InitStep::Kind::alloc, slot++, "profile_probe", kProbeBytes});
    plan.push_back({InitStep::Kind::release, probe, "profile_probe", kProbeBytes});
    return plan;
}

}  // namespace foundry
