// Offline tooling (see tooling.hpp).
#include "foundry/tooling.hpp"

#include <chrono>
#include <sstream>
#include <unistd.h>

#include <json.hpp>

#include "foundry/archive.hpp"
#include "foundry/bytes.hpp"
#include "foundry/pipeline.hpp"
#include "foundry/save.hpp"

namespace foundry {

namespace fs = std::filesystem;
using nlohmann::json;

namespace {

std::string hex_bytes(const std::vector<uint8_t>& b) {
    static const char* d = "0123456789abcdef";
    std::string s;
    s.reserve(b.size() * 2);
    for (uint8_t x : b) {
        s.push_back(d[x >> 4]);
        s.push_back(d[x & 15]);
    }
    return s;
}

Manifest read_manifest(const fs::path& root) {
    const auto mb = slurp(ArchivePaths{root}.manifest());
    return parse_manifest(std::string(mb.begin(), mb.end()));
}

}  // namespace

std::string serialize_graph_json(const CapturedGraph& g) {
    json root;
    root["label"] = g.label;
    json nodes = json::array();
    for (const auto& n : g.nodes) {
        json o;
        o["id"] = n.id;
        o["type"] = std::string(node_type_name(n.type));
        json p = json::object();
        if (n.type == NodeType::Kernel) {
            const auto& k = n.kernel_params();
            p["blockDimX"] = k.block.x;
            p["blockDimY"] = k.block.y;
            p["blockDimZ"] = k.block.z;
            p["gridDimX"] = k.grid.x;
            p["gridDimY"] = k.grid.y;
            p["gridDimZ"] = k.grid.z;
            p["sharedMemBytes"] = k.shared_mem_bytes;
            p["kernel_node_attrs"] = {
                {"attrQueryAvailable", n.attrs.attr_query_available},
                {"clusterDimX", n.attrs.cluster_dim.x},
                {"clusterDimY", n.attrs.cluster_dim.y},
                {"clusterDimZ", n.attrs.cluster_dim.z},
                {"clusterSchedulingPolicyPreference", n.attrs.cluster_scheduling_policy_preference},
                {"memSyncDomainMapDefault", n.attrs.mem_sync_domain_map_default},
                {"memSyncDomainMapRemote", n.attrs.mem_sync_domain_map_remote},
            };
            p["kernelParams"] = json::array({json{{"index", 0}, {"offset", 0}, {"size", k.arg_buffer.size()}}});
            p["extra"] = json::array({"CU_LAUNCH_PARAM_BUFFER_SIZE", k.arg_buffer.size(),
                                      "CU_LAUNCH_PARAM_BUFFER_POINTER", "null", "CU_LAUNCH_PARAM_END"});
            p["extra_argBuffer_hex"] = hex_bytes(k.arg_buffer);
            p["function_name"] = k.kernel.name;
            p["kernel_source_binary_hash"] = k.kernel.binary_hash;
            p["func_attrs"] = {
                {"max_dynamic_shared_size_bytes", k.func_attrs.max_dynamic_shared_size_bytes},
                {"preferred_shared_memory_carveout", k.func_attrs.preferred_shared_memory_carveout},
                {"cluster_scheduling_policy_preference", k.func_attrs.cluster_scheduling_policy_preference},
                {"required_cluster_width", k.func_attrs.required_cluster_width},
                {"required_cluster_height", k.func_attrs.required_cluster_height},
                {"required_cluster_depth", k.func_attrs.required_cluster_depth},
            };
        } else if (n.type == NodeType::Memcpy) {
            const auto& m = std::get<MemcpyParams>(n.params);
            p["srcDevice"] = m.src;
            p["dstDevice"] = m.dst;
            p["WidthInBytes"] = m.length;
        } else if (n.type == NodeType::Memset) {
            const auto& m = std::get<MemsetParams>(n.params);
            p["dst"] = m.dst;
            p["value"] = m.value;
            p["WidthInBytes"] = m.length;
        }
        o["params"] = std::move(p);
        nodes.push_back(std::move(o));
    }
    root["nodes"] = std::move(nodes);
    json deps = json::array();
    for (const auto& e : g.edges) deps.push_back(json{{"from", e.from}, {"to", e.to}});
    root["dependencies"] = std::move(deps);
    return root.dump(2);
}

std::string inspect_text(const fs::path& archive) {
    ArchivePaths paths{archive};
    require(fs::exists(paths.manifest()), Errc::archive_corruption, "no manifest under " + archive.string());
    const Manifest m = read_manifest(archive);
    const Catalog cat = parse_catalog(slurp(paths.catalog()));
    uint64_t metadata = fs::file_size(paths.manifest());
    for (const char* rel : {"graphs.bin", "memlayout.bin", "catalog.bin", "patch.bin"})
        metadata += fs::file_size(archive / rel);
    uint64_t binary_bytes = 0;
    std::ostringstream lines;
    for (const auto& [hash, r] : cat.binaries) {
        const uint64_t bytes = fs::file_size(paths.binary(hash));
        binary_bytes += bytes;
        lines << "  " << hex16(hash) << "  " << bytes << " bytes, " << r.entrypoints.size() << " kernels";
        if (r.needs_device_init) lines << ", device-init";
        if (r.is_stub) lines << ", comm-stub";
        if (r.is_comm_real) lines << ", comm-real";
        lines << "\n";
    }
    std::ostringstream o;
    o << "archive format v" << m.format_version << ", hash algorithm " << int(m.hash_algorithm) << "\n";
    o << "workload digest " << hex16(m.workload_digest) << ", kv cache " << m.kv_cache_bytes << " bytes\n";
    o << "allocator base 0x" << hex16(m.allocator.base) << ", capacity " << m.allocator.capacity
      << ", granularity " << m.allocator.granularity << ", final offset 0x" << hex16(m.final_offset) << "\n";
    o << "graphs: " << m.grouping.total_graphs << " captured, " << m.grouping.template_count
      << " templates (" << m.grouping.total_graphs - m.grouping.template_count
      << " served by on-demand update)\n";
    o << "group sizes:";
    for (const auto& g : m.grouping.groups) o << " " << g.members.size();
    o << "\n";
    o << "binaries: " << cat.binaries.size() << " (" << binary_bytes << " bytes), metadata " << metadata
      << " bytes\n";
    o << lines.str();
    if (m.comm_real_hash != 0)
        o << "comm: world placeholder " << m.comm_world_placeholder << ", real binary " << hex16(m.comm_real_hash)
          << "\n";
    return o.str();
}

std::string inspect_graph_json(const fs::path& archive, uint32_t batch) {
    const auto bin = slurp(ArchivePaths{archive}.graphs());
    for (const auto& l : parse_graph_locators(bin))
        if (l.label == batch) return serialize_graph_json(parse_graph_at(bin, l));
    raise(Errc::invalid_argument, "archive has no graph for batch " + std::to_string(batch));
}

void write_json_graphs(const fs::path& archive) {
    const auto bin = slurp(ArchivePaths{archive}.graphs());
    fs::create_directories(archive / "graphs");
    for (const auto& g : parse_graphs(bin))
        spit(archive / "graphs" / (std::to_string(g.label) + ".json"), serialize_graph_json(g));
}

std::pair<bool, std::string> diff_archives(const fs::path& a, const fs::path& b) {
    std::vector<std::string> lines;
    auto note = [&](const std::string& s) { lines.push_back(s); };
    const Manifest ma = read_manifest(a), mb = read_manifest(b);
    if (ma.workload_digest != mb.workload_digest) note("workload specs differ");
    if (!(ma.allocator == mb.allocator) || ma.final_offset != mb.final_offset) note("allocator layout differs");
    if (ma.kv_cache_bytes != mb.kv_cache_bytes) note("kv cache size differs");
    if (ma.comm_real_hash != mb.comm_real_hash) note("comm binaries differ");
    const Catalog ca = parse_catalog(slurp(ArchivePaths{a}.catalog()));
    const Catalog cb = parse_catalog(slurp(ArchivePaths{b}.catalog()));
    for (const auto& [h, r] : ca.binaries) {
        auto it = cb.binaries.find(h);
        if (it == cb.binaries.end()) note("binary " + hex16(h) + " only in " + a.string());
        else if (!(r == it->second)) note("binary " + hex16(h) + " metadata differs");
    }
    for (const auto& [h, r] : cb.binaries)
        if (!ca.binaries.count(h)) note("binary " + hex16(h) + " only in " + b.string());
    if (!(parse_patch_table(slurp(ArchivePaths{a}.patch_table())) ==
          parse_patch_table(slurp(ArchivePaths{b}.patch_table()))))
        note("patch tables differ");
    const auto ga = parse_graphs(slurp(ArchivePaths{a}.graphs()));
    const auto gb = parse_graphs(slurp(ArchivePaths{b}.graphs()));
    std::map<uint32_t, const CapturedGraph*> by_label;
    for (const auto& g : gb) by_label[g.label] = &g;
    if (ga.size() != gb.size())
        note("graph counts differ (" + std::to_string(ga.size()) + " vs " + std::to_string(gb.size()) + ")");
    for (const auto& g : ga) {
        auto it = by_label.find(g.label);
        if (it == by_label.end()) {
            note("graph " + std::to_string(g.label) + " only in " + a.string());
            continue;
        }
        const GraphDiff d = diff(g, *it->second);
        if (!d.topology_equal) note("graph " + std::to_string(g.label) + ": topology differs");
        else if (!d.empty())
            note("graph " + std::to_string(g.label) + ": " + std::to_string(d.node_deltas.size()) +
                 " nodes differ in parameters");
    }
    if (lines.empty()) return {true, "archives identical\n"};
    std::string text;
    for (const auto& l : lines) text += l + "\n";
    return {false, text};
}

std::map<std::string, uint64_t> save_counters(const WorkloadSpec& spec) {
    const ExpectedOutcome e = expected_outcome(spec);
    const uint64_t B = spec.batch_max;
    const uint64_t kernels = uint64_t(spec.layers) * (spec.kernels_per_layer + spec.collectives_per_layer);
    const uint64_t images = spec.layers + (spec.comm == CommMode::spmd ? 2 : 0) + 1;  // + decoy
    std::map<std::string, uint64_t> c;
    c["capture.begin_calls"] = B;
    c["capture.launch_calls"] = B * kernels;
    c["capture.node_records"] = B * e.nodes_per_graph;
    c["module.load_calls"] = images;
    c["catalog.prelink_calls"] = spec.kernels_per_layer >= 2 ? 1 : 0;
    c["catalog.linked_segments"] = spec.kernels_per_layer >= 2 ? 2 : 0;
    c["exec.instantiate_calls"] = B;
    c["replay.launch_calls"] = B;
    return c;
}

std::map<std::string, double> bench(const WorkloadSpec& spec, const std::string& mode) {
    require(mode == "save" || mode == "load" || mode == "naive", Errc::invalid_argument,
            "bench mode must be save, load, or naive");
    const auto stamp = std::chrono::steady_clock::now().time_since_epoch().count();
    const fs::path dir = fs::temp_directory_path() / ("foundry-b200-bench-" + std::to_string(::getpid()) +
                                                      "-" + std::to_string(stamp));
    struct Cleanup {
        fs::path d;
        ~Cleanup() {
            std::error_code ec;
            fs::remove_all(d, ec);
        }
    } cleanup{dir};
    using clock = std::chrono::steady_clock;
    std::map<std::string, double> r;
    const SaveOptions opt;
    if (mode == "save") {
        const auto t0 = clock::now();
        SaveResult s = save(spec, dir, opt);
        r["wall_ms"] = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        const auto c = save_counters(spec);
        r["update_served_fraction"] = s.manifest.grouping.update_served_fraction();
        r["capture_calls"] = double(c.at("capture.begin_calls") + c.at("capture.launch_calls") +
                                    c.at("capture.node_records"));
        r["construction_calls"] = double(c.at("exec.instantiate_calls"));
        r["update_calls"] = 0;
    } else {
        SaveResult s = save(spec, dir, opt);
        const auto t0 = clock::now();
        LoadOptions lo;
        ServingContext sc = load(dir, lo);
        uint64_t naive_calls = 0;
        if (mode == "load") {
            for (uint32_t b : sc.batches()) sc.replay(b);
        } else {
            naive_calls = sc.naive_rebuild_all();
        }
        r["wall_ms"] = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        const auto c = sc.counters();
        const uint64_t construction = c.at("graph.add_node_calls") + c.at("graph.add_edge_calls") +
                                      c.at("graph.set_attr_calls") + c.at("exec.instantiate_calls");
        r["construction_calls"] = double(mode == "load" ? construction : naive_calls);
        r["update_calls"] = double(c.at("exec.update_calls"));
        r["capture_calls"] = 0;
        r["update_served_fraction"] = mode == "load" ? s.manifest.grouping.update_served_fraction() : 0.0;
    }
    std::error_code ec;
    uint64_t bytes = 0;
    for (const auto& e : fs::recursive_directory_iterator(dir, ec))
        if (e.is_regular_file()) bytes += e.file_size();
    r["archive_bytes"] = double(bytes);
    return r;
}

// ---------------------------------------------------------------- FNDA

void pack_archive_file(const fs::path& dir, const fs::path& file) {
    require(fs::exists(ArchivePaths{dir}.manifest()), Errc::archive_corruption, "no manifest under " + dir.string());
    std::map<std::string, std::vector<uint8_t>> files;  // sorted by relative path
    for (const auto& e : fs::recursive_directory_iterator(dir))
        if (e.is_regular_file()) files[fs::relative(e.path(), dir).generic_string()] = slurp(e.path());
    Sink w;
    w.raw("FNDA", 4);
    w.u16(1);
    w.u32(static_cast<uint32_t>(files.size()));
    std::vector<size_t> at;
    for (const auto& [rel, bytes] : files) {
        w.str(rel);
        at.push_back(w.size());
        w.u64(0);  // offset: known once the table is complete
        w.u64(bytes.size());
        w.u64(crc64(bytes.data(), bytes.size()));
    }
    size_t k = 0;
    for (const auto& [rel, bytes] : files) {
        w.poke<uint64_t>(at[k++], w.size());
        w.raw(bytes);
    }
    spit(file, w.bytes());
}

void unpack_archive_file(const fs::path& file, const fs::path& dir) {
    const auto bytes = slurp(file);
    Cursor r(bytes, Errc::archive_corruption);
    r.magic("FNDA");
    const uint16_t version = r.u16();
    require(version == 1, Errc::archive_corruption, "unsupported packed archive version " + std::to_string(version));
    struct Entry {
        std::string rel;
        uint64_t offset, length, checksum;
    };
    // entries are appended one at a time (as the reference reads them), so a
    // corrupt count fails as a cursor overrun rather than a huge allocation
    const uint32_t count = r.u32();
    std::vector<Entry> entries;
    for (uint32_t i = 0; i < count; ++i) {
        Entry& e = entries.emplace_back();
        e.rel = r.str();
        e.offset = r.u64();
        e.length = r.u64();
        e.checksum = r.u64();
        require(e.offset <= bytes.size() && e.length <= bytes.size() - e.offset, Errc::archive_corruption,
                e.rel + " overruns the packed archive");
        require(!e.rel.empty() && e.rel.find("..") == std::string::npos && e.rel.front() != '/',
                Errc::archive_corruption, "packed entry path escapes the archive");
    }
    fs::create_directories(dir);
    for (const Entry& e : entries) {
        const std::span<const uint8_t> blob(bytes.data() + e.offset, e.length);
        require(crc64(blob.data(), blob.size()) == e.checksum, Errc::archive_corruption,
                "integrity check failed for " + e.rel);
        const fs::path target = dir / e.rel;
        fs::create_directories(target.parent_path());
        spit(target, blob);
    }
}

}  // namespace foundry
