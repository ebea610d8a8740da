// Tier-R archive writer (see save.hpp). The graph set is generated directly
// as CapturedGraphs — there is no simulated driver on this side — following
// the reference generator's deterministic recipe (workload_gen.cpp:354-531),
// the stub lowering of collectives (rank_forge.cpp:97-130), the bump
// allocator (det_alloc.cpp:71-111) and the archive layout (pipeline.cpp:341-389).
#include "foundry/save.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <sstream>

#include "foundry/bytes.hpp"
#include "foundry/template_store.hpp"
#include "foundry/trace_module.hpp"

namespace foundry {

namespace fs = std::filesystem;

std::string LaunchTrace::to_text() const {
    std::ostringstream o;
    for (const auto& r : records) {
        o << "node=" << r.node_id << " type=" << node_type_name(r.type);
        if (r.type == NodeType::Kernel) {
            o << " name=" << r.kernel_name << " grid=" << r.grid.x << "," << r.grid.y << ","
              << r.grid.z << " block=" << r.block.x << "," << r.block.y << "," << r.block.z
              << " shmem=" << r.shared_mem_bytes;
        }
        o << " args=" << hex16(r.arg_digest) << " addrs=";
        for (size_t i = 0; i < r.addresses.size(); ++i) o << (i ? "," : "") << "0x" << hex16(r.addresses[i]);
        o << "\n";
    }
    return o.str();
}

std::string traces_to_text(const std::map<uint32_t, LaunchTrace>& traces) {
    std::ostringstream o;
    for (const auto& [batch, t] : traces) o << "# batch " << batch << "\n" << t.to_text();
    return o.str();
}

namespace {

constexpr uint32_t kAddrFields[5] = {8, 16, 24, 32, 40};
constexpr uint32_t kArgHeader = 48;
const char* const kSlotNames[8] = {"fused_qkv_gemm", "paged_attn_decode", "silu_mul_gemm",
                                   "rmsnorm_residual", "moe_group_gemm", "rope_embed",
                                   "logits_gemm", "topk_softmax"};

std::string kernel_name(uint32_t l, uint32_t s, uint32_t v) {
    return std::string(kSlotNames[s % 8]) + "_l" + std::to_string(l) + "_v" + std::to_string(v);
}
uint32_t arg_size(uint32_t s) { return 192 + 32 * s; }

std::vector<uint32_t> hidden_offsets(const WorkloadSpec& spec, uint32_t l, uint32_t s) {
    std::vector<uint32_t> c(std::begin(kAddrFields), std::end(kAddrFields));
    SplitMix64 rng(mix_seed(spec.seed, 0x48494444ull + l * 131 + s));
    for (size_t i = c.size() - 1; i > 0; --i) std::swap(c[i], c[rng.below(i + 1)]);
    const auto want = static_cast<size_t>(std::lround(spec.hidden_offset_density * 5.0));
    c.resize(std::clamp<size_t>(want, 1, c.size()));
    std::sort(c.begin(), c.end());
    return c;
}

FuncAttrs slot_func_attrs(uint32_t s, uint32_t v) {
    FuncAttrs f;
    f.max_dynamic_shared_size_bytes = static_cast<int32_t>(32768 + 4096 * s + 1024 * v);
    return f;
}

KernelNodeAttrs variant_attrs(uint32_t v) {
    KernelNodeAttrs a;
    a.cluster_dim = {2 + (v % 8), 1 + (v / 8), 1};
    a.cluster_scheduling_policy_preference = static_cast<int32_t>(v % 2);
    return a;
}

struct Binary {
    std::vector<uint8_t> payload;
    uint64_t hash = 0;
    LoadVariant variant = LoadVariant::data;
    std::vector<uint8_t> options;
    KernelImage image;  // parsed form of payload
};

// Deterministic bump allocator over the capture region (det_alloc.cpp:71-111).
struct Bump {
    RegionConfig cfg;
    uint64_t offset = 0;
    bool window = false;
    std::vector<AllocationRecord> records;
    uint64_t allocate(uint64_t size) {
        require(size > 0, Errc::invalid_argument, "zero-byte allocation");
        const uint64_t len = (size + cfg.granularity - 1) / cfg.granularity * cfg.granularity;
        require(offset + len <= cfg.capacity, Errc::out_of_region,
                "allocation of " + std::to_string(size) + " bytes exceeds region capacity");
        const uint64_t addr = cfg.base + offset;
        offset += len;
        records.push_back({records.size(), size, addr, len,
                           window ? AllocWindow::capture_window : AllocWindow::pre_capture});
        return addr;
    }
};

void put_u64(std::vector<uint8_t>& buf, uint32_t at, uint64_t v) { std::memcpy(buf.data() + at, &v, 8); }

}  // namespace

SaveResult save(const WorkloadSpec& spec, const fs::path& out, const SaveOptions& options) {
    spec.validate();
    if (fs::exists(out)) {
        require(fs::is_directory(out) && fs::is_empty(out), Errc::invalid_argument,
                "archive path " + out.string() + " exists and is not empty");
    }
    fs::create_directories(out);
    try {
        const ExpectedOutcome expect = expected_outcome(spec);
        const uint32_t V = expect.group_count;
        const uint32_t K = spec.kernels_per_layer;
        const bool spmd = spec.comm == CommMode::spmd;

        // ---- binaries: one image per layer (layer 0 pre-linked from two segments)
        std::vector<Binary> layer_bin(spec.layers);
        for (uint32_t l = 0; l < spec.layers; ++l) {
            const bool split = l == 0 && K >= 2;
            std::vector<std::vector<uint8_t>> segments;
            for (uint32_t part = 0; part < (split ? 2u : 1u); ++part) {
                KernelImage seg;
                seg.relocatable = split;
                seg.link_tag = 1000 + l;
                for (uint32_t s = 0; s < K; ++s) {
                    if (split && s % 2 != part) continue;
                    for (uint32_t v = 0; v < V; ++v)
                        seg.entrypoints.push_back(
                            {kernel_name(l, s, v), arg_size(s), hidden_offsets(spec, l, s), slot_func_attrs(s, v)});
                }
                segments.push_back(encode_kernel_image(seg));
            }
            Binary& b = layer_bin[l];
            b.payload = segments.size() > 1 ? link_segments(segments) : segments.front();
            if (l == 1) {
                b.variant = LoadVariant::with_options;
                b.options = {0x4F, 0x50, 0x54, 0x01};
            }
        }
        Binary stub_bin, real_bin;
        if (spmd) {
            KernelImage stub, real;
            stub.link_tag = 2000;
            real.link_tag = 2001;
            real.requires_device_init = true;
            for (const auto& k : collective_kinds()) {
                stub.entrypoints.push_back({std::string(k.stub_name), 32, {16}, {}});
                real.entrypoints.push_back({std::string(k.real_name), 32, {16}, {}});
            }
            stub_bin.payload = encode_kernel_image(stub);
            real_bin.payload = encode_kernel_image(real);
            real_bin.variant = LoadVariant::file;
        }
        auto finish = [](Binary& b) {
            b.hash = crc64(b.payload);
            b.image = parse_kernel_image(b.payload);
        };
        for (auto& b : layer_bin) finish(b);
        if (spmd) {
            finish(stub_bin);
            finish(real_bin);
        }

        // ---- deterministic allocation sequence
        Bump region;
        if (options.base_address) region.cfg.base = *options.base_address;
        std::vector<uint64_t> slot;
        for (const InitStep& st : build_init_plan(spec)) {
            if (st.kind == InitStep::Kind::alloc) {
                if (st.slot >= slot.size()) slot.resize(st.slot + 1, 0);
                slot[st.slot] = region.allocate(st.size);
            }  // release: the granule leaks, the offset never rewinds (det_alloc.cpp:102-111)
        }
        const uint64_t kv = slot[spec.layers], io = slot[spec.layers + 1];
        const uint64_t comm = spmd ? slot[spec.layers + 2] : 0;
        region.window = true;
        const uint64_t window_start = region.offset;

        // ---- capture every batch size
        std::vector<CapturedGraph> graphs;
        std::map<uint32_t, LaunchTrace> traces;
        PatchTable patches;
        std::vector<std::vector<uint8_t>> filler(spec.layers * K);
        for (uint32_t l = 0; l < spec.layers; ++l)
            for (uint32_t s = 0; s < K; ++s) {
                auto& f = filler[l * K + s];
                f.resize(arg_size(s) - kArgHeader);
                SplitMix64 rng(mix_seed(spec.seed, 0x46494C4Cull + l * 131 + s));
                for (auto& byte : f) byte = static_cast<uint8_t>(rng.next() & 0xFF);
            }
        for (uint32_t b = 1; b <= spec.batch_max; ++b) {
            const uint64_t scratch = region.allocate(spec.scratch_bytes_per_batch * b);
            const uint32_t v = spec.variant_for_batch(b);
            CapturedGraph g;
            g.label = b;
            std::vector<CommPatchEntry> entries;
            auto add_edges = [&](const std::vector<uint32_t>& deps) {
                const uint32_t i = static_cast<uint32_t>(g.nodes.size()) - 1;
                if (deps.empty()) {
                    if (i > 0) g.edges.push_back({i - 1, i});
                } else {
                    for (uint32_t d : deps) g.edges.push_back({d, i});
                }
            };
            {
                GraphNode n;
                n.type = NodeType::Memset;
                n.params = MemsetParams{io, 0, 64ull * b};
                g.nodes.push_back(n);
                add_edges({});
            }
            std::vector<uint32_t> tail = {0};
            for (uint32_t l = 0; l < spec.layers; ++l) {
                const uint32_t layer_base = static_cast<uint32_t>(g.nodes.size());
                for (uint32_t s = 0; s < K; ++s) {
                    GraphNode n;
                    n.type = NodeType::Kernel;
                    if (s == 0) n.attrs = variant_attrs(v);
                    KernelNodeParams k;
                    k.grid = {1 + (s % 4), (b + 7) / 8, 1};
                    k.block = {128 * (1 + s % 3), 1, 1};
                    k.shared_mem_bytes = 1024 * (1 + s % 4) + 2048 * (v % 3);
                    k.kernel = {layer_bin[l].hash, kernel_name(l, s, v)};
                    k.func_attrs = slot_func_attrs(s, v);
                    k.arg_buffer.assign(arg_size(s), 0);
                    put_u64(k.arg_buffer, 0, b);
                    put_u64(k.arg_buffer, 8, slot[l]);
                    put_u64(k.arg_buffer, 16, io);
                    put_u64(k.arg_buffer, 24, kv);
                    put_u64(k.arg_buffer, 32, scratch);
                    put_u64(k.arg_buffer, 40, kv + 4096ull * s);
                    const auto& f = filler[l * K + s];
                    std::copy(f.begin(), f.end(), k.arg_buffer.begin() + kArgHeader);
                    n.params = std::move(k);
                    g.nodes.push_back(std::move(n));
                    add_edges(s == 0 ? tail : std::vector<uint32_t>{layer_base});
                }
                tail.clear();
                for (uint32_t s = 0; s < K; ++s) tail.push_back(layer_base + s);
                for (uint32_t c = 0; c < spec.collectives_per_layer; ++c) {
                    const auto& kind = collective_kinds()[c % collective_kinds().size()];
                    require(!(spec.emit_raw_collective && b == 1 && l == 0 && c == 0),
                            Errc::unpatchable_comm,
                            "graph capture: batch 1 op " + std::to_string(g.nodes.size()) +
                                ": collective reached capture outside the comm stub layer");
                    GraphNode n;
                    n.type = NodeType::Kernel;
                    KernelNodeParams k;
                    k.grid = {1, 1, 1};
                    k.block = {32, 1, 1};
                    k.kernel = {stub_bin.hash, std::string(kind.stub_name)};
                    k.arg_buffer.assign(32, 0);
                    put_u64(k.arg_buffer, 0, 0);  // single SAVE rank
                    put_u64(k.arg_buffer, 8, 1);  // world placeholder
                    put_u64(k.arg_buffer, 16, comm + 256ull * (l * spec.collectives_per_layer + c));
                    put_u64(k.arg_buffer, 24, 32ull * b + 16ull * c);
                    n.params = std::move(k);
                    const uint32_t id = static_cast<uint32_t>(g.nodes.size());
                    g.nodes.push_back(std::move(n));
                    add_edges(tail);
                    tail = {id};
                    entries.push_back({id, {stub_bin.hash, std::string(kind.stub_name)},
                                       std::string(kind.real_name), {0}, {8}, 8});
                }
            }
            {
                GraphNode n;
                n.type = NodeType::Memcpy;
                n.params = MemcpyParams{scratch, io, 64ull * b};
                g.nodes.push_back(n);
                add_edges(tail);
            }
            g.canonicalize();

            // expected replay (capture-time state), reference sim_driver.cpp:402-479
            LaunchTrace t;
            for (const auto& n : g.nodes) {
                TraceRecord r;
                r.node_id = n.id;
                r.type = n.type;
                if (n.type == NodeType::Kernel) {
                    const auto& k = n.kernel_params();
                    const Binary* bin = nullptr;
                    for (const auto& lb : layer_bin)
                        if (lb.hash == k.kernel.binary_hash) bin = &lb;
                    if (!bin) bin = &stub_bin;
                    for (const auto& e : bin->image.entrypoints)
                        if (e.name == k.kernel.name)
                            for (uint32_t off : e.hidden_offsets) {
                                uint64_t a;
                                std::memcpy(&a, k.arg_buffer.data() + off, 8);
                                r.addresses.push_back(a);
                            }
                    r.kernel_name = k.kernel.name;
                    r.grid = k.grid;
                    r.block = k.block;
                    r.shared_mem_bytes = k.shared_mem_bytes;
                    r.arg_digest = crc64(k.arg_buffer);
                } else if (n.type == NodeType::Memcpy) {
                    const auto& m = std::get<MemcpyParams>(n.params);
                    r.addresses = {m.src, m.dst};
                    const uint64_t raw[3] = {m.src, m.dst, m.length};
                    r.arg_digest = crc64(raw, sizeof raw);
                } else if (n.type == NodeType::Memset) {
                    const auto& m = std::get<MemsetParams>(n.params);
                    r.addresses = {m.dst};
                    const uint64_t raw[3] = {m.dst, m.value, m.length};
                    r.arg_digest = crc64(raw, sizeof raw);
                }
                t.records.push_back(std::move(r));
            }
            traces.emplace(b, std::move(t));
            graphs.push_back(std::move(g));
            if (!entries.empty()) patches.per_graph.emplace(b, std::move(entries));
        }

        // ---- grouping, catalog, archive files
        GroupingManifest grouping = group_graphs(graphs);
        Catalog catalog;
        auto record = [&](const Binary& b, bool stub, bool real) {
            KernelBinaryRecord r;
            r.hash = b.hash;
            r.variant = b.variant;
            r.load_options = b.options;
            r.needs_device_init = b.image.requires_device_init || real;
            r.is_stub = stub;
            r.is_comm_real = real;
            for (const auto& e : b.image.entrypoints) {
                r.entrypoints.push_back(e.name);
                r.entrypoint_attrs.push_back(e.attrs);
            }
            catalog.binaries[b.hash] = std::move(r);
        };
        std::vector<const Binary*> written;
        for (const auto& b : layer_bin) {
            record(b, false, false);
            written.push_back(&b);
        }
        if (spmd) {  // the stub binary is referenced by graphs; the real one is kept explicitly
            record(stub_bin, true, false);
            record(real_bin, false, true);
            written.push_back(&stub_bin);
            written.push_back(&real_bin);
        }

        const std::vector<uint8_t> graphs_bin = serialize_graphs(graphs);
        attach_locators(grouping, parse_graph_locators(graphs_bin));

        MemoryEventLog log;
        log.config = region.cfg;
        log.starting_offset = window_start;
        log.final_offset = region.offset;
        log.records = region.records;

        Manifest m;
        m.workload_digest = spec.digest();
        m.workload_text = spec.canonical_text();
        m.allocator = region.cfg;
        m.final_offset = region.offset;
        m.kv_cache_bytes = spec.kv_cache_bytes;
        m.comm_real_hash = spmd ? real_bin.hash : 0;
        m.grouping = std::move(grouping);

        ArchivePaths paths{out};
        const auto memlayout_bin = serialize_event_log(log);
        const auto catalog_bin = serialize_catalog(catalog);
        const auto patch_bin = serialize_patch_table(patches);
        spit(paths.graphs(), graphs_bin);
        spit(paths.memlayout(), memlayout_bin);
        spit(paths.catalog(), catalog_bin);
        spit(paths.patch_table(), patch_bin);
        m.file_digests["graphs.bin"] = crc64(graphs_bin);
        m.file_digests["memlayout.bin"] = crc64(memlayout_bin);
        m.file_digests["catalog.bin"] = crc64(catalog_bin);
        m.file_digests["patch.bin"] = crc64(patch_bin);
        fs::create_directories(paths.binaries());
        for (const Binary* b : written) {
            spit(paths.binary(b->hash), b->payload);
            m.file_digests["binaries/" + hex16(b->hash) + ".bin"] = b->hash;
        }
        spit(paths.manifest(), serialize_manifest(m));
        if (options.b200_artifacts) pack_archive(out, options.threads);

        SaveResult res;
        res.archive_dir = out;
        {
            const auto mt = slurp(paths.manifest());
            res.manifest = parse_manifest(std::string(mt.begin(), mt.end()));
        }
        res.traces = std::move(traces);
        res.allocation_records = std::move(region.records);
        return res;
    } catch (...) {
        std::error_code ec;
        fs::remove_all(out, ec);  // never leave a partial archive behind
        throw;
    }
}

void pack_archive(const fs::path& archive, unsigned threads) {
    pack_archive_store(archive, threads);
    write_trace_cubins(archive);
}

}  // namespace foundry
