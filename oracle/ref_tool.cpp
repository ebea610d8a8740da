// ref_tool — a thin command-line driver over the UNMODIFIED reference library
// (/root/reference/proj, compiled by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY. Nothing in the product path links or executes
// this; it exists so tests/ and bench.py's CPU-baseline leg can ask the
// reference itself for ground truth:
//
//   save <preset|spec-file> <out-dir> [traces-file]
//        foundry::save (pipeline.cpp:249-405); writes the SAVE self-replay
//        traces (pipeline.cpp:326-327) to traces-file.
//   prepare <archive> <rank> <world> <out.fndg>
//        the reference PrepareFn for every member (pipeline.cpp:506-514):
//        parse_graph_at (graph_model.cpp:295-303) + apply_rank_patches
//        (rank_forge.cpp:132-152), re-serialized with serialize_graphs
//        (graph_model.cpp:244-269) in graphs.bin locator order.
//   replay <archive> <graphs.fndg> <delta-hex> <traces-out>
//        replays externally materialized graphs on the reference simulated
//        driver with the region mapped at base+delta (det_alloc.cpp:169-181,
//        sim_driver.cpp:402-479): the reference's own hidden offsets decide
//        whether every embedded address is live.
//   time-load <archive> <rank> <world> <lanes> <reps> [replay]
//        best-of-reps wall time of foundry::load (pipeline.cpp:447-557),
//        optionally followed by serve+replay of every batch; prints JSON.
//   time-materialize <archive> <rank> <world> <lanes> <reps>
//        integrity CRC of every file + PrepareFn of every member, timed.
//   time-serve <archive> <rank> <world> <lanes> <reps>
//        serve + replay of every batch after one load (pipeline.cpp:876-889).
//   load-traces <archive> <rank> <world> <traces-out>
//        foundry::load + replay of every batch, traces_to_text.
//   crc <file>   CRC-64/XZ (hash.cpp:53-69) of a file, hex.
//   diff <a.fndg> <b.fndg>   reference diff() text per graph pair.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>
#include <thread>

#include "foundry/binary_catalog.hpp"
#include "foundry/det_alloc.hpp"
#include "foundry/graph_model.hpp"
#include "foundry/hash.hpp"
#include "foundry/io.hpp"
#include "foundry/pipeline.hpp"
#include "foundry/rank_forge.hpp"
#include "foundry/sim_driver.hpp"
#include "foundry/workload_gen.hpp"

using namespace foundry;
namespace fs = std::filesystem;

static int usage() {
    std::fprintf(stderr,
                 "usage: ref_tool save|prepare|replay|time-load|crc|diff ...\n");
    return 64;
}

static int cmd_save(int argc, char** argv) {
    if (argc < 4) return usage();
    const WorkloadSpec spec = resolve_workload(argv[2]);
    SaveResult result = save(spec, argv[3]);
    if (argc >= 5) {
        write_file(argv[4], traces_to_text(result.traces));
    }
    std::printf("{\"graphs\": %u, \"templates\": %u}\n", result.manifest.grouping.total_graphs,
                result.manifest.grouping.template_count);
    return 0;
}

static int cmd_prepare(int argc, char** argv) {
    if (argc < 6) return usage();
    const fs::path archive = argv[2];
    const uint32_t rank = static_cast<uint32_t>(std::stoul(argv[3]));
    const uint32_t world = static_cast<uint32_t>(std::stoul(argv[4]));
    ArchivePaths paths{archive};
    const auto manifest_bytes = read_file(paths.manifest());
    const Manifest manifest =
        parse_manifest(std::string(manifest_bytes.begin(), manifest_bytes.end()));
    const PatchTable table = parse_patch_table(read_file(paths.patch_table()));
    const auto graphs_bin = read_file(paths.graphs());
    std::vector<CapturedGraph> out;
    for (const auto& loc : parse_graph_locators(graphs_bin)) {
        CapturedGraph g = parse_graph_at(graphs_bin, loc);
        auto it = table.per_graph.find(loc.label);
        if (it != table.per_graph.end()) {
            apply_rank_patches(g, it->second, manifest.comm_real_hash, rank, world);
        }
        out.push_back(std::move(g));
    }
    write_file(argv[5], serialize_graphs(out));
    return 0;
}

static int cmd_replay(int argc, char** argv) {
    if (argc < 6) return usage();
    const fs::path archive = argv[2];
    ArchivePaths paths{archive};
    const auto manifest_bytes = read_file(paths.manifest());
    const Manifest manifest =
        parse_manifest(std::string(manifest_bytes.begin(), manifest_bytes.end()));
    const uint64_t delta = parse_hex_u64(argv[4]);
    const auto graphs = parse_graphs(read_file(argv[3]));

    SimDriver driver;
    DeviceContext& ctx = driver.create_context();
    const Catalog catalog = parse_catalog(read_file(paths.catalog()));
    restore_binaries(ctx, catalog, [&](uint64_t hash) { return read_file(paths.binary(hash)); });
    RegionConfig config = manifest.allocator;
    config.base += delta;
    VirtualRegion region(ctx, config, Phase::load);
    region.preallocate(manifest.final_offset);

    std::map<uint32_t, LaunchTrace> traces;
    try {
        for (const auto& g : graphs) {
            const GraphHandle handle = ctx.build_graph(g);
            const ExecHandle exec = ctx.instantiate(handle);
            traces.emplace(g.label, ctx.replay(exec));
        }
    } catch (const Error& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 3;
    }
    write_file(argv[5], traces_to_text(traces));
    return 0;
}

static int cmd_time_load(int argc, char** argv) {
    if (argc < 7) return usage();
    const fs::path archive = argv[2];
    LoadOptions options;
    options.rank = static_cast<uint32_t>(std::stoul(argv[3]));
    options.world = static_cast<uint32_t>(std::stoul(argv[4]));
    options.prepare_lanes = static_cast<unsigned>(std::stoul(argv[5]));
    const int reps = std::stoi(argv[6]);
    const bool replay = argc >= 8 && std::string(argv[7]) == "replay";
    using clock = std::chrono::steady_clock;
    double best = 1e300, total = 0.0;
    size_t graphs = 0;
    for (int i = 0; i < reps + 1; ++i) {  // one warm-up (page cache), then reps
        const auto t0 = clock::now();
        ServingContext sc = load(archive, options);
        if (replay) {
            for (uint32_t b : sc.batches()) sc.replay(b);
        }
        const auto t1 = clock::now();
        graphs = sc.batches().size();
        const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (i > 0) {
            best = std::min(best, ms);
            total += ms;
        }
    }
    std::printf("{\"best_ms\": %.6f, \"mean_ms\": %.6f, \"reps\": %d, \"graphs\": %zu, "
                "\"lanes\": %u, \"hw_threads\": %u}\n",
                best, total / reps, reps, graphs, options.prepare_lanes,
                std::thread::hardware_concurrency());
    return 0;
}

// load-traces <archive> <rank> <world> <traces-out>
//   the reference's own load() (pipeline.cpp:447-557) + replay of every batch
//   (pipeline.cpp:566-569), as traces_to_text.
static int cmd_load_traces(int argc, char** argv) {
    if (argc < 6) return usage();
    LoadOptions options;
    options.rank = static_cast<uint32_t>(std::stoul(argv[3]));
    options.world = static_cast<uint32_t>(std::stoul(argv[4]));
    ServingContext sc = load(argv[2], options);
    std::map<uint32_t, LaunchTrace> traces;
    for (uint32_t b : sc.batches()) traces.emplace(b, sc.replay(b));
    write_file(argv[5], traces_to_text(traces));
    return 0;
}

// time-serve <archive> <rank> <world> <lanes> <reps>
//   one foundry::load, then `reps` sweeps of ServingContext::replay over every
//   batch in label order (= ServingSet::serve + the simulated launch,
//   pipeline.cpp:566-569, the loop of bench --mode load pipeline.cpp:876-889),
//   after one untimed sweep.
static int cmd_time_serve(int argc, char** argv) {
    if (argc < 7) return usage();
    LoadOptions options;
    options.rank = static_cast<uint32_t>(std::stoul(argv[3]));
    options.world = static_cast<uint32_t>(std::stoul(argv[4]));
    options.prepare_lanes = static_cast<unsigned>(std::stoul(argv[5]));
    const int reps = std::max(1, std::stoi(argv[6]));
    using clock = std::chrono::steady_clock;
    ServingContext sc = load(argv[2], options);
    const auto batches = sc.batches();
    double best = 1e300, total = 0.0;
    for (int i = 0; i < reps + 1; ++i) {
        const auto t0 = clock::now();
        for (uint32_t b : batches) sc.replay(b);
        const double ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        if (i > 0) {
            best = std::min(best, ms);
            total += ms;
        }
    }
    std::printf("{\"best_ms\": %.6f, \"mean_ms\": %.6f, \"reps\": %d, \"batches\": %zu, "
                "\"us_per_batch\": %.3f}\n",
                best, total / reps, reps, batches.size(), 1e3 * (total / reps) / batches.size());
    return 0;
}

// time-materialize <archive> <rank> <world> <lanes> <reps> [warmup=1]
//   the reference's share of LOAD that the GPU path replaces: the integrity
//   CRC of every manifest-listed file, single-threaded as in
//   verify_archive_integrity (pipeline.cpp:411-417), then the PrepareFn of
//   every member (parse_graph_at + apply_rank_patches, pipeline.cpp:506-514)
//   on `lanes` threads like the prepare lanes (templater.cpp:102-130).
static int cmd_time_materialize(int argc, char** argv) {
    if (argc < 7) return usage();
    const fs::path archive = argv[2];
    const uint32_t rank = static_cast<uint32_t>(std::stoul(argv[3]));
    const uint32_t world = static_cast<uint32_t>(std::stoul(argv[4]));
    const unsigned lanes = static_cast<unsigned>(std::stoul(argv[5]));
    const int reps = std::stoi(argv[6]);
    const int warmup = argc > 7 ? std::max(0, std::stoi(argv[7])) : 1;
    using clock = std::chrono::steady_clock;
    double best = 1e300, total = 0.0, crc_best = 1e300;
    for (int i = 0; i < reps + warmup; ++i) {
        const auto t0 = clock::now();
        ArchivePaths paths{archive};
        const auto mb = read_file(paths.manifest());
        const Manifest m = parse_manifest(std::string(mb.begin(), mb.end()));
        for (const auto& [rel, digest] : m.file_digests) {
            if (crc64(read_file(archive / rel)) != digest) {
                std::fprintf(stderr, "integrity check failed for %s\n", rel.c_str());
                return 3;
            }
        }
        const auto t1 = clock::now();
        const PatchTable table = parse_patch_table(read_file(paths.patch_table()));
        const auto graphs_bin = read_file(paths.graphs());
        const auto locs = parse_graph_locators(graphs_bin);
        std::atomic<size_t> next{0};
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < std::max(1u, lanes); ++t)
            pool.emplace_back([&] {
                for (size_t k; (k = next.fetch_add(1)) < locs.size();) {
                    CapturedGraph g = parse_graph_at(graphs_bin, locs[k]);
                    auto it = table.per_graph.find(locs[k].label);
                    if (it != table.per_graph.end())
                        apply_rank_patches(g, it->second, m.comm_real_hash, rank, world);
                }
            });
        for (auto& t : pool) t.join();
        const auto t2 = clock::now();
        const double ms = std::chrono::duration<double, std::milli>(t2 - t0).count();
        const double crc_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (i >= warmup) {
            best = std::min(best, ms);
            crc_best = std::min(crc_best, crc_ms);
            total += ms;
        }
    }
    std::printf("{\"best_ms\": %.6f, \"mean_ms\": %.6f, \"integrity_best_ms\": %.6f, \"reps\": %d, "
                "\"lanes\": %u, \"hw_threads\": %u}\n",
                best, total / reps, crc_best, reps, lanes, std::thread::hardware_concurrency());
    return 0;
}

static int cmd_crc(int argc, char** argv) {
    if (argc < 3) return usage();
    std::printf("%s\n", to_hex(crc64(read_file(argv[2]))).c_str());
    return 0;
}

static int cmd_diff(int argc, char** argv) {
    if (argc < 4) return usage();
    const auto a = parse_graphs(read_file(argv[2]));
    const auto b = parse_graphs(read_file(argv[3]));
    for (size_t i = 0; i < std::min(a.size(), b.size()); ++i) {
        std::printf("# graph %u\n%s", a[i].label, diff(a[i], b[i]).to_text().c_str());
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "save") return cmd_save(argc, argv);
        if (cmd == "pack" && argc == 4) {  // reference pack_archive (pipeline.cpp:747-773)
            pack_archive(argv[2], argv[3]);
            return 0;
        }
        if (cmd == "unpack" && argc == 4) {  // reference unpack_archive (pipeline.cpp:775-817)
            unpack_archive(argv[2], argv[3]);
            return 0;
        }
        if (cmd == "prepare") return cmd_prepare(argc, argv);
        if (cmd == "replay") return cmd_replay(argc, argv);
        if (cmd == "time-load") return cmd_time_load(argc, argv);
        if (cmd == "time-materialize") return cmd_time_materialize(argc, argv);
        if (cmd == "time-serve") return cmd_time_serve(argc, argv);
        if (cmd == "load-traces") return cmd_load_traces(argc, argv);
        if (cmd == "crc") return cmd_crc(argc, argv);
        if (cmd == "diff") return cmd_diff(argc, argv);
    } catch (const Error& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 2;
    }
    return usage();
}
