// `foundry` — the reference's command-line front end (proj/tools/main.cpp:22-133)
// over the B200 build: same subcommands, options, output lines and exit codes
// (errors.cpp:24-39 via exit_code_for). CLI11 is not in this image, so the
// options are parsed by hand; `--name value` and `--name=value` both work.
//
//   foundry save    --workload <preset|spec> --out <dir> [--traces <file>] [--emit-json-graphs]
//   foundry load    --archive <dir> [--rank R] [--world W] [--no-prealloc] [--replay-all]
//                   [--traces <file>]                      (+ B200: --relocate --share-execs
//                                                           --device-updates --device N)
//   foundry inspect <archive> [--graph <batch>]
//   foundry diff    <a> <b>
//   foundry bench   --workload <preset|spec> [--mode save|load|naive]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "foundry/errors.hpp"
#include "foundry/pipeline.hpp"
#include "foundry/save.hpp"
#include "foundry/bytes.hpp"
#include "foundry/tooling.hpp"
#include "foundry/workload.hpp"

namespace fs = std::filesystem;
using namespace foundry;

namespace {

// FOUNDRY_BASE_ADDR (SAVE only; the manifest wins at LOAD): main.cpp:11-17
std::optional<uint64_t> base_addr_from_env() {
    const char* v = std::getenv("FOUNDRY_BASE_ADDR");
    if (v == nullptr || *v == '\0') return std::nullopt;
    return std::stoull(v, nullptr, 0);
}

struct Args {
    std::vector<std::string> positional;
    std::map<std::string, std::string> opts;  // --name -> value ("" for flags)
    bool has(const std::string& k) const { return opts.count(k) != 0; }
    std::string get(const std::string& k, const std::string& dflt = "") const {
        auto it = opts.find(k);
        return it == opts.end() ? dflt : it->second;
    }
};

int usage(const char* msg) {
    std::cerr << msg << "\n"
              << "usage: foundry {save|load|inspect|diff|bench} ...\n"
                 "  save    --workload W --out DIR [--traces FILE] [--emit-json-graphs]\n"
                 "  load    --archive DIR [--rank R] [--world N] [--no-prealloc] [--replay-all] [--traces FILE]\n"
                 "          [--relocate] [--share-execs] [--device-updates] [--device ORDINAL]\n"
                 "  inspect ARCHIVE [--graph BATCH]\n"
                 "  diff    A B\n"
                 "  bench   --workload W [--mode save|load|naive]\n";
    return 2;  // CLI11's parse-error exit code family: a usage error
}

Args parse(int argc, char** argv, const std::vector<std::string>& flags) {
    Args a;
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) != 0) {
            a.positional.push_back(s);
            continue;
        }
        const auto eq = s.find('=');
        if (eq != std::string::npos) {
            a.opts[s.substr(0, eq)] = s.substr(eq + 1);
        } else if (std::find(flags.begin(), flags.end(), s) != flags.end()) {
            a.opts[s] = "";
        } else {
            require(i + 1 < argc, Errc::invalid_argument, "option " + s + " needs a value");
            a.opts[s] = argv[++i];
        }
    }
    return a;
}

int cmd_save(const Args& a) {
    if (!a.has("--workload") || !a.has("--out")) return usage("save: --workload and --out are required");
    const WorkloadSpec spec = resolve_workload(a.get("--workload"));
    SaveOptions options;
    options.base_address = base_addr_from_env();
    SaveResult r = save(spec, a.get("--out"), options);
    if (a.has("--emit-json-graphs")) write_json_graphs(r.archive_dir);
    if (a.has("--traces")) spit(a.get("--traces"), traces_to_text(r.traces));
    uint64_t bytes = 0;
    for (const auto& e : fs::recursive_directory_iterator(r.archive_dir))
        if (e.is_regular_file()) bytes += e.file_size();
    std::cout << "archive written to " << r.archive_dir.string() << " (" << bytes << " bytes, "
              << r.manifest.grouping.total_graphs << " graphs, " << r.manifest.grouping.template_count
              << " templates)\n";
    return 0;
}

int cmd_load(const Args& a) {
    if (!a.has("--archive")) return usage("load: --archive is required");
    LoadOptions o;
    o.rank = static_cast<uint32_t>(std::stoul(a.get("--rank", "0")));
    o.world = static_cast<uint32_t>(std::stoul(a.get("--world", "1")));
    o.preallocate = !a.has("--no-prealloc");
    o.relocate = a.has("--relocate");
    o.share_execs = a.has("--share-execs");
    o.device_updates = a.has("--device-updates");
    o.device = std::stoi(a.get("--device", "0"));
    std::optional<ServingContext> held(load(a.get("--archive"), o));
    ServingContext& sc = *held;
    std::cout << "rank " << o.rank << "/" << o.world << " ready: " << sc.batches().size()
              << " batch sizes servable" << std::endl;  // flushed: callers time exec -> servable
    if (a.has("--replay-all")) {
        std::map<uint32_t, LaunchTrace> traces;
        for (uint32_t b : sc.batches()) traces.emplace(b, sc.replay(b));
        std::cout << "replayed " << traces.size() << " graphs\n";
        if (a.has("--traces")) spit(a.get("--traces"), traces_to_text(traces));
    }
    for (const auto& [key, value] : sc.counters()) std::cout << "  " << key << " = " << value << "\n";
    const auto t0 = std::chrono::steady_clock::now();
    held.reset();  // graphs, libraries, VA and the device context
    if (std::getenv("FOUNDRY_DEBUG"))
        std::cerr << "[foundry] teardown "
                  << std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count()
                  << " ms\n";
    return 0;
}

int cmd_inspect(const Args& a) {
    if (a.positional.size() != 1) return usage("inspect: one archive directory expected");
    if (a.has("--graph"))
        std::cout << inspect_graph_json(a.positional[0], static_cast<uint32_t>(std::stoul(a.get("--graph"))))
                  << "\n";
    else
        std::cout << inspect_text(a.positional[0]);
    return 0;
}

int cmd_diff(const Args& a) {
    if (a.positional.size() != 2) return usage("diff: two archive directories expected");
    const auto [identical, text] = diff_archives(a.positional[0], a.positional[1]);
    std::cout << text;
    return identical ? 0 : 1;
}

int cmd_bench(const Args& a) {
    if (!a.has("--workload")) return usage("bench: --workload is required");
    const std::string mode = a.get("--mode", "load");
    if (mode != "save" && mode != "load" && mode != "naive") return usage("bench: --mode save|load|naive");
    const auto r = bench(resolve_workload(a.get("--workload")), mode);
    // BenchReport::to_text (pipeline.cpp:831-845)
    std::cout << "mode: " << mode << "\n"
              << "wall time: " << r.at("wall_ms") << " ms\n"
              << "archive size: " << static_cast<uint64_t>(r.at("archive_bytes")) << " bytes\n"
              << "update-served fraction: " << r.at("update_served_fraction") << "\n"
              << "construction calls (graph mutation + instantiate): "
              << static_cast<uint64_t>(r.at("construction_calls")) << "\n"
              << "update calls: " << static_cast<uint64_t>(r.at("update_calls")) << "\n"
              << "capture calls: " << static_cast<uint64_t>(r.at("capture_calls")) << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage("a subcommand is required");
    const std::string cmd = argv[1];
    try {
        if (cmd == "save") return cmd_save(parse(argc, argv, {"--emit-json-graphs"}));
        if (cmd == "load")
            return cmd_load(parse(argc, argv, {"--no-prealloc", "--replay-all", "--relocate", "--share-execs",
                                               "--device-updates"}));
        if (cmd == "inspect") return cmd_inspect(parse(argc, argv, {}));
        if (cmd == "diff") return cmd_diff(parse(argc, argv, {}));
        if (cmd == "bench") return cmd_bench(parse(argc, argv, {}));
        return usage(("unknown subcommand " + cmd).c_str());
    } catch (const Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_code_for(e.code());
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
