// Generation of per-binary trace cubins (see trace_module.hpp).
#include "foundry/trace_module.hpp"

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <sstream>
#include <cstring>
#include <unistd.h>

#include "foundry/bytes.hpp"
#include "foundry/parallel.hpp"

namespace foundry {

namespace fs = std::filesystem;

namespace {

// .entry wrappers only; the device body lives in a separately compiled object
// that nvlink links in once (a whole-program compile would clone the body
// into every entry and make large modules slow to build and load).
std::string entries_ptx(const KernelImage& image, uint32_t ordinal, bool needs_init) {
    std::ostringstream o;
    o << ".version 8.8\n.target sm_100a\n.address_size 64\n\n"
      << ".extern .func fdy_trace_body(.param .b64 a0, .param .b32 a1, .param .b64 a2, "
         ".param .b32 a3, .param .b32 a4, .param .b32 a5);\n";
    for (size_t i = 0; i < image.entrypoints.size(); ++i) {
        const KernelEntry& e = image.entrypoints[i];
        require(e.arg_buffer_size > 0 && e.arg_buffer_size <= 32764, Errc::binary_format,
                "entrypoint '" + e.name + "' has an argument buffer the device ABI cannot carry");
        const uint32_t entry_id = (ordinal << 16) | static_cast<uint32_t>(i);
        const std::string h = "fdy_hidden_" + std::to_string(i);
        if (!e.hidden_offsets.empty()) {
            o << ".global .align 4 .u32 " << h << "[" << e.hidden_offsets.size() << "] = {";
            for (size_t k = 0; k < e.hidden_offsets.size(); ++k) o << (k ? ", " : "") << e.hidden_offsets[k];
            o << "};\n";
        }
        o << ".visible .entry " << e.name << "(\n\t.param .align 8 .b8 " << e.name << "_param_0["
          << e.arg_buffer_size << "]\n)\n{\n"
          << "\t.reg .b64 %rd<5>;\n"
          << "\tmov.b64 %rd1, " << e.name << "_param_0;\n"
          << "\tcvta.param.u64 %rd2, %rd1;\n";
        if (!e.hidden_offsets.empty())
            o << "\tmov.u64 %rd3, " << h << ";\n\tcvta.global.u64 %rd4, %rd3;\n";
        else
            o << "\tmov.u64 %rd4, 0;\n";
        o << "\t{\n\t.param .b64 p0;\n\t.param .b32 p1;\n\t.param .b64 p2;\n\t.param .b32 p3;\n"
          << "\t.param .b32 p4;\n\t.param .b32 p5;\n"
          << "\tst.param.b64 [p0], %rd2;\n\tst.param.b32 [p1], " << e.arg_buffer_size << ";\n"
          << "\tst.param.b64 [p2], %rd4;\n\tst.param.b32 [p3], " << e.hidden_offsets.size() << ";\n"
          << "\tst.param.b32 [p4], " << entry_id << ";\n\tst.param.b32 [p5], " << (needs_init ? 1 : 0)
          << ";\n\tcall.uni fdy_trace_body, (p0, p1, p2, p3, p4, p5);\n\t}\n\tret;\n}\n";
    }
    return o.str();
}

std::string cuda_tool(const char* name) {
    const char* home = std::getenv("CUDA_HOME");
    return std::string(home ? home : "/usr/local/cuda") + "/bin/" + name;
}

struct TempDir {
    fs::path path;
    TempDir() {
        char dir[] = "/tmp/fdy_ptx_XXXXXX";
        require(mkdtemp(dir) != nullptr, Errc::invalid_argument, "cannot create a temp dir for ptxas");
        path = dir;
    }
    ~TempDir() {
        std::error_code ec;
        fs::remove_all(path, ec);
    }
};

void run_tool(const std::string& cmd, const fs::path& log) {
    if (std::system((cmd + " > '" + log.string() + "' 2>&1").c_str()) != 0) {
        std::string err;
        if (fs::exists(log)) {
            const auto l = slurp(log);
            err.assign(l.begin(), l.end());
        }
        raise(Errc::binary_format, "device code generation failed: " + err.substr(0, 2000));
    }
}

// Relocatable object of the shared device body, built once per process.
const fs::path& body_object() {
    static std::once_flag once;
    static fs::path obj;
    static TempDir dir;
    std::call_once(once, [] {
        const fs::path ptx = dir.path / "body.ptx";
        obj = dir.path / "body.o";
        spit(ptx, std::string_view(trace_body_ptx()));
        run_tool("'" + cuda_tool("ptxas") + "' -arch=sm_100a -O3 -c '" + ptx.string() + "' -o '" +
                     obj.string() + "'",
                 dir.path / "body.log");
    });
    return obj;
}

fs::path cache_dir() {
    if (const char* env = std::getenv("FOUNDRY_CUBIN_CACHE")) return env;
    return {};
}

}  // namespace

std::string trace_module_ptx(const KernelImage& image, uint32_t ordinal, bool needs_init) {
    return entries_ptx(image, ordinal, needs_init);
}

std::vector<uint8_t> compile_ptx_to_cubin(const std::string& entries) {
    // content-addressed cache (optional): identical binaries compile once
    const uint64_t key = crc64(entries.data(), entries.size()) ^
                         (crc64(trace_body_ptx(), std::strlen(trace_body_ptx())) * 0x9E3779B97F4A7C15ull);
    const fs::path cache = cache_dir();
    if (!cache.empty()) {
        const fs::path hit = cache / (hex16(key) + ".cubin");
        if (fs::exists(hit)) return slurp(hit);
    }
    TempDir dir;
    const fs::path in = dir.path / "m.ptx", obj = dir.path / "m.o", out = dir.path / "m.cubin";
    spit(in, entries);
    run_tool("'" + cuda_tool("ptxas") + "' -arch=sm_100a -O3 -c '" + in.string() + "' -o '" +
                 obj.string() + "'",
             dir.path / "ptxas.log");
    run_tool("'" + cuda_tool("nvlink") + "' -arch=sm_100a '" + body_object().string() + "' '" +
                 obj.string() + "' -o '" + out.string() + "'",
             dir.path / "nvlink.log");
    auto cubin = slurp(out);
    if (!cache.empty()) {
        std::error_code ec;
        fs::create_directories(cache, ec);
        const fs::path tmp = cache / (hex16(key) + ".tmp" + std::to_string(::getpid()));
        spit(tmp, cubin);
        fs::rename(tmp, cache / (hex16(key) + ".cubin"), ec);
    }
    return cubin;
}

void write_trace_cubins(const fs::path& archive, unsigned threads) {
    ArchivePaths paths{archive};
    const auto mt = slurp(paths.manifest());
    Manifest m = parse_manifest(std::string(mt.begin(), mt.end()));
    const Catalog cat = parse_catalog(slurp(paths.catalog()));
    std::vector<const KernelBinaryRecord*> recs;
    for (const auto& [hash, r] : cat.binaries) recs.push_back(&r);
    std::vector<uint64_t> digests(recs.size());
    parallel_for(recs.size(), threads ? threads : default_threads(), [&](size_t i) {
        const KernelBinaryRecord& r = *recs[i];
        const KernelImage img = parse_kernel_image(slurp(paths.binary(r.hash)));
        const auto cubin = compile_ptx_to_cubin(
            trace_module_ptx(img, static_cast<uint32_t>(i), r.needs_device_init));
        spit(paths.cubin(r.hash), cubin);
        digests[i] = crc64(cubin);
    });
    for (size_t i = 0; i < recs.size(); ++i)
        m.file_digests["binaries/" + hex16(recs[i]->hash) + ".sm_100a.cubin"] = digests[i];
    spit(paths.manifest(), serialize_manifest(m));
}

}  // namespace foundry
