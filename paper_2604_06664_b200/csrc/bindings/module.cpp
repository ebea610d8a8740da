// pybind11 module `_foundry`: the reference's Python surface (reference
// proj/bindings/module.cpp:77-135, python/foundry/__init__.py:7-41) backed by
// the B200 runtime. Names, argument names/defaults and return shapes match the
// reference; B200-only knobs are extra keyword arguments with defaults that
// keep reference behaviour.
#include <cstring>

#include <pybind11/pybind11.h>
#include <pybind11/stl.h>
#include <pybind11/stl/filesystem.h>

#include <chrono>

#include "foundry/bytes.hpp"
#include "foundry/device_pack.hpp"
#include "foundry/pipeline.hpp"
#include "foundry/save.hpp"
#include "foundry/template_store.hpp"
#include "foundry/tooling.hpp"
#include "foundry/workload.hpp"

namespace py = pybind11;
using namespace foundry;

namespace {

struct SaveOutcome {
    std::string archive_dir;
    std::map<uint32_t, std::string> traces;
    std::map<std::string, uint64_t> counters;
    uint32_t total_graphs = 0;
    uint32_t template_count = 0;
    double update_served_fraction = 0.0;
    // (sequence, size, address, length, window) per allocation, SAVE's capture-time layout
    std::vector<std::tuple<uint64_t, uint64_t, uint64_t, uint64_t, int>> allocation_records;
};

std::vector<std::tuple<uint64_t, uint64_t, uint64_t, uint64_t, int>> records_tuples(
    const std::vector<AllocationRecord>& rs) {
    std::vector<std::tuple<uint64_t, uint64_t, uint64_t, uint64_t, int>> out;
    for (const auto& r : rs) out.emplace_back(r.sequence, r.size, r.address, r.length, static_cast<int>(r.window));
    return out;
}

struct ServingHandle {
    explicit ServingHandle(ServingContext&& s) : sc(std::make_unique<ServingContext>(std::move(s))) {}
    ServingContext& ctx() const {
        require(sc != nullptr, Errc::invalid_argument, "serving handle is closed");
        return *sc;
    }
    void close() { sc.reset(); }
    std::string replay(uint32_t batch) { return ctx().replay(batch).to_text(); }
    std::vector<uint32_t> batches() const { return ctx().batches(); }
    std::map<std::string, uint64_t> counters() const {
        const auto c = ctx().counters();
        return {c.begin(), c.end()};
    }
    uint32_t template_count() const { return ctx().template_count(); }
    py::dict timings() const {
        const LoadTimings& t = ctx().timings();
        py::dict d;
        d["total_ms"] = t.total_ms;
        d["manifest_ms"] = t.manifest_ms;
        d["stage_ms"] = t.stage_ms;
        d["integrity_ms"] = t.integrity_ms;
        d["restore_ms"] = t.restore_ms;
        d["region_ms"] = t.region_ms;
        d["materialize_ms"] = t.materialize_ms;
        d["download_ms"] = t.download_ms;
        d["build_ms"] = t.build_ms;
        d["function_load_ms"] = t.function_load_ms;
        d["pack_ms"] = t.pack_ms;
        d["instantiate_ms"] = t.instantiate_ms;
        d["foreground_ms"] = t.foreground_ms;
        d["crc_kernel_ms"] = t.crc_kernel_ms;
        d["materialize_kernel_ms"] = t.materialize_kernel_ms;
        d["h2d_bytes"] = t.h2d_bytes;
        d["d2h_bytes"] = t.d2h_bytes;
        d["member_bytes"] = t.member_bytes;
        d["store_bytes"] = t.store_bytes;
        d["graphs"] = t.graphs;
        d["nodes"] = t.nodes;
        d["templates"] = t.templates;
        d["relocation_delta"] = t.relocation_delta;
        return d;
    }
    py::bytes prepared_record(uint32_t batch) const {
        const auto rec = encode_graph_record(ctx().prepared_params(batch));
        return py::bytes(reinterpret_cast<const char*>(rec.data()), rec.size());
    }
    uint64_t serve(uint32_t batch) { return ctx().serve(batch); }
    uint64_t region_base() { return ctx().context().region_base(); }
    py::tuple fresh_capture_check(uint32_t batch) {
        std::string rep;
        bool ok;
        {
            py::gil_scoped_release nogil;
            ok = ctx().fresh_capture_check(batch, &rep);
        }
        return py::make_tuple(ok, rep);
    }
    // GPU-side SAVE: the FNDG record (encode_graph_record) of batch's graph as
    // stream-captured on the device and extracted back from the driver
    py::bytes capture_graph(uint32_t batch) {
        std::vector<uint8_t> rec;
        {
            py::gil_scoped_release nogil;
            rec = encode_graph_record(ctx().capture_graph(batch));
        }
        return py::bytes(reinterpret_cast<const char*>(rec.data()), rec.size());
    }
    // reference DeviceContext::exec_update (sim_driver.cpp:365-398): apply a
    // donor graph (FNDG record bytes) to the exec serving batch's template;
    // a different topology raises topology-mismatch
    void exec_update(uint32_t batch, py::bytes donor) {
        const std::string b = donor;
        const CapturedGraph g = decode_graph_record(
            std::span<const uint8_t>(reinterpret_cast<const uint8_t*>(b.data()), b.size()));
        py::gil_scoped_release nogil;
        ctx().exec_update(batch, g);
    }
    uint64_t naive_rebuild_all() {
        py::gil_scoped_release nogil;
        return ctx().naive_rebuild_all();
    }
    // GPU-side SAVE to an archive directory; returns (graphs, templates)
    py::tuple save_captured(const std::string& out) {
        SaveResult r;
        {
            py::gil_scoped_release nogil;
            r = ctx().save_captured(out);
        }
        return py::make_tuple(r.manifest.grouping.total_graphs, r.manifest.grouping.template_count);
    }
    std::unique_ptr<ServingContext> sc;
};

SaveOutcome do_save(const WorkloadSpec& spec, const std::string& out, bool emit_json_graphs,
                    bool b200_artifacts) {
    SaveOptions o;
    o.b200_artifacts = b200_artifacts;
    SaveResult r;
    {
        py::gil_scoped_release nogil;
        r = save(spec, out, o);
        if (emit_json_graphs) write_json_graphs(out);
    }
    SaveOutcome s;
    s.archive_dir = r.archive_dir.string();
    for (const auto& [b, t] : r.traces) s.traces.emplace(b, t.to_text());
    s.counters = save_counters(spec);
    s.total_graphs = r.manifest.grouping.total_graphs;
    s.template_count = r.manifest.grouping.template_count;
    s.update_served_fraction = r.manifest.grouping.update_served_fraction();
    s.allocation_records = records_tuples(r.allocation_records);
    return s;
}

ServingHandle do_load(const std::string& archive, uint32_t rank, uint32_t world, bool preallocate,
                      int device, bool relocate, unsigned prepare_lanes, bool skip_binary_restore,
                      bool skip_device_init, int64_t base_shift_granules, bool extra_prewindow_alloc,
                      bool verify_replay, bool share_execs, bool device_updates,
                      std::vector<uint64_t> comm_values, bool fail_device_serve) {
    LoadOptions o;
    o.rank = rank;
    o.world = world;
    o.preallocate = preallocate;
    o.device = device;
    o.relocate = relocate;
    o.prepare_lanes = prepare_lanes;
    o.verify_replay = verify_replay;
    o.share_execs = share_execs;
    o.device_updates = device_updates;
    o.comm_values = std::move(comm_values);
    o.faults.skip_binary_restore = skip_binary_restore;
    o.faults.skip_device_init = skip_device_init;
    o.faults.base_shift_granules = base_shift_granules;
    o.faults.extra_prewindow_alloc = extra_prewindow_alloc;
    o.faults.fail_device_serve = fail_device_serve;
    py::gil_scoped_release nogil;
    return ServingHandle(load(archive, o));
}

}  // namespace

PYBIND11_MODULE(_foundry, m) {
    m.doc() = "B200-native LOAD of template-based CUDA graph archives (Foundry drop-in)";
    m.attr("__version__") = "0.1.0";

    // FoundryError carries e.what(); a message that quotes bytes from a corrupt
    // archive (a kernel name) need not be UTF-8, so it is decoded with
    // backslash escapes instead of failing the conversion
    static PyObject* foundry_error = py::exception<Error>(m, "FoundryError").inc_ref().ptr();
    py::register_exception_translator([](std::exception_ptr p) {
        try {
            if (p) std::rethrow_exception(p);
        } catch (const Error& e) {
            const char* w = e.what();
            PyObject* msg = PyUnicode_DecodeUTF8(w, static_cast<Py_ssize_t>(std::strlen(w)), "backslashreplace");
            PyErr_SetObject(foundry_error, msg);
            Py_XDECREF(msg);
        }
    });

    py::class_<WorkloadSpec>(m, "WorkloadSpec")
        .def(py::init<>())
        .def_readwrite("seed", &WorkloadSpec::seed)
        .def_readwrite("batch_max", &WorkloadSpec::batch_max)
        .def_readwrite("layers", &WorkloadSpec::layers)
        .def_readwrite("kernels_per_layer", &WorkloadSpec::kernels_per_layer)
        .def_readwrite("thresholds", &WorkloadSpec::thresholds)
        .def_readwrite("collectives_per_layer", &WorkloadSpec::collectives_per_layer)
        .def_readwrite("hidden_offset_density", &WorkloadSpec::hidden_offset_density)
        .def("__repr__", [](const WorkloadSpec& s) {
            return "<WorkloadSpec B=" + std::to_string(s.batch_max) + " L=" + std::to_string(s.layers) + ">";
        });

    py::class_<SaveOutcome>(m, "SaveOutcome")
        .def_readonly("archive_dir", &SaveOutcome::archive_dir)
        .def_readonly("traces", &SaveOutcome::traces)
        .def_readonly("counters", &SaveOutcome::counters)
        .def_readonly("total_graphs", &SaveOutcome::total_graphs)
        .def_readonly("template_count", &SaveOutcome::template_count)
        .def_readonly("update_served_fraction", &SaveOutcome::update_served_fraction)
        .def_readonly("allocation_records", &SaveOutcome::allocation_records);

    py::class_<ServingHandle>(m, "ServingHandle")
        .def("replay", &ServingHandle::replay, py::arg("batch"), py::call_guard<py::gil_scoped_release>())
        .def("batches", &ServingHandle::batches)
        .def("allocation_records",
             [](ServingHandle& h) { return records_tuples(h.ctx().allocation_records()); },
             "(sequence, size, address, length, window) per allocation of the rank's region")
        .def("counters", &ServingHandle::counters)
        .def("template_count", &ServingHandle::template_count)
        .def("timings", &ServingHandle::timings)
        .def("prepared_record", &ServingHandle::prepared_record, py::arg("batch"))
        .def("serve", &ServingHandle::serve, py::arg("batch"), py::call_guard<py::gil_scoped_release>())
        .def("region_base", &ServingHandle::region_base)
        .def("fresh_capture_check", &ServingHandle::fresh_capture_check, py::arg("batch"))
        .def("capture_graph", &ServingHandle::capture_graph, py::arg("batch"),
             "GPU-side SAVE: stream-capture the batch's graph and extract it (FNDG record bytes)")
        .def("naive_rebuild_all", &ServingHandle::naive_rebuild_all)
        .def("save_captured", &ServingHandle::save_captured, py::arg("out"),
             "GPU-side SAVE: capture every batch on the device and write a reference-layout archive")
        .def("exec_update", &ServingHandle::exec_update, py::arg("batch"), py::arg("donor"),
             "Apply a donor graph (FNDG record bytes) to the exec of batch's template")
        .def("close", &ServingHandle::close, "Release the rank's graphs, libraries and VA region now")
        .def("__enter__", [](py::object self) { return self; })
        .def("__exit__", [](ServingHandle& h, py::args) { h.close(); });

    m.def("preset_names", &preset_names);
    m.def("preset", &preset, py::arg("name"));
    m.def("workload_from_text", [](const std::string& t) { return WorkloadSpec::parse_text(t); },
          py::arg("text"));
    m.def("spec_text", [](const WorkloadSpec& s) { return s.canonical_text(); }, py::arg("spec"));
    m.def("save", &do_save, py::arg("spec"), py::arg("out"), py::arg("emit_json_graphs") = false,
          py::arg("b200_artifacts") = true);
    m.def("load", &do_load, py::arg("archive"), py::arg("rank") = 0, py::arg("world") = 1,
          py::arg("preallocate") = true, py::arg("device") = 0, py::arg("relocate") = false,
          py::arg("prepare_lanes") = 4, py::arg("skip_binary_restore") = false,
          py::arg("skip_device_init") = false, py::arg("base_shift_granules") = 0,
          py::arg("extra_prewindow_alloc") = false, py::arg("verify_replay") = true,
          py::arg("share_execs") = false, py::arg("device_updates") = false,
          py::arg("comm_values") = std::vector<uint64_t>{}, py::arg("fail_device_serve") = false);
    // The stub layer's comm-slot authoring (archive.hpp CommSlotTable): writes
    // comm_slots.bin, records its digest in the manifest and re-packs the
    // template store if the archive has one.
    m.def("write_comm_slots", [](const std::string& archive, uint32_t n_values,
                                 const std::map<uint32_t, std::vector<std::tuple<uint32_t, uint32_t, uint32_t, uint8_t>>>& slots) {
        CommSlotTable t;
        t.n_values = n_values;
        for (const auto& [label, list] : slots)
            for (const auto& [node, off, idx, width] : list) t.per_graph[label].push_back(CommSlot{node, off, idx, width});
        py::gil_scoped_release nogil;
        write_comm_slots(archive, t);
    }, py::arg("archive"), py::arg("n_values"), py::arg("slots"));
    m.def("pack", [](const std::string& archive) {
        py::gil_scoped_release nogil;
        pack_archive(archive);
    }, py::arg("archive"));
    m.def("pack_archive", [](const std::string& dir, const std::string& file) {
        py::gil_scoped_release nogil;
        pack_archive_file(dir, file);
    }, py::arg("archive"), py::arg("file"), "Single-file FNDA archive (reference pack_archive)");
    m.def("unpack_archive", [](const std::string& file, const std::string& dir) {
        py::gil_scoped_release nogil;
        unpack_archive_file(file, dir);
    }, py::arg("file"), py::arg("archive"), "Inverse of pack_archive (reference unpack_archive)");
    m.def("inspect_text", [](const std::string& a) { return inspect_text(a); }, py::arg("archive"));
    m.def("inspect_graph_json", [](const std::string& a, uint32_t b) { return inspect_graph_json(a, b); },
          py::arg("archive"), py::arg("batch"));
    m.def("diff_archives",
          [](const std::string& a, const std::string& b) {
              const auto r = diff_archives(a, b);
              return py::make_tuple(r.first, r.second);
          },
          py::arg("a"), py::arg("b"));
    m.def("bench", [](const WorkloadSpec& spec, const std::string& mode) {
        py::gil_scoped_release nogil;
        return bench(spec, mode);
    }, py::arg("spec"), py::arg("mode") = "load");
    m.def("cuda_device_count", &cuda_device_count);

    // --- internals used by the test-suite (not part of the reference surface) ---
    m.def("_crc64", [](py::bytes b) {
        const std::string s = b;
        return crc64(s.data(), s.size());
    });
    m.def("_crc64_combine", &crc64_combine);
    m.def("_manifest_fast_path_agrees", [](const std::string& text) { return manifest_fast_path_agrees(text); });
    m.def("_pack_store", [](const std::string& archive) {
        py::gil_scoped_release nogil;
        const PackStats st = pack_archive_store(archive);
        return std::map<std::string, uint64_t>{{"store_bytes", st.store_bytes},
                                               {"template_bytes", st.template_bytes},
                                               {"diff_entries", st.diff_entries},
                                               {"rank_ops", st.rank_ops},
                                               {"member_image_bytes", st.member_image_bytes}};
    });
    // The template store of an archive as bytes, packed on the host
    // (pack_template_store) or on the GPU (pack_template_store_device, from a
    // device copy of graphs.bin); with the GPU packer's phase timings.
    m.def("_pack_store_bytes", [](const std::string& archive, bool gpu, int device) {
        ArchivePaths paths{archive};
        std::vector<uint8_t> out;
        std::map<std::string, double> t;
        {
            py::gil_scoped_release nogil;
            if (!gpu) {
                const auto mtext = slurp(paths.manifest());
                const Manifest man = parse_manifest(std::string(mtext.begin(), mtext.end()));
                const bool has_slots = man.file_digests.count("comm_slots.bin") != 0;
                out = pack_template_store(slurp(paths.graphs()), slurp(paths.patch_table()), man, 0, nullptr,
                                          has_slots ? slurp(paths.comm_slots()) : std::vector<uint8_t>{});
            } else {
                Device dev(device);
                DevicePackTimings tm;
                out = pack_archive_store_device(dev, archive, &tm);
                t = {{"prep_ms", tm.prep_ms}, {"patch_parse_ms", tm.patch_parse_ms}, {"tiles_ms", tm.tiles_ms}, {"layout_ms", tm.layout_ms}, {"checks_ms", tm.checks_ms},
                     {"kernel_table_ms", tm.kernel_table_ms}, {"rank_ops_ms", tm.rank_ops_ms}, {"pass1_ms", tm.pass1_ms}, {"pass1_upload_ms", tm.pass1_upload_ms}, {"pass1_launch_ms", tm.pass1_launch_ms}, {"pass1_sync_ms", tm.pass1_sync_ms}, {"host1_ms", tm.host1_ms}, {"pass2_ms", tm.pass2_ms},
                     {"host2_ms", tm.host2_ms}, {"pass3_ms", tm.pass3_ms}, {"total_ms", tm.total_ms},
                     {"kernel_keys", double(tm.kernel_keys)}, {"retries", double(tm.retries)}};
            }
        }
        return py::make_tuple(py::bytes(reinterpret_cast<const char*>(out.data()), out.size()), t);
    }, py::arg("archive"), py::arg("gpu") = true, py::arg("device") = 0);
    // parse_patch_view against parse_patch_table: the same entries (or the same
    // error) for a patch.bin's bytes
    m.def("_patch_view_matches_table", [](py::bytes raw) {
        const std::string b = raw;
        const std::span<const uint8_t> bytes(reinterpret_cast<const uint8_t*>(b.data()), b.size());
        const PatchTable t = parse_patch_table(bytes);  // raises like the reference
        const PatchView v = parse_patch_view(bytes);
        if (v.world_placeholder != t.world_placeholder || v.graphs.size() != t.per_graph.size()) return false;
        for (const auto& [label, entries] : t.per_graph) {
            if (!v.has(label)) return false;
            const auto got = v.find(label);
            if (got.size() != entries.size()) return false;
            for (size_t i = 0; i < entries.size(); ++i) {
                const CommPatchEntry& e = entries[i];
                const PatchEntryView& g = got[i];
                if (g.node_id != e.node_id || g.stub_hash != e.stub.binary_hash || g.stub_name != e.stub.name ||
                    g.real_name != e.real_name || g.n_rank != e.rank_offsets.size() ||
                    g.n_world != e.world_offsets.size() || g.patch_width != e.patch_width)
                    return false;
                for (uint32_t k = 0; k < g.n_rank; ++k)
                    if (g.rank_offset(k) != e.rank_offsets[k]) return false;
                for (uint32_t k = 0; k < g.n_world; ++k)
                    if (g.world_offset(k) != e.world_offsets[k]) return false;
            }
        }
        return true;
    });
    m.def("_parse_patch_view", [](py::bytes raw) {
        const std::string b = raw;
        (void)parse_patch_view({reinterpret_cast<const uint8_t*>(b.data()), b.size()});
    });
    // member-image arena (the kernel's output layout) -> FNDG container in
    // graphs.bin locator order
    m.def("_decode_member_images", [](const std::string& archive, py::bytes arena_bytes) {
        const std::string arena = arena_bytes;
        ArchivePaths paths{archive};
        const auto blob = slurp(paths.template_store());
        StoreView view(blob);
        const auto graphs_bin = slurp(paths.graphs());
        std::vector<CapturedGraph> out;
        for (const auto& loc : parse_graph_locators(graphs_bin)) {
            const int64_t mi = view.member_of(loc.label);
            require(mi >= 0, Errc::archive_corruption, "store has no member " + std::to_string(loc.label));
            const auto& M = view.member(static_cast<uint32_t>(mi));
            const auto& G = view.group(M.group);
            require(M.out_off + G.image_bytes <= arena.size(), Errc::invalid_argument, "arena too small");
            out.push_back(view.image_to_graph(
                static_cast<uint32_t>(mi),
                {reinterpret_cast<const uint8_t*>(arena.data()) + M.out_off, G.image_bytes}));
        }
        const auto c = serialize_graphs(out);
        return py::bytes(reinterpret_cast<const char*>(c.data()), c.size());
    });
}
