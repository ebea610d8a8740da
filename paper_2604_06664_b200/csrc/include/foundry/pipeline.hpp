// LOAD: the drop-in entry point of the B200 build.
//
// Signatures and semantics mirror the reference (pipeline.hpp:73-119,
// pipeline.cpp:447-569): load(archive, LoadOptions) -> ServingContext whose
// replay(batch) returns the LaunchTrace of that batch's graph. What happens
// underneath is B200-native:
//
//   stage     every manifest-listed file is read (prepare_lanes host threads)
//             into pinned staging and DMAed to HBM in one copy
//   verify    GPU CRC-64/XZ of every file against the manifest digests
//             (verify_archive_integrity, pipeline.cpp:411-417)
//   restore   cuLibraryLoadData of each cataloged binary's sm_100a cubin;
//             device-side init where flagged (restore_binaries)
//   region    real VA reservation at the captured base + physical backing
//             (VirtualRegion + preallocate, det_alloc.cpp)
//   prepare   ONE fused K2+K1+K3 kernel materializes every member graph of
//             this rank in HBM straight from the template store (the GPU
//             replacement of PrepareFn, pipeline.cpp:506-514); member images
//             stream back to pinned host memory for the driver
//   build     one cuGraph per topology group, instantiated once
//             (ServingSet::build, templater.cpp:70-159) — concurrently with
//   fore      the deterministic init plan + capture-window replay on the
//             region (pipeline.cpp:527-542)
//
// serve(b) applies member b to its group's exec with per-node
// cuGraphExec*SetParams on exactly the nodes whose parameters differ
// (ServingSet::serve, templater.cpp:177-188); replay(b) launches the exec and
// verifies the on-device trace records against the expected launches.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "foundry/archive.hpp"
#include "foundry/gpu_context.hpp"
#include "foundry/save.hpp"

namespace foundry {

struct FaultInjection {
    bool skip_binary_restore = false;
    bool skip_device_init = false;
    int64_t base_shift_granules = 0;
    bool extra_prewindow_alloc = false;
    // B200 addition: the device serve kernel reports every update as failed
    // (exercises the error word replay() checks; device_updates only)
    bool fail_device_serve = false;
};

struct LoadOptions {
    uint32_t rank = 0;
    uint32_t world = 1;
    bool preallocate = true;
    unsigned prepare_lanes = 4;  // host threads staging archive files
    FaultInjection faults;
    // --- B200 additions (defaults keep reference behaviour) ---
    int device = 0;
    bool relocate = false;       // rebase embedded addresses if the VA region moves
    bool verify_replay = true;   // check on-device trace records at replay
    // Templates whose CUDA graphs have the same shape (node types, edges and the
    // launch attributes the build applies) share ONE instantiated exec; serve()
    // switches it between them with cuGraphExec*NodeSetParams on the nodes that
    // differ. Cold start pays one cuGraphInstantiate per shape instead of one per
    // template (the driver-bound part of LOAD); a serve that crosses templates
    // pays a larger update. Off = the reference's one exec per template.
    bool share_execs = false;
    // Kernel nodes are built device-updatable: serve() applies a member from
    // the GPU (kernels/serve.cu: cudaGraphKernelNodeSetParam / SetGridDim
    // straight from the HBM member images, one thread per node); only memcpy /
    // memset nodes (and any node whose function, block or shared memory would
    // change) go through the host. Excludes share_execs.
    bool device_updates = false;
    // This rank's communication state for the archive's comm slots
    // (comm_slots.bin, archive.hpp: comm handles, peer buffer addresses, ...);
    // at least the store's n_values entries when the archive carries slots.
    std::vector<uint64_t> comm_values;
};

// Wall/kernel time of each LOAD phase (milliseconds) and the DMA volume.
struct LoadTimings {
    double total_ms = 0, manifest_ms = 0, stage_ms = 0, integrity_ms = 0, restore_ms = 0,
           region_ms = 0, materialize_ms = 0, download_ms = 0, build_ms = 0, instantiate_ms = 0,
           foreground_ms = 0,
           function_load_ms = 0,  // share_execs: loading the functions of exec-sharing templates
           pack_ms = 0;           // reference-written archive: the GPU packer (graphs.bin -> store)
    float crc_kernel_ms = 0, materialize_kernel_ms = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0, member_bytes = 0, store_bytes = 0;
    uint64_t graphs = 0, nodes = 0, templates = 0;
    uint64_t relocation_delta = 0;
};

class ServingContext {
public:
    ServingContext(ServingContext&&) noexcept;
    ServingContext& operator=(ServingContext&&) noexcept;
    ~ServingContext();

    LaunchTrace replay(uint32_t batch);
    std::vector<uint32_t> batches() const;
    const Manifest& manifest() const;
    std::vector<AllocationRecord> allocation_records() const;
    CounterSnapshot counters() const;
    GpuContext& context();
    const LoadTimings& timings() const;

    // B200 extras
    uint32_t template_count() const;
    // The prepared (materialized) parameter set of a batch, decoded from the
    // member image the GPU produced (ServingSet::prepared_params analogue).
    CapturedGraph prepared_params(uint32_t batch) const;
    // In-place update of a group's exec from an arbitrary donor graph; the
    // topology must match (DeviceContext::exec_update, sim_driver.cpp:365-398).
    void exec_update(uint32_t batch_in_group, const CapturedGraph& donor);
    // serve(b) only (no launch); returns the number of nodes touched.
    uint64_t serve(uint32_t batch);
    // The naive comparator (reference bench "naive", pipeline.cpp:890-918):
    // build, instantiate and launch a separate graph for EVERY member, no
    // templates. Returns the construction calls issued (nodes+edges+attrs+inst).
    uint64_t naive_rebuild_all();

    // "Replaying the materialized graphs must reproduce the outputs of freshly
    // captured graphs": runs batch b once through the materialized exec and
    // once through a graph stream-captured from the same launches, each from a
    // zeroed region, and compares the device trace records and a GPU CRC-64 of
    // the whole region. Returns true when both agree (details in *report).
    bool fresh_capture_check(uint32_t batch, std::string* report = nullptr);
    // GPU-side SAVE: stream-captures batch's materialized work
    // with the template's dependencies (cudaStreamUpdateCaptureDependencies per
    // node) and extracts the driver's graph back into the portable model.
    CapturedGraph capture_graph(uint32_t batch);
    // GPU-side SAVE to an archive: capture_graph of every batch, comm nodes
    // lowered back to stubs, grouped, serialized and written with the catalog,
    // memory log, patch table, binaries and a packed template store. The
    // archive loads in the reference and here. Needs a LOAD at the captured
    // base and no comm slots.
    SaveResult save_captured(const std::filesystem::path& out);

    struct Impl;

private:
    friend ServingContext load(Device&, const std::filesystem::path&, const LoadOptions&);
    friend ServingContext load(const std::filesystem::path&, const LoadOptions&);
    explicit ServingContext(std::unique_ptr<Impl> impl);
    std::unique_ptr<Impl> impl_;
};

ServingContext load(const std::filesystem::path& archive, const LoadOptions& options = {});
// Several ranks sharing one device (the reference's shared-SimDriver overload,
// pipeline.hpp:118-119).
ServingContext load(Device& device, const std::filesystem::path& archive,
                    const LoadOptions& options = {});

}  // namespace foundry
