// Per-rank execution context on a real B200: the counterpart of the
// reference's simulated DeviceContext (sim_driver.hpp:94-211) + VirtualRegion
// (det_alloc.hpp:61-95), built on the CUDA driver API.
//
//  * libraries:  one cuLibraryLoadData per cataloged binary (restore_binaries,
//                binary_catalog.cpp:200-227); device-side init sets the
//                module's init flag (run_device_init, sim_driver.cpp:90-98).
//  * region:     the deterministic VA range is a real reservation
//                (cuMemAddressReserve at the captured base) backed by
//                cuMemCreate/cuMemMap; the bump allocator, capture-window
//                replay and allocation records follow det_alloc.cpp:71-181
//                exactly. A logical per-granule map mirrors the reference's
//                mapped_ ranges and is mirrored to HBM for the trace kernels.
//  * relocation: if the reservation cannot land at the captured base (or a
//                fault shifts it), and relocation is enabled, the region's
//                logical base follows the real one and materialization
//                rebases embedded addresses (K1).
//  * counters:   same keys as the reference (sim_driver.cpp:483-503).
#pragma once

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <string>
#include <unordered_map>
#include <vector>

#include "foundry/archive.hpp"
#include "foundry/device.hpp"
#include "foundry/driver_api.hpp"
#include "foundry/trace_abi.h"

namespace foundry {

// Summed wall time and count of the driver calls GpuContext issues per kind
// (thread time: concurrent calls add up); diagnostics for FOUNDRY_DEBUG.
std::string driver_call_stats(bool reset);

using CounterSnapshot = std::map<std::string, uint64_t>;

class GpuContext {
public:
    explicit GpuContext(Device& dev);
    ~GpuContext();
    GpuContext(const GpuContext&) = delete;
    GpuContext& operator=(const GpuContext&) = delete;

    Device& device() { return dev_; }

    // ------------------------------------------------------------ libraries
    struct Kernel {
        CUkernel kern = nullptr;           // context-independent handle (graph nodes use this)
        mutable CUfunction fn = nullptr;   // loaded on demand, see function()
        mutable int max_dynamic_smem = 0;  // attribute values already applied
        mutable int carveout = -1;
        mutable bool loaded = false;       // function forced into the context (ensure_loaded)
        uint32_t library = 0;
        uint32_t entry_index = 0;
        uint32_t entry_id = 0;
        uint32_t arg_buffer_size = 0;
        std::vector<uint32_t> hidden_offsets;
        std::string name;
        uint64_t binary_hash = 0;
        FuncAttrs attrs;                   // the catalog entry's captured attributes
    };
    // A loaded library before registration: only driver calls, so several
    // host threads may open libraries concurrently (cuLibraryLoadData scales
    // with threads). Entry functions are not forced into the context here:
    // graph nodes reference the CUkernel and the driver loads each function
    // when a graph is instantiated (lazy loading).
    struct OpenedLibrary {
        CUlibrary lib = nullptr;
        CUdeviceptr ctx_global = 0;
        CUdeviceptr init_global = 0;
        std::vector<CUkernel> kernels;  // image.entrypoints order
    };
    OpenedLibrary open_library(const KernelImage& image, std::span<const uint8_t> cubin) const;
    // Registers an opened library and its entrypoints (single thread).
    uint32_t register_library(uint64_t hash, const KernelImage& image, OpenedLibrary&& opened,
                              uint32_t ordinal, bool requires_device_init);
    // open_library + register_library.
    uint32_t load_library(uint64_t hash, const KernelImage& image, std::span<const uint8_t> cubin,
                          uint32_t ordinal, bool requires_device_init);
    // The kernel's CUfunction in this context (cuKernelGetFunction on first use).
    CUfunction function(const Kernel& k) const;
    // Forces the (lazily loaded) function into the context now (cuFuncLoad),
    // so a later graph update or launch of it does not stall on the load.
    void ensure_loaded(const Kernel& k) const;
    void set_kernel_attribute(const Kernel& k, CUfunction_attribute attr, int value) const;
    // Per-kernel launch attributes, applied once: the dynamic shared memory
    // limit only ever grows (every node of the kernel must fit).
    void require_dynamic_smem(const Kernel& k, int bytes) const;
    void set_carveout(const Kernel& k, int percent) const;
    // cuFuncGetAttribute of the kernel's function in this context
    int function_attribute(const Kernel& k, CUfunction_attribute attr) const;
    void run_device_init(uint32_t library);
    bool library_device_inited(uint32_t library) const;
    bool library_requires_init(uint32_t library) const;
    const Kernel* find_kernel(uint64_t hash, std::string_view name) const;
    const Kernel* kernel_by_entry_id(uint32_t entry_id) const;
    // Reverse lookup for graph extraction: the restored kernel a node's
    // function (or context-independent kernel handle) belongs to.
    const Kernel* kernel_by_handle(CUfunction fn, CUkernel kern) const;
    bool has_library(uint64_t hash) const;

    // ------------------------------------------------------------ region
    // Reserves the VA range and backs [base, base + backed_bytes).
    void reserve_region(const RegionConfig& logical, uint64_t backed_bytes, bool allow_relocation);
    uint64_t region_base() const { return logical_.base; }      // where allocations land
    uint64_t captured_base() const { return captured_base_; }  // manifest base
    const RegionConfig& region_config() const { return logical_; }
    uint64_t allocate(uint64_t size);
    void free(uint64_t address);
    void preallocate(uint64_t final_offset);
    void begin_capture_window();
    void replay_capture_window(const MemoryEventLog& log);
    uint64_t offset() const { return offset_; }
    std::vector<AllocationRecord> records() const { return records_; }
    bool address_mapped(uint64_t addr) const;  // logical (reference mapped_ ranges)
    bool physically_backed(uint64_t addr) const {
        return addr >= phys_at_ && addr < phys_at_ + phys_bytes_;
    }
    uint64_t backing_base() const { return phys_at_; }
    uint64_t backed_bytes() const { return phys_bytes_; }
    void zero_region();  // cuMemsetD8 over the backed range (deterministic replay outputs)

    // ------------------------------------------------------------ trace
    // Device trace context (pointer published to every library's global).
    void ensure_trace_arena(uint64_t bytes);
    void sync_trace_state();  // upload mapping bitmap; publish ctx to libraries
    fdy_trace_ctx* device_trace_ctx() const { return d_ctx_; }
    void reset_trace();
    std::vector<uint8_t> read_trace();

    // ------------------------------------------------------------ counters
    std::atomic<uint64_t> c_reserve{0}, c_map{0}, c_unmap{0}, c_grants{0}, c_module_load{0},
        c_device_init{0}, c_add_node{0}, c_add_edge{0}, c_set_attr{0}, c_instantiate{0},
        c_update{0}, c_update_touched{0}, c_replay{0};
    CounterSnapshot counters() const;

private:
    struct Library {
        CUlibrary lib = nullptr;
        uint64_t hash = 0;
        bool requires_init = false;
        bool inited = false;
        CUdeviceptr ctx_global = 0;
        CUdeviceptr init_global = 0;
    };
    void mark(uint64_t addr, uint64_t len, bool on);

    Device& dev_;
    int cu_device_ = 0;
    mutable std::mutex fn_mu_;
    std::vector<Library> libs_;
    std::unordered_map<std::string, uint32_t> kernel_index_;  // hash|name -> kernels_
    std::vector<Kernel> kernels_;
    std::unordered_map<uint32_t, uint32_t> by_entry_id_;

    // region state
    RegionConfig logical_{};
    uint64_t captured_base_ = 0;
    CUdeviceptr va_ = 0;
    size_t va_bytes_ = 0;
    CUmemGenericAllocationHandle phys_ = 0;
    CUdeviceptr phys_at_ = 0;
    size_t phys_bytes_ = 0;
    bool reserved_ = false;
    uint64_t offset_ = 0;
    bool recording_window_ = false;
    std::optional<uint64_t> prealloc_limit_;
    std::vector<AllocationRecord> records_;
    std::vector<std::pair<uint64_t, uint64_t>> live_;
    std::vector<uint64_t> bitmap_;  // logical granule map
    bool bitmap_dirty_ = true;

    // trace state
    DeviceBuffer trace_arena_;
    DeviceBuffer trace_meta_;  // fdy_trace_ctx + cursor + bitmap
    fdy_trace_ctx* d_ctx_ = nullptr;
    unsigned long long* d_cursor_ = nullptr;
    uint64_t* d_bitmap_ = nullptr;
    std::vector<uint32_t> published_;  // libraries that already hold d_ctx_
};

}  // namespace foundry
