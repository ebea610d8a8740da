// B200 device runtime: one CUDA device, its streams, HBM buffers, and the
// launches of the sm_100a kernels (materialize, CRC-64). No CPU fallback:
// every entry point raises Errc::device_unavailable when no GPU/driver exists.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "foundry/archive.hpp"
#include "foundry/errors.hpp"
#include "foundry/store_format.h"

typedef struct CUstream_st* cudaStream_t;
typedef struct CUevent_st* cudaEvent_t;

namespace foundry {

// Raises Errc::cuda_error (or device_unavailable) for a failed runtime call.
void cuda_check(int err, const char* what);
bool cuda_available();
int cuda_device_count();

class Device {
public:
    explicit Device(int ordinal);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    int ordinal() const { return ordinal_; }
    int sm_count() const { return sm_count_; }
    cudaStream_t stream() const { return stream_; }
    cudaStream_t copy_stream() const { return copy_stream_; }
    cudaStream_t side_stream() const { return side_stream_; }  // integrity CRC work
    void make_current() const;
    void sync() const;

    // HBM. Ordinary buffers come from the device's stream-ordered pool
    // (cudaMallocAsync on stream(); the pool keeps freed memory, so a second
    // LOAD / prepare in the process does not pay cudaMalloc + cudaFree of
    // ~400 MB again). `shareable` buffers (CUDA IPC export) use cudaMalloc.
    void* alloc(size_t bytes, bool shareable = false);
    void release(void* p, bool shareable = false);
    void* alloc_host_pinned(size_t bytes);
    void release_host_pinned(void* p);

private:
    int ordinal_;
    int sm_count_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaStream_t copy_stream_ = nullptr;
    cudaStream_t side_stream_ = nullptr;
};

// Device-resident buffer with RAII release.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    DeviceBuffer(Device& dev, size_t bytes, bool shareable = false);
    ~DeviceBuffer();
    DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;

    unsigned char* data() const { return p_; }
    size_t size() const { return n_; }
    Device* device() const { return dev_; }

private:
    Device* dev_ = nullptr;
    unsigned char* p_ = nullptr;
    size_t n_ = 0;
    bool shareable_ = false;
};

class PinnedBuffer {
public:
    PinnedBuffer() = default;
    PinnedBuffer(Device& dev, size_t bytes);
    ~PinnedBuffer();
    PinnedBuffer(PinnedBuffer&& o) noexcept { *this = std::move(o); }
    PinnedBuffer& operator=(PinnedBuffer&& o) noexcept;
    PinnedBuffer(const PinnedBuffer&) = delete;
    PinnedBuffer& operator=(const PinnedBuffer&) = delete;

    unsigned char* data() const { return p_; }
    size_t size() const { return n_; }

private:
    Device* dev_ = nullptr;
    unsigned char* p_ = nullptr;
    size_t n_ = 0;
};

// A template store resident in HBM (blob uploaded verbatim).
struct DeviceStore {
    Device* dev = nullptr;
    DeviceBuffer blob;   // owning, unless `borrowed` is set
    const unsigned char* data = nullptr;
    size_t bytes = 0;
    fdt_header header{};
    // Relocated template images of the launch in flight (delta != 0); one per
    // store, so materializations of a store are ordered on its device stream.
    DeviceBuffer rtimages;
    // The per-rank value table of the launch in flight (FDT_ROP_VALUE ops).
    mutable DeviceBuffer values;
};

// The store's source digests must be the archive's (graphs.bin, patch.bin,
// comm_slots.bin when present); a store with rank ops needs a real comm binary.
void check_store_sources(const fdt_header& h, const Manifest& manifest);

struct MaterializeRequest {
    uint32_t rank = 0;
    uint32_t world = 1;
    uint64_t new_base = 0;  // 0 = keep the captured base
    std::vector<uint64_t> values;  // FDT_ROP_VALUE table (>= header.n_values entries)
};

struct MaterializeTiming {
    bool gate = true;       // hold the stream while submitting (events = device time only)
    bool split = false;     // time the relocation prepass and the member pass separately
    float kernel_ms = 0.f;  // CUDA-event time of the fused kernel, launching stream
    float reloc_ms = 0.f;   // split: relocation grid (delta != 0)
    float member_ms = 0.f;  // split: member pass alone
    int grid = 0;
    int blocks_per_sm = 0;
};

// Checks a device-resident store blob's header (host copy) and prepares pointers.
DeviceStore adopt_store(Device& dev, const unsigned char* d_blob, size_t bytes,
                        const fdt_header& host_header);
DeviceStore upload_store(Device& dev, const void* host_blob, size_t bytes);

// Launches K2+K1+K3 into `out` (must hold header.members_image_bytes bytes).
// Asynchronous on dev.stream(); timing (if non-null) is filled after a sync.
// req.values is copied to the store's value scratch first (stream ordered).
void launch_materialize(Device& dev, const DeviceStore& store, const MaterializeRequest& req,
                        unsigned char* out, MaterializeTiming* timing, int grid_override = 0);

struct Segment {
    uint64_t offset = 0;  // within the device buffer
    uint64_t length = 0;
};

// GPU CRC-64/XZ of byte ranges in device memory; returns one digest per range.
// Blocking (one small D2H of the digests).
std::vector<uint64_t> crc64_device(Device& dev, const unsigned char* d_base,
                                   std::span<const Segment> segments, float* kernel_ms = nullptr);

}  // namespace foundry
