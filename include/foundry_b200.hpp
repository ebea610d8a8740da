// foundry_b200.hpp — header-only C++ convenience layer over the C-ABI
// (foundry_b200.h). No dependency on this build's internals or on the
// reference: a reference maintainer includes it next to the reference's own
// headers and gets the GPU replacement of its PrepareFn
// (reference templater.hpp:48, built at pipeline.cpp:506-514).
//
//   foundry_b200::GpuPrepare gpu(archive, rank, world);      // integrity + fused kernel, once
//   PrepareFn prepare = [&](uint32_t label, const GraphLocator&) {
//       const auto r = gpu.record(label);                     // FNDG record bytes + CRC
//       return parse_graph_at(r.bytes, GraphLocator{label, 0, r.bytes.size(), r.crc});
//   };
//   ServingSet::build(ctx, manifest.grouping, prepare, lanes); // reference templater.hpp:62-64
//
// Errors are thrown as foundry_b200::Error carrying the C-ABI code
// (1 + the reference Errc, errors.hpp:9-23) and fdy_last_error()'s text
// ("<errc>: <step>: <detail>").
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "foundry_b200.h"

namespace foundry_b200 {

class Error : public std::runtime_error {
public:
    Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
    int code() const { return code_; }  // 1 + reference Errc; FDY_ERR_CUDA / FDY_ERR_NO_DEVICE
private:
    int code_;
};

inline void check(int rc) {
    if (rc != FDY_OK) throw Error(rc, fdy_last_error());
}

// One CUDA device (fdy_device), move-only.
class Device {
public:
    explicit Device(int ordinal = 0) { check(fdy_device_open(ordinal, &d_)); }
    ~Device() {
        if (d_) fdy_device_close(d_);
    }
    Device(Device&& o) noexcept : d_(o.d_) { o.d_ = nullptr; }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    fdy_device* get() const { return d_; }

private:
    fdy_device* d_ = nullptr;
};

struct Record {
    std::vector<uint8_t> bytes;  // encode_graph_record layout (graph_model.cpp:205-218)
    uint64_t crc = 0;            // CRC-64/XZ of bytes (the GraphLocator checksum)
};

// The GPU PrepareFn: every member of `archive` materialized for (rank, world)
// in HBM by one fdy_load_members call; record(label) then returns the member
// graph the reference PrepareFn would return. record() is safe to call from
// several prepare lanes at once.
class GpuPrepare {
public:
    struct Options {
        int device = 0;
        uint64_t new_base = 0;             // 0: keep the captured VA base
        std::vector<uint64_t> comm_values; // per-rank comm slot values (comm_slots.bin)
        uint32_t lanes = 4;                // host threads staging/hashing archive files
    };

    GpuPrepare(const std::string& archive, uint32_t rank, uint32_t world) : GpuPrepare(archive, rank, world, Options{}) {}
    GpuPrepare(const std::string& archive, uint32_t rank, uint32_t world, const Options& o) : dev_(o.device) {
        fdy_materialize_desc desc{};
        desc.rank = rank;
        desc.world = world;
        desc.new_base = o.new_base;
        desc.values = o.comm_values.empty() ? nullptr : o.comm_values.data();
        desc.n_values = static_cast<uint32_t>(o.comm_values.size());
        check(fdy_load_members(dev_.get(), archive.c_str(), &desc, o.lanes, &m_, &timings_));
    }
    ~GpuPrepare() {
        if (m_) fdy_members_free(m_);
    }
    GpuPrepare(const GpuPrepare&) = delete;
    GpuPrepare& operator=(const GpuPrepare&) = delete;

    Record record(uint32_t label) const {
        Record r;
        size_t len = 0;
        check(fdy_members_record(m_, label, nullptr, 0, &len, &r.crc));
        r.bytes.resize(len);
        check(fdy_members_record(m_, label, r.bytes.data(), len, &len, &r.crc));
        return r;
    }

    const fdy_prepare_timings& timings() const { return timings_; }
    fdy_members* members() const { return m_; }

private:
    Device dev_;
    fdy_members* m_ = nullptr;
    fdy_prepare_timings timings_{};
};

}  // namespace foundry_b200
