// C-ABI, kernel layer (declarations and reference anchors: include/foundry_b200.h).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "capi_common.hpp"
#include "../kernels/fdy_kernels.h"
#include "foundry/device.hpp"
#include "foundry/graph_model.hpp"
#include "foundry/hash.hpp"
#include "foundry/staging.hpp"
#include "foundry/template_store.hpp"
#include "foundry_b200.h"

using namespace foundry;

struct fdy_device {
    std::unique_ptr<Device> dev;
};

struct fdy_store {
    fdy_device* owner = nullptr;
    DeviceStore store;
    // host copy of the blob, fetched from HBM on first decode (its host
    // sections turn member images back into graphs)
    std::mutex mu;
    std::vector<uint8_t> host;
    std::unique_ptr<StoreView> view;

    const StoreView& host_view() {
        std::lock_guard lock(mu);
        if (!view) {
            host.resize(store.bytes);
            owner->dev->make_current();
            cuda_check(cudaMemcpy(host.data(), store.data, store.bytes, cudaMemcpyDeviceToHost), "store D2H");
            view = std::make_unique<StoreView>(host);
        }
        return *view;
    }
};

struct fdy_members {
    fdy_device* owner = nullptr;
    DeviceBuffer out;
    fdy_store* store = nullptr;  // the store the images were materialized from
    // fdy_load_members: the archive's own store, kept with its images
    std::vector<uint8_t> store_host;
    std::unique_ptr<StoreView> own_view;
    uint64_t generation = 0;     // bumped whenever the arena is rewritten

    const StoreView& view() { return own_view ? *own_view : store->host_view(); }
};

namespace {
std::atomic<uint64_t> g_generation{1};
}

extern "C" {

int fdy_device_count(void) { return cuda_device_count(); }

int fdy_device_open(int ordinal, fdy_device** out) {
    return fdy_guard([&] {
        require(out != nullptr, Errc::invalid_argument, "fdy_device_open: null out");
        auto d = std::make_unique<fdy_device>();
        d->dev = std::make_unique<Device>(ordinal);
        *out = d.release();
    });
}

void fdy_device_close(fdy_device* dev) { delete dev; }

int fdy_sync(fdy_device* dev) {
    return fdy_guard([&] {
        require(dev != nullptr, Errc::invalid_argument, "fdy_sync: null device");
        dev->dev->sync();
    });
}

int fdy_store_upload(fdy_device* dev, const void* host_blob, size_t bytes, fdy_store** out) {
    return fdy_guard([&] {
        require(dev && host_blob && out, Errc::invalid_argument, "fdy_store_upload: null argument");
        auto s = std::make_unique<fdy_store>();
        s->owner = dev;
        s->store = upload_store(*dev->dev, host_blob, bytes);
        *out = s.release();
    });
}

int fdy_store_fanout(const fdy_store* src, fdy_device* dst_dev, fdy_store** out) {
    return fdy_guard([&] {
        require(src && dst_dev && out, Errc::invalid_argument, "fdy_store_fanout: null argument");
        Device& d = *dst_dev->dev;
        Device& s = *src->owner->dev;
        DeviceBuffer buf(d, src->store.bytes, /*shareable=*/true);
        src->owner->dev->sync();  // the source upload must have landed
        d.make_current();
        int can = 0;
        if (d.ordinal() != s.ordinal()) {
            cuda_check(cudaDeviceCanAccessPeer(&can, d.ordinal(), s.ordinal()), "cudaDeviceCanAccessPeer");
            if (can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(s.ordinal(), 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else cuda_check(e, "cudaDeviceEnablePeerAccess");
            }
        }
        // peer copy: NVLink when P2P is enabled, otherwise the driver stages it
        cuda_check(cudaMemcpyPeerAsync(buf.data(), d.ordinal(), src->store.data, s.ordinal(),
                                       src->store.bytes, d.stream()),
                   "cudaMemcpyPeerAsync(store fan-out)");
        auto o = std::make_unique<fdy_store>();
        o->owner = dst_dev;
        o->store = adopt_store(d, buf.data(), src->store.bytes, src->store.header);
        o->store.blob = std::move(buf);
        *out = o.release();
    });
}

namespace {

constexpr uint64_t kChainChunk = 2ull << 20;
// a link gives up on a predecessor that publishes nothing for this long (per
// chunk; FOUNDRY_CHAIN_TIMEOUT_MS overrides, for tests)
uint64_t chain_timeout_ns() {
    if (const char* v = std::getenv("FOUNDRY_CHAIN_TIMEOUT_MS")) return std::strtoull(v, nullptr, 10) * 1000000ull;
    return 60ull * 1000 * 1000 * 1000;
}

void enable_peer(Device& d, Device& s) {
    if (d.ordinal() == s.ordinal()) return;
    int can = 0;
    cuda_check(cudaDeviceCanAccessPeer(&can, d.ordinal(), s.ordinal()), "cudaDeviceCanAccessPeer");
    if (!can) return;
    d.make_current();
    const cudaError_t e = cudaDeviceEnablePeerAccess(s.ordinal(), 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else cuda_check(e, "cudaDeviceEnablePeerAccess");
}

}  // namespace

int fdy_store_fanout_chain(const fdy_store* src, fdy_device* const* dsts, uint32_t n, uint64_t chunk_bytes,
                           fdy_store** outs) {
    return fdy_guard([&] {
        require(src && (dsts || n == 0) && (outs || n == 0), Errc::invalid_argument,
                "fdy_store_fanout_chain: null argument");
        for (uint32_t i = 0; i < n; ++i)
            require(dsts[i] != nullptr, Errc::invalid_argument, "fdy_store_fanout_chain: null device");
        const uint64_t bytes = src->store.bytes;
        const uint64_t chunk = chunk_bytes ? chunk_bytes : kChainChunk;
        const uint64_t nchunks = (bytes + chunk - 1) / chunk;
        src->owner->dev->sync();  // the head's bytes have landed
        std::vector<DeviceBuffer> bufs;
        bufs.reserve(n);
        for (uint32_t i = 0; i < n; ++i) {
            Device& d = *dsts[i]->dev;
            Device& up = i == 0 ? *src->owner->dev : *dsts[i - 1]->dev;
            enable_peer(d, up);
            d.make_current();
            bufs.emplace_back(d, bytes, /*shareable=*/true);
        }
        // events[i * nchunks + k]: chunk k has landed on dsts[i]
        std::vector<cudaEvent_t> events(size_t(n) * nchunks, nullptr);
        auto cleanup = [&] {
            for (cudaEvent_t e : events)
                if (e) cudaEventDestroy(e);
        };
        try {
            for (uint32_t i = 0; i < n; ++i) {
                dsts[i]->dev->make_current();
                for (uint64_t k = 0; k < nchunks; ++k)
                    cuda_check(cudaEventCreateWithFlags(&events[i * nchunks + k], cudaEventDisableTiming),
                               "cudaEventCreate");
            }
            for (uint64_t k = 0; k < nchunks; ++k) {
                const uint64_t off = k * chunk, len = std::min(chunk, bytes - off);
                for (uint32_t i = 0; i < n; ++i) {
                    Device& d = *dsts[i]->dev;
                    d.make_current();
                    const unsigned char* from = i == 0 ? src->store.data : bufs[i - 1].data();
                    const int from_dev = i == 0 ? src->owner->dev->ordinal() : dsts[i - 1]->dev->ordinal();
                    if (i > 0)
                        cuda_check(cudaStreamWaitEvent(d.stream(), events[(i - 1) * nchunks + k], 0),
                                   "cudaStreamWaitEvent");
                    cuda_check(cudaMemcpyPeerAsync(bufs[i].data() + off, d.ordinal(), from + off, from_dev, len,
                                                   d.stream()),
                               "cudaMemcpyPeerAsync(chain fan-out)");
                    cuda_check(cudaEventRecord(events[i * nchunks + k], d.stream()), "cudaEventRecord");
                }
            }
            for (uint32_t i = 0; i < n; ++i) dsts[i]->dev->sync();
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
        for (uint32_t i = 0; i < n; ++i) {
            auto o = std::make_unique<fdy_store>();
            o->owner = dsts[i];
            o->store = adopt_store(*dsts[i]->dev, bufs[i].data(), bytes, src->store.header);
            o->store.blob = std::move(bufs[i]);
            outs[i] = o.release();
        }
    });
}

// Cross-process chain link: the store bytes, then a progress word (chunks
// landed), in one shareable allocation whose IPC handle the next link opens.
struct fdy_chain {
    fdy_device* dev = nullptr;
    DeviceBuffer buf;
    uint64_t bytes = 0, chunk = 0, progress_off = 0;
    uint32_t nchunks = 0;
    void* upstream = nullptr;  // opened IPC mapping of the previous link
    bool fed = false;
    uint32_t* progress() { return reinterpret_cast<uint32_t*>(buf.data() + progress_off); }
    uint32_t* failed() { return progress() + 1; }  // set by a wait that timed out
    ~fdy_chain() {
        if (upstream) {
            dev->dev->make_current();
            cudaIpcCloseMemHandle(upstream);
        }
    }
};

int fdy_chain_create(fdy_device* dev, uint64_t bytes, uint64_t chunk_bytes, fdy_chain** out,
                     unsigned char handle[64]) {
    return fdy_guard([&] {
        require(dev && out && handle && bytes >= sizeof(fdt_header), Errc::invalid_argument,
                "fdy_chain_create: null argument or store smaller than its header");
        auto c = std::make_unique<fdy_chain>();
        c->dev = dev;
        c->bytes = bytes;
        c->chunk = chunk_bytes ? chunk_bytes : kChainChunk;
        c->nchunks = static_cast<uint32_t>((bytes + c->chunk - 1) / c->chunk);
        c->progress_off = (bytes + 255) / 256 * 256;
        Device& d = *dev->dev;
        d.make_current();
        c->buf = DeviceBuffer(d, c->progress_off + 256, /*shareable=*/true);
        // zeroed before the handle leaves this process: a link never sees a stale count
        cuda_check(cudaMemset(c->progress(), 0, 256), "cudaMemset(chain progress)");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, c->buf.data()), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof h);
        *out = c.release();
    });
}

int fdy_chain_seed(fdy_chain* c, const void* host_blob) {
    return fdy_guard([&] {
        require(c && host_blob && !c->fed, Errc::invalid_argument, "fdy_chain_seed: null argument or fed twice");
        Device& d = *c->dev->dev;
        d.make_current();
        const auto* src = static_cast<const unsigned char*>(host_blob);
        for (uint32_t k = 0; k < c->nchunks; ++k) {
            const uint64_t off = uint64_t(k) * c->chunk, len = std::min(c->chunk, c->bytes - off);
            cuda_check(cudaMemcpyAsync(c->buf.data() + off, src + off, len, cudaMemcpyHostToDevice, d.stream()),
                       "cudaMemcpyAsync(chain seed)");
            cuda_check(fdy_launch_chain_publish(c->progress(), k + 1, nullptr, d.stream()), "chain publish");
        }
        c->fed = true;
    });
}

int fdy_chain_pull(fdy_chain* c, const unsigned char upstream[64]) {
    return fdy_guard([&] {
        require(c && upstream && !c->fed, Errc::invalid_argument, "fdy_chain_pull: null argument or fed twice");
        Device& d = *c->dev->dev;
        d.make_current();
        cudaIpcMemHandle_t h;
        std::memcpy(&h, upstream, sizeof h);
        cuda_check(cudaIpcOpenMemHandle(&c->upstream, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        const auto* up = static_cast<const unsigned char*>(c->upstream);
        const auto* up_progress = reinterpret_cast<const uint32_t*>(up + c->progress_off);
        const uint64_t timeout = chain_timeout_ns();
        for (uint32_t k = 0; k < c->nchunks; ++k) {
            const uint64_t off = uint64_t(k) * c->chunk, len = std::min(c->chunk, c->bytes - off);
            cuda_check(fdy_launch_chain_wait(up_progress, k + 1, timeout, c->failed(), d.stream()),
                       "chain wait");
            cuda_check(cudaMemcpyAsync(c->buf.data() + off, up + off, len, cudaMemcpyDeviceToDevice, d.stream()),
                       "cudaMemcpyAsync(chain link)");
            cuda_check(fdy_launch_chain_publish(c->progress(), k + 1, c->failed(), d.stream()), "chain publish");
        }
        c->fed = true;
    });
}

int fdy_chain_finish(fdy_chain* c, fdy_store** out) {
    return fdy_guard([&] {
        require(c && out && c->fed, Errc::invalid_argument, "fdy_chain_finish: null argument or nothing fed");
        Device& d = *c->dev->dev;
        d.make_current();
        cuda_check(cudaStreamSynchronize(d.stream()), "chain fan-out");
        if (c->upstream) {
            cuda_check(cudaIpcCloseMemHandle(c->upstream), "cudaIpcCloseMemHandle");
            c->upstream = nullptr;
        }
        uint32_t failed = 0;
        cuda_check(cudaMemcpy(&failed, c->failed(), sizeof failed, cudaMemcpyDeviceToHost), "chain status D2H");
        require(failed == 0, Errc::cuda_error,
                "chain fan-out: the predecessor published no progress within the timeout (did its process exit?)");
        fdt_header hdr;
        cuda_check(cudaMemcpy(&hdr, c->buf.data(), sizeof hdr, cudaMemcpyDeviceToHost), "store header D2H");
        auto o = std::make_unique<fdy_store>();
        o->owner = c->dev;
        o->store = adopt_store(d, c->buf.data(), c->bytes, hdr);
        o->store.blob = std::move(c->buf);  // the next link may still be reading it: free after a barrier
        *out = o.release();
    });
}

void fdy_chain_free(fdy_chain* c) { delete c; }

int fdy_store_export(const fdy_store* store, unsigned char handle[64], uint64_t* bytes) {
    return fdy_guard([&] {
        require(store && handle && bytes, Errc::invalid_argument, "fdy_store_export: null argument");
        require(store->store.blob.data() == store->store.data, Errc::invalid_argument,
                "fdy_store_export: only stores uploaded with fdy_store_upload can be exported");
        store->owner->dev->sync();  // the upload must have landed before a peer reads it
        cudaIpcMemHandle_t h;
        static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
        cuda_check(cudaIpcGetMemHandle(&h, const_cast<unsigned char*>(store->store.data)),
                   "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof h);
        *bytes = store->store.bytes;
    });
}

int fdy_store_import(fdy_device* dev, const unsigned char handle[64], uint64_t bytes, fdy_store** out) {
    return fdy_guard([&] {
        require(dev && handle && out, Errc::invalid_argument, "fdy_store_import: null argument");
        Device& d = *dev->dev;
        d.make_current();
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        void* peer = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&peer, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        DeviceBuffer buf(d, bytes, /*shareable=*/true);  // may be exported onwards
        // GPU -> GPU pull; NVLink P2P between the two devices
        const cudaError_t e = cudaMemcpyAsync(buf.data(), peer, bytes, cudaMemcpyDeviceToDevice, d.stream());
        const cudaError_t s = e == cudaSuccess ? cudaStreamSynchronize(d.stream()) : e;
        cudaIpcCloseMemHandle(peer);
        cuda_check(s, "store fan-out copy");
        fdt_header hdr;
        cuda_check(cudaMemcpy(&hdr, buf.data(), sizeof hdr, cudaMemcpyDeviceToHost), "store header D2H");
        auto o = std::make_unique<fdy_store>();
        o->owner = dev;
        o->store = adopt_store(d, buf.data(), bytes, hdr);
        o->store.blob = std::move(buf);
        *out = o.release();
    });
}

void fdy_store_free(fdy_store* store) { delete store; }

size_t fdy_store_members_bytes(const fdy_store* store) {
    return store ? store->store.header.members_image_bytes : 0;
}

static void copy_timings(const ArchiveMaterializeTimings& t, fdy_prepare_timings* timings) {
    if (!timings) return;
    timings->total_ms = t.total_ms;
    timings->read_ms = t.read_ms;
    timings->integrity_ms = t.integrity_ms;
    timings->materialize_ms = t.materialize_ms;
    timings->d2h_ms = t.d2h_ms;
    timings->crc_kernel_ms = t.crc_kernel_ms;
    timings->kernel_ms = t.kernel_ms;
    timings->h2d_bytes = t.h2d_bytes;
    timings->d2h_bytes = t.d2h_bytes;
    timings->member_bytes = t.member_bytes;
    timings->graphs = t.graphs;
    timings->nodes = t.nodes;
}

// The request a descriptor describes; the value table (FDT_ROP_VALUE ops) is
// part of it on every entry point.
static MaterializeRequest request_of(const fdy_materialize_desc* desc) {
    MaterializeRequest req;
    req.rank = desc->rank;
    req.world = desc->world;
    req.new_base = desc->new_base;
    if (desc->n_values) {
        require(desc->values != nullptr, Errc::invalid_argument, "fdy_materialize: null value table");
        req.values.assign(desc->values, desc->values + desc->n_values);
    }
    return req;
}

static void materialize_into(fdy_device* dev, const fdy_store* store,
                             const fdy_materialize_desc* desc, fdy_members* m, float* kernel_ms) {
    require(dev && store && desc && m, Errc::invalid_argument, "fdy_materialize: null argument");
    require(store->owner == dev, Errc::invalid_argument, "fdy_materialize: store lives on another device");
    m->store = const_cast<fdy_store*>(store);
    m->own_view.reset();
    m->generation = g_generation.fetch_add(1);
    const MaterializeRequest req = request_of(desc);
    MaterializeTiming t;
    launch_materialize(*dev->dev, store->store, req, m->out.data(), kernel_ms ? &t : nullptr, desc->grid);
    if (kernel_ms) *kernel_ms = t.kernel_ms;
}

int fdy_materialize(fdy_device* dev, const fdy_store* store, const fdy_materialize_desc* desc,
                    fdy_members** out, float* kernel_ms) {
    return fdy_guard([&] {
        require(dev && store && out, Errc::invalid_argument, "fdy_materialize: null argument");
        auto m = std::make_unique<fdy_members>();
        m->owner = dev;
        m->out = DeviceBuffer(*dev->dev, store->store.header.members_image_bytes);
        materialize_into(dev, store, desc, m.get(), kernel_ms);
        *out = m.release();
    });
}

int fdy_materialize_into(fdy_device* dev, const fdy_store* store, const fdy_materialize_desc* desc,
                         fdy_members* members, float* kernel_ms) {
    return fdy_guard([&] {
        require(members && store, Errc::invalid_argument, "fdy_materialize_into: null argument");
        require(members->out.size() >= store->store.header.members_image_bytes,
                Errc::invalid_argument, "fdy_materialize_into: arena too small for this store");
        materialize_into(dev, store, desc, members, kernel_ms);
    });
}

int fdy_materialize_timed_split(fdy_device* dev, const fdy_store* store, const fdy_materialize_desc* desc,
                                fdy_members* m, float* reloc_ms, float* member_ms) {
    return fdy_guard([&] {
        require(dev && store && desc && m, Errc::invalid_argument, "fdy_materialize_timed_split: null argument");
        require(store->owner == dev, Errc::invalid_argument, "fdy_materialize: store lives on another device");
        require(m->out.size() >= store->store.header.members_image_bytes, Errc::invalid_argument,
                "fdy_materialize_timed_split: arena too small for this store");
        const MaterializeRequest req = request_of(desc);
        m->store = const_cast<fdy_store*>(store);
        m->own_view.reset();
        m->generation = g_generation.fetch_add(1);
        MaterializeTiming t;
        t.split = true;
        launch_materialize(*dev->dev, store->store, req, m->out.data(), &t, desc->grid);
        if (reloc_ms) *reloc_ms = t.reloc_ms;
        if (member_ms) *member_ms = t.member_ms;
    });
}

int fdy_members_write_probe(fdy_members* m, float* ms) {
    return fdy_guard([&] {
        require(m && ms, Errc::invalid_argument, "fdy_members_write_probe: null argument");
        Device& d = *m->owner->dev;
        d.make_current();
        m->generation = g_generation.fetch_add(1);  // the arena no longer holds member images
        cudaEvent_t e0, e1;
        cuda_check(cudaEventCreate(&e0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&e1), "cudaEventCreate");
        cuda_check(cudaEventRecord(e0, d.stream()), "cudaEventRecord");
        cuda_check(fdy_launch_write_probe(m->out.data(), m->out.size(), d.stream()), "write probe launch");
        cuda_check(cudaEventRecord(e1, d.stream()), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(e1), "cudaEventSynchronize");
        cuda_check(cudaEventElapsedTime(ms, e0, e1), "cudaEventElapsedTime");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

size_t fdy_members_bytes(const fdy_members* m) { return m ? m->out.size() : 0; }

int fdy_members_download(fdy_members* m, void* host_dst, size_t offset, size_t bytes) {
    return fdy_guard([&] {
        require(m && host_dst, Errc::invalid_argument, "fdy_members_download: null argument");
        require(offset <= m->out.size() && bytes <= m->out.size() - offset, Errc::invalid_argument,
                "fdy_members_download: range outside the arena");
        Device& d = *m->owner->dev;
        d.make_current();
        cuda_check(cudaMemcpyAsync(host_dst, m->out.data() + offset, bytes, cudaMemcpyDeviceToHost,
                                   d.stream()),
                   "cudaMemcpyAsync(members D2H)");
        cuda_check(cudaStreamSynchronize(d.stream()), "cudaStreamSynchronize");
    });
}

void fdy_members_free(fdy_members* m) { delete m; }

int fdy_members_record(fdy_members* m, uint32_t label, unsigned char* buf, size_t cap, size_t* len,
                       uint64_t* crc) {
    return fdy_guard([&] {
        require(m != nullptr, Errc::invalid_argument, "fdy_members_record: null members");
        require(m->own_view || m->store, Errc::invalid_argument, "fdy_members_record: arena holds no materialization");
        // the last record this thread decoded: the size query and the copy are one decode
        thread_local struct {
            uint64_t generation = 0;
            uint32_t label = 0;
            std::vector<uint8_t> rec;
            uint64_t crc = 0;
        } last;
        if (last.generation != m->generation || last.label != label || last.rec.empty()) {
            const StoreView& v = m->view();
            const int64_t mi = v.member_of(label);
            require(mi >= 0, Errc::invalid_argument,
                    "label " + std::to_string(label) + " is not a member of the materialized graph set");
            const fdt_member& M = v.member(static_cast<uint32_t>(mi));
            std::vector<uint8_t> image(v.group(M.group).image_bytes);
            m->owner->dev->make_current();
            cuda_check(cudaMemcpy(image.data(), m->out.data() + M.out_off, image.size(), cudaMemcpyDeviceToHost),
                       "cudaMemcpy(member image D2H)");
            last.rec = encode_graph_record(v.image_to_graph(static_cast<uint32_t>(mi), image));
            last.crc = crc64(last.rec);
            last.generation = m->generation;
            last.label = label;
        }
        if (len) *len = last.rec.size();
        if (crc) *crc = last.crc;
        if (buf && cap >= last.rec.size()) std::memcpy(buf, last.rec.data(), last.rec.size());
    });
}

int fdy_load_members(fdy_device* dev, const char* archive, const fdy_materialize_desc* desc, uint32_t lanes,
                     fdy_members** out, fdy_prepare_timings* timings) {
    return fdy_guard([&] {
        require(dev && archive && desc && out, Errc::invalid_argument, "fdy_load_members: null argument");
        auto m = std::make_unique<fdy_members>();
        m->owner = dev;
        MaterializedArchive keep;
        ArchiveMaterializeTimings t;
        materialize_archive(*dev->dev, archive, request_of(desc), lanes ? lanes : 4, nullptr, 0, &t, &keep);
        m->out = std::move(keep.images);
        m->store_host = std::move(keep.store_host);
        m->own_view = std::make_unique<StoreView>(m->store_host);
        m->generation = g_generation.fetch_add(1);
        copy_timings(t, timings);
        *out = m.release();
    });
}

int fdy_prepare_archive(fdy_device* dev, const char* archive, const fdy_materialize_desc* desc,
                        uint32_t lanes, void* host_out, size_t cap, size_t* out_len,
                        fdy_prepare_timings* timings) {
    return fdy_guard([&] {
        require(dev && archive && desc, Errc::invalid_argument, "fdy_prepare_archive: null argument");
        ArchiveMaterializeTimings t;
        const MaterializeRequest req = request_of(desc);
        const uint64_t n = materialize_archive(*dev->dev, archive, req, lanes ? lanes : 4, host_out, cap, &t);
        if (out_len) *out_len = n;
        copy_timings(t, timings);
    });
}

void* fdy_host_alloc(fdy_device* dev, size_t bytes) {
    void* p = nullptr;
    fdy_guard([&] {
        require(dev != nullptr, Errc::invalid_argument, "fdy_host_alloc: null device");
        p = dev->dev->alloc_host_pinned(bytes);
    });
    return p;
}

void fdy_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int fdy_crc64_segments(fdy_device* dev, const void* host, size_t bytes, const uint64_t* offsets,
                       const uint64_t* lengths, uint32_t n, uint64_t* digests, float* kernel_ms) {
    return fdy_guard([&] {
        require(dev && (host || !bytes) && (offsets || !n) && (lengths || !n) && (digests || !n),
                Errc::invalid_argument, "fdy_crc64_segments: null argument");
        // pack every range at a 16-byte aligned offset of one device buffer
        std::vector<Segment> segs(n);
        uint64_t total = 0;
        for (uint32_t i = 0; i < n; ++i) {
            require(offsets[i] <= bytes && lengths[i] <= bytes - offsets[i], Errc::invalid_argument,
                    "fdy_crc64_segments: range outside the buffer");
            segs[i] = {total, lengths[i]};
            total += (lengths[i] + 255) / 256 * 256;
        }
        Device& d = *dev->dev;
        DeviceBuffer buf(d, total);
        for (uint32_t i = 0; i < n; ++i)
            if (lengths[i])
                cuda_check(cudaMemcpyAsync(buf.data() + segs[i].offset,
                                           static_cast<const unsigned char*>(host) + offsets[i],
                                           lengths[i], cudaMemcpyHostToDevice, d.stream()),
                           "cudaMemcpyAsync(crc H2D)");
        const auto out = crc64_device(d, buf.data(), segs, kernel_ms);
        std::memcpy(digests, out.data(), n * sizeof(uint64_t));
    });
}

}  // extern "C"
