// C-ABI, session layer: foundry::load / ServingContext behind opaque handles
// (declarations and reference anchors: include/foundry_b200.h).
#include <cstring>
#include <sstream>
#include <string>

#include "capi_common.hpp"
#include "foundry/pipeline.hpp"
#include "foundry_b200.h"

using namespace foundry;

struct fdy_serving {
    explicit fdy_serving(ServingContext&& s) : sc(std::move(s)) {}
    ServingContext sc;
};

namespace {
int copy_out(const std::string& text, char* buf, size_t cap, size_t* len) {
    if (len) *len = text.size();
    if (buf && cap) {
        const size_t n = std::min(cap - 1, text.size());
        std::memcpy(buf, text.data(), n);
        buf[n] = '\0';
    }
    return 0;
}
}  // namespace

extern "C" {

void fdy_load_options_init(fdy_load_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->world = 1;
    o->preallocate = 1;
    o->prepare_lanes = 4;
}

int fdy_load(const char* archive, const fdy_load_options* o, fdy_serving** out) {
    return fdy_guard([&] {
        require(archive && out, Errc::invalid_argument, "fdy_load: null argument");
        LoadOptions opts;
        if (o) {
            opts.rank = o->rank;
            opts.world = o->world;
            opts.preallocate = o->preallocate != 0;
            opts.prepare_lanes = o->prepare_lanes ? o->prepare_lanes : 4;
            opts.device = o->device;
            opts.relocate = o->relocate != 0;
            opts.faults.skip_binary_restore = o->skip_binary_restore != 0;
            opts.faults.skip_device_init = o->skip_device_init != 0;
            opts.faults.base_shift_granules = o->base_shift_granules;
            opts.faults.extra_prewindow_alloc = o->extra_prewindow_alloc != 0;
            opts.share_execs = o->share_execs != 0;
            opts.device_updates = o->device_updates != 0;
            if (o->n_comm_values) {
                require(o->comm_values != nullptr, Errc::invalid_argument, "fdy_load: null comm_values");
                opts.comm_values.assign(o->comm_values, o->comm_values + o->n_comm_values);
            }
        }
        *out = new fdy_serving(load(archive, opts));
    });
}

int fdy_serving_replay(fdy_serving* s, uint32_t batch, char* buf, size_t cap, size_t* len) {
    return fdy_guard([&] {
        require(s != nullptr, Errc::invalid_argument, "fdy_serving_replay: null handle");
        copy_out(s->sc.replay(batch).to_text(), buf, cap, len);
    });
}

int fdy_serving_capture_graph(fdy_serving* s, uint32_t batch, unsigned char* buf, size_t cap, size_t* len) {
    return fdy_guard([&] {
        require(s != nullptr, Errc::invalid_argument, "fdy_serving_capture_graph: null handle");
        const std::vector<uint8_t> rec = encode_graph_record(s->sc.capture_graph(batch));
        if (len) *len = rec.size();
        if (buf) std::memcpy(buf, rec.data(), std::min(cap, rec.size()));
    });
}

int fdy_serving_save_captured(fdy_serving* s, const char* out_dir) {
    return fdy_guard([&] {
        require(s && out_dir, Errc::invalid_argument, "fdy_serving_save_captured: null argument");
        s->sc.save_captured(out_dir);
    });
}

int fdy_serving_batches(fdy_serving* s, uint32_t* out, size_t cap, size_t* count) {
    return fdy_guard([&] {
        require(s != nullptr, Errc::invalid_argument, "fdy_serving_batches: null handle");
        const auto b = s->sc.batches();
        if (count) *count = b.size();
        if (out) std::memcpy(out, b.data(), std::min(cap, b.size()) * sizeof(uint32_t));
    });
}

int fdy_serving_counter(fdy_serving* s, const char* key, uint64_t* value) {
    return fdy_guard([&] {
        require(s && key && value, Errc::invalid_argument, "fdy_serving_counter: null argument");
        const auto c = s->sc.counters();
        auto it = c.find(key);
        *value = it == c.end() ? 0 : it->second;
    });
}

int fdy_serving_counters(fdy_serving* s, char* buf, size_t cap, size_t* len) {
    return fdy_guard([&] {
        require(s != nullptr, Errc::invalid_argument, "fdy_serving_counters: null handle");
        std::ostringstream o;
        for (const auto& [k, v] : s->sc.counters()) o << k << "=" << v << "\n";
        copy_out(o.str(), buf, cap, len);
    });
}

uint32_t fdy_serving_template_count(const fdy_serving* s) { return s ? s->sc.template_count() : 0; }

void fdy_serving_close(fdy_serving* s) { delete s; }

}  // extern "C"
