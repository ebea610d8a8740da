// Host side of the GPU packer (kernels/pack.cu; format: store_format.h).
//
// The offline packer (template_store.cpp pack_template_store) decodes every
// member with parse_graph_at on host threads; here the members stay in HBM and
// the kernels decode, validate, lay out, diff and compact them. The host works
// on what is per group or per kernel and on patch.bin:
//   pass 1 (GPU)  node walk, validation, topology, slot capacities, kernel keys
//   host          error checks in the offline packer's order, kernel table
//                 (first-occurrence order), group layouts, stub swaps, rank ops
//   pass 2 (GPU)  member images + relocation meta, diff counts per tile
//   host          tile table (relocation-free tiles first), host sections
//   pass 3 (GPU)  diff streams (ballot / scan compaction), template images
// The result is byte-identical to pack_template_store's (tests/test_gpu_pack.py).
#include "foundry/device_pack.hpp"

#include <algorithm>
#include <array>
#include <exception>
#include <future>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <optional>
#include <unordered_map>

#include "../kernels/fdy_kernels.h"
#include "foundry/bytes.hpp"
#include "foundry/hash.hpp"
#include "foundry/parallel.hpp"
#include "foundry/staging.hpp"

namespace foundry {

namespace {

using Clock = std::chrono::steady_clock;
double ms_of(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

constexpr uint32_t kNoKernel = 0xFFFFFFFFu;
constexpr size_t kSectionAlign = 256;

uint32_t rd32(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}
uint64_t rd64(const uint8_t* p) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    return v;
}

// Bump allocator over one device allocation (256-byte aligned pieces).
class Scratch {
public:
    Scratch(Device& dev, size_t bytes) : buf_(dev, bytes + 256) {}
    template <typename T>
    T* take(size_t count) {
        at_ = (at_ + 255) / 256 * 256;
        T* p = reinterpret_cast<T*>(buf_.data() + at_);
        at_ += count * sizeof(T);
        return p;
    }
    static size_t need(std::initializer_list<size_t> sizes) {
        size_t n = 0;
        for (size_t s : sizes) n += (s + 255) / 256 * 256;
        return n;
    }

private:
    DeviceBuffer buf_;
    size_t at_ = 0;
};

// Host arrays bound for one contiguous device range, gathered into one pinned
// buffer and sent with one copy (each pageable copy blocks the host for
// ~10-20 us). The gaps between the arrays are alignment padding only.
class Upload {
public:
    template <typename T>
    void add(T* dst, const T* src, size_t count) {
        if (count) items_.push_back({reinterpret_cast<unsigned char*>(dst), src, count * sizeof(T)});
    }
    template <typename T>
    void add(T* dst, const std::vector<T>& v) { add(dst, v.data(), v.size()); }
    void send(Device& dev, cudaStream_t st) {
        if (items_.empty()) return;
        unsigned char* lo = items_[0].dst;
        unsigned char* hi = lo;
        for (const Item& it : items_) {
            lo = std::min(lo, it.dst);
            hi = std::max(hi, it.dst + it.bytes);
        }
        lease_ = PinnedLease(dev, size_t(hi - lo));
        // the patch-entry arrays are a few MB: gathered on host threads
        parallel_for(items_.size(), size_t(hi - lo) > (1u << 20) ? 0u : 1u, [&](size_t i) {
            std::memcpy(lease_.data() + (items_[i].dst - lo), items_[i].src, items_[i].bytes);
        });
        cuda_check(cudaMemcpyAsync(lo, lease_.data(), size_t(hi - lo), cudaMemcpyHostToDevice, st), "GPU pack H2D");
    }

private:
    struct Item {
        unsigned char* dst;
        const void* src;
        size_t bytes;
    };
    std::vector<Item> items_;
    PinnedLease lease_;  // alive until the owner has synchronized the stream
};

template <typename T>
void h2d(T* dst, const std::vector<T>& src, cudaStream_t st) {
    if (!src.empty())
        cuda_check(cudaMemcpyAsync(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, st),
                   "GPU pack H2D");
}
template <typename T>
void d2h(std::vector<T>& dst, const T* src, size_t count, cudaStream_t st) {
    dst.resize(count);
    if (count)
        cuda_check(cudaMemcpyAsync(dst.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost, st), "GPU pack D2H");
}

struct NodeView {  // a kernel node's fields, read from the host copy
    const uint8_t* q;
    uint32_t name_len() const { return rd32(q + 62); }
    std::string_view name() const { return {reinterpret_cast<const char*>(q + 66), name_len()}; }
    uint64_t hash() const { return rd64(q + 54); }
    const uint8_t* fattrs() const { return q + 66 + name_len(); }
    uint32_t arg_size() const { return rd32(q + 90 + name_len()); }
};

// The GPU packer's state and phases, in order (run()). Host arrays are
// members so each phase reads what the earlier ones produced.
class DevicePacker {
public:
    DevicePacker(Device& dev, std::span<const uint8_t> graphs_host, const unsigned char* d_graphs,
                 std::span<const uint8_t> patch_bin, const Manifest& manifest, std::span<const uint8_t> slots_bin,
                 bool full_host_copy, const uint64_t* verified_graphs_crc, std::future<PatchView>* patch_view)
        : dev_(dev), graphs_host_(graphs_host), G_(graphs_host.data()), gsize_(graphs_host.size()),
          d_graphs_(d_graphs), patch_bin_(patch_bin), manifest_(manifest), slots_bin_(slots_bin),
          full_host_copy_(full_host_copy), verified_graphs_crc_(verified_graphs_crc), patch_view_(patch_view) {}

    DevicePackResult run(PackStats* stats, DevicePackTimings* timings) {
        t_all_ = Clock::now();
        patches_ = patch_view_ ? patch_view_->get() : parse_patch_view(patch_bin_);
        tm_.patch_parse_ms = ms_of(t_all_);
        slots_ = slots_bin_.empty() ? CommSlotTable{} : parse_comm_slots(slots_bin_);
        if (!patches_.empty())
            require(manifest_.comm_real_hash != 0, Errc::unresolved_kernel,
                    "archive carries comm patches but no real comm binary");
        dev_.make_current();
        st_ = dev_.stream();
        load_members();
        flatten_entries();
        tm_.prep_ms = ms_of(t_all_);

        auto t0 = Clock::now();
        pass1();
        tm_.pass1_ms = ms_of(t0);

        t0 = Clock::now();
        check_errors();
        tm_.checks_ms = ms_of(t0);
        layout();
        // rank ops need only the layouts: host threads build them while the
        // kernel table is assembled and pass 2 runs
        std::future<void> rops_done = std::async(std::launch::async, [this] { build_rank_ops(); });
        const auto tk = Clock::now();
        build_kernel_table();
        tm_.kernel_table_ms = ms_of(tk);
        tm_.host1_ms = ms_of(t0);

        t0 = Clock::now();
        pass2();
        rops_done.get();
        tm_.pass2_ms = ms_of(t0);

        t0 = Clock::now();
        build_tables();
        tm_.tiles_ms = ms_of(t0);
        place_sections();
        tm_.layout_ms = ms_of(t0) - tm_.tiles_ms;
        DevicePackResult out = host_sections();
        tm_.host2_ms = ms_of(t0);

        t0 = Clock::now();
        pass3(out);
        tm_.pass3_ms = ms_of(t0);

        if (stats) {
            stats->template_bytes = timages_bytes_;
            stats->diff_entries = n_diffs_;
            stats->rank_ops = rops_.size();
            stats->member_image_bytes = arena_bytes_;
            stats->store_bytes = blob_bytes_;
        }
        tm_.total_ms = ms_of(t_all_);
        if (timings) *timings = tm_;
        return out;
    }

private:
    const uint8_t* node_ptr(uint32_t m, uint32_t n) const { return G_ + rec_off_[m] + node_off_[node_base_[m] + n]; }
    uint32_t group_end(uint32_t g) const { return g + 1 < n_groups_ ? group_first_[g + 1] : nm_; }

    // ------------------------------------------------ members, group-major
    void load_members() {
        const auto& groups_in = manifest_.grouping.groups;
        n_groups_ = static_cast<uint32_t>(groups_in.size());
        uint64_t total = 0;
        for (uint32_t g = 0; g < n_groups_; ++g) {
            const TemplateGroup& grp = groups_in[g];
            require(grp.locators.size() == grp.members.size() && !grp.members.empty(), Errc::invalid_argument,
                    "grouping manifest is missing member locators");
            group_first_.push_back(static_cast<uint32_t>(rec_off_.size()));
            size_t rep = 0;  // the offline packer keeps the last member whose label is the representative
            for (size_t i = 0; i < grp.locators.size(); ++i)
                if (grp.locators[i].label == grp.representative) rep = i;
            group_rep_.push_back(group_first_.back() + static_cast<uint32_t>(rep));
            for (const GraphLocator& l : grp.locators) {
                require(l.offset <= gsize_ && l.length <= gsize_ - l.offset, Errc::binary_format,
                        "graph record for label " + std::to_string(l.label) + " overruns the container");
                require(l.length < (1ull << 32), Errc::invalid_argument, "graph record exceeds 4 GiB");
                uint32_t nn = 0, ne = 0;
                bool bad = l.length < 12;
                if (!bad) {
                    const uint8_t* r = G_ + l.offset;
                    nn = rd32(r + 4);
                    ne = rd32(r + 8);
                    bad = rd32(r) != l.label || nn > l.length - 12 || ne > (l.length - 12) / 8;
                }
                if (bad) nn = ne = 0;
                rec_off_.push_back(l.offset);
                rec_len_.push_back(l.length);
                node_base_.push_back(static_cast<uint32_t>(total));
                n_nodes_.push_back(nn);
                n_edges_.push_back(ne);
                member_group_.push_back(g);
                loc_of_.push_back(&l);
                suspect_.push_back(bad ? 1 : 0);
                total += nn;
            }
        }
        nm_ = static_cast<uint32_t>(rec_off_.size());
        require(total < (1ull << 31), Errc::invalid_argument, "graph set exceeds 2^31 nodes");
        total_nodes_ = total;
        TN_ = static_cast<uint32_t>(total);
        gnode_base_.assign(n_groups_ + 1, 0);
        for (uint32_t g = 0; g < n_groups_; ++g) gnode_base_[g + 1] = gnode_base_[g] + n_nodes_[group_rep_[g]];
        GN_ = gnode_base_[n_groups_];
    }

    uint32_t intern(std::string_view n) {
        for (uint32_t i = 0; i < name_list_.size(); ++i)
            if (name_list_[i].size() == n.size() && std::memcmp(name_list_[i].data(), n.data(), n.size()) == 0)
                return i;
        name_list_.push_back(n);
        name_off_.push_back(static_cast<uint32_t>(name_bytes_.size()));
        name_len_.push_back(static_cast<uint32_t>(n.size()));
        name_bytes_.append(n);
        return static_cast<uint32_t>(name_list_.size() - 1);
    }

    // patch entries, flattened in member order (apply_rank_patches' table);
    // names interned (a handful of distinct stub / real comm names)
    void flatten_entries() {
        entry_base_.assign(nm_ + 1, 0);
        patch_bad_.assign(nm_, 0);
        if (!patches_.empty() || !slots_.empty()) {
            // entry ranges per member, then the entries filled on host threads
            std::vector<std::span<const PatchEntryView>> entries_of(nm_);
            uint32_t ne = 0;
            for (uint32_t m = 0; m < nm_; ++m) {
                entries_of[m] = patches_.find(loc_of_[m]->label);
                entry_base_[m] = ne;
                ne += static_cast<uint32_t>(entries_of[m].size());
            }
            pe_node_.resize(ne);
            pe_stub_hash_.resize(ne);
            pe_stub_name_.resize(ne);
            pe_real_name_.resize(ne);
            pe_need_.resize(ne);
            // the distinct names (a handful), seen on the first few patched members;
            // any other name goes through the fix-up below
            for (uint32_t m = 0, seen = 0; m < nm_ && seen < 4; ++m) {
                for (const PatchEntryView& e : entries_of[m]) {
                    intern(e.stub_name);
                    intern(e.real_name);
                }
                seen += entries_of[m].empty() ? 0 : 1;
            }
            // the name table is frozen during the parallel fill: a name the scan
            // above did not see leaves the member for a sequential fix-up
            std::vector<uint8_t> unnamed(nm_, 0);
            parallel_for(nm_, 0, [&](size_t mi) {
                const uint32_t m = static_cast<uint32_t>(mi);
                const uint32_t label = loc_of_[m]->label;
                const auto entries = entries_of[m];
                uint32_t last_stub = 0, last_real = 0;
                auto id_of = [&](std::string_view n, uint32_t& last) {
                    if (last < name_list_.size() && name_list_[last] == n) return last;
                    for (uint32_t i = 0; i < name_list_.size(); ++i)
                        if (name_list_[i] == n) return last = i;
                    unnamed[m] = 1;
                    return kNoKernel;
                };
                for (uint32_t j = 0; j < entries.size(); ++j) {
                    const PatchEntryView& e = entries[j];
                    const uint32_t i = entry_base_[m] + j;
                    const bool in = e.node_id < n_nodes_[m];
                    if (!in) patch_bad_[m] = 1;
                    pe_node_[i] = in ? node_base_[m] + e.node_id : kNoKernel;
                    pe_stub_hash_[i] = e.stub_hash;
                    pe_stub_name_[i] = id_of(e.stub_name, last_stub);
                    pe_real_name_[i] = id_of(e.real_name, last_real);
                    uint64_t need = 0;
                    for (uint32_t k = 0; k < e.n_rank; ++k) need = std::max<uint64_t>(need, e.rank_offset(k) + 8ull);
                    for (uint32_t k = 0; k < e.n_world; ++k)
                        need = std::max<uint64_t>(need, e.world_offset(k) + 8ull);
                    if (need > UINT32_MAX) patch_bad_[m] = 1;
                    pe_need_[i] = static_cast<uint32_t>(std::min<uint64_t>(need, UINT32_MAX));
                }
                auto sit = slots_.per_graph.find(label);
                if (sit == slots_.per_graph.end()) return;
                if (!patches_.has(label)) {
                    patch_bad_[m] = 1;
                    return;
                }
                std::vector<std::pair<uint32_t, uint32_t>> by_node;  // (node id, entry)
                for (uint32_t j = 0; j < entries.size(); ++j) by_node.push_back({entries[j].node_id, entry_base_[m] + j});
                std::sort(by_node.begin(), by_node.end());
                for (const CommSlot& c : sit->second) {
                    auto it = std::lower_bound(by_node.begin(), by_node.end(), std::make_pair(c.node_id, 0u));
                    const uint64_t end = uint64_t(c.offset) + c.width;
                    if (it == by_node.end() || it->first != c.node_id || end > UINT32_MAX) {
                        patch_bad_[m] = 1;
                        continue;
                    }
                    pe_need_[it->second] = std::max<uint32_t>(pe_need_[it->second], static_cast<uint32_t>(end));
                }
            });
            for (uint32_t m = 0; m < nm_; ++m) {
                if (!unnamed[m]) continue;
                for (uint32_t j = 0; j < entries_of[m].size(); ++j) {
                    pe_stub_name_[entry_base_[m] + j] = intern(entries_of[m][j].stub_name);
                    pe_real_name_[entry_base_[m] + j] = intern(entries_of[m][j].real_name);
                }
            }
            entry_base_[nm_] = ne;
        }
        NE_ = entry_base_[nm_];
        tslots_ = 1024;
        while (tslots_ < 2ull * (uint64_t(TN_) + NE_)) tslots_ <<= 1;
    }

    // ------------------------------------------------ pass 1
    void pass1() {
        const uint32_t nm = nm_, TN = TN_, GN = GN_, NE = NE_, tslots = tslots_;
        const auto tp = Clock::now();
        static const bool debug = std::getenv("FOUNDRY_DEBUG") != nullptr;
        cudaEvent_t ev[6] = {};  // upload done, read-back done, pass-1 kernels done, CRC done, entry, scratch
        if (debug) {
            for (auto& e : ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
            cuda_check(cudaEventRecord(ev[4], dev_.stream()), "cudaEventRecord");
        }
        s1_.emplace(dev_, Scratch::need({8ull * nm, 8ull * nm, 4ull * nm, 4ull * nm, 4ull * nm, 4ull * nm, 4ull * nm,
                                         4ull * n_groups_, 4ull * n_groups_, 4ull * TN, 4ull * TN, 4ull * TN,
                                         4ull * GN, sizeof(fdt_node_attrs) * GN, GN, 8ull * tslots, 8ull * tslots,
                                         4ull * tslots, 8ull * tslots, 8ull * tslots, 16, 4ull * NE, 8ull * NE,
                                         4ull * NE, 4ull * NE, 4ull * NE, 4ull * NE, 4ull * (nm + 1),
                                         name_bytes_.size() + 1, 4ull * name_off_.size(), 4ull * name_len_.size(),
                                         size_t(std::min<uint64_t>(tslots, uint64_t(TN) + NE + 1)) *
                                             FDY_PACK_KEY_BYTES}));
        Scratch& s1 = *s1_;
        if (debug) cuda_check(cudaEventRecord(ev[5], dev_.stream()), "cudaEventRecord");
        FdyPackArgs& a = a_;
        a.graphs = d_graphs_;
        a.graphs_bytes = gsize_;
        // uploaded arrays first (one contiguous range, one copy), then the results
        // read back (one contiguous range), then the device-only scratch
        auto* d_rec_off = s1.take<uint64_t>(nm);
        auto* d_rec_len = s1.take<uint64_t>(nm);
        auto* d_node_base = s1.take<uint32_t>(nm);
        auto* d_n_nodes = s1.take<uint32_t>(nm);
        auto* d_n_edges = s1.take<uint32_t>(nm);
        auto* d_member_group = s1.take<uint32_t>(nm);
        auto* d_group_rep = s1.take<uint32_t>(n_groups_);
        auto* d_gnode_base = s1.take<uint32_t>(n_groups_);
        auto* d_pe_node = s1.take<uint32_t>(NE);
        auto* d_pe_stub_hash = s1.take<uint64_t>(NE);
        auto* d_pe_stub_name = s1.take<uint32_t>(NE);
        auto* d_pe_real_name = s1.take<uint32_t>(NE);
        auto* d_pe_need = s1.take<uint32_t>(NE);
        auto* d_entry_base = s1.take<uint32_t>(nm + 1);
        auto* d_names = s1.take<unsigned char>(name_bytes_.size() + 1);
        auto* d_name_off = s1.take<uint32_t>(name_off_.size());
        auto* d_name_len = s1.take<uint32_t>(name_len_.size());
        auto* d_status = s1.take<uint32_t>(nm);
        a.cap = s1.take<uint32_t>(GN);
        a.rep_attrs = s1.take<fdt_node_attrs>(GN);
        a.rep_type = s1.take<uint8_t>(GN);
        a.node_off = s1.take<uint32_t>(TN);
        unsigned char* const back_end = reinterpret_cast<unsigned char*>(a.node_off + TN);
        a.node_member = s1.take<uint32_t>(TN);
        a.node_slot = s1.take<uint32_t>(TN);
        a.tkey = s1.take<unsigned long long>(tslots);
        a.tpos = s1.take<unsigned long long>(tslots);
        a.tuniq = s1.take<uint32_t>(tslots);
        a.upos = s1.take<unsigned long long>(tslots);
        a.uoff = s1.take<uint64_t>(tslots);
        const uint32_t key_cap = std::min<uint32_t>(tslots, TN + NE + 1);  // distinct keys <= key uses
        a.ukey = s1.take<unsigned char>(size_t(key_cap) * FDY_PACK_KEY_BYTES);
        auto* d_small = s1.take<uint32_t>(4);  // ucount, flags
        a.pe_slot = s1.take<uint32_t>(NE);
        a.pe_node = d_pe_node;
        a.pe_stub_hash = d_pe_stub_hash;
        a.pe_stub_name = d_pe_stub_name;
        a.pe_real_name = d_pe_real_name;
        a.pe_need = d_pe_need;
        a.entry_base = d_entry_base;
        a.names = d_names;
        a.name_off = d_name_off;
        a.name_len = d_name_len;
        a.comm_real_hash = manifest_.comm_real_hash;
        a.n_entries = NE;
        a.rec_off = d_rec_off;
        a.rec_len = d_rec_len;
        a.node_base = d_node_base;
        a.n_nodes = d_n_nodes;
        a.n_edges = d_n_edges;
        a.member_group = d_member_group;
        a.group_rep = d_group_rep;
        a.gnode_base = d_gnode_base;
        a.status = d_status;
        a.ucount = d_small;
        a.flags = d_small + 1;
        a.tmask = tslots - 1;
        a.n_members = nm;
        a.total_nodes = TN;
        Upload up1;
        up1.add(d_rec_off, rec_off_);
        up1.add(d_rec_len, rec_len_);
        up1.add(d_node_base, node_base_);
        up1.add(d_n_nodes, n_nodes_);
        up1.add(d_n_edges, n_edges_);
        up1.add(d_member_group, member_group_);
        up1.add(d_group_rep, group_rep_);
        up1.add(d_gnode_base, gnode_base_.data(), n_groups_);
        up1.add(d_pe_node, pe_node_);
        up1.add(d_pe_stub_hash, pe_stub_hash_);
        up1.add(d_pe_stub_name, pe_stub_name_);
        up1.add(d_pe_real_name, pe_real_name_);
        up1.add(d_pe_need, pe_need_);
        up1.add(d_entry_base, entry_base_);
        up1.add(d_names, reinterpret_cast<const unsigned char*>(name_bytes_.data()), name_bytes_.size());
        up1.add(d_name_off, name_off_);
        up1.add(d_name_len, name_len_);
        up1.send(dev_, st_);
        const double t_up = ms_of(tp);
        // record CRCs (parse_graph_at's per-record check) and the whole file's
        // digest (the store header's source_graphs_crc), on the GPU; the whole
        // file only when the caller has not already verified it. A record rarely
        // starts on a 16-byte boundary: its head (up to 15 bytes) and its aligned
        // body are CRCed as two segments, so the body takes the kernel's
        // vectorized path, and the host combines them
        // (crc(A||B) = crc64_combine(crc(A), crc(B), |B|)).
        std::vector<Segment> segs;
        segs.push_back({0, verified_graphs_crc_ ? 0 : gsize_});
        for (uint32_t m = 0; m < nm; ++m) {
            const uint64_t head = std::min<uint64_t>(rec_len_[m], (16 - rec_off_[m] % 16) % 16);
            segs.push_back({rec_off_[m], head});
            segs.push_back({rec_off_[m] + head, rec_len_[m] - head});
        }
        if (debug) cuda_check(cudaEventRecord(ev[0], st_), "cudaEventRecord");
        // on the side stream, concurrent with pass 1 (the record walk is latency
        // bound, the CRC bandwidth bound); joined before the pass-1 sync
        crc_.launch(dev_, d_graphs_, segs, dev_.side_stream());
        if (debug) cuda_check(cudaEventRecord(ev[3], dev_.side_stream()), "cudaEventRecord");
        const double t_crc = ms_of(tp);
        // status | cap | rep_attrs | rep_type | node_off: one copy into pinned memory,
        // read back with the key count
        unsigned char* const back_lo = reinterpret_cast<unsigned char*>(d_status);
        back_ = PinnedLease(dev_, size_t(back_end - back_lo));
        std::vector<uint32_t> small;
        for (uint32_t attempt = 0;; ++attempt) {
            a.seed = 0x46445450ull + 0x9E3779B97F4A7C15ull * attempt;  // "FDTP"
            cuda_check(cudaMemsetAsync(d_status, 0, 4ull * nm, st_), "GPU pack memset");
            cuda_check(cudaMemsetAsync(a.node_member, 0xFF, 4ull * TN, st_), "GPU pack memset");
            cuda_check(cudaMemsetAsync(a.cap, 0, 4ull * GN, st_), "GPU pack memset");
            cuda_check(cudaMemsetAsync(a.tkey, 0, 8ull * tslots, st_), "GPU pack memset");
            cuda_check(cudaMemsetAsync(a.tpos, 0xFF, 8ull * tslots, st_), "GPU pack memset");
            cuda_check(cudaMemsetAsync(d_small, 0, 16, st_), "GPU pack memset");
            cuda_check(fdy_launch_pack_pass1(&a, st_), "GPU pack pass 1");
            if (attempt == 0) crc_.join(st_);
            if (debug) cuda_check(cudaEventRecord(ev[2], st_), "cudaEventRecord");
            d2h(small, d_small, 2, st_);
            cuda_check(cudaMemcpyAsync(back_.data(), back_lo, size_t(back_end - back_lo), cudaMemcpyDeviceToHost, st_),
                       "GPU pack D2H");
            if (debug) cuda_check(cudaEventRecord(ev[1], st_), "cudaEventRecord");
            cuda_check(cudaStreamSynchronize(st_), "GPU pack pass 1");
            tm_.pass1_sync_ms = ms_of(tp);
            if (small[1] == 0) break;
            require(attempt < 4, Errc::cuda_error, "GPU pack: kernel key fingerprints keep colliding");
            ++tm_.retries;
        }
        if (debug) {
            float crc = 0, all = 0, pre = 0, tail = 0;
            cuda_check(cudaEventElapsedTime(&pre, ev[4], ev[0]), "cudaEventElapsedTime");
            float alloc = 0;
            cuda_check(cudaEventElapsedTime(&alloc, ev[4], ev[5]), "cudaEventElapsedTime");
            tm_.pass1_gpu_alloc_ms = alloc;
            cuda_check(cudaEventElapsedTime(&crc, ev[0], ev[3]), "cudaEventElapsedTime");
            cuda_check(cudaEventElapsedTime(&all, ev[0], ev[2]), "cudaEventElapsedTime");
            cuda_check(cudaEventElapsedTime(&tail, ev[2], ev[1]), "cudaEventElapsedTime");
            tm_.pass1_gpu_crc_ms = crc;
            tm_.pass1_gpu_ms = all;
            tm_.pass1_gpu_pre_ms = pre;
            tm_.pass1_gpu_tail_ms = tail;
            for (auto& e : ev) cudaEventDestroy(e);
        }
        nu_ = small[0];
        tm_.kernel_keys = nu_;
        d2h(upos_, a.upos, nu_, st_);
        d2h(uoff_, a.uoff, nu_, st_);
        ukeys_ = PinnedLease(dev_, std::max<size_t>(size_t(nu_) * FDY_PACK_KEY_BYTES, 16));
        if (nu_)
            cuda_check(cudaMemcpyAsync(ukeys_.data(), a.ukey, size_t(nu_) * FDY_PACK_KEY_BYTES,
                                       cudaMemcpyDeviceToHost, st_),
                       "GPU pack D2H");
        cuda_check(cudaStreamSynchronize(st_), "GPU pack pass 1 keys");
        tm_.pass1_upload_ms = t_up;
        tm_.pass1_launch_ms = t_crc;
        auto host_of = [&](const void* d) {
            return back_.data() + (static_cast<const unsigned char*>(d) - back_lo);
        };
        status_ = reinterpret_cast<const uint32_t*>(host_of(d_status));
        cap_ = reinterpret_cast<const uint32_t*>(host_of(a.cap));
        rep_attrs_ = reinterpret_cast<const fdt_node_attrs*>(host_of(a.rep_attrs));
        rep_type_ = host_of(a.rep_type);
        node_off_ = reinterpret_cast<const uint32_t*>(host_of(a.node_off));
        const auto parts = crc_.digests();  // launched ahead of pass 1: complete
        digests_.assign(1 + nm, 0);
        digests_[0] = parts[0];
        // ~1 us per combine (GF(2) powers): 512 records on the worker pool
        parallel_for(nm, nm >= 64 ? 0u : 1u, [&](size_t m) {
            digests_[1 + m] = crc64_combine(parts[1 + 2 * m], parts[2 + 2 * m], segs[2 + 2 * m].length);
        });
    }

    // ------------------------------------------------ host: checks, kernel table, layout

    // apply_rank_patches' checks with the reference's messages, reading the
    // node bytes on the host: only run for a group whose entries the GPU (or
    // the host's table scan) rejected
    void check_patches_exact(uint32_t m) const {
        const uint32_t label = loc_of_[m]->label;
        const bool patched = patches_.has(label);
        auto sit = slots_.per_graph.find(label);
        require(sit == slots_.per_graph.end() || patched, Errc::archive_corruption,
                "comm slot table lists graph " + std::to_string(label) + ", which has no comm patches");
        if (!patched) return;
        const auto entries = patches_.find(label);
        for (const PatchEntryView& e : entries) {
            require(e.node_id < n_nodes_[m], Errc::archive_corruption, "patch entry references missing node");
            const uint8_t* q = node_ptr(m, e.node_id);
            require(q[0] == 0, Errc::archive_corruption, "patch entry references a non-kernel node");
            const NodeView v{q};
            require(v.hash() == e.stub_hash && v.name() == e.stub_name, Errc::archive_corruption,
                    "node " + std::to_string(e.node_id) + " is not the recorded stub " +
                        KernelRef{e.stub_hash, std::string(e.stub_name)}.describe());
            for (uint32_t i = 0; i < e.n_rank; ++i)
                require(uint64_t(e.rank_offset(i)) + 8 <= v.arg_size(), Errc::invalid_argument,
                        "patch offset outside the argument buffer");
            for (uint32_t i = 0; i < e.n_world; ++i)
                require(uint64_t(e.world_offset(i)) + 8 <= v.arg_size(), Errc::invalid_argument,
                        "patch offset outside the argument buffer");
        }
        if (sit == slots_.per_graph.end()) return;
        for (const CommSlot& c : sit->second) {
            bool stub = false;
            for (const PatchEntryView& e : entries) stub = stub || e.node_id == c.node_id;
            require(stub && c.node_id < n_nodes_[m] && node_ptr(m, c.node_id)[0] == 0, Errc::archive_corruption,
                    "comm slot references node " + std::to_string(c.node_id) + ", which is not a patched comm node");
            require(uint64_t(c.offset) + c.width <= NodeView{node_ptr(m, c.node_id)}.arg_size(),
                    Errc::invalid_argument, "comm slot offset outside the argument buffer");
        }
    }

    // errors in the offline packer's order: group by group, decode, topology,
    // patches (representative first)
    void check_errors() const {
        auto decode_error = [&](uint32_t m) {
            const bool crc_bad = digests_[1 + m] != loc_of_[m]->checksum;
            return suspect_[m] || crc_bad || (status_[m] & FDY_PACK_DECODE);
        };
        for (uint32_t g = 0; g < n_groups_; ++g) {
            const uint32_t f = group_first_[g], e = group_end(g);
            for (uint32_t m = f; m < e; ++m) {
                if (!decode_error(m)) continue;
                (void)parse_graph_at(graphs_host_, *loc_of_[m]);  // raises the reference's message
                raise(Errc::binary_format, "graph record for label " + std::to_string(loc_of_[m]->label) +
                                               " failed to decode on the GPU");
            }
            for (uint32_t m = f; m < e; ++m) {
                if (!(status_[m] & FDY_PACK_TOPO)) continue;
                const TopologyKey k = topology_key(parse_graph_at(graphs_host_, *loc_of_[m]));
                const TopologyKey want = topology_key(parse_graph_at(graphs_host_, *loc_of_[group_rep_[g]]));
                require(k == want, Errc::topology_mismatch,
                        "donor topology " + k.hex() + " does not match exec topology " + want.hex());
            }
            bool patch_error = false;
            for (uint32_t m = f; m < e; ++m) patch_error |= patch_bad_[m] || (status_[m] & FDY_PACK_PATCH);
            if (!patch_error) continue;
            check_patches_exact(group_rep_[g]);
            for (uint32_t m = f; m < e; ++m)
                if (m != group_rep_[g]) check_patches_exact(m);
            raise(Errc::archive_corruption, "a patch entry of group " + std::to_string(g) + " was rejected on the GPU");
        }
    }

    // kernel table: every distinct (hash, func attrs, name) in first-occurrence
    // order, where a graph's patch entries' real comm kernels follow its nodes
    // (the GPU table holds both; positions order them)
    void build_kernel_table() {
        std::vector<std::pair<unsigned long long, uint32_t>> order(nu_);  // positions are unique
        for (uint32_t u = 0; u < nu_; ++u) order[u] = {upos_[u], u};
        std::sort(order.begin(), order.end());
        kernels_.assign(nu_, fdt_kernel{});
        ukidx_.assign(nu_, kNoKernel);
        strings_.reserve(size_t(nu_) * 48);
        for (uint32_t k = 0; k < nu_; ++k) {
            const uint32_t u = order[k].second;
            const uint8_t* r = ukeys_.data() + size_t(u) * FDY_PACK_KEY_BYTES;  // hash | fattrs | nl | name
            fdt_kernel& K = kernels_[k];
            const uint32_t nl = rd32(r + 32);
            std::string_view name(reinterpret_cast<const char*>(r + 36), std::min<uint32_t>(nl, FDY_PACK_KEY_NAME));
            if (nl > FDY_PACK_KEY_NAME) {  // a long name: from the host copy (node) or the name table (entry)
                const uint32_t m = uint32_t(upos_[u] >> 32), local = uint32_t(upos_[u]);
                name = local < n_nodes_[m] ? NodeView{G_ + uoff_[u]}.name()
                                           : name_list_[pe_real_name_[entry_base_[m] + (local - n_nodes_[m])]];
            }
            K.binary_hash = rd64(r);
            K.name_off = static_cast<uint32_t>(strings_.size());
            K.name_len = static_cast<uint32_t>(name.size());
            std::memcpy(K.func_attrs, r + 8, 24);
            strings_.append(name);
            ukidx_[u] = k;
        }
    }

    // group layouts (slot capacity = group-wide maximum, round16, in node
    // order), member image offsets and the natural-order tile list
    void layout() {
        blob_off_.assign(GN_, 0);
        g_image_.assign(n_groups_, 0);
        g_desc_.assign(n_groups_, 0);
        for (uint32_t g = 0; g < n_groups_; ++g) {
            uint64_t pool = 0;
            for (uint32_t i = gnode_base_[g]; i < gnode_base_[g + 1]; ++i) {
                blob_off_[i] = static_cast<uint32_t>(pool);
                pool += cap_[i];
            }
            g_desc_[g] = 48ull * n_nodes_[group_rep_[g]];
            g_image_[g] = g_desc_[g] + pool;
        }
        out_off_.assign(nm_, 0);
        tile_base_.assign(nm_, 0);
        for (uint32_t m = 0; m < nm_; ++m) {
            const uint64_t img = g_image_[member_group_[m]];
            out_off_[m] = arena_bytes_;
            arena_bytes_ += img;
            const uint64_t ntiles = (img / 16 + FDT_TILE_CHUNKS - 1) / FDT_TILE_CHUNKS;
            require(ntiles <= UINT32_MAX && img / 8 <= UINT32_MAX, Errc::invalid_argument,
                    "graph image exceeds the store's 32 GiB limit");
            tile_base_[m] = static_cast<uint32_t>(tile_member_.size());
            tile_member_.insert(tile_member_.end(), ntiles, m);
        }
        n_tiles_ = static_cast<uint32_t>(tile_member_.size());
    }

    // rank ops (apply_rank_patches' rank / world writes, then comm slots as
    // value ops), per member in table order, stably sorted by chunk; the stub
    // -> real kernel swap is the GPU's (pack_swaps_kernel)
    void build_rank_ops() {
        const auto t_r = Clock::now();
        rops_of_.assign(nm_, {});
        if (!NE_ && slots_.empty()) return;
        parallel_for(nm_, 0, [&](size_t mi) {
            const uint32_t m = static_cast<uint32_t>(mi);
            const uint32_t label = loc_of_[m]->label;
            const uint32_t gi0 = gnode_base_[member_group_[m]];
            const uint64_t desc = g_desc_[member_group_[m]];
            auto& ops = rops_of_[m];
            const auto entries = patches_.find(label);
            ops.reserve(entries.size() * 4);
            for (const PatchEntryView& e : entries) {
                const uint64_t blob = desc + blob_off_[gi0 + e.node_id];
                for (uint32_t i = 0; i < e.n_rank; ++i)
                    store_detail::emit_write(ops, blob + e.rank_offset(i), 8, FDT_ROP_RANK, 0);
                for (uint32_t i = 0; i < e.n_world; ++i)
                    store_detail::emit_write(ops, blob + e.world_offset(i), 8, FDT_ROP_WORLD, 0);
            }
            auto sit = slots_.per_graph.find(label);
            if (sit != slots_.per_graph.end())
                for (const CommSlot& c : sit->second)
                    store_detail::emit_write(ops, desc + blob_off_[gi0 + c.node_id] + c.offset, c.width,
                                             FDT_ROP_VALUE, c.value_index);
            const auto by_chunk = [](const fdt_rank_op& x, const fdt_rank_op& y) { return x.chunk < y.chunk; };
            if (!std::is_sorted(ops.begin(), ops.end(), by_chunk))  // entries usually come in node order
                std::stable_sort(ops.begin(), ops.end(), by_chunk);
        });
        tm_.rank_ops_ms = ms_of(t_r);
    }

    // ------------------------------------------------ pass 2: images, swaps, diff counts
    void pass2() {
        const uint32_t nm = nm_, n_tiles = n_tiles_, nu = nu_;
        s2_.emplace(dev_, Scratch::need({4ull * GN_, 8ull * nm, 4ull * nm, 8ull * n_groups_, 4ull * std::max(nu, 1u),
                                         4ull * n_tiles, 4ull * n_tiles, n_tiles, 4ull * n_tiles, arena_bytes_,
                                         arena_bytes_ / 16}));
        Scratch& s2 = *s2_;
        FdyPackArgs& a = a_;
        auto* d_blob_off = s2.take<uint32_t>(GN_);  // uploaded: one contiguous range
        auto* d_out_off = s2.take<uint64_t>(nm);
        auto* d_tile_base = s2.take<uint32_t>(nm);
        auto* d_g_image = s2.take<uint64_t>(n_groups_);
        auto* d_ukidx = s2.take<uint32_t>(std::max(nu, 1u));
        auto* d_tile_member = s2.take<uint32_t>(n_tiles);
        a.tile_count = s2.take<uint32_t>(n_tiles);  // read back: one contiguous range
        a.tile_reloc = s2.take<uint8_t>(n_tiles);
        d_diff_lo_ = s2.take<uint32_t>(n_tiles);
        a.arena = s2.take<unsigned char>(arena_bytes_);
        a.meta = s2.take<uint8_t>(arena_bytes_ / 16);
        a.blob_off = d_blob_off;
        a.out_off = d_out_off;
        a.tile_base = d_tile_base;
        a.g_image = d_g_image;
        a.ukidx = d_ukidx;
        a.tile_member = d_tile_member;
        a.diff_lo = d_diff_lo_;
        a.n_tiles = n_tiles;
        Upload up2;
        up2.add(d_blob_off, blob_off_);
        up2.add(d_out_off, out_off_);
        up2.add(d_tile_base, tile_base_);
        up2.add(d_g_image, g_image_);
        up2.add(d_ukidx, ukidx_);
        up2.add(d_tile_member, tile_member_);
        up2.send(dev_, st_);
        cuda_check(fdy_launch_pack_pass2(&a, st_), "GPU pack pass 2");
        const auto* back2_lo = reinterpret_cast<const unsigned char*>(a.tile_count);
        const size_t back2_bytes = size_t(reinterpret_cast<const unsigned char*>(a.tile_reloc + n_tiles) - back2_lo);
        back2_ = PinnedLease(dev_, std::max<size_t>(back2_bytes, 16));
        if (n_tiles)
            cuda_check(cudaMemcpyAsync(back2_.data(), back2_lo, back2_bytes, cudaMemcpyDeviceToHost, st_),
                       "GPU pack D2H");
        cuda_check(cudaStreamSynchronize(st_), "GPU pack pass 2");
        tile_count_ = reinterpret_cast<const uint32_t*>(back2_.data());
        tile_reloc_ = back2_.data() + (reinterpret_cast<const unsigned char*>(a.tile_reloc) - back2_lo);
    }

    // ------------------------------------------------ host: tables and sections

    // groups (layout, node attributes, edges, topology key), members, tiles with
    // their diff and shared rank-op ranges, relocation-free tiles first
    void build_tables() {
        diff_lo_.assign(n_tiles_, 0);
        n_diffs_ = 0;
        for (uint32_t t = 0; t < n_tiles_; ++t) {
            diff_lo_[t] = static_cast<uint32_t>(n_diffs_);
            n_diffs_ += tile_count_[t];
        }
        require(n_diffs_ < (1ull << 32), Errc::invalid_argument, "template store exceeds 2^32 diff entries");
        groups_.assign(n_groups_, fdt_group{});
        members_.assign(nm_, fdt_member{});
        const auto& groups_in = manifest_.grouping.groups;
        // section offsets first (prefix sums), then every group's attributes, edges
        // and topology key on host threads
        size_t n_attrs = 0, n_edge_words = 0;
        for (uint32_t g = 0; g < n_groups_; ++g) {
            const uint32_t rep = group_rep_[g];
            fdt_group& Gp = groups_[g];
            Gp.image_bytes = g_image_[g];
            Gp.n_nodes = n_nodes_[rep];
            Gp.n_edges = n_edges_[rep];
            Gp.first_member = group_first_[g];
            Gp.n_members = group_end(g) - group_first_[g];
            Gp.representative = groups_in[g].representative;
            Gp.attrs_first = static_cast<uint32_t>(n_attrs);
            Gp.edges_off = n_edge_words * sizeof(uint32_t);
            n_attrs += gnode_base_[g + 1] - gnode_base_[g];
            n_edge_words += 2ull * Gp.n_edges;
            timages_bytes_ = (timages_bytes_ + 15) / 16 * 16;
            Gp.timage_off = timages_bytes_;  // TIMAGES-relative until rebased
            timages_bytes_ += g_image_[g];
        }
        attrs_.resize(n_attrs);
        edges_.resize(n_edge_words);
        parallel_for(n_groups_, 0, [&](size_t gi) {
            const uint32_t g = static_cast<uint32_t>(gi);
            fdt_group& Gp = groups_[g];
            const uint32_t rep = group_rep_[g], N = Gp.n_nodes, E = Gp.n_edges;
            std::copy(rep_attrs_ + gnode_base_[g], rep_attrs_ + gnode_base_[g + 1], attrs_.begin() + Gp.attrs_first);
            const uint8_t* etab = G_ + rec_off_[rep] + rec_len_[rep] - 8ull * E;
            if (E) std::memcpy(edges_.data() + Gp.edges_off / sizeof(uint32_t), etab, 8ull * E);
            // topology key of the representative (topology_key, graph_model.cpp)
            Sink k;
            k.u64(N);
            for (uint32_t n = 0; n < N; ++n) {
                const uint8_t t = rep_type_[gnode_base_[g] + n];  // read back with the attributes
                k.u8(t);
                if (t == 0) {
                    const fdt_node_attrs& at = rep_attrs_[gnode_base_[g] + n];
                    k.u32(at.cluster[0]);
                    k.u32(at.cluster[1]);
                    k.u32(at.cluster[2]);
                    k.i32(at.sched_policy);
                    k.i32(at.sync_default);
                    k.i32(at.sync_remote);
                    k.u8(at.attr_query ? 1 : 0);
                }
            }
            k.u64(E);
            k.raw(etab, 8ull * E);
            const Digest128 key = murmur3_x64_128(k.bytes().data(), k.size(), 0x464E4447ull);
            Gp.key_hi = key.hi;
            Gp.key_lo = key.lo;
        });
        // members' tiles, group by group on host threads: rank-op ranges are shared
        // per (group, tile index), so each group builds its own op list, which are
        // then concatenated in group order (the offline packer's single list)
        tiles_.assign(n_tiles_, fdt_tile{});
        std::vector<std::vector<fdt_rank_op>> grops(n_groups_);
        parallel_for(n_groups_, 0, [&](size_t gi) {
            const uint32_t g = static_cast<uint32_t>(gi);
            const fdt_group& Gp = groups_[g];
            std::vector<fdt_rank_op>& gops = grops[g];
            // per tile index: the distinct op slices stored so far, as ranges of gops
            std::vector<std::vector<std::pair<uint32_t, uint32_t>>> shared_ops;
            for (uint32_t m = Gp.first_member; m < Gp.first_member + Gp.n_members; ++m) {
                fdt_member& M = members_[m];
                M.label = loc_of_[m]->label;
                M.group = g;
                M.out_off = out_off_[m];
                M.n_nodes = Gp.n_nodes;
                M.first_tile = tile_base_[m];
                const uint64_t nchunks = g_image_[g] / 16;
                const uint32_t ntiles = static_cast<uint32_t>((nchunks + FDT_TILE_CHUNKS - 1) / FDT_TILE_CHUNKS);
                M.n_tiles = ntiles;
                shared_ops.resize(std::max<size_t>(shared_ops.size(), ntiles));
                const auto& ops = rops_of_[m];
                size_t rpos = 0;
                for (uint32_t t = 0; t < ntiles; ++t) {
                    const uint64_t cb = uint64_t(t) * FDT_TILE_CHUNKS;
                    const uint64_t ce = std::min<uint64_t>(nchunks, cb + FDT_TILE_CHUNKS);
                    fdt_tile& T = tiles_[tile_base_[m] + t];
                    T.src_off = Gp.timage_off + 16 * cb;
                    T.dst_off = out_off_[m] + 16 * cb;
                    T.nchunks = static_cast<uint32_t>(ce - cb);
                    T.member = m;
                    T.chunk_base = static_cast<uint32_t>(cb);
                    T.diff_lo = diff_lo_[tile_base_[m] + t];
                    T.diff_hi = T.diff_lo + tile_count_[tile_base_[m] + t];
                    const size_t r_begin = rpos;
                    while (rpos < ops.size() && ops[rpos].chunk < ce) ++rpos;
                    const size_t n_ops = rpos - r_begin;
                    const std::pair<uint32_t, uint32_t>* hit = nullptr;
                    for (const auto& c : shared_ops[t])
                        if (c.second - c.first == n_ops &&
                            std::memcmp(gops.data() + c.first, ops.data() + r_begin, n_ops * sizeof(fdt_rank_op)) ==
                                0) {
                            hit = &c;
                            break;
                        }
                    if (!hit) {
                        const uint32_t lo = static_cast<uint32_t>(gops.size());
                        gops.insert(gops.end(), ops.begin() + static_cast<long>(r_begin),
                                    ops.begin() + static_cast<long>(rpos));
                        shared_ops[t].push_back({lo, static_cast<uint32_t>(gops.size())});
                        hit = &shared_ops[t].back();
                    }
                    T.rop_lo = hit->first;  // group-relative until the lists are joined
                    T.rop_hi = hit->second;
                }
            }
        });
        for (uint32_t g = 0; g < n_groups_; ++g) {
            const uint32_t base = static_cast<uint32_t>(rops_.size());
            rops_.insert(rops_.end(), grops[g].begin(), grops[g].end());
            const fdt_group& Gp = groups_[g];
            if (Gp.n_members == 0) continue;
            const uint32_t last = Gp.first_member + Gp.n_members - 1;
            for (uint32_t t = tile_base_[Gp.first_member]; t < tile_base_[last] + members_[last].n_tiles; ++t) {
                tiles_[t].rop_lo += base;
                tiles_[t].rop_hi += base;
            }
        }
        // relocation-free template tiles first (stable), as the offline packer orders them
        uint32_t n_plain = 0;
        for (uint32_t t = 0; t < n_tiles_; ++t) n_plain += tile_reloc_[t] ? 0 : 1;
        std::vector<fdt_tile> ordered(n_tiles_);
        for (uint32_t t = 0, p = 0, r = n_plain; t < n_tiles_; ++t) ordered[tile_reloc_[t] ? r++ : p++] = tiles_[t];
        n_plain_ = n_plain;
        tiles_ = std::move(ordered);
    }

    // the header and the section layout, in the offline packer's order
    void place_sections() {
        fdt_header& h = h_;
        h = fdt_header{};
        std::memcpy(h.magic, "FNDT", 4);
        h.version = FDT_VERSION;
        h.header_bytes = sizeof(fdt_header);
        h.n_groups = n_groups_;
        h.n_members = nm_;
        h.n_kernels = static_cast<uint32_t>(kernels_.size());
        h.n_tiles = n_tiles_;
        h.tile_chunks = FDT_TILE_CHUNKS;
        h.n_diffs = static_cast<uint32_t>(n_diffs_);
        h.n_rank_ops = static_cast<uint32_t>(rops_.size());
        h.source_graphs_crc = verified_graphs_crc_ ? *verified_graphs_crc_ : digests_[0];
        // a caller that verified graphs.bin verified every input against the manifest
        const auto digest_of = [&](const char* rel, std::span<const uint8_t> bytes) {
            if (verified_graphs_crc_) {
                auto it = manifest_.file_digests.find(rel);
                if (it != manifest_.file_digests.end()) return it->second;
            }
            return crc64(bytes);
        };
        h.source_patch_crc = digest_of("patch.bin", patch_bin_);
        h.old_base = manifest_.allocator.base;
        h.final_offset = manifest_.final_offset;
        h.real_comm_hash = manifest_.comm_real_hash;
        h.members_image_bytes = arena_bytes_;
        h.total_nodes = total_nodes_;
        h.n_plain_tiles = n_plain_;
        h.n_values = slots_.empty() ? 0u : slots_.n_values;
        h.source_slots_crc = slots_bin_.empty() ? 0ull : digest_of("comm_slots.bin", slots_bin_);
        uint64_t at = sizeof(fdt_header);
        auto place = [&](int id, uint64_t bytes) {
            at = (at + kSectionAlign - 1) / kSectionAlign * kSectionAlign;
            h.sec[id] = {at, bytes};
            at += bytes;
        };
        place(FDT_SEC_TIMAGES, timages_bytes_);
        timg_base_ = h.sec[FDT_SEC_TIMAGES].offset;
        for (auto& Gp : groups_) Gp.timage_off += timg_base_;
        for (auto& T : tiles_) T.src_off += timg_base_;
        place(FDT_SEC_GROUPS, groups_.size() * sizeof(fdt_group));
        place(FDT_SEC_CMETA, timages_bytes_ / 16);
        place(FDT_SEC_MEMBERS, members_.size() * sizeof(fdt_member));
        place(FDT_SEC_TILES, tiles_.size() * sizeof(fdt_tile));
        place(FDT_SEC_DIDX, n_diffs_ * sizeof(uint16_t));
        place(FDT_SEC_DDATA, n_diffs_ * sizeof(uint64_t));
        place(FDT_SEC_ROPS, rops_.size() * sizeof(fdt_rank_op));
        place(FDT_SEC_KERNELS, kernels_.size() * sizeof(fdt_kernel));
        place(FDT_SEC_NODEATTRS, attrs_.size() * sizeof(fdt_node_attrs));
        place(FDT_SEC_EDGES, edges_.size() * sizeof(uint32_t));
        place(FDT_SEC_STRINGS, strings_.size());
        blob_bytes_ = (at + kSectionAlign - 1) / kSectionAlign * kSectionAlign;
    }

    // the host copy: header, host sections, zero padding (device sections are
    // filled by pass 3's read-back, or left out)
    DevicePackResult host_sections() {
        const fdt_header& h = h_;
        DevicePackResult out;
        out.host_bytes.reset(new uint8_t[blob_bytes_]);  // not zeroed: every byte is written below
        out.host_size = blob_bytes_;
        out.host_complete = full_host_copy_;
        uint8_t* hb = out.host_bytes.get();
        uint64_t at0 = sizeof h;
        std::vector<int> by_offset(FDT_NSEC);
        for (int i = 0; i < FDT_NSEC; ++i) by_offset[i] = i;
        std::sort(by_offset.begin(), by_offset.end(), [&](int x, int y) { return h.sec[x].offset < h.sec[y].offset; });
        for (int id : by_offset) {
            std::memset(hb + at0, 0, h.sec[id].offset - at0);
            at0 = h.sec[id].offset + h.sec[id].bytes;
        }
        std::memset(hb + at0, 0, blob_bytes_ - at0);
        std::memcpy(hb, &h, sizeof h);
        auto put = [&](int id, const void* src) {
            if (h.sec[id].bytes) std::memcpy(hb + h.sec[id].offset, src, h.sec[id].bytes);
        };
        put(FDT_SEC_GROUPS, groups_.data());
        put(FDT_SEC_MEMBERS, members_.data());
        put(FDT_SEC_TILES, tiles_.data());
        put(FDT_SEC_ROPS, rops_.data());
        put(FDT_SEC_KERNELS, kernels_.data());
        put(FDT_SEC_NODEATTRS, attrs_.data());
        put(FDT_SEC_EDGES, edges_.data());
        put(FDT_SEC_STRINGS, strings_.data());
        return out;
    }

    // ------------------------------------------------ pass 3: device sections
    void pass3(DevicePackResult& out) {
        const fdt_header& h = h_;
        FdyPackArgs& a = a_;
        uint8_t* hb = out.host_bytes.get();
        out.blob = DeviceBuffer(dev_, blob_bytes_);
        unsigned char* db = out.blob.data();
        cuda_check(cudaMemsetAsync(db, 0, blob_bytes_, st_), "GPU pack memset");
        // the host-built sections (header .. strings, without the device ones)
        cuda_check(cudaMemcpyAsync(db, hb, sizeof h, cudaMemcpyHostToDevice, st_), "GPU pack H2D");
        for (int id : {FDT_SEC_GROUPS, FDT_SEC_MEMBERS, FDT_SEC_TILES, FDT_SEC_ROPS, FDT_SEC_KERNELS,
                       FDT_SEC_NODEATTRS, FDT_SEC_EDGES, FDT_SEC_STRINGS})
            if (h.sec[id].bytes)
                cuda_check(cudaMemcpyAsync(db + h.sec[id].offset, hb + h.sec[id].offset, h.sec[id].bytes,
                                           cudaMemcpyHostToDevice, st_),
                           "GPU pack H2D");
        a.didx = reinterpret_cast<uint16_t*>(db + h.sec[FDT_SEC_DIDX].offset);
        a.ddata = reinterpret_cast<uint64_t*>(db + h.sec[FDT_SEC_DDATA].offset);
        h2d(d_diff_lo_, diff_lo_, st_);
        cuda_check(fdy_launch_pack_pass3(&a, st_), "GPU pack pass 3");
        // template images = the representatives' pack images (+ their relocation meta)
        for (uint32_t g = 0; g < n_groups_; ++g) {
            const uint64_t src = out_off_[group_rep_[g]];
            const uint64_t dst = groups_[g].timage_off;  // blob-relative now
            cuda_check(cudaMemcpyAsync(db + dst, a.arena + src, g_image_[g], cudaMemcpyDeviceToDevice, st_),
                       "GPU pack template image");
            cuda_check(cudaMemcpyAsync(db + h.sec[FDT_SEC_CMETA].offset + (dst - timg_base_) / 16, a.meta + src / 16,
                                       g_image_[g] / 16, cudaMemcpyDeviceToDevice, st_),
                       "GPU pack template meta");
        }
        for (int id : {FDT_SEC_TIMAGES, FDT_SEC_CMETA, FDT_SEC_DIDX, FDT_SEC_DDATA})
            if (h.sec[id].bytes && full_host_copy_)
                cuda_check(cudaMemcpyAsync(hb + h.sec[id].offset, db + h.sec[id].offset, h.sec[id].bytes,
                                           cudaMemcpyDeviceToHost, st_),
                           "GPU pack D2H");
        cuda_check(cudaStreamSynchronize(st_), "GPU pack pass 3");
    }

    // inputs
    Device& dev_;
    std::span<const uint8_t> graphs_host_;
    const uint8_t* G_;
    uint64_t gsize_;
    const unsigned char* d_graphs_;
    std::span<const uint8_t> patch_bin_;
    const Manifest& manifest_;
    std::span<const uint8_t> slots_bin_;
    bool full_host_copy_;
    const uint64_t* verified_graphs_crc_;
    std::future<PatchView>* patch_view_;
    cudaStream_t st_ = nullptr;
    Clock::time_point t_all_;
    DevicePackTimings tm_;
    PatchView patches_;
    CommSlotTable slots_;
    // members, group-major
    uint32_t n_groups_ = 0, nm_ = 0, TN_ = 0, GN_ = 0;
    uint64_t total_nodes_ = 0;
    std::vector<uint64_t> rec_off_, rec_len_;
    std::vector<uint32_t> node_base_, n_nodes_, n_edges_, member_group_, group_rep_, group_first_, gnode_base_;
    std::vector<const GraphLocator*> loc_of_;
    std::vector<uint8_t> suspect_;  // the host already sees the record is malformed
    // patch entries
    std::vector<uint32_t> pe_node_, pe_stub_name_, pe_real_name_, pe_need_, entry_base_;
    std::vector<uint64_t> pe_stub_hash_;
    std::vector<uint8_t> patch_bad_;  // the host already sees a patch / slot problem
    std::vector<std::string_view> name_list_;
    std::string name_bytes_;
    std::vector<uint32_t> name_off_, name_len_;
    uint32_t NE_ = 0, tslots_ = 1024;
    // pass 1
    std::optional<Scratch> s1_;
    FdyPackArgs a_{};
    uint32_t nu_ = 0;
    std::vector<unsigned long long> upos_;
    std::vector<uint64_t> uoff_, digests_;
    PinnedLease ukeys_, back_;
    CrcJob crc_;
    const uint32_t *status_ = nullptr, *cap_ = nullptr, *node_off_ = nullptr;
    const fdt_node_attrs* rep_attrs_ = nullptr;
    const uint8_t* rep_type_ = nullptr;
    // kernel table, layout, rank ops
    std::vector<fdt_kernel> kernels_;
    std::string strings_;
    std::vector<uint32_t> ukidx_, blob_off_, tile_base_, tile_member_;
    std::vector<uint64_t> g_image_, g_desc_, out_off_;
    uint64_t arena_bytes_ = 0;
    uint32_t n_tiles_ = 0;
    std::vector<std::vector<fdt_rank_op>> rops_of_;
    // pass 2
    std::optional<Scratch> s2_;
    PinnedLease back2_;
    const uint32_t* tile_count_ = nullptr;
    const uint8_t* tile_reloc_ = nullptr;
    uint32_t* d_diff_lo_ = nullptr;
    // tables and sections
    std::vector<uint32_t> diff_lo_;
    uint64_t n_diffs_ = 0, timages_bytes_ = 0, timg_base_ = 0, blob_bytes_ = 0;
    uint32_t n_plain_ = 0;
    std::vector<fdt_group> groups_;
    std::vector<fdt_member> members_;
    std::vector<fdt_tile> tiles_;
    std::vector<fdt_rank_op> rops_;
    std::vector<uint32_t> edges_;
    std::vector<fdt_node_attrs> attrs_;
    fdt_header h_{};
};

}  // namespace

DevicePackResult pack_template_store_device(Device& dev, std::span<const uint8_t> graphs_host,
                                            const unsigned char* d_graphs, std::span<const uint8_t> patch_bin,
                                            const Manifest& manifest, std::span<const uint8_t> slots_bin,
                                            PackStats* stats, DevicePackTimings* timings, bool full_host_copy,
                                            const uint64_t* verified_graphs_crc,
                                            std::future<PatchView>* patch_view) {
    DevicePacker packer(dev, graphs_host, d_graphs, patch_bin, manifest, slots_bin, full_host_copy,
                        verified_graphs_crc, patch_view);
    try {
        return packer.run(stats, timings);
    } catch (...) {
        // copies into the packer's pinned leases may still be in flight: they
        // must land before the leases go back to the pool
        cudaStreamSynchronize(dev.stream());
        throw;
    }
}

std::vector<uint8_t> pack_archive_store_device(Device& dev, const std::filesystem::path& archive,
                                               DevicePackTimings* timings) {
    ArchivePaths paths{archive};
    const auto mtext = slurp(paths.manifest());
    const Manifest man = parse_manifest(std::string(mtext.begin(), mtext.end()));
    const auto graphs = slurp(paths.graphs());
    const auto patch = slurp(paths.patch_table());
    const bool has_slots = man.file_digests.count("comm_slots.bin") != 0;
    const auto slots = has_slots ? slurp(paths.comm_slots()) : std::vector<uint8_t>{};
    dev.make_current();
    DeviceBuffer d(dev, (graphs.size() + 256) / 256 * 256);  // kernels read whole 16-byte units
    cuda_check(cudaMemcpyAsync(d.data(), graphs.data(), graphs.size(), cudaMemcpyHostToDevice, dev.stream()),
               "cudaMemcpyAsync(graphs.bin)");
    DevicePackResult r = pack_template_store_device(dev, graphs, d.data(), patch, man, slots, nullptr, timings);
    const auto h = r.host();
    return std::vector<uint8_t>(h.begin(), h.end());
}

}  // namespace foundry
