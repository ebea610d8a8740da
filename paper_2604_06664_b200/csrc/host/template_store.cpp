// Template store packer + host view (format and semantics: store_format.h).
#include "foundry/template_store.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <unordered_map>

#include "foundry/bytes.hpp"
#include "foundry/parallel.hpp"

namespace foundry {

namespace {

constexpr uint32_t kNoKernel = 0xFFFFFFFFu;
constexpr size_t kSectionAlign = 256;

uint32_t round16(uint64_t v) { return static_cast<uint32_t>((v + 15) / 16 * 16); }

uint32_t blob_len_of(const GraphNode& n) {
    switch (n.type) {
        case NodeType::Kernel: return static_cast<uint32_t>(n.kernel_params().arg_buffer.size());
        case NodeType::Memcpy:
        case NodeType::Memset: return 24;
        default: return 0;
    }
}

// Kernel table: unique (KernelRef, FuncAttrs) pairs.
// Indices are assigned by a sequential pre-pass (intern) so the store is
// deterministic; the parallel phases only call lookup() on a frozen table.
class KernelTable {
public:
    uint32_t intern(const KernelRef& ref, const FuncAttrs& fa) {
        auto [it, fresh] = index_.try_emplace(key(ref, fa), static_cast<uint32_t>(refs_.size()));
        if (fresh) {
            refs_.push_back(ref);
            attrs_.push_back(fa);
        }
        return it->second;
    }
    uint32_t lookup(const KernelRef& ref, const FuncAttrs& fa) const {
        auto it = index_.find(key(ref, fa));
        require(it != index_.end(), Errc::invalid_argument, "kernel table: missing entry");
        return it->second;
    }
    size_t size() const { return refs_.size(); }
    const KernelRef& ref(size_t i) const { return refs_[i]; }
    const FuncAttrs& attrs(size_t i) const { return attrs_[i]; }

private:
    static std::string key(const KernelRef& ref, const FuncAttrs& fa) {
        std::string k(sizeof(uint64_t) + sizeof(FuncAttrs), '\0');
        std::memcpy(k.data(), &ref.binary_hash, 8);
        std::memcpy(k.data() + 8, &fa, sizeof(FuncAttrs));
        return k + ref.name;
    }
    std::unordered_map<std::string, uint32_t> index_;
    std::vector<KernelRef> refs_;
    std::vector<FuncAttrs> attrs_;
};

struct GroupLayout {
    uint32_t n_nodes = 0;
    std::vector<uint32_t> blob_off;  // per node, from pool start
    std::vector<uint32_t> cap;       // per node slot capacity (multiple of 16)
    uint64_t pool_bytes = 0;
    uint64_t image_bytes() const { return 48ull * n_nodes + pool_bytes; }
    uint64_t desc_bytes() const { return 48ull * n_nodes; }
};

// Image of one graph under a group layout, plus per-chunk relocation meta.
void build_image(const CapturedGraph& g, const GroupLayout& L, const KernelTable& kt,
                 std::vector<uint8_t>& img, std::vector<uint8_t>& meta) {
    img.assign(L.image_bytes(), 0);
    meta.assign(L.image_bytes() / 16, 0);
    uint8_t* pool = img.data() + L.desc_bytes();
    const uint64_t pool_chunk0 = L.desc_bytes() / 16;
    for (uint32_t i = 0; i < L.n_nodes; ++i) {
        const GraphNode& n = g.nodes[i];
        fdt_node d{};
        d.type = static_cast<uint8_t>(n.type);
        d.kernel = kNoKernel;
        d.blob_off = L.blob_off[i];
        d.blob_len = blob_len_of(n);
        uint8_t* blob = pool + d.blob_off;
        const uint64_t c0 = pool_chunk0 + d.blob_off / 16;
        if (n.type == NodeType::Kernel) {
            const auto& k = n.kernel_params();
            d.kernel = kt.lookup(k.kernel, k.func_attrs);
            d.grid[0] = k.grid.x, d.grid[1] = k.grid.y, d.grid[2] = k.grid.z;
            d.block[0] = k.block.x, d.block[1] = k.block.y, d.block[2] = k.block.z;
            d.shmem = k.shared_mem_bytes;
            std::memcpy(blob, k.arg_buffer.data(), k.arg_buffer.size());
            // every 8-aligned slot with o + 8 <= len is a relocation candidate
            for (uint32_t o = 0; o + 8 <= d.blob_len; o += 8)
                meta[c0 + o / 16] |= (o % 16 == 0) ? FDT_CMETA_LANE0 : FDT_CMETA_LANE1;
        } else if (n.type == NodeType::Memcpy) {
            const auto& m = std::get<MemcpyParams>(n.params);
            std::memcpy(blob, &m.src, 8);
            std::memcpy(blob + 8, &m.dst, 8);
            std::memcpy(blob + 16, &m.length, 8);
            meta[c0] |= FDT_CMETA_LANE0 | FDT_CMETA_LANE1;  // src, dst
        } else if (n.type == NodeType::Memset) {
            const auto& m = std::get<MemsetParams>(n.params);
            std::memcpy(blob, &m.dst, 8);
            std::memcpy(blob + 8, &m.value, 8);
            std::memcpy(blob + 16, &m.length, 8);
            meta[c0] |= FDT_CMETA_LANE0;  // dst only
        }
        std::memcpy(img.data() + 48ull * i, &d, sizeof d);
    }
}

struct MemberOut {
    std::vector<uint32_t> dlane;  // 8-byte lane index within the member image
    std::vector<uint8_t> dreloc;  // the lane's relocation flag in the member
    std::vector<uint64_t> dval;   // the member's lane value
    std::vector<fdt_rank_op> rops;
};

bool lane_flag(const std::vector<uint8_t>& meta, uint64_t lane) {
    return (meta[lane / 2] >> (lane % 2)) & 1u;
}

}  // namespace

namespace store_detail {

// Splits a little-endian write of `width` bytes at image byte offset `at`
// into per-chunk ops.
void emit_write(std::vector<fdt_rank_op>& ops, uint64_t at, uint32_t width, uint8_t kind,
                uint32_t aux) {
    uint64_t b = at;
    while (b < at + width) {
        const uint64_t chunk = b / 16;
        const uint64_t end = std::min<uint64_t>(at + width, (chunk + 1) * 16);
        fdt_rank_op op{};
        op.chunk = static_cast<uint32_t>(chunk);
        op.kind = kind;
        op.shift = static_cast<int8_t>(int64_t(at) - int64_t(chunk * 16));
        // bytes [b, end) of the chunk (at most 16)
        op.mask = static_cast<uint16_t>(((1u << (end - b)) - 1u) << (b - chunk * 16));
        op.aux = aux;
        ops.push_back(op);
        b = end;
    }
}

}  // namespace store_detail

namespace {

using store_detail::emit_write;

template <typename T>
uint64_t put_section(Sink& s, fdt_header& h, int id, const T* data, size_t count) {
    s.align(kSectionAlign);
    h.sec[id].offset = s.size();
    h.sec[id].bytes = count * sizeof(T);
    s.raw(data, count * sizeof(T));
    return h.sec[id].offset;
}

// parallel_for whose failure is the lowest failing index's, not the first in
// time: when several members of a group are bad, the store build reports the
// same one on every run, in the order the GPU packer checks them (member order
// within each phase). The reference's prepare lanes keep whichever failure
// lands first (templater.cpp:100-116), so any one of them is a faithful
// report; this build fixes which.
template <typename Fn>
void parallel_for_first_error(size_t n, unsigned threads, Fn&& fn) {
    std::vector<std::exception_ptr> err(n);
    parallel_for(n, threads, [&](size_t i) {
        try {
            fn(i);
        } catch (...) {
            err[i] = std::current_exception();
        }
    });
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

// apply_rank_patches (rank_forge.cpp:132-152) for graph g, split by what it
// depends on: the stub -> real kernel swap is rank-independent, so it is
// written into g's image here (and so lands in the template / diffs); the
// rank and world writes become rank ops, in table order.
// Comm slots (archive.hpp) follow the rank/world writes as value ops, with
// the checks apply_comm_slots performs.
void patch_graph(const CapturedGraph& g, const PatchTable& patches, const CommSlotTable& slots,
                 const GroupLayout& L, const KernelTable& kt, uint64_t comm_real_hash,
                 std::vector<uint8_t>& img, std::vector<fdt_rank_op>* rops) {
    auto pit = patches.per_graph.find(g.label);
    auto sit = slots.per_graph.find(g.label);
    require(sit == slots.per_graph.end() || pit != patches.per_graph.end(), Errc::archive_corruption,
            "comm slot table lists graph " + std::to_string(g.label) + ", which has no comm patches");
    if (pit == patches.per_graph.end()) return;
    for (const CommPatchEntry& e : pit->second) {
        // the checks apply_rank_patches performs (rank_forge.cpp:136-150)
        require(e.node_id < g.nodes.size(), Errc::archive_corruption,
                "patch entry references missing node");
        const GraphNode& n = g.nodes[e.node_id];
        require(n.type == NodeType::Kernel, Errc::archive_corruption,
                "patch entry references a non-kernel node");
        const auto& kp = n.kernel_params();
        require(kp.kernel == e.stub, Errc::archive_corruption,
                "node " + std::to_string(e.node_id) + " is not the recorded stub " + e.stub.describe());
        const uint32_t real = kt.lookup(KernelRef{comm_real_hash, e.real_name}, kp.func_attrs);
        std::memcpy(img.data() + 48ull * e.node_id + offsetof(fdt_node, kernel), &real, 4);
        const uint64_t blob = L.desc_bytes() + L.blob_off[e.node_id];
        for (uint32_t off : e.rank_offsets) {
            require(uint64_t(off) + 8 <= kp.arg_buffer.size(), Errc::invalid_argument,
                    "patch offset outside the argument buffer");
            if (rops) emit_write(*rops, blob + off, 8, FDT_ROP_RANK, 0);
        }
        for (uint32_t off : e.world_offsets) {
            require(uint64_t(off) + 8 <= kp.arg_buffer.size(), Errc::invalid_argument,
                    "patch offset outside the argument buffer");
            if (rops) emit_write(*rops, blob + off, 8, FDT_ROP_WORLD, 0);
        }
    }
    if (sit != slots.per_graph.end()) {
        for (const CommSlot& c : sit->second) {
            bool stub = false;
            for (const CommPatchEntry& e : pit->second) stub = stub || e.node_id == c.node_id;
            require(stub && c.node_id < g.nodes.size() && g.nodes[c.node_id].type == NodeType::Kernel,
                    Errc::archive_corruption,
                    "comm slot references node " + std::to_string(c.node_id) + ", which is not a patched comm node");
            require(uint64_t(c.offset) + c.width <= g.nodes[c.node_id].kernel_params().arg_buffer.size(),
                    Errc::invalid_argument, "comm slot offset outside the argument buffer");
            if (rops)
                emit_write(*rops, L.desc_bytes() + L.blob_off[c.node_id] + c.offset, c.width, FDT_ROP_VALUE,
                           c.value_index);
        }
    }
    if (rops)
        std::stable_sort(rops->begin(), rops->end(),
                         [](const fdt_rank_op& a, const fdt_rank_op& b) { return a.chunk < b.chunk; });
}

}  // namespace

std::vector<uint8_t> pack_template_store(std::span<const uint8_t> graphs_bin,
                                         std::span<const uint8_t> patch_bin,
                                         const Manifest& manifest, unsigned threads,
                                         PackStats* stats, std::span<const uint8_t> slots_bin) {
    const PatchTable patches = parse_patch_table(patch_bin);
    const CommSlotTable slots = slots_bin.empty() ? CommSlotTable{} : parse_comm_slots(slots_bin);
    KernelTable kt;
    const bool has_patches = !patches.empty();
    if (has_patches) {
        require(manifest.comm_real_hash != 0, Errc::unresolved_kernel,
                "archive carries comm patches but no real comm binary");
    }

    std::vector<fdt_group> groups;
    std::vector<fdt_member> members;
    std::vector<fdt_node_attrs> attrs;
    std::vector<uint32_t> edges;
    Sink timages;
    std::vector<uint8_t> cmeta;
    std::vector<uint16_t> didx;
    std::vector<uint64_t> ddata;
    std::vector<fdt_rank_op> rops;
    std::vector<fdt_tile> tiles;
    uint64_t out_off = 0, total_nodes = 0;

    for (const TemplateGroup& grp : manifest.grouping.groups) {
        require(grp.locators.size() == grp.members.size() && !grp.members.empty(),
                Errc::invalid_argument, "grouping manifest is missing member locators");
        const size_t nm = grp.members.size();
        std::vector<CapturedGraph> graphs(nm);
        parallel_for_first_error(nm, threads, [&](size_t i) {
            graphs[i] = parse_graph_at(graphs_bin, grp.locators[i]);
        });
        // representative = smallest label (templater.hpp:16); members ascending
        size_t rep = 0;
        for (size_t i = 0; i < nm; ++i)
            if (graphs[i].label == grp.representative) rep = i;
        const CapturedGraph& T = graphs[rep];
        const TopologyKey tkey = topology_key(T);
        parallel_for_first_error(nm, threads, [&](size_t i) {
            if (i == rep) return;
            const TopologyKey k = topology_key(graphs[i]);
            require(k == tkey, Errc::topology_mismatch,
                    "donor topology " + k.hex() + " does not match exec topology " + tkey.hex());
        });

        // deterministic kernel-table pre-pass (member order, then real comm kernels)
        for (const auto& g : graphs) {
            for (const auto& n : g.nodes)
                if (n.type == NodeType::Kernel)
                    kt.intern(n.kernel_params().kernel, n.kernel_params().func_attrs);
            auto pit = patches.per_graph.find(g.label);
            if (pit == patches.per_graph.end()) continue;
            for (const CommPatchEntry& e : pit->second)
                if (e.node_id < g.nodes.size() && g.nodes[e.node_id].type == NodeType::Kernel)
                    kt.intern(KernelRef{manifest.comm_real_hash, e.real_name},
                              g.nodes[e.node_id].kernel_params().func_attrs);
        }

        GroupLayout L;
        L.n_nodes = static_cast<uint32_t>(T.nodes.size());
        L.cap.assign(L.n_nodes, 0);
        L.blob_off.assign(L.n_nodes, 0);
        for (const auto& g : graphs)
            for (uint32_t n = 0; n < L.n_nodes; ++n)
                L.cap[n] = std::max(L.cap[n], round16(blob_len_of(g.nodes[n])));
        for (uint32_t n = 0; n < L.n_nodes; ++n) {
            L.blob_off[n] = static_cast<uint32_t>(L.pool_bytes);
            L.pool_bytes += L.cap[n];
        }

        fdt_group G{};
        G.image_bytes = L.image_bytes();
        G.n_nodes = L.n_nodes;
        G.n_edges = static_cast<uint32_t>(T.edges.size());
        G.first_member = static_cast<uint32_t>(members.size());
        G.n_members = static_cast<uint32_t>(nm);
        G.representative = grp.representative;
        G.attrs_first = static_cast<uint32_t>(attrs.size());
        G.edges_off = edges.size() * sizeof(uint32_t);
        G.key_hi = tkey.digest.hi;
        G.key_lo = tkey.digest.lo;
        for (const auto& n : T.nodes) {
            fdt_node_attrs a{};
            a.cluster[0] = n.attrs.cluster_dim.x;
            a.cluster[1] = n.attrs.cluster_dim.y;
            a.cluster[2] = n.attrs.cluster_dim.z;
            a.sched_policy = n.attrs.cluster_scheduling_policy_preference;
            a.sync_default = n.attrs.mem_sync_domain_map_default;
            a.sync_remote = n.attrs.mem_sync_domain_map_remote;
            a.attr_query = n.attrs.attr_query_available ? 1 : 0;
            attrs.push_back(a);
        }
        for (const auto& e : T.edges) {
            edges.push_back(e.from);
            edges.push_back(e.to);
        }

        std::vector<uint8_t> timg, tmeta;
        build_image(T, L, kt, timg, tmeta);
        patch_graph(T, patches, slots, L, kt, manifest.comm_real_hash, timg, nullptr);
        timages.align(16);
        G.timage_off = timages.size();  // rebased onto the section below
        timages.raw(timg);
        cmeta.resize(timages.size() / 16, 0);
        std::copy(tmeta.begin(), tmeta.end(), cmeta.begin() + G.timage_off / 16);

        std::vector<MemberOut> outs(nm);
        parallel_for_first_error(nm, threads, [&](size_t i) {
            const CapturedGraph& g = graphs[i];
            MemberOut& o = outs[i];
            std::vector<uint8_t> img, meta;
            build_image(g, L, kt, img, meta);
            patch_graph(g, patches, slots, L, kt, manifest.comm_real_hash, img, &o.rops);
            // every 8-byte lane whose bytes or relocation flag differ from the
            // template's becomes a diff entry (store_format.h)
            const uint64_t nlanes = img.size() / 8;
            for (uint64_t l = 0; l < nlanes; ++l) {
                const bool f = lane_flag(meta, l);
                if (f == lane_flag(tmeta, l) && std::memcmp(img.data() + 8 * l, timg.data() + 8 * l, 8) == 0)
                    continue;
                uint64_t v;
                std::memcpy(&v, img.data() + 8 * l, 8);
                o.dlane.push_back(static_cast<uint32_t>(l));
                o.dreloc.push_back(f ? 1 : 0);
                o.dval.push_back(v);
            }
        });

        // members of a group whose rank ops for a tile are identical share
        // one stored range (tile index -> op bytes -> range)
        std::vector<std::map<std::string, std::pair<uint32_t, uint32_t>>> shared_ops;
        for (size_t i = 0; i < nm; ++i) {
            MemberOut& o = outs[i];
            fdt_member M{};
            M.label = graphs[i].label;
            M.group = static_cast<uint32_t>(groups.size());
            M.out_off = out_off;
            M.n_nodes = L.n_nodes;
            M.first_tile = static_cast<uint32_t>(tiles.size());
            const uint64_t nchunks = L.image_bytes() / 16;
            const uint64_t ntiles = (nchunks + FDT_TILE_CHUNKS - 1) / FDT_TILE_CHUNKS;
            M.n_tiles = static_cast<uint32_t>(ntiles);
            require(ntiles <= UINT32_MAX && L.image_bytes() / 8 <= UINT32_MAX, Errc::invalid_argument,
                    "graph image exceeds the store's 32 GiB limit");
            shared_ops.resize(std::max<size_t>(shared_ops.size(), ntiles));
            size_t dpos = 0, rpos = 0;
            for (uint64_t t = 0; t < ntiles; ++t) {
                const uint64_t cb = t * FDT_TILE_CHUNKS;
                const uint64_t ce = std::min<uint64_t>(nchunks, cb + FDT_TILE_CHUNKS);
                fdt_tile T{};
                T.src_off = G.timage_off + 16 * cb;  // rebased below
                T.dst_off = out_off + 16 * cb;
                T.nchunks = static_cast<uint32_t>(ce - cb);
                T.member = static_cast<uint32_t>(members.size());
                T.chunk_base = static_cast<uint32_t>(cb);
                T.diff_lo = static_cast<uint32_t>(didx.size());
                for (; dpos < o.dlane.size() && o.dlane[dpos] < 2 * ce; ++dpos) {
                    didx.push_back(static_cast<uint16_t>((o.dlane[dpos] - 2 * cb) |
                                                         (o.dreloc[dpos] ? FDT_DIDX_RELOC : 0u)));
                    ddata.push_back(o.dval[dpos]);
                }
                T.diff_hi = static_cast<uint32_t>(didx.size());
                const size_t r_begin = rpos;
                while (rpos < o.rops.size() && o.rops[rpos].chunk < ce) ++rpos;
                const std::string key(reinterpret_cast<const char*>(o.rops.data() + r_begin),
                                      (rpos - r_begin) * sizeof(fdt_rank_op));
                auto [it, fresh] = shared_ops[t].try_emplace(key);
                if (fresh) {
                    it->second.first = static_cast<uint32_t>(rops.size());
                    rops.insert(rops.end(), o.rops.begin() + static_cast<long>(r_begin),
                                o.rops.begin() + static_cast<long>(rpos));
                    it->second.second = static_cast<uint32_t>(rops.size());
                }
                T.rop_lo = it->second.first;
                T.rop_hi = it->second.second;
                tiles.push_back(T);
            }
            members.push_back(M);
            out_off += L.image_bytes();
            total_nodes += L.n_nodes;
        }
        groups.push_back(G);
    }

    // tiles whose template chunks hold no relocatable lane go first (stable)
    uint32_t n_plain = 0;
    {
        std::vector<fdt_tile> plain, rest;
        for (const fdt_tile& t : tiles) {
            const uint64_t c0 = t.src_off / 16;  // TIMAGES-relative until rebased below
            bool reloc = false;
            for (uint64_t c = c0; !reloc && c < c0 + t.nchunks; ++c) reloc = cmeta[c] != 0;
            (reloc ? rest : plain).push_back(t);
        }
        n_plain = static_cast<uint32_t>(plain.size());
        plain.insert(plain.end(), rest.begin(), rest.end());
        tiles = std::move(plain);
    }

    // kernel table + strings
    std::vector<fdt_kernel> kernels(kt.size());
    std::string strings;
    for (size_t k = 0; k < kt.size(); ++k) {
        kernels[k].binary_hash = kt.ref(k).binary_hash;
        kernels[k].name_off = static_cast<uint32_t>(strings.size());
        kernels[k].name_len = static_cast<uint32_t>(kt.ref(k).name.size());
        std::memcpy(kernels[k].func_attrs, &kt.attrs(k), sizeof(FuncAttrs));
        strings += kt.ref(k).name;
    }

    fdt_header h{};
    std::memcpy(h.magic, "FNDT", 4);
    h.version = FDT_VERSION;
    h.header_bytes = sizeof(fdt_header);
    h.n_groups = static_cast<uint32_t>(groups.size());
    h.n_members = static_cast<uint32_t>(members.size());
    h.n_kernels = static_cast<uint32_t>(kernels.size());
    h.n_tiles = static_cast<uint32_t>(tiles.size());
    h.tile_chunks = FDT_TILE_CHUNKS;
    h.n_diffs = static_cast<uint32_t>(didx.size());
    h.n_rank_ops = static_cast<uint32_t>(rops.size());
    h.source_graphs_crc = crc64(graphs_bin);
    h.source_patch_crc = crc64(patch_bin);
    h.old_base = manifest.allocator.base;
    h.final_offset = manifest.final_offset;
    h.real_comm_hash = manifest.comm_real_hash;
    h.members_image_bytes = out_off;
    h.total_nodes = total_nodes;
    h.n_plain_tiles = n_plain;
    h.n_values = slots.empty() ? 0u : slots.n_values;
    h.source_slots_crc = slots_bin.empty() ? 0ull : crc64(slots_bin);

    Sink s;
    s.zeros(sizeof(fdt_header));
    // TIMAGES first so the group/tile offsets can be rebased before writing them.
    s.align(kSectionAlign);
    const uint64_t timg_base = s.size();
    h.sec[FDT_SEC_TIMAGES] = {timg_base, timages.size()};
    s.raw(timages.bytes());
    for (auto& G : groups) G.timage_off += timg_base;
    for (auto& T : tiles) T.src_off += timg_base;
    put_section(s, h, FDT_SEC_GROUPS, groups.data(), groups.size());
    put_section(s, h, FDT_SEC_CMETA, cmeta.data(), cmeta.size());
    put_section(s, h, FDT_SEC_MEMBERS, members.data(), members.size());
    put_section(s, h, FDT_SEC_TILES, tiles.data(), tiles.size());
    put_section(s, h, FDT_SEC_DIDX, didx.data(), didx.size());
    put_section(s, h, FDT_SEC_DDATA, ddata.data(), ddata.size());
    put_section(s, h, FDT_SEC_ROPS, rops.data(), rops.size());
    put_section(s, h, FDT_SEC_KERNELS, kernels.data(), kernels.size());
    put_section(s, h, FDT_SEC_NODEATTRS, attrs.data(), attrs.size());
    put_section(s, h, FDT_SEC_EDGES, edges.data(), edges.size());
    put_section(s, h, FDT_SEC_STRINGS, strings.data(), strings.size());
    s.align(kSectionAlign);
    s.poke(0, h);

    if (stats) {
        stats->template_bytes = timages.size();
        stats->diff_entries = didx.size();
        stats->rank_ops = rops.size();
        stats->member_image_bytes = out_off;
        stats->store_bytes = s.size();
    }
    return s.release();
}

PackStats pack_archive_store(const std::filesystem::path& archive, unsigned threads) {
    ArchivePaths paths{archive};
    const auto mtext = slurp(paths.manifest());
    Manifest m = parse_manifest(std::string(mtext.begin(), mtext.end()));
    const auto graphs = slurp(paths.graphs());
    const auto patch = slurp(paths.patch_table());
    const bool has_slots = m.file_digests.count("comm_slots.bin") != 0;
    const auto slots = has_slots ? slurp(paths.comm_slots()) : std::vector<uint8_t>{};
    PackStats st;
    const auto store = pack_template_store(graphs, patch, m, threads, &st, slots);
    spit(paths.template_store(), store);
    m.file_digests["templates.fdt"] = crc64(store);
    spit(paths.manifest(), serialize_manifest(m));
    return st;
}

void write_comm_slots(const std::filesystem::path& archive, const CommSlotTable& table) {
    ArchivePaths paths{archive};
    const auto mtext = slurp(paths.manifest());
    Manifest m = parse_manifest(std::string(mtext.begin(), mtext.end()));
    const auto bytes = serialize_comm_slots(table);
    // validate against the graphs it patches before touching the archive
    (void)pack_template_store(slurp(paths.graphs()), slurp(paths.patch_table()), m, 0, nullptr, bytes);
    spit(paths.comm_slots(), bytes);
    m.file_digests["comm_slots.bin"] = crc64(bytes);
    spit(paths.manifest(), serialize_manifest(m));
    if (m.file_digests.count("templates.fdt")) pack_archive_store(archive);
}

// ------------------------------------------------------------------ StoreView

StoreView::StoreView(std::span<const uint8_t> blob) : blob_(blob) {
    require(blob.size() >= sizeof(fdt_header), Errc::archive_corruption,
            "template store: truncated input");
    std::memcpy(&h_, blob.data(), sizeof h_);
    require(std::memcmp(h_.magic, "FNDT", 4) == 0, Errc::archive_corruption,
            "template store: bad magic, expected 'FNDT'");
    require(h_.version == FDT_VERSION, Errc::archive_corruption,
            "template store: unsupported version " + std::to_string(h_.version));
    for (int i = 0; i < FDT_NSEC; ++i)
        require(h_.sec[i].offset <= blob.size() && h_.sec[i].bytes <= blob.size() - h_.sec[i].offset,
                Errc::archive_corruption, "template store: section overruns the blob");
    auto at = [&](int id) { return blob.data() + h_.sec[id].offset; };
    require(h_.sec[FDT_SEC_GROUPS].bytes == h_.n_groups * sizeof(fdt_group) &&
                h_.sec[FDT_SEC_MEMBERS].bytes == h_.n_members * sizeof(fdt_member) &&
                h_.sec[FDT_SEC_KERNELS].bytes == h_.n_kernels * sizeof(fdt_kernel) &&
                h_.sec[FDT_SEC_TILES].bytes == h_.n_tiles * sizeof(fdt_tile),
            Errc::archive_corruption, "template store: section sizes disagree with the header");
    groups_ = reinterpret_cast<const fdt_group*>(at(FDT_SEC_GROUPS));
    members_ = reinterpret_cast<const fdt_member*>(at(FDT_SEC_MEMBERS));
    kernels_ = reinterpret_cast<const fdt_kernel*>(at(FDT_SEC_KERNELS));
    attrs_ = reinterpret_cast<const fdt_node_attrs*>(at(FDT_SEC_NODEATTRS));
    edges_ = at(FDT_SEC_EDGES);
    strings_ = reinterpret_cast<const char*>(at(FDT_SEC_STRINGS));
    validate_tables();
    uint32_t max_label = 0;
    for (uint32_t m = 0; m < h_.n_members; ++m) max_label = std::max(max_label, members_[m].label);
    if (max_label <= 4ull * h_.n_members + 4096) {  // batch labels: dense table
        by_label_.assign(size_t(max_label) + 1, -1);
        for (uint32_t m = 0; m < h_.n_members; ++m) by_label_[members_[m].label] = int32_t(m);
    } else {  // sparse labels: sorted (label, member), the last member of a label wins as above
        for (uint32_t m = 0; m < h_.n_members; ++m) sparse_labels_.push_back({members_[m].label, m});
        std::stable_sort(sparse_labels_.begin(), sparse_labels_.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
    }
}

// Every index and range the kernels and the host readers follow, checked once:
// a store whose digest matches but whose tables do not (a writer bug, a forged
// file) fails here with archive-corruption instead of reading or writing out
// of bounds on the device. Linear in groups + members + kernels + tiles + edges.
void StoreView::validate_tables() const {
    auto bad = [](const std::string& what) { raise(Errc::archive_corruption, "template store: " + what); };
    const fdt_section& ti = h_.sec[FDT_SEC_TIMAGES];
    const uint64_t n_attrs = h_.sec[FDT_SEC_NODEATTRS].bytes / sizeof(fdt_node_attrs);
    const uint64_t edge_bytes = h_.sec[FDT_SEC_EDGES].bytes, string_bytes = h_.sec[FDT_SEC_STRINGS].bytes;
    if (h_.tile_chunks != FDT_TILE_CHUNKS) bad("tile size disagrees with this build");
    if (h_.sec[FDT_SEC_CMETA].bytes != ti.bytes / 16 || h_.sec[FDT_SEC_DIDX].bytes != uint64_t(h_.n_diffs) * 2 ||
        h_.sec[FDT_SEC_DDATA].bytes != uint64_t(h_.n_diffs) * 8 ||
        h_.sec[FDT_SEC_ROPS].bytes != uint64_t(h_.n_rank_ops) * sizeof(fdt_rank_op))
        bad("section sizes disagree with the header");
    if (h_.n_plain_tiles > h_.n_tiles) bad("more relocation-free tiles than tiles");
    const auto in_timages = [&](uint64_t off, uint64_t bytes) {
        return off % 16 == 0 && off >= ti.offset && bytes <= ti.bytes && off - ti.offset <= ti.bytes - bytes;
    };
    for (uint32_t g = 0; g < h_.n_groups; ++g) {
        const fdt_group& G = groups_[g];
        const std::string at = "group " + std::to_string(g) + ": ";
        if (G.image_bytes % 16 || G.image_bytes < 48ull * G.n_nodes || !in_timages(G.timage_off, G.image_bytes))
            bad(at + "template image outside its section");
        if (uint64_t(G.attrs_first) + G.n_nodes > n_attrs) bad(at + "node attributes outside their section");
        if (G.edges_off % 4 || G.edges_off > edge_bytes || 8ull * G.n_edges > edge_bytes - G.edges_off)
            bad(at + "edges outside their section");
        if (uint64_t(G.first_member) + G.n_members > h_.n_members) bad(at + "members outside the member table");
        const uint8_t* e = edges_ + G.edges_off;
        for (uint64_t i = 0; i < 2ull * G.n_edges; ++i) {
            uint32_t v;
            std::memcpy(&v, e + 4 * i, 4);
            if (v >= G.n_nodes) bad(at + "edge endpoint " + std::to_string(v) + " is not a node");
        }
    }
    for (uint32_t k = 0; k < h_.n_kernels; ++k)
        if (kernels_[k].name_off > string_bytes || kernels_[k].name_len > string_bytes - kernels_[k].name_off)
            bad("kernel " + std::to_string(k) + ": name outside the string section");
    for (uint32_t m = 0; m < h_.n_members; ++m) {
        const fdt_member& M = members_[m];
        if (M.group >= h_.n_groups) bad("member " + std::to_string(m) + ": no such group");
        const fdt_group& G = groups_[M.group];
        if (M.n_nodes != G.n_nodes || M.out_off % 16 || M.out_off > h_.members_image_bytes ||
            G.image_bytes > h_.members_image_bytes - M.out_off ||
            uint64_t(M.first_tile) + M.n_tiles > h_.n_tiles)
            bad("member " + std::to_string(m) + ": image or tiles outside the arena");
    }
    for (uint32_t t = 0; t < h_.n_tiles; ++t) {
        fdt_tile T;
        std::memcpy(&T, blob_.data() + h_.sec[FDT_SEC_TILES].offset + uint64_t(t) * sizeof T, sizeof T);
        const uint64_t bytes = 16ull * T.nchunks;
        if (T.nchunks == 0 || T.nchunks > FDT_TILE_CHUNKS || T.member >= h_.n_members ||
            !in_timages(T.src_off, bytes) || T.dst_off % 16 || T.dst_off > h_.members_image_bytes ||
            bytes > h_.members_image_bytes - T.dst_off || T.diff_lo > T.diff_hi || T.diff_hi > h_.n_diffs ||
            T.rop_lo > T.rop_hi || T.rop_hi > h_.n_rank_ops)
            bad("tile " + std::to_string(t) + " reaches outside the store or the arena");
    }
}

std::string_view StoreView::kernel_name(uint32_t k) const {
    return {strings_ + kernels_[k].name_off, kernels_[k].name_len};
}

KernelRef StoreView::kernel_ref(uint32_t k) const {
    return KernelRef{kernels_[k].binary_hash, std::string(kernel_name(k))};
}

FuncAttrs StoreView::kernel_func_attrs(uint32_t k) const {
    FuncAttrs f;
    std::memcpy(&f, kernels_[k].func_attrs, sizeof f);
    return f;
}

const fdt_node_attrs& StoreView::node_attrs(uint32_t g, uint32_t n) const {
    return attrs_[groups_[g].attrs_first + n];
}

std::span<const uint32_t> StoreView::edges(uint32_t g) const {
    return {reinterpret_cast<const uint32_t*>(edges_ + groups_[g].edges_off),
            size_t(groups_[g].n_edges) * 2};
}

int64_t StoreView::member_of(uint32_t label) const {
    if (sparse_labels_.empty()) return label < by_label_.size() ? by_label_[label] : -1;
    auto it = std::upper_bound(sparse_labels_.begin(), sparse_labels_.end(), label,
                               [](uint32_t l, const auto& p) { return l < p.first; });
    return it != sparse_labels_.begin() && (it - 1)->first == label ? int64_t((it - 1)->second) : -1;
}

void StoreView::check_image(uint32_t m, const uint8_t* image) const {
    const fdt_member& M = members_[m];
    const fdt_group& G = groups_[M.group];
    const uint64_t pool = G.image_bytes - 48ull * G.n_nodes;
    for (uint32_t i = 0; i < G.n_nodes; ++i) {
        fdt_node d;
        std::memcpy(&d, image + 48ull * i, sizeof d);
        const uint64_t need = d.type == 1 || d.type == 2 ? 24 : d.type == 0 ? d.blob_len : 0;
        const bool dims = d.type != 0 || (d.grid[0] && d.grid[1] && d.grid[2] && d.block[0] && d.block[1] &&
                                          d.block[2]);  // decode_node's "launch dims must be >= 1"
        if (d.type > 3 || (d.type == 0 && d.kernel >= h_.n_kernels) || !dims || d.blob_off > pool ||
            need > pool - d.blob_off)
            raise(Errc::archive_corruption, "template store: member " + std::to_string(M.label) + " node " +
                                                std::to_string(i) + ": descriptor outside its image");
    }
}

CapturedGraph StoreView::image_to_graph(uint32_t m, std::span<const uint8_t> image) const {
    const fdt_member& M = members_[m];
    const fdt_group& G = groups_[M.group];
    require(image.size() >= G.image_bytes, Errc::invalid_argument, "member image too small");
    check_image(m, image.data());
    CapturedGraph g;
    g.label = M.label;
    g.nodes.resize(G.n_nodes);
    const uint8_t* pool = image.data() + 48ull * G.n_nodes;
    for (uint32_t i = 0; i < G.n_nodes; ++i) {
        fdt_node d;
        std::memcpy(&d, image.data() + 48ull * i, sizeof d);
        GraphNode& n = g.nodes[i];
        n.id = i;
        n.type = static_cast<NodeType>(d.type);
        const uint8_t* blob = pool + d.blob_off;
        if (n.type == NodeType::Kernel) {
            const fdt_node_attrs& a = node_attrs(M.group, i);
            n.attrs.cluster_dim = {a.cluster[0], a.cluster[1], a.cluster[2]};
            n.attrs.cluster_scheduling_policy_preference = a.sched_policy;
            n.attrs.mem_sync_domain_map_default = a.sync_default;
            n.attrs.mem_sync_domain_map_remote = a.sync_remote;
            n.attrs.attr_query_available = a.attr_query != 0;
            KernelNodeParams k;
            require(d.kernel < h_.n_kernels, Errc::archive_corruption,
                    "template store: kernel index out of range");
            k.kernel = kernel_ref(d.kernel);
            k.func_attrs = kernel_func_attrs(d.kernel);
            k.grid = {d.grid[0], d.grid[1], d.grid[2]};
            k.block = {d.block[0], d.block[1], d.block[2]};
            k.shared_mem_bytes = d.shmem;
            k.arg_buffer.assign(blob, blob + d.blob_len);
            n.params = std::move(k);
        } else if (n.type == NodeType::Memcpy) {
            MemcpyParams p;
            std::memcpy(&p.src, blob, 8);
            std::memcpy(&p.dst, blob + 8, 8);
            std::memcpy(&p.length, blob + 16, 8);
            n.params = p;
        } else if (n.type == NodeType::Memset) {
            MemsetParams p;
            std::memcpy(&p.dst, blob, 8);
            std::memcpy(&p.value, blob + 8, 8);
            std::memcpy(&p.length, blob + 16, 8);
            n.params = p;
        } else {
            n.params = EmptyParams{};
        }
    }
    const auto e = edges(M.group);
    g.edges.resize(G.n_edges);
    for (uint32_t i = 0; i < G.n_edges; ++i) g.edges[i] = {e[2 * i], e[2 * i + 1]};
    return g;
}

}  // namespace foundry
