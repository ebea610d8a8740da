// FNDG codec, topology key and structural diff.
// Byte layout and validation order follow the reference (graph_model.cpp:41-303,
// :578-629) so both builds read each other's archives and raise the same errors.
#include "foundry/graph_model.hpp"

#include <algorithm>
#include <sstream>

#include "foundry/bytes.hpp"

namespace foundry {

std::string_view node_type_name(NodeType t) {
    switch (t) {
        case NodeType::Kernel: return "KernelNode";
        case NodeType::Memcpy: return "MemcpyNode";
        case NodeType::Memset: return "MemsetNode";
        case NodeType::Empty: return "EmptyNode";
    }
    return "UnknownNode";
}

void CapturedGraph::canonicalize() {
    for (uint32_t i = 0; i < nodes.size(); ++i) nodes[i].id = i;
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    validate();
}

void CapturedGraph::validate() const {
    for (uint32_t i = 0; i < nodes.size(); ++i) {
        require(nodes[i].id == i, Errc::invalid_argument, "node ids must be dense");
        if (nodes[i].type != NodeType::Kernel) continue;
        const auto& kp = nodes[i].kernel_params();
        require(!kp.arg_buffer.empty(), Errc::invalid_argument,
                "kernel node " + std::to_string(i) + " has empty argument buffer");
        const bool dims_ok = kp.grid.x && kp.grid.y && kp.grid.z && kp.block.x && kp.block.y &&
                             kp.block.z;
        require(dims_ok, Errc::invalid_argument, "launch dims must be >= 1");
    }
    for (size_t i = 0; i < edges.size(); ++i) {
        const GraphEdge& e = edges[i];
        require(e.from < nodes.size() && e.to < nodes.size(), Errc::invalid_argument,
                "edge references missing node");
        require(e.from < e.to, Errc::invalid_argument,
                "edge must go from an earlier node to a later one");
        require(i == 0 || edges[i - 1] < e, Errc::invalid_argument,
                "edges must be in canonical order");
    }
}

namespace {

void put_attrs(Sink& s, const KernelNodeAttrs& a) {
    s.u32(a.cluster_dim.x);
    s.u32(a.cluster_dim.y);
    s.u32(a.cluster_dim.z);
    s.i32(a.cluster_scheduling_policy_preference);
    s.i32(a.mem_sync_domain_map_default);
    s.i32(a.mem_sync_domain_map_remote);
    s.u8(a.attr_query_available ? 1 : 0);
}

KernelNodeAttrs get_attrs(Cursor& c) {
    KernelNodeAttrs a;
    a.cluster_dim = {c.u32(), 0, 0};
    a.cluster_dim.y = c.u32();
    a.cluster_dim.z = c.u32();
    a.cluster_scheduling_policy_preference = c.i32();
    a.mem_sync_domain_map_default = c.i32();
    a.mem_sync_domain_map_remote = c.i32();
    a.attr_query_available = c.u8() != 0;
    return a;
}

void put_dim(Sink& s, const Dim3& d) {
    s.u32(d.x);
    s.u32(d.y);
    s.u32(d.z);
}

Dim3 get_dim(Cursor& c) {
    Dim3 d;
    d.x = c.u32();
    d.y = c.u32();
    d.z = c.u32();
    return d;
}

void put_fattrs(Sink& s, const FuncAttrs& f) {
    for (int32_t v : {f.max_dynamic_shared_size_bytes, f.preferred_shared_memory_carveout,
                      f.cluster_scheduling_policy_preference, f.required_cluster_width,
                      f.required_cluster_height, f.required_cluster_depth})
        s.i32(v);
}

FuncAttrs get_fattrs(Cursor& c) {
    FuncAttrs f;
    f.max_dynamic_shared_size_bytes = c.i32();
    f.preferred_shared_memory_carveout = c.i32();
    f.cluster_scheduling_policy_preference = c.i32();
    f.required_cluster_width = c.i32();
    f.required_cluster_height = c.i32();
    f.required_cluster_depth = c.i32();
    return f;
}

void put_node(Sink& s, const GraphNode& n) {
    s.u8(static_cast<uint8_t>(n.type));
    if (n.type == NodeType::Kernel) {
        const auto& k = n.kernel_params();
        put_attrs(s, n.attrs);
        put_dim(s, k.grid);
        put_dim(s, k.block);
        s.u32(k.shared_mem_bytes);
        s.u64(k.kernel.binary_hash);
        s.str(k.kernel.name);
        put_fattrs(s, k.func_attrs);
        s.u32(static_cast<uint32_t>(k.arg_buffer.size()));
        s.raw(k.arg_buffer);
    } else if (n.type == NodeType::Memcpy) {
        const auto& m = std::get<MemcpyParams>(n.params);
        s.u64(m.src);
        s.u64(m.dst);
        s.u64(m.length);
    } else if (n.type == NodeType::Memset) {
        const auto& m = std::get<MemsetParams>(n.params);
        s.u64(m.dst);
        s.u64(m.value);
        s.u64(m.length);
    }
}

GraphNode get_node(Cursor& c, uint32_t id) {
    GraphNode n;
    n.id = id;
    const uint8_t tag = c.u8();
    n.type = static_cast<NodeType>(tag);
    switch (n.type) {
        case NodeType::Kernel: {
            n.attrs = get_attrs(c);
            KernelNodeParams k;
            k.grid = get_dim(c);
            k.block = get_dim(c);
            k.shared_mem_bytes = c.u32();
            k.kernel.binary_hash = c.u64();
            k.kernel.name = c.str();
            k.func_attrs = get_fattrs(c);
            const uint32_t len = c.u32();
            const uint8_t* p = c.take(len);
            k.arg_buffer.assign(p, p + len);
            n.params = std::move(k);
            break;
        }
        case NodeType::Memcpy: {
            MemcpyParams m;
            m.src = c.u64();
            m.dst = c.u64();
            m.length = c.u64();
            n.params = m;
            break;
        }
        case NodeType::Memset: {
            MemsetParams m;
            m.dst = c.u64();
            m.value = c.u64();
            m.length = c.u64();
            n.params = m;
            break;
        }
        case NodeType::Empty: n.params = EmptyParams{}; break;
        default: raise(Errc::binary_format, "unknown node type tag");
    }
    return n;
}

}  // namespace

TopologyKey topology_key(const CapturedGraph& g) {
    Sink s;
    s.u64(g.nodes.size());
    for (const auto& n : g.nodes) {
        s.u8(static_cast<uint8_t>(n.type));
        if (n.type == NodeType::Kernel) put_attrs(s, n.attrs);
    }
    s.u64(g.edges.size());
    for (const auto& e : g.edges) {
        s.u32(e.from);
        s.u32(e.to);
    }
    return TopologyKey{murmur3_x64_128(s.bytes().data(), s.size(), 0x464E4447ull)};
}

std::vector<uint8_t> encode_graph_record(const CapturedGraph& g) {
    Sink s;
    s.u32(g.label);
    s.u32(static_cast<uint32_t>(g.nodes.size()));
    s.u32(static_cast<uint32_t>(g.edges.size()));
    for (const auto& n : g.nodes) put_node(s, n);
    for (const auto& e : g.edges) {
        s.u32(e.from);
        s.u32(e.to);
    }
    return s.release();
}

CapturedGraph decode_graph_record(std::span<const uint8_t> record) {
    Cursor c(record, Errc::binary_format);
    CapturedGraph g;
    g.label = c.u32();
    const uint32_t nn = c.u32();
    const uint32_t ne = c.u32();
    g.nodes.reserve(std::min<size_t>(nn, record.size()));
    for (uint32_t i = 0; i < nn; ++i) g.nodes.push_back(get_node(c, i));
    g.edges.reserve(std::min<size_t>(ne, record.size() / 8));
    for (uint32_t i = 0; i < ne; ++i) {
        GraphEdge e;
        e.from = c.u32();
        e.to = c.u32();
        g.edges.push_back(e);
    }
    require(c.at_end(), Errc::binary_format, "trailing bytes in graph record");
    g.validate();
    return g;
}

std::vector<uint8_t> serialize_graphs(const std::vector<CapturedGraph>& graphs) {
    Sink s;
    s.raw("FNDG", 4);
    s.u16(1);
    s.u32(static_cast<uint32_t>(graphs.size()));
    const size_t table = s.size();
    for (const auto& g : graphs) {
        s.u32(g.label);
        s.zeros(24);
    }
    for (size_t i = 0; i < graphs.size(); ++i) {
        const auto rec = encode_graph_record(graphs[i]);
        const size_t at = table + 28 * i;
        s.poke<uint64_t>(at + 4, s.size());
        s.poke<uint64_t>(at + 12, rec.size());
        s.poke<uint64_t>(at + 20, crc64(rec));
        s.raw(rec);
    }
    return s.release();
}

std::vector<GraphLocator> parse_graph_locators(std::span<const uint8_t> bytes) {
    Cursor c(bytes, Errc::binary_format);
    c.magic("FNDG");
    const uint16_t version = c.u16();
    require(version == 1, Errc::binary_format,
            "unsupported graph container version " + std::to_string(version));
    const uint32_t count = c.u32();
    std::vector<GraphLocator> out;
    out.reserve(std::min<size_t>(count, bytes.size() / 28));
    for (uint32_t i = 0; i < count; ++i) {
        GraphLocator l;
        l.label = c.u32();
        l.offset = c.u64();
        l.length = c.u64();
        l.checksum = c.u64();
        require(l.offset <= bytes.size() && l.length <= bytes.size() - l.offset,
                Errc::binary_format,
                "graph record for label " + std::to_string(l.label) + " overruns the container");
        out.push_back(l);
    }
    return out;
}

CapturedGraph parse_graph_at(std::span<const uint8_t> bytes, const GraphLocator& loc) {
    const auto rec = bytes.subspan(loc.offset, loc.length);
    require(crc64(rec) == loc.checksum, Errc::binary_format,
            "checksum failure in graph record for label " + std::to_string(loc.label));
    CapturedGraph g = decode_graph_record(rec);
    require(g.label == loc.label, Errc::binary_format, "label mismatch in graph record");
    return g;
}

std::vector<CapturedGraph> parse_graphs(std::span<const uint8_t> bytes) {
    std::vector<CapturedGraph> out;
    for (const auto& l : parse_graph_locators(bytes)) out.push_back(parse_graph_at(bytes, l));
    return out;
}

// ----------------------------------------------------------------------- diff

std::vector<ByteRange> differing_ranges(std::span<const uint8_t> a, std::span<const uint8_t> b) {
    std::vector<ByteRange> runs;
    const size_t common = std::min(a.size(), b.size());
    size_t i = 0;
    while (i < common) {
        if (a[i] == b[i]) {
            ++i;
            continue;
        }
        const size_t start = i;
        while (i < common && a[i] != b[i]) ++i;
        runs.push_back({static_cast<uint32_t>(start), static_cast<uint32_t>(i)});
    }
    if (a.size() != b.size())
        runs.push_back({static_cast<uint32_t>(common),
                        static_cast<uint32_t>(std::max(a.size(), b.size()))});
    return runs;
}

GraphDiff diff(const CapturedGraph& a, const CapturedGraph& b) {
    GraphDiff d;
    d.topology_equal = topology_key(a) == topology_key(b);
    d.label_equal = a.label == b.label;
    const size_t n = std::min(a.nodes.size(), b.nodes.size());
    for (size_t i = 0; i < n; ++i) {
        const GraphNode& x = a.nodes[i];
        const GraphNode& y = b.nodes[i];
        NodeDelta nd;
        nd.node_id = static_cast<uint32_t>(i);
        if (x.type != y.type) {
            nd.memop_changed = true;
        } else if (x.type == NodeType::Kernel) {
            const auto& kx = x.kernel_params();
            const auto& ky = y.kernel_params();
            nd.kernel_changed = !(kx.kernel == ky.kernel) || !(kx.func_attrs == ky.func_attrs);
            nd.dims_changed = !(kx.grid == ky.grid) || !(kx.block == ky.block);
            nd.shared_mem_changed = kx.shared_mem_bytes != ky.shared_mem_bytes;
            nd.arg_byte_ranges = differing_ranges(kx.arg_buffer, ky.arg_buffer);
        } else {
            nd.memop_changed = !(x.params == y.params);
        }
        if (!nd.empty()) d.node_deltas.push_back(std::move(nd));
    }
    return d;
}

std::string GraphDiff::to_text() const {
    std::ostringstream o;
    if (empty()) return "graphs identical\n";
    o << "topology: " << (topology_equal ? "equal" : "DIFFERS") << "\n";
    if (!label_equal) o << "labels differ\n";
    for (const auto& nd : node_deltas) {
        o << "node " << nd.node_id << ":";
        if (nd.kernel_changed) o << " kernel";
        if (nd.dims_changed) o << " dims";
        if (nd.shared_mem_changed) o << " shared-mem";
        if (nd.memop_changed) o << " memop-params";
        if (!nd.arg_byte_ranges.empty()) {
            o << " arg-bytes";
            for (const auto& r : nd.arg_byte_ranges) o << " [" << r.begin << "," << r.end << ")";
        }
        o << "\n";
    }
    return o.str();
}

}  // namespace foundry
