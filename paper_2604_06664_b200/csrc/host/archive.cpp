// Archive side-file codecs (anchors in foundry/archive.hpp).
#include "foundry/archive.hpp"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <memory>
#include <optional>
#include <type_traits>
#include <string_view>
#include <unordered_map>
#include <unordered_set>

#include <json.hpp>

#include "foundry/bytes.hpp"
#include "foundry/parallel.hpp"

namespace foundry {

using nlohmann::json;

// ------------------------------------------------------------ memlayout

std::vector<uint8_t> serialize_event_log(const MemoryEventLog& log) {
    Sink s;
    for (uint64_t v : {log.config.base, log.config.capacity, log.config.granularity,
                       log.starting_offset, log.final_offset, uint64_t(log.records.size())})
        s.u64(v);
    for (const auto& r : log.records) {
        s.u64(r.sequence);
        s.u64(r.size);
        s.u64(r.address);
        s.u64(r.length);
        s.u8(static_cast<uint8_t>(r.window));
    }
    return s.release();
}

MemoryEventLog parse_event_log(std::span<const uint8_t> bytes) {
    Cursor c(bytes, Errc::archive_corruption);
    MemoryEventLog log;
    log.config.base = c.u64();
    log.config.capacity = c.u64();
    log.config.granularity = c.u64();
    log.starting_offset = c.u64();
    log.final_offset = c.u64();
    const uint64_t n = c.u64();
    require(n <= bytes.size() / 33, Errc::archive_corruption, "truncated input");
    log.records.resize(n);
    for (auto& r : log.records) {
        r.sequence = c.u64();
        r.size = c.u64();
        r.address = c.u64();
        r.length = c.u64();
        r.window = static_cast<AllocWindow>(c.u8());
    }
    require(c.at_end(), Errc::archive_corruption, "trailing bytes in event log");
    return log;
}

// ------------------------------------------------------------ grouping

GroupingManifest group_graphs(const std::vector<CapturedGraph>& graphs) {
    struct KeyHash {
        size_t operator()(const TopologyKey& k) const {
            return size_t(k.digest.hi ^ (k.digest.lo * 0x9E3779B97F4A7C15ull));
        }
    };
    GroupingManifest m;
    std::unordered_map<TopologyKey, size_t, KeyHash> slot;
    std::unordered_set<uint32_t> labels;
    for (const auto& g : graphs) {
        require(labels.insert(g.label).second, Errc::invalid_argument,
                "duplicate graph label " + std::to_string(g.label));
        const TopologyKey key = topology_key(g);
        auto [it, fresh] = slot.try_emplace(key, m.groups.size());
        if (fresh) {
            TemplateGroup grp;
            grp.key = key;
            m.groups.push_back(std::move(grp));
        }
        m.groups[it->second].members.push_back(g.label);
    }
    for (auto& grp : m.groups) {
        std::sort(grp.members.begin(), grp.members.end());
        grp.representative = grp.members.front();
    }
    std::sort(m.groups.begin(), m.groups.end(),
              [](const TemplateGroup& a, const TemplateGroup& b) {
                  return a.representative < b.representative;
              });
    m.total_graphs = static_cast<uint32_t>(graphs.size());
    m.template_count = static_cast<uint32_t>(m.groups.size());
    return m;
}

void attach_locators(GroupingManifest& m, const std::vector<GraphLocator>& locators) {
    std::unordered_map<uint32_t, GraphLocator> by_label;
    for (const auto& l : locators) by_label[l.label] = l;
    for (auto& grp : m.groups) {
        grp.locators.clear();
        for (uint32_t label : grp.members) {
            auto it = by_label.find(label);
            require(it != by_label.end(), Errc::archive_corruption,
                    "container has no record for graph " + std::to_string(label));
            grp.locators.push_back(it->second);
        }
    }
}

// ------------------------------------------------------------ manifest

std::string serialize_manifest(const Manifest& m) {
    json groups = json::array();
    for (const auto& g : m.grouping.groups) {
        json locs = json::array();
        for (const auto& l : g.locators) locs.push_back({l.label, l.offset, l.length, l.checksum});
        groups.push_back(json{{"key", g.key.hex()},
                              {"representative", g.representative},
                              {"members", g.members},
                              {"locators", std::move(locs)}});
    }
    json root;
    root["format_version"] = m.format_version;
    root["hash_algorithm"] = m.hash_algorithm;
    root["workload_digest"] = m.workload_digest;
    root["workload"] = m.workload_text;
    root["allocator"] = {{"base", m.allocator.base},
                         {"capacity", m.allocator.capacity},
                         {"granularity", m.allocator.granularity},
                         {"final_offset", m.final_offset}};
    root["kv_cache_bytes"] = m.kv_cache_bytes;
    root["comm"] = {{"world_placeholder", m.comm_world_placeholder},
                    {"real_binary_hash", m.comm_real_hash}};
    root["grouping"] = {{"total", m.grouping.total_graphs},
                        {"templates", m.grouping.template_count},
                        {"groups", std::move(groups)}};
    root["memlayout"] = m.memlayout_ref;
    root["catalog"] = m.catalog_ref;
    root["patch_table"] = m.patch_table_ref;
    root["files"] = m.file_digests;
    return root.dump(2) + "\n";
}

namespace {

// Fast path of parse_manifest: a minimal JSON reader for the shape every
// writer of this format emits (objects, arrays, unsigned integers, strings).
// Anything else -- a float, a negative number, a duplicate key, a missing or
// mistyped field, a failed check -- returns nullopt and the nlohmann path
// below parses the text again and reports exactly as before. The 44 KB
// manifest of the headline archive sits on the critical path of LOAD and
// fdy_prepare_archive (the store digest is checked against it): ~1.2 ms with
// the DOM parser, well under 0.1 ms here.
struct FastJson {
    enum class T : uint8_t { uint, str, arr, obj };
    T t = T::uint;
    uint64_t u = 0;
    std::string s;                                   // str (unescaped)
    std::vector<FastJson> a;                         // arr
    std::vector<std::pair<std::string_view, FastJson>> o;  // obj (keys without escapes)

    const FastJson* at(std::string_view k) const {
        if (t != T::obj) return nullptr;
        for (const auto& [key, v] : o)
            if (key == k) return &v;
        return nullptr;
    }
};

class FastReader {
public:
    explicit FastReader(std::string_view text) : p_(text.data()), e_(text.data() + text.size()) {}

    bool document(FastJson& out) {
        if (!value(out, 0)) return false;
        ws();
        return p_ == e_;
    }

private:
    const char* p_;
    const char* e_;

    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
    }

    bool string(std::string& out, bool allow_escapes) {
        if (p_ >= e_ || *p_ != '"') return false;
        ++p_;
        const char* start = p_;
        while (p_ < e_ && *p_ != '"' && *p_ != '\\' && static_cast<unsigned char>(*p_) >= 0x20 &&
               static_cast<unsigned char>(*p_) < 0x80)
            ++p_;
        out.assign(start, p_);
        while (p_ < e_ && *p_ != '"') {
            const unsigned char c = static_cast<unsigned char>(*p_);
            if (c < 0x20 || c >= 0x80) return false;  // non-ASCII: the full parser validates UTF-8
            if (c != '\\') {
                out.push_back(static_cast<char>(c));
                ++p_;
                continue;
            }
            if (!allow_escapes || ++p_ >= e_) return false;
            switch (*p_++) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                default: return false;  // \uXXXX: left to the full parser
            }
        }
        if (p_ >= e_) return false;
        ++p_;  // closing quote
        return true;
    }

    bool key(std::string_view& out) {
        if (p_ >= e_ || *p_ != '"') return false;
        const char* start = ++p_;
        while (p_ < e_ && *p_ != '"') {
            if (*p_ == '\\' || static_cast<unsigned char>(*p_) < 0x20 || static_cast<unsigned char>(*p_) >= 0x80)
                return false;
            ++p_;
        }
        if (p_ >= e_) return false;
        out = std::string_view(start, static_cast<size_t>(p_ - start));
        ++p_;
        return true;
    }

    bool value(FastJson& v, int depth) {
        if (depth > 16) return false;
        ws();
        if (p_ >= e_) return false;
        const char c = *p_;
        if (c == '{') {
            v.t = FastJson::T::obj;
            ++p_;
            ws();
            if (p_ < e_ && *p_ == '}') return ++p_, true;
            for (;;) {
                ws();
                std::string_view k;
                if (!key(k)) return false;
                ws();
                if (p_ >= e_ || *p_ != ':') return false;
                ++p_;
                v.o.emplace_back(k, FastJson{});
                if (!value(v.o.back().second, depth + 1)) return false;
                ws();
                if (p_ < e_ && *p_ == ',') { ++p_; continue; }
                if (p_ < e_ && *p_ == '}') { ++p_; break; }
                return false;
            }
            // duplicate keys: the full parser decides which one wins
            std::vector<std::string_view> keys;
            keys.reserve(v.o.size());
            for (const auto& kv : v.o) keys.push_back(kv.first);
            std::sort(keys.begin(), keys.end());
            return std::adjacent_find(keys.begin(), keys.end()) == keys.end();
        }
        if (c == '[') {
            v.t = FastJson::T::arr;
            ++p_;
            ws();
            if (p_ < e_ && *p_ == ']') return ++p_, true;
            for (;;) {
                v.a.emplace_back();
                if (!value(v.a.back(), depth + 1)) return false;
                ws();
                if (p_ < e_ && *p_ == ',') { ++p_; continue; }
                if (p_ < e_ && *p_ == ']') { ++p_; return true; }
                return false;
            }
        }
        if (c == '"') {
            v.t = FastJson::T::str;
            return string(v.s, true);
        }
        if (c >= '0' && c <= '9') {
            v.t = FastJson::T::uint;
            if (c == '0' && p_ + 1 < e_ && p_[1] >= '0' && p_[1] <= '9') return false;  // leading zero
            uint64_t x = 0;
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') {
                const uint64_t d = static_cast<uint64_t>(*p_ - '0');
                if (x > (UINT64_MAX - d) / 10) return false;  // overflow: the full parser's float
                x = x * 10 + d;
                ++p_;
            }
            if (p_ < e_ && (*p_ == '.' || *p_ == 'e' || *p_ == 'E')) return false;
            v.u = x;
            return true;
        }
        return false;  // negative numbers, floats, true/false/null
    }
};

bool fast_uint(const FastJson* v, uint64_t& out) {
    if (v == nullptr || v->t != FastJson::T::uint) return false;
    out = v->u;
    return true;
}

bool fast_str(const FastJson* v, std::string& out) {
    if (v == nullptr || v->t != FastJson::T::str) return false;
    out = v->s;
    return true;
}

bool hex16(std::string_view t, uint64_t& out) {
    uint64_t v = 0;
    for (char c : t) {
        int d;
        if (c >= '0' && c <= '9') d = c - '0';
        else if (c >= 'a' && c <= 'f') d = c - 'a' + 10;
        else if (c >= 'A' && c <= 'F') d = c - 'A' + 10;
        else return false;
        v = (v << 4) | static_cast<uint64_t>(d);
    }
    out = v;
    return true;
}

std::optional<Manifest> parse_manifest_fast(std::string_view text) {
    FastJson root;
    if (!FastReader(text).document(root) || root.t != FastJson::T::obj) return std::nullopt;
    Manifest m;
    uint64_t u = 0;
    if (!fast_uint(root.at("format_version"), u)) return std::nullopt;
    m.format_version = static_cast<uint32_t>(u);
    if (m.format_version != Manifest::kFormatVersion) return std::nullopt;
    if (!fast_uint(root.at("hash_algorithm"), u)) return std::nullopt;
    m.hash_algorithm = static_cast<uint8_t>(u);
    if (m.hash_algorithm != kContentHashAlgorithm) return std::nullopt;
    if (!fast_uint(root.at("workload_digest"), m.workload_digest)) return std::nullopt;
    if (!fast_str(root.at("workload"), m.workload_text)) return std::nullopt;
    const FastJson* a = root.at("allocator");
    if (a == nullptr || !fast_uint(a->at("base"), m.allocator.base) ||
        !fast_uint(a->at("capacity"), m.allocator.capacity) ||
        !fast_uint(a->at("granularity"), m.allocator.granularity) ||
        !fast_uint(a->at("final_offset"), m.final_offset))
        return std::nullopt;
    if (!fast_uint(root.at("kv_cache_bytes"), m.kv_cache_bytes)) return std::nullopt;
    const FastJson* comm = root.at("comm");
    if (comm == nullptr || !fast_uint(comm->at("world_placeholder"), m.comm_world_placeholder) ||
        !fast_uint(comm->at("real_binary_hash"), m.comm_real_hash))
        return std::nullopt;
    const FastJson* gr = root.at("grouping");
    if (gr == nullptr || !fast_uint(gr->at("total"), u)) return std::nullopt;
    m.grouping.total_graphs = static_cast<uint32_t>(u);
    if (!fast_uint(gr->at("templates"), u)) return std::nullopt;
    m.grouping.template_count = static_cast<uint32_t>(u);
    const FastJson* groups = gr->at("groups");
    if (groups == nullptr || groups->t != FastJson::T::arr) return std::nullopt;
    for (const FastJson& gj : groups->a) {
        TemplateGroup g;
        std::string key;
        if (!fast_str(gj.at("key"), key) || key.size() != 32 || !hex16(std::string_view(key).substr(0, 16), g.key.digest.hi) ||
            !hex16(std::string_view(key).substr(16), g.key.digest.lo))
            return std::nullopt;
        if (!fast_uint(gj.at("representative"), u)) return std::nullopt;
        g.representative = static_cast<uint32_t>(u);
        const FastJson* members = gj.at("members");
        if (members == nullptr || members->t != FastJson::T::arr) return std::nullopt;
        g.members.reserve(members->a.size());
        for (const FastJson& x : members->a) {
            if (x.t != FastJson::T::uint) return std::nullopt;
            g.members.push_back(static_cast<uint32_t>(x.u));
        }
        const FastJson* locs = gj.at("locators");
        if (locs == nullptr || locs->t != FastJson::T::arr) return std::nullopt;
        g.locators.reserve(locs->a.size());
        for (const FastJson& lj : locs->a) {
            // nlohmann's at(i) reads the first four entries of a longer array too
            if (lj.t != FastJson::T::arr || lj.a.size() < 4) return std::nullopt;
            for (int i = 0; i < 4; ++i)
                if (lj.a[i].t != FastJson::T::uint) return std::nullopt;
            g.locators.push_back({static_cast<uint32_t>(lj.a[0].u), lj.a[1].u, lj.a[2].u, lj.a[3].u});
        }
        m.grouping.groups.push_back(std::move(g));
    }
    if (!fast_str(root.at("memlayout"), m.memlayout_ref) || !fast_str(root.at("catalog"), m.catalog_ref) ||
        !fast_str(root.at("patch_table"), m.patch_table_ref))
        return std::nullopt;
    const FastJson* files = root.at("files");
    if (files == nullptr || files->t != FastJson::T::obj) return std::nullopt;
    for (const auto& [k, v] : files->o) {
        if (v.t != FastJson::T::uint) return std::nullopt;
        m.file_digests.emplace(std::string(k), v.u);
    }
    return m;
}

}  // namespace

namespace {
Manifest parse_manifest_json(const std::string& text);
}

Manifest parse_manifest(const std::string& text) {
    if (auto fast = parse_manifest_fast(text)) return std::move(*fast);
    return parse_manifest_json(text);
}

int manifest_fast_path_agrees(const std::string& text) {
    const auto fast = parse_manifest_fast(text);
    if (!fast) return -1;
    return *fast == parse_manifest_json(text) ? 1 : 0;
}

namespace {
Manifest parse_manifest_json(const std::string& text) {
    json root;
    try {
        root = json::parse(text);
    } catch (const json::exception& e) {
        raise(Errc::archive_corruption, std::string("manifest is not valid JSON: ") + e.what());
    }
    try {
        Manifest m;
        m.format_version = root.at("format_version").get<uint32_t>();
        require(m.format_version == Manifest::kFormatVersion, Errc::archive_corruption,
                "unsupported archive format version " + std::to_string(m.format_version));
        m.hash_algorithm = root.at("hash_algorithm").get<uint8_t>();
        require(m.hash_algorithm == kContentHashAlgorithm, Errc::archive_corruption,
                "archive pins hash algorithm " + std::to_string(m.hash_algorithm) +
                    ", this build implements " + std::to_string(kContentHashAlgorithm));
        m.workload_digest = root.at("workload_digest").get<uint64_t>();
        m.workload_text = root.at("workload").get<std::string>();
        const json& a = root.at("allocator");
        m.allocator.base = a.at("base").get<uint64_t>();
        m.allocator.capacity = a.at("capacity").get<uint64_t>();
        m.allocator.granularity = a.at("granularity").get<uint64_t>();
        m.final_offset = a.at("final_offset").get<uint64_t>();
        m.kv_cache_bytes = root.at("kv_cache_bytes").get<uint64_t>();
        m.comm_world_placeholder = root.at("comm").at("world_placeholder").get<uint64_t>();
        m.comm_real_hash = root.at("comm").at("real_binary_hash").get<uint64_t>();
        const json& gr = root.at("grouping");
        m.grouping.total_graphs = gr.at("total").get<uint32_t>();
        m.grouping.template_count = gr.at("templates").get<uint32_t>();
        for (const json& gj : gr.at("groups")) {
            TemplateGroup g;
            const std::string key = gj.at("key").get<std::string>();
            require(key.size() == 32, Errc::archive_corruption, "bad topology key literal");
            g.key.digest.hi = parse_hex(key.substr(0, 16));
            g.key.digest.lo = parse_hex(key.substr(16));
            g.representative = gj.at("representative").get<uint32_t>();
            g.members = gj.at("members").get<std::vector<uint32_t>>();
            for (const json& lj : gj.at("locators")) {
                GraphLocator l;
                l.label = lj.at(0).get<uint32_t>();
                l.offset = lj.at(1).get<uint64_t>();
                l.length = lj.at(2).get<uint64_t>();
                l.checksum = lj.at(3).get<uint64_t>();
                g.locators.push_back(l);
            }
            m.grouping.groups.push_back(std::move(g));
        }
        m.memlayout_ref = root.at("memlayout").get<std::string>();
        m.catalog_ref = root.at("catalog").get<std::string>();
        m.patch_table_ref = root.at("patch_table").get<std::string>();
        m.file_digests = root.at("files").get<std::map<std::string, uint64_t>>();
        return m;
    } catch (const json::exception& e) {
        raise(Errc::archive_corruption, std::string("manifest field error: ") + e.what());
    }
}
}  // namespace

// ------------------------------------------------------------ FNDB

namespace {
constexpr uint8_t kImgRelocatable = 0x01;
constexpr uint8_t kImgDeviceInit = 0x02;

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
}  // namespace

std::vector<uint8_t> encode_kernel_image(const KernelImage& img) {
    Sink s;
    s.raw("FNDB", 4);
    s.u16(1);
    s.u8((img.relocatable ? kImgRelocatable : 0) | (img.requires_device_init ? kImgDeviceInit : 0));
    s.u32(img.link_tag);
    s.u32(static_cast<uint32_t>(img.entrypoints.size()));
    for (const auto& e : img.entrypoints) {
        s.str(e.name);
        s.u32(e.arg_buffer_size);
        s.u32(static_cast<uint32_t>(e.hidden_offsets.size()));
        for (uint32_t o : e.hidden_offsets) s.u32(o);
        put_fattrs(s, e.attrs);
    }
    s.u32(static_cast<uint32_t>(img.aux.size()));
    s.raw(img.aux);
    return s.release();
}

KernelImage parse_kernel_image(std::span<const uint8_t> payload) {
    Cursor c(payload, Errc::binary_format);
    c.magic("FNDB");
    const uint16_t version = c.u16();
    require(version == 1, Errc::binary_format, "unsupported image version " + std::to_string(version));
    KernelImage img;
    const uint8_t flags = c.u8();
    img.relocatable = flags & kImgRelocatable;
    img.requires_device_init = flags & kImgDeviceInit;
    img.link_tag = c.u32();
    const uint32_t n = c.u32();
    std::unordered_set<std::string> seen;
    for (uint32_t i = 0; i < n; ++i) {
        KernelEntry e;
        e.name = c.str();
        require(!e.name.empty(), Errc::binary_format, "empty entrypoint name");
        require(seen.insert(e.name).second, Errc::binary_format,
                "duplicate entrypoint '" + e.name + "'");
        e.arg_buffer_size = c.u32();
        const uint32_t k = c.u32();
        for (uint32_t j = 0; j < k; ++j) {
            const uint32_t off = c.u32();
            require(uint64_t(off) + 8 <= e.arg_buffer_size, Errc::binary_format,
                    "hidden offset " + std::to_string(off) + " out of range in '" + e.name + "'");
            e.hidden_offsets.push_back(off);
        }
        e.attrs = get_fattrs(c);
        img.entrypoints.push_back(std::move(e));
    }
    const uint32_t aux = c.u32();
    const uint8_t* p = c.take(aux);
    img.aux.assign(p, p + aux);
    require(c.at_end(), Errc::binary_format, "trailing bytes after image");
    return img;
}

std::vector<uint8_t> link_segments(const std::vector<std::vector<uint8_t>>& segments) {
    require(!segments.empty(), Errc::invalid_argument, "no segments to link");
    KernelImage out;
    std::unordered_set<std::string> names;
    for (size_t i = 0; i < segments.size(); ++i) {
        KernelImage seg = parse_kernel_image(segments[i]);
        if (i == 0) {
            out.link_tag = seg.link_tag;
            out.requires_device_init = seg.requires_device_init;
        } else {
            require(seg.link_tag == out.link_tag, Errc::binary_format,
                    "link tag mismatch across segments");
            out.requires_device_init = out.requires_device_init || seg.requires_device_init;
        }
        for (auto& e : seg.entrypoints) {
            require(names.insert(e.name).second, Errc::binary_format,
                    "conflicting entrypoint '" + e.name + "' across segments");
            out.entrypoints.push_back(std::move(e));
        }
    }
    out.relocatable = false;
    return encode_kernel_image(out);
}

// ------------------------------------------------------------ catalog

namespace {
constexpr uint8_t kCatInit = 0x01, kCatStub = 0x02, kCatReal = 0x04;
}

std::vector<uint8_t> serialize_catalog(const Catalog& cat) {
    Sink s;
    s.raw("FNDC", 4);
    s.u16(1);
    s.u8(kContentHashAlgorithm);
    s.u32(static_cast<uint32_t>(cat.binaries.size()));
    for (const auto& [hash, r] : cat.binaries) {
        s.u64(hash);
        s.u8(static_cast<uint8_t>(r.variant));
        s.u8((r.needs_device_init ? kCatInit : 0) | (r.is_stub ? kCatStub : 0) |
             (r.is_comm_real ? kCatReal : 0));
        s.u32(static_cast<uint32_t>(r.load_options.size()));
        s.raw(r.load_options);
        s.u32(static_cast<uint32_t>(r.entrypoints.size()));
        for (size_t i = 0; i < r.entrypoints.size(); ++i) {
            s.str(r.entrypoints[i]);
            put_fattrs(s, r.entrypoint_attrs[i]);
        }
    }
    return s.release();
}

Catalog parse_catalog(std::span<const uint8_t> bytes) {
    Cursor c(bytes, Errc::archive_corruption);
    c.magic("FNDC");
    const uint16_t version = c.u16();
    require(version == 1, Errc::archive_corruption,
            "unsupported catalog version " + std::to_string(version));
    const uint8_t algo = c.u8();
    require(algo == kContentHashAlgorithm, Errc::archive_corruption,
            "archive uses hash algorithm " + std::to_string(algo) + ", this build implements " +
                std::to_string(kContentHashAlgorithm));
    Catalog cat;
    const uint32_t n = c.u32();
    for (uint32_t i = 0; i < n; ++i) {
        KernelBinaryRecord r;
        r.hash = c.u64();
        r.variant = static_cast<LoadVariant>(c.u8());
        const uint8_t f = c.u8();
        r.needs_device_init = f & kCatInit;
        r.is_stub = f & kCatStub;
        r.is_comm_real = f & kCatReal;
        const uint32_t no = c.u32();
        const uint8_t* p = c.take(no);
        r.load_options.assign(p, p + no);
        const uint32_t ne = c.u32();
        for (uint32_t j = 0; j < ne; ++j) {
            r.entrypoints.push_back(c.str());
            r.entrypoint_attrs.push_back(get_fattrs(c));
        }
        const uint64_t h = r.hash;
        cat.binaries.emplace(h, std::move(r));
    }
    require(c.at_end(), Errc::archive_corruption, "trailing bytes in catalog");
    return cat;
}

// ------------------------------------------------------------ patch table

size_t PatchTable::total_entries() const {
    size_t n = 0;
    for (const auto& [label, entries] : per_graph) n += entries.size();
    return n;
}

std::vector<uint8_t> serialize_patch_table(const PatchTable& t) {
    Sink s;
    s.raw("FNDP", 4);
    s.u16(1);
    s.u64(t.world_placeholder);
    s.u32(static_cast<uint32_t>(t.per_graph.size()));
    for (const auto& [label, entries] : t.per_graph) {
        s.u32(label);
        s.u32(static_cast<uint32_t>(entries.size()));
        for (const auto& e : entries) {
            s.u32(e.node_id);
            s.u64(e.stub.binary_hash);
            s.str(e.stub.name);
            s.str(e.real_name);
            s.u32(static_cast<uint32_t>(e.rank_offsets.size()));
            for (uint32_t o : e.rank_offsets) s.u32(o);
            s.u32(static_cast<uint32_t>(e.world_offsets.size()));
            for (uint32_t o : e.world_offsets) s.u32(o);
            s.u8(e.patch_width);
        }
    }
    return s.release();
}

PatchTable parse_patch_table(std::span<const uint8_t> bytes) {
    Cursor c(bytes, Errc::archive_corruption);
    c.magic("FNDP");
    const uint16_t version = c.u16();
    require(version == 1, Errc::archive_corruption,
            "unsupported patch table version " + std::to_string(version));
    PatchTable t;
    t.world_placeholder = c.u64();
    const uint32_t ng = c.u32();
    for (uint32_t g = 0; g < ng; ++g) {
        const uint32_t label = c.u32();
        const uint32_t n = c.u32();
        std::vector<CommPatchEntry> entries;
        for (uint32_t i = 0; i < n; ++i) {
            CommPatchEntry e;
            e.node_id = c.u32();
            e.stub.binary_hash = c.u64();
            e.stub.name = c.str();
            e.real_name = c.str();
            const uint32_t nr = c.u32();
            for (uint32_t j = 0; j < nr; ++j) e.rank_offsets.push_back(c.u32());
            const uint32_t nw = c.u32();
            for (uint32_t j = 0; j < nw; ++j) e.world_offsets.push_back(c.u32());
            e.patch_width = c.u8();
            entries.push_back(std::move(e));
        }
        t.per_graph.emplace(label, std::move(entries));
    }
    require(c.at_end(), Errc::archive_corruption, "trailing bytes in patch table");
    return t;
}

uint32_t PatchEntryView::rank_offset(uint32_t i) const {
    uint32_t v;
    std::memcpy(&v, rank_offsets + 4ull * i, 4);
    return v;
}
uint32_t PatchEntryView::world_offset(uint32_t i) const {
    uint32_t v;
    std::memcpy(&v, world_offsets + 4ull * i, 4);
    return v;
}

namespace {

// The reference-order parse (one pass, Cursor bounds checks): the exact error
// for a malformed table, and the parse itself for a small one.
PatchView parse_patch_view_sequential(std::span<const uint8_t> bytes) {
    Cursor c(bytes, Errc::archive_corruption);
    c.magic("FNDP");
    const uint16_t version = c.u16();
    require(version == 1, Errc::archive_corruption,
            "unsupported patch table version " + std::to_string(version));
    PatchView t;
    t.world_placeholder = c.u64();
    const uint32_t ng = c.u32();
    t.graphs.reserve(std::min<size_t>(ng, bytes.size() / 8));
    t.entries.reserve(bytes.size() / 29);  // an entry is at least 29 bytes: no regrowth
    for (uint32_t g = 0; g < ng; ++g) {
        const uint32_t label = c.u32();
        const uint32_t n = c.u32();
        const uint32_t first = static_cast<uint32_t>(t.entries.size());
        for (uint32_t i = 0; i < n; ++i) {
            PatchEntryView e;
            e.node_id = c.u32();
            e.stub_hash = c.u64();
            e.stub_name = c.str_view();
            e.real_name = c.str_view();
            e.n_rank = c.u32();
            e.rank_offsets = c.take(4ull * e.n_rank);
            e.n_world = c.u32();
            e.world_offsets = c.take(4ull * e.n_world);
            e.patch_width = c.u8();
            t.entries.push_back(e);
        }
        t.graphs.push_back({label, first, n});
    }
    require(c.at_end(), Errc::archive_corruption, "trailing bytes in patch table");
    return t;
}

uint32_t rd32le(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}

// Pooled storage for large PatchViews' entries (raw bytes; PatchEntryView is
// trivially destructible, so a block is returned without running destructors).
std::mutex g_entry_pool_mu;
std::vector<std::pair<void*, size_t>> g_entry_pool;

static_assert(std::is_trivially_destructible_v<PatchEntryView>, "pooled entries are released without destructors");

std::shared_ptr<PatchEntryView> pooled_entries(size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(PatchEntryView);
    void* p = nullptr;
    size_t cap = 0;
    {
        std::lock_guard lock(g_entry_pool_mu);
        for (size_t i = 0; i < g_entry_pool.size(); ++i)
            if (g_entry_pool[i].second >= bytes && (!p || g_entry_pool[i].second < cap)) {
                p = g_entry_pool[i].first;
                cap = g_entry_pool[i].second;
            }
        if (p)
            g_entry_pool.erase(std::find(g_entry_pool.begin(), g_entry_pool.end(), std::make_pair(p, cap)));
    }
    if (!p) {
        cap = bytes;
        p = ::operator new(cap);
    }
    return std::shared_ptr<PatchEntryView>(static_cast<PatchEntryView*>(p), [cap](PatchEntryView* q) {
        std::lock_guard lock(g_entry_pool_mu);
        g_entry_pool.push_back({q, cap});
        if (g_entry_pool.size() > 2) {  // keep the two largest
            std::sort(g_entry_pool.begin(), g_entry_pool.end(),
                      [](const auto& a, const auto& b) { return a.second > b.second; });
            ::operator delete(g_entry_pool.back().first);
            g_entry_pool.pop_back();
        }
    });
}

}  // namespace

// Large tables (10 MB, 144K entries on the headline set) parse in two passes: a
// sequential walk over the entry sizes finds every graph's byte range, then the
// graphs are decoded on the worker pool into a pre-sized entry array. Anything
// the walk cannot account for falls back to the sequential parse, so a
// malformed table raises exactly the reference-order error.
PatchView parse_patch_view(std::span<const uint8_t> bytes) {
    PatchView t;
    const uint8_t* p = bytes.data();
    const uint64_t n = bytes.size();
    if (n < (256u << 10) || std::memcmp(p, "FNDP", 4) != 0 || p[4] != 1 || p[5] != 0) {
        t = parse_patch_view_sequential(bytes);
    } else {
        std::memcpy(&t.world_placeholder, p + 6, 8);
        const uint32_t ng = rd32le(p + 14);
        struct Span {
            uint64_t at;
            uint32_t label, count, first;
        };
        std::vector<Span> spans;
        spans.reserve(std::min<uint64_t>(ng, n / 8));
        uint64_t at = 18, total = 0;
        bool ok = true;
        auto fits = [&](uint64_t k) { return k <= n - at; };
        for (uint32_t g = 0; g < ng && ok; ++g) {
            if (!fits(8)) { ok = false; break; }
            Span sp{at + 8, rd32le(p + at), rd32le(p + at + 4), static_cast<uint32_t>(total)};
            at += 8;
            for (uint32_t i = 0; i < sp.count; ++i) {
                // node_id u32, stub_hash u64, two names (u32 + bytes), two u32 lists, u8
                if (!fits(16)) { ok = false; break; }
                at += 12;
                uint64_t k = rd32le(p + at);
                at += 4;
                if (!fits(k) || !fits(k + 4)) { ok = false; break; }
                at += k;
                k = rd32le(p + at);
                at += 4;
                if (!fits(k) || !fits(k + 4)) { ok = false; break; }
                at += k;
                k = 4ull * rd32le(p + at);
                at += 4;
                if (!fits(k) || !fits(k + 4)) { ok = false; break; }
                at += k;
                k = 4ull * rd32le(p + at);
                at += 4;
                if (!fits(k) || !fits(k + 1)) { ok = false; break; }
                at += k + 1;
            }
            total += sp.count;
            spans.push_back(sp);
        }
        if (!ok || at != n || total >= (1ull << 32)) {
            t = parse_patch_view_sequential(bytes);  // raises the reference's error
        } else {
            t.pooled = pooled_entries(total);
            PatchEntryView* const out = t.pooled.get();
            parallel_for(spans.size(), spans.size() >= 64 ? 0u : 1u, [&](size_t g) {
                const Span& sp = spans[g];
                Cursor c(p + sp.at, n - sp.at, Errc::archive_corruption);
                for (uint32_t i = 0; i < sp.count; ++i) {
                    PatchEntryView& e = *new (out + sp.first + i) PatchEntryView;
                    e.node_id = c.u32();
                    e.stub_hash = c.u64();
                    e.stub_name = c.str_view();
                    e.real_name = c.str_view();
                    e.n_rank = c.u32();
                    e.rank_offsets = c.take(4ull * e.n_rank);
                    e.n_world = c.u32();
                    e.world_offsets = c.take(4ull * e.n_world);
                    e.patch_width = c.u8();
                }
            });
            t.graphs.reserve(spans.size());
            for (const Span& sp : spans) t.graphs.push_back({sp.label, sp.first, sp.count});
        }
    }
    std::stable_sort(t.graphs.begin(), t.graphs.end(),
                     [](const auto& a, const auto& b) { return a[0] < b[0]; });
    t.graphs.erase(std::unique(t.graphs.begin(), t.graphs.end(),
                               [](const auto& a, const auto& b) { return a[0] == b[0]; }),
                   t.graphs.end());
    return t;
}

std::span<const PatchEntryView> PatchView::find(uint32_t label) const {
    auto it = std::lower_bound(graphs.begin(), graphs.end(), label,
                               [](const std::array<uint32_t, 3>& g, uint32_t l) { return g[0] < l; });
    if (it == graphs.end() || (*it)[0] != label) return {};
    return {entry_data() + (*it)[1], (*it)[2]};
}

bool PatchView::has(uint32_t label) const {
    auto it = std::lower_bound(graphs.begin(), graphs.end(), label,
                               [](const std::array<uint32_t, 3>& g, uint32_t l) { return g[0] < l; });
    return it != graphs.end() && (*it)[0] == label;
}

void apply_rank_patches(CapturedGraph& graph, std::span<const CommPatchEntry> entries,
                        uint64_t real_comm_hash, uint32_t rank, uint32_t world) {
    auto put = [](std::vector<uint8_t>& buf, uint32_t off, uint64_t v) {
        require(uint64_t(off) + 8 <= buf.size(), Errc::invalid_argument,
                "patch offset outside the argument buffer");
        std::memcpy(buf.data() + off, &v, 8);
    };
    for (const auto& e : entries) {
        require(e.node_id < graph.nodes.size(), Errc::archive_corruption,
                "patch entry references missing node");
        GraphNode& n = graph.nodes[e.node_id];
        require(n.type == NodeType::Kernel, Errc::archive_corruption,
                "patch entry references a non-kernel node");
        auto& k = n.kernel_params();
        require(k.kernel == e.stub, Errc::archive_corruption,
                "node " + std::to_string(e.node_id) + " is not the recorded stub " +
                    e.stub.describe());
        k.kernel = KernelRef{real_comm_hash, e.real_name};
        for (uint32_t o : e.rank_offsets) put(k.arg_buffer, o, rank);
        for (uint32_t o : e.world_offsets) put(k.arg_buffer, o, world);
    }
}

// ------------------------------------------------------------------ comm slots

std::vector<uint8_t> serialize_comm_slots(const CommSlotTable& t) {
    Sink s;
    s.raw("FNDS", 4);
    s.u16(1);
    s.u32(t.n_values);
    s.u32(static_cast<uint32_t>(t.per_graph.size()));
    for (const auto& [label, slots] : t.per_graph) {
        s.u32(label);
        s.u32(static_cast<uint32_t>(slots.size()));
        for (const CommSlot& c : slots) {
            s.u32(c.node_id);
            s.u32(c.offset);
            s.u32(c.value_index);
            s.u8(c.width);
        }
    }
    return s.release();
}

CommSlotTable parse_comm_slots(std::span<const uint8_t> bytes) {
    Cursor c(bytes, Errc::archive_corruption);
    c.magic("FNDS");
    const uint16_t version = c.u16();
    require(version == 1, Errc::archive_corruption, "unsupported comm slot table version " + std::to_string(version));
    CommSlotTable t;
    t.n_values = c.u32();
    const uint32_t graphs = c.u32();
    for (uint32_t g = 0; g < graphs; ++g) {
        const uint32_t label = c.u32();
        const uint32_t count = c.u32();
        std::vector<CommSlot> slots;
        for (uint32_t i = 0; i < count; ++i) {  // one at a time: a short table is a cursor overrun
            CommSlot s;
            s.node_id = c.u32();
            s.offset = c.u32();
            s.value_index = c.u32();
            s.width = c.u8();
            require(s.width >= 1 && s.width <= 8, Errc::archive_corruption,
                    "comm slot width " + std::to_string(s.width) + " is not 1..8");
            require(s.value_index < t.n_values, Errc::archive_corruption,
                    "comm slot value index " + std::to_string(s.value_index) + " is outside the " +
                        std::to_string(t.n_values) + "-entry value table");
            slots.push_back(s);
        }
        require(t.per_graph.emplace(label, std::move(slots)).second, Errc::archive_corruption,
                "comm slot table lists label " + std::to_string(label) + " twice");
    }
    require(c.at_end(), Errc::archive_corruption, "trailing bytes in comm slot table");
    return t;
}

void apply_comm_slots(CapturedGraph& graph, std::span<const CommSlot> slots,
                      std::span<const CommPatchEntry> patches, std::span<const uint64_t> values) {
    for (const CommSlot& s : slots) {
        bool stub = false;
        for (const auto& e : patches) stub = stub || e.node_id == s.node_id;
        require(stub && s.node_id < graph.nodes.size() && graph.nodes[s.node_id].type == NodeType::Kernel,
                Errc::archive_corruption,
                "comm slot references node " + std::to_string(s.node_id) + ", which is not a patched comm node");
        auto& args = graph.nodes[s.node_id].kernel_params().arg_buffer;
        require(uint64_t(s.offset) + s.width <= args.size(), Errc::invalid_argument,
                "comm slot offset outside the argument buffer");
        require(s.value_index < values.size(), Errc::invalid_argument,
                "comm slot value index " + std::to_string(s.value_index) + " has no value");
        const uint64_t v = values[s.value_index];
        std::memcpy(args.data() + s.offset, &v, s.width);
    }
}

}  // namespace foundry
