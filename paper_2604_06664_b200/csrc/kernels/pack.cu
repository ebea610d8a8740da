// GPU packer for sm_100a: a reference-written archive (graphs.bin + patch.bin,
// no templates.fdt) becomes the FNDT template store on the device, so the
// drop-in LOAD of such an archive does no per-member work on the CPU.
//
// It replaces, per member, the reference's prepare step parse_graph_at ->
// decode_graph_record -> decode_node (graph_model.cpp:146-240,295-303) and the
// template diff (differing_ranges / diff, graph_model.cpp:578-629), and it
// produces byte for byte what the offline packer (host/template_store.cpp)
// writes. The host only lays out what is per group or per kernel (slot
// capacities -> offsets, the kernel table order, rank ops from patch.bin).
//
// Record layout (graph_model.cpp:205-218): u32 label, u32 nodes, u32 edges,
// nodes, edges (u32 from, u32 to). Kernel node: type u8 @0, cluster 3 x u32
// @1, policy / sync_default / sync_remote i32 @13, attr_query u8 @25, grid
// @26, block @38, shmem @50, binary hash u64 @54, name u32 @62 + bytes @66,
// func attrs 6 x i32 @66+nl, arg size u32 @90+nl, args @94+nl. Memcpy /
// memset: type + 3 x u64 (25 bytes). Empty: 1 byte. Nothing is aligned.
//
// Pass 1
//   walk     one thread per record hops node to node (a node's length is only
//            known from its own name and argument sizes) through a ring of
//            8 KiB shared-memory windows that TMA bulk copies keep filled
//            ahead of it; emits node offsets, checks tags, bounds and the
//            edge-table size.
//   fields   one thread per node: launch-dim / argument validation, topology
//            against the representative's node, slot capacity (atomicMax per
//            group node), kernel key (binary hash, func attrs, name) into an
//            open-addressing table keyed by a 64-bit fingerprint with the
//            first position (atomicMin) as the key's order.
//   edges    one CTA per record: canonical order, bounds, equality with the
//            representative's edges.
//   entries  one thread per patch entry: apply_rank_patches' checks (stub
//            node, offsets inside its arguments), then the real comm kernel's
//            key into the table at the entry's position.
//   verify   one thread per kernel node / entry: its key bytes equal the first
//            occurrence's (a fingerprint collision is reported, never merged).
//   compact  warp-ballot / popc compaction of the occupied table slots.
// Pass 2
//   images   one warp per node writes the node descriptor and its 16-byte
//            slot chunks into the member's image, plus per-chunk relocation
//            meta (the offline packer's build_image).
//   swaps    stub -> real comm kernel index (apply_rank_patches' kernel swap).
//   count    one CTA per member tile: lanes that differ from the template
//            (bytes or relocation flag), warp ballot + popc, block sum.
// Pass 3
//   diffs    the same ballots; a warp scan of the per-warp counts gives each
//            differing lane its slot after the tile's first entry, so the
//            compacted (lane | reloc, value) streams land in lane order.
#include <cstdint>

#include "fdy_kernels.h"

namespace {

constexpr uint32_t kWalkWin = 8192;                  // walk: TMA window
constexpr uint32_t kWalkWins = 4;                    //       windows in the ring
constexpr uint32_t kWalkRing = kWalkWin * kWalkWins; //       (a power of two)
constexpr uint32_t kThreads = 256;
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t ld32(const unsigned char* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}
__device__ __forceinline__ uint64_t ld64(const unsigned char* p) {
    return uint64_t(ld32(p)) | uint64_t(ld32(p + 4)) << 32;
}

__device__ __forceinline__ uint64_t u64min(uint64_t x, uint64_t y) { return x < y ? x : y; }

__device__ __forceinline__ uint64_t mix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h;
}

// Kernel key (binary hash, func attrs, name): the offline packer's
// KernelTable key, for a kernel node or a patch entry's real comm kernel.
__device__ uint64_t key_fingerprint(uint64_t hash, const unsigned char* fa, const unsigned char* name, uint32_t nl,
                                    uint64_t seed) {
    uint64_t h = mix64(seed ^ (uint64_t(nl) << 1));
    h = mix64(h ^ hash);
    h = mix64(h ^ ld64(fa));
    h = mix64(h ^ ld64(fa + 8));
    h = mix64(h ^ ld64(fa + 16));
    uint32_t i = 0;
    for (; i + 8 <= nl; i += 8) h = mix64(h ^ ld64(name + i));
    uint64_t tail = 0;
    for (uint32_t k = 0; i + k < nl; ++k) tail |= uint64_t(name[i + k]) << (8 * k);
    h = mix64(h ^ tail ^ 0x9E3779B97F4A7C15ull);
    return h ? h : 1;
}

struct KeyParts {
    uint64_t hash;
    const unsigned char* fa;
    const unsigned char* name;
    uint32_t nl;
};

__device__ __forceinline__ KeyParts node_key(const unsigned char* q) {
    const uint32_t nl = ld32(q + 62);
    return {ld64(q + 54), q + 66 + nl, q + 66, nl};
}

__device__ __forceinline__ const unsigned char* node_at(const FdyPackArgs& a, uint32_t m, uint32_t n) {
    return a.graphs + a.rec_off[m] + a.node_off[a.node_base[m] + n];
}

__device__ __forceinline__ const unsigned char* gnode_at(const FdyPackArgs& a, uint32_t gn) {
    return a.graphs + a.rec_off[a.node_member[gn]] + a.node_off[gn];
}

// Patch entry e's real comm kernel key: (comm_real_hash, the stub node's func
// attrs, real name).
__device__ __forceinline__ KeyParts entry_key(const FdyPackArgs& a, uint32_t e) {
    const unsigned char* q = gnode_at(a, a.pe_node[e]);
    const uint32_t r = a.pe_real_name[e];
    return {a.comm_real_hash, q + 66 + ld32(q + 62), a.names + a.name_off[r], a.name_len[r]};
}

// The key at a table position: a node (local < its member's node count) or
// the member's patch entry local - nodes.
__device__ __forceinline__ KeyParts key_at(const FdyPackArgs& a, unsigned long long pos) {
    const uint32_t m = uint32_t(pos >> 32), local = uint32_t(pos);
    if (local < a.n_nodes[m]) return node_key(node_at(a, m, local));
    return entry_key(a, a.entry_base[m] + (local - a.n_nodes[m]));
}

__device__ __forceinline__ bool same_key(const KeyParts& x, const KeyParts& y) {
    if (x.hash != y.hash || x.nl != y.nl) return false;
    for (uint32_t i = 0; i < 24; ++i)
        if (x.fa[i] != y.fa[i]) return false;
    for (uint32_t i = 0; i < x.nl; ++i)
        if (x.name[i] != y.name[i]) return false;
    return true;
}

__device__ __forceinline__ uint32_t table_insert(const FdyPackArgs& a, uint64_t fp, unsigned long long pos) {
    uint32_t s = uint32_t(fp >> 20) & a.tmask;
    for (;;) {
        const unsigned long long old = atomicCAS(&a.tkey[s], 0ull, fp);
        if (old == 0ull || old == fp) {
            atomicMin(&a.tpos[s], pos);
            return s;
        }
        s = (s + 1) & a.tmask;
    }
}

// ------------------------------------------------------------------- pass 1

__device__ __forceinline__ uint32_t smem_u32addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One thread per record walks it node to node. The record streams through a
// ring of kWalkWins 8 KiB windows in shared memory, filled by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx) issued as far ahead as the ring
// allows, so the walk's reads (type byte, name length, argument size: the
// only fields a node's length depends on) hit shared memory and the next
// windows are already in flight. Window k of the record holds bytes
// [w0 + k * kWalkWin, ...) at ring offset (k mod kWalkWins) * kWalkWin.
__global__ void __launch_bounds__(32) pack_walk_kernel(const FdyPackArgs a) {
    __shared__ __align__(128) unsigned char ring[kWalkRing];
    __shared__ __align__(8) unsigned long long bar[kWalkWins];
    if (threadIdx.x != 0) return;
    const uint32_t m = blockIdx.x;
    const uint64_t rb = a.rec_off[m], rl = a.rec_len[m];
    const uint32_t N = a.n_nodes[m], E = a.n_edges[m], nb = a.node_base[m];
    if (rl < 12) {
        atomicOr(&a.status[m], FDY_PACK_DECODE);
        return;
    }
    const uint64_t w0 = rb & ~15ull;                 // windows start 16-byte aligned
    const uint64_t span = rb + rl - w0;              // bytes of the record's windows
    const uint32_t n_wins = uint32_t((span + kWalkWin - 1) / kWalkWin);
    for (uint32_t i = 0; i < kWalkWins; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32addr(&bar[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t issued = 0, waited = 0;  // windows [0, issued) requested, [0, waited) landed
    auto issue = [&](uint32_t k) {
        const uint32_t slot = k % kWalkWins;
        const uint64_t off = uint64_t(k) * kWalkWin;
        // whole 16-byte units; the staged buffer is padded past every file
        const uint32_t bytes = uint32_t((u64min(kWalkWin, span - off) + 15) & ~15ull);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32addr(&bar[slot])),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32addr(ring + slot * kWalkWin)),
            "l"(a.graphs + w0 + off), "r"(bytes), "r"(smem_u32addr(&bar[slot]))
            : "memory");
    };
    auto wait = [&](uint32_t k) {
        const uint32_t slot = k % kWalkWins, parity = (k / kWalkWins) & 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WALK_WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WALK_WAIT_%=;\n}" ::"r"(smem_u32addr(&bar[slot])),
            "r"(parity)
            : "memory");
    };
    // bytes [x, x + n) of the record (record-relative) are in shared memory
    // once this returns; the ring is refilled ahead of x as far as it reaches
    uint64_t ready = 0;  // window-relative bytes [0, ready) have landed (the walk only moves forward,
                         // and no window at or after the walker's is refilled before it moves on)
    auto ensure = [&](uint64_t x, uint32_t n) {
        const uint64_t ax = rb + x - w0;
        if (ax + n <= ready) return;  // the common case: inside the windows already waited for
        const uint32_t lo = uint32_t(ax / kWalkWin), hi = uint32_t((ax + n - 1) / kWalkWin);
        while (issued < n_wins && issued < lo + kWalkWins) {
            if (issued >= kWalkWins && waited <= issued - kWalkWins) {  // its slot's last window
                wait(waited);
                ++waited;
            }
            issue(issued++);
        }
        while (waited <= hi) {
            wait(waited);
            ++waited;
        }
        ready = uint64_t(waited) * kWalkWin;
    };
    auto byte_at = [&](uint64_t x) -> uint32_t { return ring[(rb + x - w0) & (kWalkRing - 1)]; };
    auto u32_at = [&](uint64_t x) {
        return byte_at(x) | byte_at(x + 1) << 8 | byte_at(x + 2) << 16 | byte_at(x + 3) << 24;
    };
    uint64_t p = 12;
    bool bad = false;
    for (uint32_t n = 0; n < N && !bad; ++n) {
        if (p + 1 > rl) { bad = true; break; }
        ensure(p, 1);
        const uint32_t t = byte_at(p);
        uint64_t len;
        if (t == 0) {
            if (p + 66 > rl) { bad = true; break; }
            ensure(p + 62, 4);
            const uint32_t nl = u32_at(p + 62);
            if (p + 94 + uint64_t(nl) > rl) { bad = true; break; }
            ensure(p + 90 + nl, 4);
            len = 94ull + nl + u32_at(p + 90 + nl);
        } else if (t <= 3) {
            len = t == 3 ? 1u : 25u;
        } else {
            bad = true;
            break;
        }
        if (p + len > rl) { bad = true; break; }
        a.node_off[nb + n] = uint32_t(p);
        a.node_member[nb + n] = m;
        p += len;
    }
    // the edge table must end the record exactly
    if (bad || p + 8ull * E != rl) atomicOr(&a.status[m], FDY_PACK_DECODE);
    while (waited < issued) {  // no bulk copy may still target this CTA's shared memory
        wait(waited);
        ++waited;
    }
}

__device__ __forceinline__ bool member_ok(const FdyPackArgs& a, uint32_t m) {
    return m != kNone && (a.status[m] & FDY_PACK_DECODE) == 0;
}

__global__ void __launch_bounds__(kThreads) pack_fields_kernel(const FdyPackArgs a) {
    for (uint32_t gn = blockIdx.x * kThreads + threadIdx.x; gn < a.total_nodes; gn += gridDim.x * kThreads) {
        const uint32_t m = a.node_member[gn];
        if (!member_ok(a, m)) continue;
        const uint32_t n = gn - a.node_base[m];
        const unsigned char* q = a.graphs + a.rec_off[m] + a.node_off[gn];
        const uint32_t g = a.member_group[m], rep = a.group_rep[g];
        const uint8_t t = q[0];
        // topology_key covers the node type and, for kernels, the launch attributes
        const bool rep_ok = member_ok(a, rep) && n < a.n_nodes[rep];
        bool same = rep_ok;
        if (rep_ok && m != rep) {
            const unsigned char* r = node_at(a, rep, n);
            same = r[0] == t;
            if (same && t == 0) {
                for (int i = 1; i < 25; ++i) same &= q[i] == r[i];
                same &= (q[25] != 0) == (r[25] != 0);
            }
        }
        if (!same) atomicOr(&a.status[m], FDY_PACK_TOPO);
        uint32_t blob_len = (t == 1 || t == 2) ? 24u : 0u;
        if (t == 0) {
            const uint32_t nl = ld32(q + 62);
            blob_len = ld32(q + 90 + nl);
            bool valid = blob_len != 0;  // CapturedGraph::validate
            for (int i = 0; i < 6; ++i) valid &= ld32(q + 26 + 4 * i) != 0;
            if (!valid) atomicOr(&a.status[m], FDY_PACK_DECODE);
            const KeyParts k = node_key(q);
            a.node_slot[gn] = table_insert(a, key_fingerprint(k.hash, k.fa, k.name, k.nl, a.seed),
                                           (uint64_t(m) << 32) | n);
        }
        if (!rep_ok) continue;
        const uint32_t gi = a.gnode_base[g] + n;
        atomicMax(&a.cap[gi], (blob_len + 15u) & ~15u);
        if (m == rep) {
            fdt_node_attrs at{};
            at.cluster[0] = at.cluster[1] = at.cluster[2] = 1;  // KernelNodeAttrs defaults
            at.attr_query = 1;
            if (t == 0) {
                at.cluster[0] = ld32(q + 1);
                at.cluster[1] = ld32(q + 5);
                at.cluster[2] = ld32(q + 9);
                at.sched_policy = int32_t(ld32(q + 13));
                at.sync_default = int32_t(ld32(q + 17));
                at.sync_remote = int32_t(ld32(q + 21));
                at.attr_query = q[25] != 0;
            }
            a.rep_attrs[gi] = at;
            a.rep_type[gi] = t;
        }
    }
}

// CapturedGraph::validate's edge rules + topology equality of the edge lists.
__global__ void __launch_bounds__(kThreads) pack_edges_kernel(const FdyPackArgs a) {
    const uint32_t m = blockIdx.x;
    if (a.status[m] & FDY_PACK_DECODE) return;
    const uint32_t N = a.n_nodes[m], E = a.n_edges[m];
    const unsigned char* e = a.graphs + a.rec_off[m] + a.rec_len[m] - 8ull * E;
    const uint32_t rep = a.group_rep[a.member_group[m]];
    const bool rep_ok = (a.status[rep] & FDY_PACK_DECODE) == 0;
    const bool same_shape = rep_ok && a.n_nodes[rep] == N && a.n_edges[rep] == E;
    const unsigned char* re = a.graphs + a.rec_off[rep] + a.rec_len[rep] - 8ull * a.n_edges[rep];
    bool bad = false, differs = !same_shape;
    for (uint32_t i = threadIdx.x; i < E; i += kThreads) {
        const uint32_t from = ld32(e + 8ull * i), to = ld32(e + 8ull * i + 4);
        bad |= from >= N || to >= N || from >= to;
        if (i > 0) {
            const uint32_t pf = ld32(e + 8ull * i - 8), pt = ld32(e + 8ull * i - 4);
            bad |= !(pf < from || (pf == from && pt < to));
        }
        if (same_shape && m != rep) differs |= from != ld32(re + 8ull * i) || to != ld32(re + 8ull * i + 4);
    }
    if (bad) atomicOr(&a.status[m], FDY_PACK_DECODE);
    if (differs && m != rep) atomicOr(&a.status[m], FDY_PACK_TOPO);
    if (!same_shape && m != rep && threadIdx.x == 0) atomicOr(&a.status[m], FDY_PACK_TOPO);
}

// apply_rank_patches' checks (rank_forge.cpp:136-150) per patch entry: the
// node is a kernel node carrying the recorded stub, and its argument buffer
// holds every rank / world offset and comm slot; then the real comm kernel's
// key goes into the table at the entry's position (after its graph's nodes).
__global__ void __launch_bounds__(kThreads) pack_entries_kernel(const FdyPackArgs a) {
    for (uint32_t e = blockIdx.x * kThreads + threadIdx.x; e < a.n_entries; e += gridDim.x * kThreads) {
        const uint32_t gn = a.pe_node[e];
        if (gn == kNone) continue;  // the host saw the node id out of range
        const uint32_t m = a.node_member[gn];
        if (!member_ok(a, m)) continue;
        const unsigned char* q = gnode_at(a, gn);
        bool ok = q[0] == 0;
        if (ok) {
            const KeyParts k = node_key(q);
            const uint32_t sn = a.pe_stub_name[e];
            ok = k.hash == a.pe_stub_hash[e] && k.nl == a.name_len[sn] && ld32(q + 90 + k.nl) >= a.pe_need[e];
            for (uint32_t i = 0; ok && i < k.nl; ++i) ok = k.name[i] == a.names[a.name_off[sn] + i];
        }
        if (!ok) {
            atomicOr(&a.status[m], FDY_PACK_PATCH);
            continue;
        }
        const KeyParts k = entry_key(a, e);
        const uint32_t local = a.n_nodes[m] + (e - a.entry_base[m]);
        a.pe_slot[e] = table_insert(a, key_fingerprint(k.hash, k.fa, k.name, k.nl, a.seed),
                                    (uint64_t(m) << 32) | local);
    }
}

// Every key equals its slot's first occurrence byte for byte (a fingerprint
// collision is reported, never merged). Threads [0, total_nodes) take nodes,
// the rest patch entries.
__global__ void __launch_bounds__(kThreads) pack_verify_kernel(const FdyPackArgs a) {
    const uint32_t n_items = a.total_nodes + a.n_entries;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < n_items; i += gridDim.x * kThreads) {
        KeyParts k;
        uint32_t slot;
        if (i < a.total_nodes) {
            const uint32_t m = a.node_member[i];
            if (!member_ok(a, m)) continue;
            const unsigned char* q = a.graphs + a.rec_off[m] + a.node_off[i];
            if (q[0] != 0) continue;
            k = node_key(q);
            slot = a.node_slot[i];
        } else {
            const uint32_t e = i - a.total_nodes;
            const uint32_t gn = a.pe_node[e];
            if (gn == kNone || !member_ok(a, a.node_member[gn]) || (a.status[a.node_member[gn]] & FDY_PACK_PATCH))
                continue;
            k = entry_key(a, e);
            slot = a.pe_slot[e];
        }
        if (!same_key(k, key_at(a, a.tpos[slot]))) atomicOr(&a.flags[0], 1u);
    }
}

__global__ void __launch_bounds__(kThreads) pack_compact_kernel(const FdyPackArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t slots = a.tmask + 1;
    for (uint32_t base = blockIdx.x * kThreads; base < slots; base += gridDim.x * kThreads) {
        const uint32_t s = base + threadIdx.x;  // slots is a multiple of kThreads
        const bool used = a.tkey[s] != 0ull;
        const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, used);
        uint32_t first = 0;
        if (lane == 0 && ballot) first = atomicAdd(a.ucount, __popc(ballot));
        first = __shfl_sync(0xFFFFFFFFu, first, 0);
        if (used) {
            const uint32_t u = first + __popc(ballot & ((1u << lane) - 1u));
            const unsigned long long pos = a.tpos[s];
            const uint32_t m = uint32_t(pos >> 32), n = uint32_t(pos);
            // the node, or for a real comm kernel the stub node it replaces
            const uint32_t gn = n < a.n_nodes[m] ? a.node_base[m] + n
                                                 : a.pe_node[a.entry_base[m] + (n - a.n_nodes[m])];
            a.upos[u] = pos;
            a.uoff[u] = a.rec_off[m] + a.node_off[gn];
            a.tuniq[s] = u;
            // the key's bytes, so the host builds the kernel table from one
            // contiguous read-back instead of 9,000 scattered ones
            const KeyParts k = key_at(a, pos);
            unsigned char* r = a.ukey + uint64_t(u) * FDY_PACK_KEY_BYTES;
            *reinterpret_cast<uint64_t*>(r) = k.hash;
            for (int i = 0; i < 24; ++i) r[8 + i] = k.fa[i];
            *reinterpret_cast<uint32_t*>(r + 32) = k.nl;
            for (uint32_t i = 0; i < k.nl && i < FDY_PACK_KEY_NAME; ++i) r[36 + i] = k.name[i];
        }
    }
}

// ------------------------------------------------------------------- pass 2

// One warp per node: descriptor + slot chunks + relocation meta.
__global__ void __launch_bounds__(kThreads) pack_images_kernel(const FdyPackArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kThreads / 32);
    for (uint32_t gn = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); gn < a.total_nodes; gn += warps) {
        const uint32_t m = a.node_member[gn];
        const uint32_t g = a.member_group[m];
        const uint32_t n = gn - a.node_base[m];
        const uint32_t N = a.n_nodes[m];
        const uint32_t gi = a.gnode_base[g] + n;
        const unsigned char* q = a.graphs + a.rec_off[m] + a.node_off[gn];
        const uint8_t t = q[0];
        const uint32_t cap = a.cap[gi], boff = a.blob_off[gi];
        uint32_t nl = 0, blob_len = 0;
        const unsigned char* src = q + 1;
        if (t == 0) {
            nl = ld32(q + 62);
            blob_len = ld32(q + 90 + nl);
            src = q + 94 + nl;
        } else if (t == 1 || t == 2) {
            blob_len = 24;
        }
        unsigned char* img = a.arena + a.out_off[m];
        uint8_t* meta = a.meta + a.out_off[m] / 16;
        if (lane < 3) {  // the 48-byte descriptor as three 16-byte stores
            union {
                fdt_node d;
                uint4 v[3];
            } u;
            u.v[0] = u.v[1] = u.v[2] = make_uint4(0, 0, 0, 0);
            fdt_node& d = u.d;
            d.type = t;
            d.kernel = kNone;
            d.blob_len = blob_len;
            d.blob_off = boff;
            if (t == 0) {
                d.kernel = a.ukidx[a.tuniq[a.node_slot[gn]]];
                for (int i = 0; i < 3; ++i) {
                    d.grid[i] = ld32(q + 26 + 4 * i);
                    d.block[i] = ld32(q + 38 + 4 * i);
                }
                d.shmem = ld32(q + 50);
            }
            reinterpret_cast<uint4*>(img + 48ull * n)[lane] = u.v[lane];
            meta[3ull * n + lane] = 0;
        }
        const uint64_t pool = 48ull * N + boff;
        const uint32_t chunks = cap / 16;
        for (uint32_t j = lane; j < chunks; j += 32) {
            // the chunk's 16 source bytes start anywhere: five aligned 32-bit
            // loads and funnel shifts (lanes read consecutive words), bytes
            // past the blob zeroed; the buffer is padded, so the last word may
            // run past the record
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (16 * j < blob_len) {
                const uintptr_t at = reinterpret_cast<uintptr_t>(src + 16 * j);
                const uint32_t* wp = reinterpret_cast<const uint32_t*>(at & ~uintptr_t(3));
                const uint32_t sh = uint32_t(at & 3u) * 8u;
                uint32_t r[5];
#pragma unroll
                for (int k = 0; k < 5; ++k) r[k] = __ldg(wp + k);
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = __funnelshift_r(r[k], r[k + 1], sh);
                const uint32_t valid = blob_len - 16 * j;  // bytes of this chunk inside the blob
                if (valid < 16) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t lo = 4u * k;
                        if (valid <= lo) w[k] = 0u;
                        else if (valid < lo + 4) w[k] &= (1u << (8 * (valid - lo))) - 1u;
                    }
                }
            }
            *reinterpret_cast<uint4*>(img + pool + 16ull * j) = make_uint4(w[0], w[1], w[2], w[3]);
            uint8_t f = 0;
            if (t == 0) {
                if (16 * j + 8 <= blob_len) f |= FDT_CMETA_LANE0;
                if (16 * j + 16 <= blob_len) f |= FDT_CMETA_LANE1;
            } else if (j == 0 && t == 1) {
                f = FDT_CMETA_LANE0 | FDT_CMETA_LANE1;  // src, dst
            } else if (j == 0 && t == 2) {
                f = FDT_CMETA_LANE0;  // dst
            }
            meta[pool / 16 + j] = f;
        }
    }
}

// apply_rank_patches' kernel swap: each entry's stub node gets the real comm
// kernel's store index.
__global__ void __launch_bounds__(kThreads) pack_swaps_kernel(const FdyPackArgs a) {
    const uint32_t e = blockIdx.x * kThreads + threadIdx.x;
    if (e >= a.n_entries) return;
    const uint32_t gn = a.pe_node[e];
    const uint32_t m = a.node_member[gn];
    const uint32_t n = gn - a.node_base[m];
    *reinterpret_cast<uint32_t*>(a.arena + a.out_off[m] + 48ull * n + offsetof(fdt_node, kernel)) =
        a.ukidx[a.tuniq[a.pe_slot[e]]];
}

struct TileRef {
    const uint64_t* mem;    // member lanes
    const uint64_t* tpl;    // template (representative) lanes
    const uint8_t* mmeta;
    const uint8_t* tmeta;
    uint32_t lanes;         // 2 x chunks in the tile
};

__device__ __forceinline__ TileRef tile_ref(const FdyPackArgs& a, uint32_t tn) {
    const uint32_t m = a.tile_member[tn];
    const uint32_t g = a.member_group[m];
    const uint32_t t = tn - a.tile_base[m];
    const uint64_t nchunks = a.g_image[g] / 16;
    const uint64_t cb = uint64_t(t) * FDT_TILE_CHUNKS;
    const uint64_t ce = u64min(nchunks, cb + FDT_TILE_CHUNKS);
    const uint64_t mo = a.out_off[m], to = a.out_off[a.group_rep[g]];
    TileRef r;
    r.mem = reinterpret_cast<const uint64_t*>(a.arena + mo) + 2 * cb;
    r.tpl = reinterpret_cast<const uint64_t*>(a.arena + to) + 2 * cb;
    r.mmeta = a.meta + mo / 16 + cb;
    r.tmeta = a.meta + to / 16 + cb;
    r.lanes = uint32_t(2 * (ce - cb));
    return r;
}

__device__ __forceinline__ bool lane_differs(const TileRef& r, uint32_t l, bool* reloc) {
    const bool mf = (r.mmeta[l >> 1] >> (l & 1)) & 1u;
    const bool tf = (r.tmeta[l >> 1] >> (l & 1)) & 1u;
    *reloc = mf;
    return mf != tf || r.mem[l] != r.tpl[l];
}

__global__ void __launch_bounds__(kThreads) pack_count_kernel(const FdyPackArgs a) {
    __shared__ uint32_t wsum[kThreads / 32];
    __shared__ uint32_t wrel[kThreads / 32];
    const uint32_t tn = blockIdx.x;
    const TileRef r = tile_ref(a, tn);
    uint32_t count = 0, rel = 0;
    for (uint32_t l = threadIdx.x; l < ((r.lanes + 31) & ~31u); l += kThreads) {
        bool f = false, d = false;
        if (l < r.lanes) {
            d = lane_differs(r, l, &f);
            rel |= (r.tmeta[l >> 1] >> (l & 1)) & 1u;
        }
        count += __popc(__ballot_sync(0xFFFFFFFFu, d));
    }
    rel = __any_sync(0xFFFFFFFFu, rel != 0);
    if ((threadIdx.x & 31) == 0) {
        wsum[threadIdx.x >> 5] = count;
        wrel[threadIdx.x >> 5] = rel;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0, any = 0;
        for (int w = 0; w < int(kThreads / 32); ++w) c += wsum[w], any |= wrel[w];
        a.tile_count[tn] = c;
        a.tile_reloc[tn] = uint8_t(any != 0);
    }
}

// ------------------------------------------------------------------- pass 3

__global__ void __launch_bounds__(kThreads) pack_diffs_kernel(const FdyPackArgs a) {
    __shared__ uint32_t wcount[kThreads / 32];
    const uint32_t tn = blockIdx.x;
    const TileRef r = tile_ref(a, tn);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t next = a.diff_lo[tn];
    for (uint32_t l0 = 0; l0 < r.lanes; l0 += kThreads) {
        const uint32_t l = l0 + threadIdx.x;
        bool f = false, d = false;
        if (l < r.lanes) d = lane_differs(r, l, &f);
        const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, d);
        if (lane == 0) wcount[warp] = __popc(ballot);
        __syncthreads();
        // warp scan of the per-warp counts (every warp computes it)
        const uint32_t c = lane < kThreads / 32 ? wcount[lane] : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= uint32_t(o)) incl += v;
        }
        const uint32_t before = __shfl_sync(0xFFFFFFFFu, incl - c, warp);
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, kThreads / 32 - 1);
        if (d) {
            const uint32_t at = next + before + __popc(ballot & ((1u << lane) - 1u));
            a.didx[at] = uint16_t(l | (f ? FDT_DIDX_RELOC : 0u));
            a.ddata[at] = r.mem[l];
        }
        next += total;
        __syncthreads();  // wcount is reused
    }
}

int grid_for(uint32_t items, uint32_t per_cta) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t need = (uint64_t(items) + per_cta - 1) / per_cta;
    return int(need == 0 ? 1 : need < uint64_t(sms) * 16 ? need : uint64_t(sms) * 16);
}

}  // namespace

extern "C" cudaError_t fdy_launch_pack_pass1(const FdyPackArgs* args, cudaStream_t stream) {
    const FdyPackArgs& a = *args;
    if (a.n_members == 0) return cudaSuccess;
    pack_walk_kernel<<<a.n_members, 32, 0, stream>>>(a);
    if (a.total_nodes) {
        pack_fields_kernel<<<grid_for(a.total_nodes, kThreads), kThreads, 0, stream>>>(a);
    }
    pack_edges_kernel<<<a.n_members, kThreads, 0, stream>>>(a);
    if (a.n_entries) pack_entries_kernel<<<grid_for(a.n_entries, kThreads), kThreads, 0, stream>>>(a);
    if (a.total_nodes + a.n_entries) {
        pack_verify_kernel<<<grid_for(a.total_nodes + a.n_entries, kThreads), kThreads, 0, stream>>>(a);
    }
    pack_compact_kernel<<<grid_for(a.tmask + 1, kThreads), kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_pack_pass2(const FdyPackArgs* args, cudaStream_t stream) {
    const FdyPackArgs& a = *args;
    if (a.total_nodes) pack_images_kernel<<<grid_for(a.total_nodes, kThreads / 32), kThreads, 0, stream>>>(a);
    if (a.n_entries) pack_swaps_kernel<<<(a.n_entries + kThreads - 1) / kThreads, kThreads, 0, stream>>>(a);
    if (a.n_tiles) pack_count_kernel<<<a.n_tiles, kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_pack_pass3(const FdyPackArgs* args, cudaStream_t stream) {
    const FdyPackArgs& a = *args;
    if (a.n_tiles) pack_diffs_kernel<<<a.n_tiles, kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}
