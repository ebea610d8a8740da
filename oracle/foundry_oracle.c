/* foundry_oracle.c — plain-C restatement of the reference LOAD-side member
 * preparation, used ONLY as the checker in tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg. The product never links or calls this.
 *
 * Parity is pinned (not "unpinned"): tests/test_oracle.py checks this file
 * against the reference's CRC KATs and, byte for byte, against the compiled
 * reference (oracle/_ref/ref_tool prepare / replay).
 *
 * Reference anchors (paths under /root/reference/proj):
 *   CRC-64/XZ ............ src/hash.cpp:13-25 (table), :53-69 (update/finish)
 *   FNDG container ....... src/graph_model.cpp:244-269 (serialize), :271-293 (locators)
 *   record decode ........ src/graph_model.cpp:146-203 (node), :220-240 (record), :41-64 (validate)
 *   record encode ........ src/graph_model.cpp:96-144 (node), :205-218 (record)
 *   parse_graph_at ....... src/graph_model.cpp:295-303
 *   patch table .......... src/rank_forge.cpp:70-102 (parse), :132-152 (apply_rank_patches)
 *   relocation rule ...... SURVEY.md §8(c) (no reference function; anchors det_alloc.cpp:152,
 *                          pipeline.cpp:434, range = manifest allocator.base + final_offset,
 *                          pipeline.hpp:38-39)
 *   comm slots ........... B200 extension, no reference function (the stub layer authors
 *                          the stub argument layout, rank_forge.cpp:18-22, and its patch
 *                          entries, :132-152; slot format and rule: archive.hpp CommSlot).
 *                          Pinned by property: the output equals ref_tool prepare's except
 *                          at exactly the slot bytes, which hold the rank's values.
 */
#define _GNU_SOURCE
#include "foundry_oracle.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ CRC */

static uint64_t crc_table[256];
static pthread_once_t crc_once = PTHREAD_ONCE_INIT;

static void crc_init(void) {
    const uint64_t poly = 0xC96C5795D7870F42ull; /* reflected 0x42F0E1EBA9EA3693 */
    for (uint64_t i = 0; i < 256; ++i) {
        uint64_t c = i;
        for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ poly : c >> 1;
        crc_table[i] = c;
    }
}

uint64_t fo_crc64(const uint8_t* data, size_t len) {
    pthread_once(&crc_once, crc_init);
    uint64_t c = ~0ull;
    for (size_t i = 0; i < len; ++i) c = (c >> 8) ^ crc_table[(c ^ data[i]) & 0xFF];
    return ~c;
}

uint64_t fo_crc64_bitwise(const uint8_t* data, size_t len) {
    uint64_t c = ~0ull;
    for (size_t i = 0; i < len; ++i) {
        c ^= data[i];
        for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ 0xC96C5795D7870F42ull : c >> 1;
    }
    return ~c;
}

/* ------------------------------------------------------- byte cursors */

typedef struct {
    const uint8_t* p;
    size_t n, pos;
    int err; /* sticky: set on overrun */
} rd_t;

static int rd_need(rd_t* r, size_t k) {
    if (r->err || r->pos + k > r->n) { r->err = 1; return 0; }
    return 1;
}
static uint8_t rd_u8(rd_t* r) { return rd_need(r, 1) ? r->p[r->pos++] : 0; }
static uint32_t rd_u32(rd_t* r) {
    uint32_t v = 0;
    if (rd_need(r, 4)) { memcpy(&v, r->p + r->pos, 4); r->pos += 4; }
    return v;
}
static uint64_t rd_u64(rd_t* r) {
    uint64_t v = 0;
    if (rd_need(r, 8)) { memcpy(&v, r->p + r->pos, 8); r->pos += 8; }
    return v;
}
static uint16_t rd_u16(rd_t* r) {
    uint16_t v = 0;
    if (rd_need(r, 2)) { memcpy(&v, r->p + r->pos, 2); r->pos += 2; }
    return v;
}
static const uint8_t* rd_bytes(rd_t* r, size_t k) {
    if (!rd_need(r, k)) return NULL;
    const uint8_t* q = r->p + r->pos;
    r->pos += k;
    return q;
}

typedef struct {
    uint8_t* p;
    size_t n, cap;
} wr_t;

static void wr_put(wr_t* w, const void* src, size_t k) {
    if (w->n + k > w->cap) {
        size_t c = w->cap ? w->cap * 2 : 4096;
        while (c < w->n + k) c *= 2;
        w->p = (uint8_t*)realloc(w->p, c);
        w->cap = c;
    }
    memcpy(w->p + w->n, src, k);
    w->n += k;
}
static void wr_u8(wr_t* w, uint8_t v) { wr_put(w, &v, 1); }
static void wr_u16(wr_t* w, uint16_t v) { wr_put(w, &v, 2); }
static void wr_u32(wr_t* w, uint32_t v) { wr_put(w, &v, 4); }
static void wr_u64(wr_t* w, uint64_t v) { wr_put(w, &v, 8); }

/* --------------------------------------------------------------- errors */

typedef struct {
    int code;
    char msg[512];
} err_t;

static int fail(err_t* e, int code, const char* fmt, ...) {
    if (e->code) return e->code;
    e->code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(e->msg, sizeof e->msg, fmt, ap);
    va_end(ap);
    return code;
}

/* ---------------------------------------------------------- patch table */

typedef struct {
    uint32_t node_id;
    uint64_t stub_hash;
    const uint8_t* stub_name;
    uint32_t stub_len;
    const uint8_t* real_name;
    uint32_t real_len;
    uint32_t n_rank, n_world;
    const uint8_t* rank_offs; /* u32 LE each */
    const uint8_t* world_offs;
} patch_entry_t;

typedef struct {
    uint32_t label;
    uint32_t count;
    patch_entry_t* entries;
} patch_graph_t;

typedef struct {
    uint32_t n_graphs;
    patch_graph_t* graphs;
} patch_table_t;

/* rank_forge.cpp:70-102; overruns are archive_corruption (ByteReader mode :71). */
static int parse_patch(const uint8_t* p, size_t n, patch_table_t* t, err_t* e) {
    memset(t, 0, sizeof *t);
    rd_t r = {p, n, 0, 0};
    const uint8_t* magic = rd_bytes(&r, 4);
    if (!magic || memcmp(magic, "FNDP", 4) != 0)
        return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: bad magic, expected 'FNDP'");
    uint16_t ver = rd_u16(&r);
    if (!r.err && ver != 1)
        return fail(e, FO_ARCHIVE_CORRUPTION,
                    "archive-corruption: unsupported patch table version %u", ver);
    (void)rd_u64(&r); /* world placeholder */
    t->n_graphs = rd_u32(&r);
    if (r.err) return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: truncated input");
    t->graphs = (patch_graph_t*)calloc(t->n_graphs ? t->n_graphs : 1, sizeof(patch_graph_t));
    for (uint32_t g = 0; g < t->n_graphs && !r.err; ++g) {
        patch_graph_t* pg = &t->graphs[g];
        pg->label = rd_u32(&r);
        pg->count = rd_u32(&r);
        if (r.err) break;
        pg->entries = (patch_entry_t*)calloc(pg->count ? pg->count : 1, sizeof(patch_entry_t));
        for (uint32_t i = 0; i < pg->count && !r.err; ++i) {
            patch_entry_t* pe = &pg->entries[i];
            pe->node_id = rd_u32(&r);
            pe->stub_hash = rd_u64(&r);
            pe->stub_len = rd_u32(&r);
            pe->stub_name = rd_bytes(&r, pe->stub_len);
            pe->real_len = rd_u32(&r);
            pe->real_name = rd_bytes(&r, pe->real_len);
            pe->n_rank = rd_u32(&r);
            pe->rank_offs = rd_bytes(&r, (size_t)pe->n_rank * 4);
            pe->n_world = rd_u32(&r);
            pe->world_offs = rd_bytes(&r, (size_t)pe->n_world * 4);
            (void)rd_u8(&r); /* patch_width: stored, never honoured (rank_forge.cpp:145-150) */
        }
    }
    if (r.err) return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: truncated input");
    if (r.pos != r.n)
        return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: trailing bytes in patch table");
    return 0;
}

static void free_patch(patch_table_t* t) {
    if (!t->graphs) return;
    for (uint32_t g = 0; g < t->n_graphs; ++g) free(t->graphs[g].entries);
    free(t->graphs);
    t->graphs = NULL;
}

static const patch_graph_t* patch_for(const patch_table_t* t, uint32_t label) {
    for (uint32_t g = 0; g < t->n_graphs; ++g)
        if (t->graphs[g].label == label) return &t->graphs[g];
    return NULL;
}

/* ----------------------------------------------------------- comm slots */

typedef struct {
    uint32_t node_id, offset, value_index;
    uint8_t width;
} slot_t;

typedef struct {
    uint32_t label, count;
    slot_t* slots;
} slot_graph_t;

typedef struct {
    uint32_t n_values, n_graphs;
    slot_graph_t* graphs;
} slot_table_t;

/* "FNDS" u16 version=1 u32 n_values u32 n_graphs, per graph u32 label u32 count,
 * per slot u32 node_id u32 offset u32 value_index u8 width (archive.hpp). */
static int parse_slots(const uint8_t* p, size_t n, slot_table_t* t, err_t* e) {
    memset(t, 0, sizeof *t);
    if (n == 0) return 0; /* no comm_slots.bin */
    rd_t r = {p, n, 0, 0};
    const uint8_t* magic = rd_bytes(&r, 4);
    if (!magic || memcmp(magic, "FNDS", 4) != 0)
        return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: bad magic, expected 'FNDS'");
    uint16_t ver = rd_u16(&r);
    if (!r.err && ver != 1)
        return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: unsupported comm slot table version %u", ver);
    t->n_values = rd_u32(&r);
    t->n_graphs = rd_u32(&r);
    if (r.err) return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: truncated input");
    if ((uint64_t)t->n_graphs * 8 > n) return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: truncated input");
    t->graphs = (slot_graph_t*)calloc(t->n_graphs ? t->n_graphs : 1, sizeof(slot_graph_t));
    for (uint32_t g = 0; g < t->n_graphs && !r.err; ++g) {
        slot_graph_t* sg = &t->graphs[g];
        sg->label = rd_u32(&r);
        sg->count = rd_u32(&r);
        if (r.err || (uint64_t)sg->count * 13 > n) { r.err = 1; break; }
        sg->slots = (slot_t*)calloc(sg->count ? sg->count : 1, sizeof(slot_t));
        for (uint32_t i = 0; i < sg->count && !r.err; ++i) {
            slot_t* s = &sg->slots[i];
            s->node_id = rd_u32(&r);
            s->offset = rd_u32(&r);
            s->value_index = rd_u32(&r);
            s->width = rd_u8(&r);
            if (r.err) break;
            if (s->width < 1 || s->width > 8)
                return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: comm slot width %u is not 1..8", s->width);
            if (s->value_index >= t->n_values)
                return fail(e, FO_ARCHIVE_CORRUPTION,
                            "archive-corruption: comm slot value index %u is outside the %u-entry value table",
                            s->value_index, t->n_values);
        }
        for (uint32_t h = 0; h < g && !r.err; ++h)
            if (t->graphs[h].label == sg->label)
                return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: comm slot table lists label %u twice",
                            sg->label);
    }
    if (r.err) return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: truncated input");
    if (r.pos != r.n) return fail(e, FO_ARCHIVE_CORRUPTION, "archive-corruption: trailing bytes in comm slot table");
    return 0;
}

static void free_slots(slot_table_t* t) {
    if (!t->graphs) return;
    for (uint32_t g = 0; g < t->n_graphs; ++g) free(t->graphs[g].slots);
    free(t->graphs);
    t->graphs = NULL;
}

static const slot_graph_t* slots_for(const slot_table_t* t, uint32_t label) {
    for (uint32_t g = 0; g < t->n_graphs; ++g)
        if (t->graphs[g].label == label) return &t->graphs[g];
    return NULL;
}

/* ---------------------------------------------------------------- nodes */

enum { NT_KERNEL = 0, NT_MEMCPY = 1, NT_MEMSET = 2, NT_EMPTY = 3 };

typedef struct {
    uint8_t type;
    uint8_t attrs[25];   /* cluster 3xu32, 3xi32, u8 — copied verbatim */
    uint32_t dims[7];    /* grid xyz, block xyz, shmem */
    uint64_t hash;
    const uint8_t* name; /* points into the record or the patch table */
    uint32_t name_len;
    uint8_t fattrs[24];  /* 6 x i32, verbatim */
    uint32_t arg_len;
    uint8_t* args;       /* owned copy */
    uint64_t mem[3];     /* memcpy src,dst,len | memset dst,value,len */
} node_t;

typedef struct {
    uint32_t label, n_nodes, n_edges;
    node_t* nodes;
    const uint8_t* edges; /* n_edges x (u32 from, u32 to), verbatim */
} graph_t;

static void free_graph(graph_t* g) {
    if (!g->nodes) return;
    for (uint32_t i = 0; i < g->n_nodes; ++i) free(g->nodes[i].args);
    free(g->nodes);
    g->nodes = NULL;
}

/* decode_graph_record graph_model.cpp:220-240 + decode_node :146-203 + validate :41-64 */
static int decode_record(const uint8_t* p, size_t n, graph_t* g, err_t* e) {
    memset(g, 0, sizeof *g);
    rd_t r = {p, n, 0, 0};
    g->label = rd_u32(&r);
    g->n_nodes = rd_u32(&r);
    g->n_edges = rd_u32(&r);
    if (r.err) return fail(e, FO_BINARY_FORMAT, "binary-format: truncated input");
    /* every node is at least one byte: bound the allocation by the record size */
    if (g->n_nodes > n) return fail(e, FO_BINARY_FORMAT, "binary-format: truncated input");
    g->nodes = (node_t*)calloc(g->n_nodes ? g->n_nodes : 1, sizeof(node_t));
    for (uint32_t i = 0; i < g->n_nodes; ++i) {
        node_t* nd = &g->nodes[i];
        nd->type = rd_u8(&r);
        if (r.err) break;
        switch (nd->type) {
            case NT_KERNEL: {
                const uint8_t* a = rd_bytes(&r, 25);
                if (a) memcpy(nd->attrs, a, 25);
                for (int k = 0; k < 7; ++k) nd->dims[k] = rd_u32(&r);
                nd->hash = rd_u64(&r);
                nd->name_len = rd_u32(&r);
                nd->name = rd_bytes(&r, nd->name_len);
                const uint8_t* fa = rd_bytes(&r, 24);
                if (fa) memcpy(nd->fattrs, fa, 24);
                nd->arg_len = rd_u32(&r);
                const uint8_t* args = rd_bytes(&r, nd->arg_len);
                if (r.err) break;
                nd->args = (uint8_t*)malloc(nd->arg_len ? nd->arg_len : 1);
                memcpy(nd->args, args, nd->arg_len);
                break;
            }
            case NT_MEMCPY:
            case NT_MEMSET:
                nd->mem[0] = rd_u64(&r);
                nd->mem[1] = rd_u64(&r);
                nd->mem[2] = rd_u64(&r);
                break;
            case NT_EMPTY:
                break;
            default:
                return fail(e, FO_BINARY_FORMAT, "binary-format: unknown node type tag");
        }
        if (r.err) break;
    }
    if (!r.err) g->edges = rd_bytes(&r, (size_t)g->n_edges * 8);
    if (r.err) return fail(e, FO_BINARY_FORMAT, "binary-format: truncated input");
    if (r.pos != r.n) return fail(e, FO_BINARY_FORMAT, "binary-format: trailing bytes in graph record");
    for (uint32_t i = 0; i < g->n_nodes; ++i) {
        const node_t* nd = &g->nodes[i];
        if (nd->type != NT_KERNEL) continue;
        if (nd->arg_len == 0)
            return fail(e, FO_INVALID_ARGUMENT,
                        "invalid-argument: kernel node %u has empty argument buffer", i);
        for (int k = 0; k < 6; ++k)
            if (nd->dims[k] < 1)
                return fail(e, FO_INVALID_ARGUMENT, "invalid-argument: launch dims must be >= 1");
    }
    uint32_t pf = 0, pt = 0;
    for (uint32_t i = 0; i < g->n_edges; ++i) {
        uint32_t f, t;
        memcpy(&f, g->edges + 8 * i, 4);
        memcpy(&t, g->edges + 8 * i + 4, 4);
        if (f >= g->n_nodes || t >= g->n_nodes)
            return fail(e, FO_INVALID_ARGUMENT, "invalid-argument: edge references missing node");
        if (f >= t)
            return fail(e, FO_INVALID_ARGUMENT,
                        "invalid-argument: edge must go from an earlier node to a later one");
        if (i > 0 && !(pf < f || (pf == f && pt < t)))
            return fail(e, FO_INVALID_ARGUMENT, "invalid-argument: edges must be in canonical order");
        pf = f;
        pt = t;
    }
    return 0;
}

/* encode_node graph_model.cpp:96-144 / encode_graph_record :205-218 */
static void encode_record(const graph_t* g, wr_t* w) {
    wr_u32(w, g->label);
    wr_u32(w, g->n_nodes);
    wr_u32(w, g->n_edges);
    for (uint32_t i = 0; i < g->n_nodes; ++i) {
        const node_t* nd = &g->nodes[i];
        wr_u8(w, nd->type);
        if (nd->type == NT_KERNEL) {
            wr_put(w, nd->attrs, 25);
            for (int k = 0; k < 7; ++k) wr_u32(w, nd->dims[k]);
            wr_u64(w, nd->hash);
            wr_u32(w, nd->name_len);
            wr_put(w, nd->name, nd->name_len);
            wr_put(w, nd->fattrs, 24);
            wr_u32(w, nd->arg_len);
            wr_put(w, nd->args, nd->arg_len);
        } else if (nd->type == NT_MEMCPY || nd->type == NT_MEMSET) {
            wr_u64(w, nd->mem[0]);
            wr_u64(w, nd->mem[1]);
            wr_u64(w, nd->mem[2]);
        }
    }
    wr_put(w, g->edges, (size_t)g->n_edges * 8);
}

/* ------------------------------------------------------ member transforms */

/* SURVEY.md §8(c) relocation rule. */
static uint64_t relocate(graph_t* g, uint64_t lo, uint64_t span, uint64_t delta) {
    uint64_t count = 0;
    if (delta == 0) return 0;
#define FO_MOVE(v) do { if ((v) - lo < span) { (v) += delta; ++count; } } while (0)
    for (uint32_t i = 0; i < g->n_nodes; ++i) {
        node_t* nd = &g->nodes[i];
        if (nd->type == NT_KERNEL) {
            for (uint32_t o = 0; o + 8 <= nd->arg_len; o += 8) {
                uint64_t v;
                memcpy(&v, nd->args + o, 8);
                uint64_t before = v;
                FO_MOVE(v);
                if (v != before) memcpy(nd->args + o, &v, 8);
            }
        } else if (nd->type == NT_MEMCPY) {
            FO_MOVE(nd->mem[0]);
            FO_MOVE(nd->mem[1]);
        } else if (nd->type == NT_MEMSET) {
            FO_MOVE(nd->mem[0]);
        }
    }
#undef FO_MOVE
    return count;
}

static int write_u64_at(node_t* nd, uint32_t off, uint64_t v, err_t* e) {
    if ((uint64_t)off + 8 > nd->arg_len)
        return fail(e, FO_INVALID_ARGUMENT,
                    "invalid-argument: patch offset outside the argument buffer");
    memcpy(nd->args + off, &v, 8);
    return 0;
}

/* apply_rank_patches rank_forge.cpp:132-152 */
static int rank_patch(graph_t* g, const patch_graph_t* pg, uint64_t real_hash, uint32_t rank,
                      uint32_t world, err_t* e) {
    for (uint32_t i = 0; i < pg->count; ++i) {
        const patch_entry_t* pe = &pg->entries[i];
        if (pe->node_id >= g->n_nodes)
            return fail(e, FO_ARCHIVE_CORRUPTION,
                        "archive-corruption: patch entry references missing node");
        node_t* nd = &g->nodes[pe->node_id];
        if (nd->type != NT_KERNEL)
            return fail(e, FO_ARCHIVE_CORRUPTION,
                        "archive-corruption: patch entry references a non-kernel node");
        if (nd->hash != pe->stub_hash || nd->name_len != pe->stub_len ||
            memcmp(nd->name, pe->stub_name, pe->stub_len) != 0)
            return fail(e, FO_ARCHIVE_CORRUPTION,
                        "archive-corruption: node %u is not the recorded stub (%016llx, %.*s)",
                        pe->node_id, (unsigned long long)pe->stub_hash, (int)pe->stub_len,
                        (const char*)pe->stub_name);
        nd->hash = real_hash;
        nd->name = pe->real_name;
        nd->name_len = pe->real_len;
        for (uint32_t k = 0; k < pe->n_rank; ++k) {
            uint32_t off;
            memcpy(&off, pe->rank_offs + 4 * k, 4);
            if (write_u64_at(nd, off, rank, e)) return e->code;
        }
        for (uint32_t k = 0; k < pe->n_world; ++k) {
            uint32_t off;
            memcpy(&off, pe->world_offs + 4 * k, 4);
            if (write_u64_at(nd, off, world, e)) return e->code;
        }
    }
    return 0;
}

/* Comm slot writes of one (already rank-patched) graph, in table order: only
 * nodes the graph's patch entries name; little-endian low `width` bytes. */
static int apply_slots(graph_t* g, const slot_graph_t* sg, const patch_graph_t* pg, const uint64_t* values,
                       uint32_t n_values, err_t* e) {
    for (uint32_t i = 0; i < sg->count; ++i) {
        const slot_t* s = &sg->slots[i];
        int stub = 0;
        for (uint32_t k = 0; pg && k < pg->count; ++k) stub |= pg->entries[k].node_id == s->node_id;
        if (!stub || s->node_id >= g->n_nodes || g->nodes[s->node_id].type != NT_KERNEL)
            return fail(e, FO_ARCHIVE_CORRUPTION,
                        "archive-corruption: comm slot references node %u, which is not a patched comm node",
                        s->node_id);
        node_t* nd = &g->nodes[s->node_id];
        if ((uint64_t)s->offset + s->width > nd->arg_len)
            return fail(e, FO_INVALID_ARGUMENT, "invalid-argument: comm slot offset outside the argument buffer");
        if (s->value_index >= n_values)
            return fail(e, FO_INVALID_ARGUMENT, "invalid-argument: comm slot value index %u has no value",
                        s->value_index);
        for (uint32_t b = 0; b < s->width; ++b) nd->args[s->offset + b] = (uint8_t)(values[s->value_index] >> (8 * b));
    }
    return 0;
}

/* ------------------------------------------------------- container walk */

typedef struct {
    uint32_t label;
    uint64_t offset, length, checksum;
} loc_t;

/* parse_graph_locators graph_model.cpp:271-293 */
static int parse_locators(const uint8_t* p, size_t n, loc_t** out, uint32_t* count, err_t* e) {
    rd_t r = {p, n, 0, 0};
    const uint8_t* magic = rd_bytes(&r, 4);
    if (!magic || memcmp(magic, "FNDG", 4) != 0)
        return fail(e, FO_BINARY_FORMAT, "binary-format: bad magic, expected 'FNDG'");
    uint16_t ver = rd_u16(&r);
    if (!r.err && ver != 1)
        return fail(e, FO_BINARY_FORMAT, "binary-format: unsupported graph container version %u",
                    ver);
    uint32_t c = rd_u32(&r);
    if (r.err) return fail(e, FO_BINARY_FORMAT, "binary-format: truncated input");
    if ((uint64_t)c * 28 > n) return fail(e, FO_BINARY_FORMAT, "binary-format: truncated input");
    loc_t* locs = (loc_t*)calloc(c ? c : 1, sizeof(loc_t));
    for (uint32_t i = 0; i < c; ++i) {
        locs[i].label = rd_u32(&r);
        locs[i].offset = rd_u64(&r);
        locs[i].length = rd_u64(&r);
        locs[i].checksum = rd_u64(&r);
        if (r.err) { free(locs); return fail(e, FO_BINARY_FORMAT, "binary-format: truncated input"); }
        if (!(locs[i].offset <= n && locs[i].length <= n - locs[i].offset)) {
            const uint32_t label = locs[i].label;
            free(locs);
            return fail(e, FO_BINARY_FORMAT,
                        "binary-format: graph record for label %u overruns the container", label);
        }
    }
    *out = locs;
    *count = c;
    return 0;
}

int64_t fo_graph_count(const uint8_t* graphs, size_t len) {
    err_t e = {0, {0}};
    loc_t* locs = NULL;
    uint32_t c = 0;
    if (parse_locators(graphs, len, &locs, &c, &e)) return -(int64_t)e.code;
    free(locs);
    return c;
}

typedef struct {
    const uint8_t* graphs;
    const loc_t* locs;
    uint32_t count;
    const patch_table_t* patch;
    const slot_table_t* slots;
    const uint64_t* values;
    uint32_t n_values;
    uint64_t real_hash, lo, span, delta;
    uint32_t rank, world;
    wr_t* records;       /* per member encoded record */
    uint64_t* relocated; /* per member */
    err_t* errs;         /* per member */
    uint32_t next;       /* shared task counter */
    pthread_mutex_t mu;
} job_t;

static void do_member(job_t* j, uint32_t i) {
    err_t* e = &j->errs[i];
    const loc_t* loc = &j->locs[i];
    const uint8_t* rec = j->graphs + loc->offset;
    /* parse_graph_at graph_model.cpp:295-303 */
    if (fo_crc64(rec, loc->length) != loc->checksum) {
        fail(e, FO_BINARY_FORMAT, "binary-format: checksum failure in graph record for label %u",
             loc->label);
        return;
    }
    graph_t g;
    if (decode_record(rec, loc->length, &g, e)) { free_graph(&g); return; }
    if (g.label != loc->label) {
        fail(e, FO_BINARY_FORMAT, "binary-format: label mismatch in graph record");
        free_graph(&g);
        return;
    }
    j->relocated[i] = relocate(&g, j->lo, j->span, j->delta);
    const patch_graph_t* pg = patch_for(j->patch, loc->label);
    if (pg && rank_patch(&g, pg, j->real_hash, j->rank, j->world, e)) { free_graph(&g); return; }
    const slot_graph_t* sg = slots_for(j->slots, loc->label);
    if (sg && apply_slots(&g, sg, pg, j->values, j->n_values, e)) { free_graph(&g); return; }
    encode_record(&g, &j->records[i]);
    free_graph(&g);
}

static void* worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        uint32_t i = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->count) break;
        do_member(j, i);
    }
    return NULL;
}

int fo_materialize_container(const uint8_t* graphs, size_t graphs_len,
                             const uint8_t* patch, size_t patch_len,
                             uint64_t real_comm_hash, uint32_t rank, uint32_t world,
                             uint64_t old_base, uint64_t final_offset, uint64_t new_base,
                             unsigned lanes, uint8_t** out, size_t* out_len,
                             uint64_t* n_relocated, char* err_msg, size_t err_cap) {
    return fo_materialize_container_ex(graphs, graphs_len, patch, patch_len, NULL, 0, NULL, 0, real_comm_hash,
                                       rank, world, old_base, final_offset, new_base, lanes, out, out_len,
                                       n_relocated, err_msg, err_cap);
}

int fo_materialize_container_ex(const uint8_t* graphs, size_t graphs_len,
                                const uint8_t* patch, size_t patch_len,
                                const uint8_t* slots, size_t slots_len,
                                const uint64_t* values, uint32_t n_values,
                                uint64_t real_comm_hash, uint32_t rank, uint32_t world,
                                uint64_t old_base, uint64_t final_offset, uint64_t new_base,
                                unsigned lanes, uint8_t** out, size_t* out_len,
                                uint64_t* n_relocated, char* err_msg, size_t err_cap) {
    err_t e = {0, {0}};
    patch_table_t pt = {0, NULL};
    slot_table_t stab = {0, 0, NULL};
    loc_t* locs = NULL;
    uint32_t count = 0;
    int rc = 0;
    *out = NULL;
    *out_len = 0;
    if (!(world >= 1 && rank < world)) {
        rc = fail(&e, FO_INVALID_ARGUMENT, "invalid-argument: rank %u is outside world size %u",
                  rank, world);
        goto done;
    }
    if ((rc = parse_patch(patch, patch_len, &pt, &e))) goto done;
    if ((rc = parse_slots(slots, slots_len, &stab, &e))) goto done;
    for (uint32_t g = 0; g < stab.n_graphs; ++g)
        if (!patch_for(&pt, stab.graphs[g].label)) {
            rc = fail(&e, FO_ARCHIVE_CORRUPTION,
                      "archive-corruption: comm slot table lists graph %u, which has no comm patches",
                      stab.graphs[g].label);
            goto done;
        }
    if (stab.n_graphs && n_values < stab.n_values) {
        rc = fail(&e, FO_INVALID_ARGUMENT,
                  "invalid-argument: the archive's comm slots read %u per-rank values, %u given", stab.n_values,
                  n_values);
        goto done;
    }
    if (pt.n_graphs > 0 && real_comm_hash == 0) {
        /* instantiate_rank rank_forge.cpp:162-163 */
        rc = fail(&e, FO_UNRESOLVED_KERNEL,
                  "unresolved-kernel: archive carries comm patches but no real comm binary");
        goto done;
    }
    if ((rc = parse_locators(graphs, graphs_len, &locs, &count, &e))) goto done;

    job_t j;
    memset(&j, 0, sizeof j);
    j.graphs = graphs;
    j.locs = locs;
    j.count = count;
    j.patch = &pt;
    j.slots = &stab;
    j.values = values;
    j.n_values = n_values;
    j.real_hash = real_comm_hash;
    j.lo = old_base;
    j.span = final_offset;
    j.delta = new_base - old_base;
    j.rank = rank;
    j.world = world;
    j.records = (wr_t*)calloc(count ? count : 1, sizeof(wr_t));
    j.relocated = (uint64_t*)calloc(count ? count : 1, sizeof(uint64_t));
    j.errs = (err_t*)calloc(count ? count : 1, sizeof(err_t));
    pthread_mutex_init(&j.mu, NULL);
    if (lanes < 1) lanes = 1;
    if (lanes > 256) lanes = 256;
    pthread_t th[256];
    for (unsigned t = 0; t < lanes; ++t) pthread_create(&th[t], NULL, worker, &j);
    for (unsigned t = 0; t < lanes; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&j.mu);

    uint64_t total_reloc = 0;
    for (uint32_t i = 0; i < count; ++i) {
        if (j.errs[i].code && !e.code) e = j.errs[i];
        total_reloc += j.relocated[i];
    }
    if (!e.code) {
        /* serialize_graphs graph_model.cpp:244-269 */
        wr_t w = {NULL, 0, 0};
        wr_put(&w, "FNDG", 4);
        wr_u16(&w, 1);
        wr_u32(&w, count);
        size_t table = w.n;
        for (uint32_t i = 0; i < count; ++i) {
            wr_u32(&w, locs[i].label);
            wr_u64(&w, 0);
            wr_u64(&w, 0);
            wr_u64(&w, 0);
        }
        for (uint32_t i = 0; i < count; ++i) {
            uint64_t off = w.n, len = j.records[i].n, crc = fo_crc64(j.records[i].p, j.records[i].n);
            memcpy(w.p + table + 28 * i + 4, &off, 8);
            memcpy(w.p + table + 28 * i + 12, &len, 8);
            memcpy(w.p + table + 28 * i + 20, &crc, 8);
            wr_put(&w, j.records[i].p, j.records[i].n);
        }
        *out = w.p;
        *out_len = w.n;
        if (n_relocated) *n_relocated = total_reloc;
    }
    rc = e.code;
    for (uint32_t i = 0; i < count; ++i) free(j.records[i].p);
    free(j.records);
    free(j.relocated);
    free(j.errs);
done:
    free(locs);
    free_patch(&pt);
    free_slots(&stab);
    if (rc && err_msg && err_cap) snprintf(err_msg, err_cap, "%s", e.msg);
    return rc;
}

void fo_free(void* p) { free(p); }
