// errors, file I/O and host hashes (see the headers for the reference anchors).
#include <array>
#include <cstdio>
#include <fstream>

#include "foundry/bytes.hpp"
#include "foundry/errors.hpp"
#include "foundry/hash.hpp"

namespace foundry {

// ---------------------------------------------------------------- errors

std::string_view errc_name(Errc code) noexcept {
    static constexpr std::string_view names[] = {
        "invalid-argument",   "spec-violation",     "binary-format",
        "unresolved-kernel",  "unmapped-address",   "topology-mismatch",
        "layout-divergence",  "archive-corruption", "out-of-region",
        "unknown-address",    "device-state-uninitialized",
        "unpatchable-comm",   "schema-violation",   "cuda-error",
        "device-unavailable",
    };
    const auto i = static_cast<size_t>(code);
    return i < std::size(names) ? names[i] : std::string_view("unknown");
}

int exit_code_for(Errc code) noexcept {
    // reference errors.cpp:24-39
    switch (code) {
        case Errc::archive_corruption:
        case Errc::binary_format:
        case Errc::schema_violation: return 2;
        case Errc::layout_divergence: return 3;
        case Errc::unresolved_kernel: return 4;
        case Errc::topology_mismatch: return 5;
        default: return 1;
    }
}

void rethrow_in_step(const char* step) {
    try {
        throw;
    } catch (const Error& e) {
        throw Error(e.code(), std::string(step) + ": " + e.detail());
    }
}

// ---------------------------------------------------------------- files

std::vector<uint8_t> slurp(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    require(in.good(), Errc::archive_corruption, "cannot open " + path.string());
    const auto n = static_cast<size_t>(in.tellg());
    in.seekg(0);
    std::vector<uint8_t> out(n);
    if (n) in.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(n));
    require(in.good() || n == 0, Errc::archive_corruption, "short read on " + path.string());
    return out;
}

void spit(const std::filesystem::path& path, std::span<const uint8_t> data) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    require(out.good(), Errc::invalid_argument, "cannot write " + path.string());
    out.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(data.size()));
    require(out.good(), Errc::invalid_argument, "short write on " + path.string());
}

void spit(const std::filesystem::path& path, std::string_view text) {
    spit(path, std::span<const uint8_t>(reinterpret_cast<const uint8_t*>(text.data()), text.size()));
}

// ---------------------------------------------------------------- CRC-64

namespace {

struct SliceTables {
    uint64_t t[8][256];
    uint64_t x2k[64];
    SliceTables() {
        for (uint64_t i = 0; i < 256; ++i) {
            uint64_t c = i;
            for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ kCrc64Poly : c >> 1;
            t[0][i] = c;
        }
        for (int k = 1; k < 8; ++k)
            for (int i = 0; i < 256; ++i) t[k][i] = (t[k - 1][i] >> 8) ^ t[0][t[k - 1][i] & 0xFF];
        x2k[0] = 1ull << 62;  // x^1
        for (int k = 1; k < 64; ++k) x2k[k] = crc64_mulmod(x2k[k - 1], x2k[k - 1]);
    }
};

const SliceTables& tables() {
    static const SliceTables s;
    return s;
}

}  // namespace

void Crc64::update(const void* data, size_t len) {
    const auto& T = tables().t;
    const auto* p = static_cast<const uint8_t*>(data);
    uint64_t c = state_;
    while (len >= 8) {
        uint64_t w;
        std::memcpy(&w, p, 8);
        c ^= w;
        c = T[7][c & 0xFF] ^ T[6][(c >> 8) & 0xFF] ^ T[5][(c >> 16) & 0xFF] ^
            T[4][(c >> 24) & 0xFF] ^ T[3][(c >> 32) & 0xFF] ^ T[2][(c >> 40) & 0xFF] ^
            T[1][(c >> 48) & 0xFF] ^ T[0][c >> 56];
        p += 8;
        len -= 8;
    }
    while (len--) c = (c >> 8) ^ T[0][(c ^ *p++) & 0xFF];
    state_ = c;
}

uint64_t crc64(const void* data, size_t len) {
    Crc64 c;
    c.update(data, len);
    return c.value();
}

uint64_t crc64_mulmod(uint64_t a, uint64_t b) {
    uint64_t prod = 0;
    for (uint64_t m = 1ull << 63; m; m >>= 1) {
        if (a & m) prod ^= b;
        b = (b & 1) ? (b >> 1) ^ kCrc64Poly : b >> 1;
    }
    return prod;
}

uint64_t crc64_x8n(uint64_t nbytes) {
    const auto& x2k = tables().x2k;
    uint64_t p = 1ull << 63;  // x^0
    for (int k = 3; nbytes; nbytes >>= 1, ++k)
        if (nbytes & 1) p = crc64_mulmod(x2k[k & 63], p);
    return p;
}

uint64_t crc64_combine(uint64_t crc_a, uint64_t crc_b, uint64_t len_b) {
    return crc64_mulmod(crc64_x8n(len_b), crc_a) ^ crc_b;
}

const uint64_t* crc64_x2k_table() { return tables().x2k; }

// ---------------------------------------------------------------- murmur3

namespace {
inline uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline uint64_t fmix(uint64_t k) {
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDull;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ull;
    return k ^ (k >> 33);
}
}  // namespace

Digest128 murmur3_x64_128(const void* data, size_t len, uint64_t seed) {
    constexpr uint64_t c1 = 0x87C37B91114253D5ull, c2 = 0x4CF5AD432745937Full;
    const auto* p = static_cast<const uint8_t*>(data);
    uint64_t h1 = seed, h2 = seed;
    const size_t blocks = len / 16;
    for (size_t i = 0; i < blocks; ++i) {
        uint64_t k1, k2;
        std::memcpy(&k1, p + 16 * i, 8);
        std::memcpy(&k2, p + 16 * i + 8, 8);
        h1 ^= rotl(k1 * c1, 31) * c2;
        h1 = (rotl(h1, 27) + h2) * 5 + 0x52DCE729;
        h2 ^= rotl(k2 * c2, 33) * c1;
        h2 = (rotl(h2, 31) + h1) * 5 + 0x38495AB5;
    }
    const uint8_t* tail = p + 16 * blocks;
    const size_t rest = len & 15;
    uint64_t k1 = 0, k2 = 0;
    for (size_t i = rest; i > 8; --i) k2 ^= static_cast<uint64_t>(tail[i - 1]) << (8 * (i - 9));
    if (rest > 8) h2 ^= rotl(k2 * c2, 33) * c1;
    for (size_t i = std::min<size_t>(rest, 8); i > 0; --i)
        k1 ^= static_cast<uint64_t>(tail[i - 1]) << (8 * (i - 1));
    if (rest > 0) h1 ^= rotl(k1 * c1, 31) * c2;
    h1 ^= len;
    h2 ^= len;
    h1 += h2;
    h2 += h1;
    h1 = fmix(h1);
    h2 = fmix(h2);
    h1 += h2;
    h2 += h1;
    return {h1, h2};
}

std::string Digest128::hex() const { return hex16(hi) + hex16(lo); }

std::string hex16(uint64_t v) {
    char b[17];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
    return b;
}

uint64_t parse_hex(std::string_view text) {
    require(!text.empty() && text.size() <= 16, Errc::invalid_argument,
            "bad hex literal '" + std::string(text) + "'");
    uint64_t v = 0;
    for (char c : text) {
        int d;
        if (c >= '0' && c <= '9') d = c - '0';
        else if (c >= 'a' && c <= 'f') d = c - 'a' + 10;
        else if (c >= 'A' && c <= 'F') d = c - 'A' + 10;
        else raise(Errc::invalid_argument, "bad hex digit in '" + std::string(text) + "'");
        v = (v << 4) | static_cast<uint64_t>(d);
    }
    return v;
}

}  // namespace foundry
