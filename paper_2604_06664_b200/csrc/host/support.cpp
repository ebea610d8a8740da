// errors, file I/O and host hashes (see the headers for the reference anchors).
#include <array>
#include <cstring>
#include <immintrin.h>
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

// ---- carry-less multiply folding (PCLMULQDQ) for long inputs
//
// In the reflected representation (x^0 is bit 63 of a u64; a 16-byte LE
// load has x^127 in bit 0), clmul(a, b) of two reflected 64-bit operands is
// the reflected 128-bit form of a(x) b(x) x. A 128-bit state X = Xh x^64 + Xl
// (Xh = low lane) moves d bits further down the message as
//     X x^d == clmul(Xh, x^(d+63) mod P) ^ clmul(Xl, x^(d-1) mod P)   (mod P),
// and a final 128-bit state reduces to the CRC register by feeding its 16
// bytes through the table walk from a zero register (register = W x^64 mod P).
// Four accumulators fold 64 bytes per step.

uint64_t x_pow_mod(unsigned n) {  // x^n mod P, reflected
    uint64_t p = 1ull << 63;
    while (n--) p = (p & 1) ? (p >> 1) ^ kCrc64Poly : p >> 1;
    return p;
}

struct FoldConstants {
    uint64_t k[4][2];  // fold distances 128, 256, 384, 512 bits: {x^(d+63), x^(d-1)}
    FoldConstants() {
        for (int i = 0; i < 4; ++i) {
            const unsigned d = 128u * static_cast<unsigned>(i + 1);
            k[i][0] = x_pow_mod(d + 63);
            k[i][1] = x_pow_mod(d - 1);
        }
    }
};

const FoldConstants& fold_constants() {
    static const FoldConstants f;
    return f;
}

bool have_pclmul() {
    static const bool ok = __builtin_cpu_supports("pclmul") && __builtin_cpu_supports("sse4.1");
    return ok;
}

__attribute__((target("pclmul,sse4.1"))) inline __m128i fold128(__m128i x, const uint64_t* k) {
    const __m128i kk = _mm_set_epi64x(static_cast<long long>(k[1]), static_cast<long long>(k[0]));
    return _mm_xor_si128(_mm_clmulepi64_si128(x, kk, 0x00), _mm_clmulepi64_si128(x, kk, 0x11));
}

// Consumes floor(len / 64) * 64 bytes (len >= 64); returns the register.
__attribute__((target("pclmul,sse4.1"))) uint64_t fold_blocks(uint64_t c, const uint8_t* p, size_t n64) {
    const FoldConstants& K = fold_constants();
    __m128i x0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
    __m128i x1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16));
    __m128i x2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 32));
    __m128i x3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 48));
    x0 = _mm_xor_si128(x0, _mm_set_epi64x(0, static_cast<long long>(c)));  // register into the first 8 bytes
    for (size_t i = 1; i < n64; ++i) {
        const uint8_t* q = p + 64 * i;
        x0 = _mm_xor_si128(fold128(x0, K.k[3]), _mm_loadu_si128(reinterpret_cast<const __m128i*>(q)));
        x1 = _mm_xor_si128(fold128(x1, K.k[3]), _mm_loadu_si128(reinterpret_cast<const __m128i*>(q + 16)));
        x2 = _mm_xor_si128(fold128(x2, K.k[3]), _mm_loadu_si128(reinterpret_cast<const __m128i*>(q + 32)));
        x3 = _mm_xor_si128(fold128(x3, K.k[3]), _mm_loadu_si128(reinterpret_cast<const __m128i*>(q + 48)));
    }
    __m128i x = _mm_xor_si128(_mm_xor_si128(fold128(x0, K.k[2]), fold128(x1, K.k[1])),
                              _mm_xor_si128(fold128(x2, K.k[0]), x3));
    // 16 bytes through the table walk from a zero register
    const auto& T = tables().t;
    uint64_t r = 0;
    for (int lane = 0; lane < 2; ++lane) {
        r ^= static_cast<uint64_t>(lane ? _mm_extract_epi64(x, 1) : _mm_cvtsi128_si64(x));
        r = T[7][r & 0xFF] ^ T[6][(r >> 8) & 0xFF] ^ T[5][(r >> 16) & 0xFF] ^ T[4][(r >> 24) & 0xFF] ^
            T[3][(r >> 32) & 0xFF] ^ T[2][(r >> 40) & 0xFF] ^ T[1][(r >> 48) & 0xFF] ^ T[0][r >> 56];
    }
    return r;
}

// ---- the same fold four 128-bit lanes at a time (VPCLMULQDQ on 512-bit
// registers): four accumulators fold 256 bytes per step, then the 16 lanes
// (lane i = bytes 16i..16i+15 of the last window) fold to the end of it.

struct WideFoldConstants {
    uint64_t step[2];      // d = 2048 bits
    uint64_t tail[16][2];  // d = 128 * (15 - i) bits for lane i (lane 15: unused)
    WideFoldConstants() {
        step[0] = x_pow_mod(2048 + 63);
        step[1] = x_pow_mod(2048 - 1);
        for (int i = 0; i < 15; ++i) {
            const unsigned d = 128u * static_cast<unsigned>(15 - i);
            tail[i][0] = x_pow_mod(d + 63);
            tail[i][1] = x_pow_mod(d - 1);
        }
    }
};

const WideFoldConstants& wide_fold_constants() {
    static const WideFoldConstants f;
    return f;
}

bool have_vpclmul() {
    static const bool ok = __builtin_cpu_supports("vpclmulqdq") && __builtin_cpu_supports("avx512f") &&
                           __builtin_cpu_supports("pclmul") && __builtin_cpu_supports("sse4.1");
    return ok;
}

__attribute__((target("avx512f,vpclmulqdq"))) inline __m512i fold512(__m512i x, __m512i k) {
    return _mm512_xor_si512(_mm512_clmulepi64_epi128(x, k, 0x00), _mm512_clmulepi64_epi128(x, k, 0x11));
}

// Consumes n256 * 256 bytes (n256 >= 1); returns the register.
__attribute__((target("avx512f,vpclmulqdq,pclmul,sse4.1"))) uint64_t fold_blocks_wide(uint64_t c, const uint8_t* p,
                                                                                       size_t n256) {
    const WideFoldConstants& K = wide_fold_constants();
    const __m512i k = _mm512_broadcast_i32x4(
        _mm_set_epi64x(static_cast<long long>(K.step[1]), static_cast<long long>(K.step[0])));
    __m512i x0 = _mm512_loadu_si512(p);
    __m512i x1 = _mm512_loadu_si512(p + 64);
    __m512i x2 = _mm512_loadu_si512(p + 128);
    __m512i x3 = _mm512_loadu_si512(p + 192);
    x0 = _mm512_xor_si512(x0, _mm512_set_epi64(0, 0, 0, 0, 0, 0, 0, static_cast<long long>(c)));
    for (size_t i = 1; i < n256; ++i) {
        const uint8_t* q = p + 256 * i;
        x0 = _mm512_xor_si512(fold512(x0, k), _mm512_loadu_si512(q));
        x1 = _mm512_xor_si512(fold512(x1, k), _mm512_loadu_si512(q + 64));
        x2 = _mm512_xor_si512(fold512(x2, k), _mm512_loadu_si512(q + 128));
        x3 = _mm512_xor_si512(fold512(x3, k), _mm512_loadu_si512(q + 192));
    }
    alignas(64) __m128i lane[16];
    _mm512_store_si512(lane, x0);
    _mm512_store_si512(lane + 4, x1);
    _mm512_store_si512(lane + 8, x2);
    _mm512_store_si512(lane + 12, x3);
    __m128i x = lane[15];
    for (int i = 0; i < 15; ++i) x = _mm_xor_si128(x, fold128(lane[i], K.tail[i]));
    const auto& T = tables().t;
    uint64_t r = 0;
    for (int l = 0; l < 2; ++l) {
        r ^= static_cast<uint64_t>(l ? _mm_extract_epi64(x, 1) : _mm_cvtsi128_si64(x));
        r = T[7][r & 0xFF] ^ T[6][(r >> 8) & 0xFF] ^ T[5][(r >> 16) & 0xFF] ^ T[4][(r >> 24) & 0xFF] ^
            T[3][(r >> 32) & 0xFF] ^ T[2][(r >> 40) & 0xFF] ^ T[1][(r >> 48) & 0xFF] ^ T[0][r >> 56];
    }
    return r;
}

}  // namespace

void Crc64::update(const void* data, size_t len) {
    const auto& T = tables().t;
    const auto* p = static_cast<const uint8_t*>(data);
    uint64_t c = state_;
    if (len >= 1024 && have_vpclmul()) {
        const size_t n256 = len / 256;
        c = fold_blocks_wide(c, p, n256);
        p += 256 * n256;
        len -= 256 * n256;
    }
    if (len >= 256 && have_pclmul()) {
        const size_t n64 = len / 64;
        c = fold_blocks(c, p, n64);
        p += 64 * n64;
        len -= 64 * n64;
    }
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
