// Host-side hashes.
//
// CRC-64/XZ (reflected poly 0x42F0E1EBA9EA3693, init = xorout = ~0) is the
// archive content hash (reference hash.hpp:14-26). On the LOAD hot path it is
// computed on the GPU (csrc/kernels/crc64.cu); this host version serves the
// offline tools (save, pack) and small control records. It is a
// slicing-by-8 implementation, bit-identical to the reference's byte-at-a-time
// table walk (hash.cpp:53-61).
//
// crc64_combine / x8n_mod_p implement the GF(2) algebra the GPU kernel uses to
// stitch chunk CRCs: crc(A||B) = mulmod(x^(8|B|), crc(A)) ^ crc(B).
//
// murmur3_x64_128 keys topologies (reference hash.cpp:73-148); SAVE-side only.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <string>

namespace foundry {

inline constexpr uint64_t kCrc64Poly = 0xC96C5795D7870F42ull;  // reflected
inline constexpr uint8_t kContentHashAlgorithm = 1;

class Crc64 {
public:
    void update(const void* data, size_t len);
    uint64_t value() const { return ~state_; }

private:
    uint64_t state_ = ~0ull;
};

uint64_t crc64(const void* data, size_t len);
inline uint64_t crc64(std::span<const uint8_t> s) { return crc64(s.data(), s.size()); }

// a(x) * b(x) mod P(x), reflected representation (x^0 is bit 63).
uint64_t crc64_mulmod(uint64_t a, uint64_t b);
// x^(8 * nbytes) mod P(x).
uint64_t crc64_x8n(uint64_t nbytes);
// CRC-64/XZ of A||B from crc(A), crc(B) and |B|.
uint64_t crc64_combine(uint64_t crc_a, uint64_t crc_b, uint64_t len_b);
// x^(2^k) mod P for k = 0..63 (the GPU kernel's constant table).
const uint64_t* crc64_x2k_table();

struct Digest128 {
    uint64_t hi = 0, lo = 0;
    bool operator==(const Digest128&) const = default;
    auto operator<=>(const Digest128&) const = default;
    std::string hex() const;
};

Digest128 murmur3_x64_128(const void* data, size_t len, uint64_t seed);

std::string hex16(uint64_t v);
uint64_t parse_hex(std::string_view text);

}  // namespace foundry
