// Little-endian byte cursors shared by every on-disk codec (FNDG graphs,
// FNDB images, FNDC catalog, FNDP patch table, memlayout, FNDT template store).
#pragma once

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "foundry/errors.hpp"

namespace foundry {

class Cursor {
public:
    Cursor(const uint8_t* p, size_t n, Errc on_overrun = Errc::binary_format)
        : p_(p), n_(n), err_(on_overrun) {}
    explicit Cursor(std::span<const uint8_t> s, Errc on_overrun = Errc::binary_format)
        : Cursor(s.data(), s.size(), on_overrun) {}

    template <typename T>
    T get() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, p_ + at_, sizeof(T));
        at_ += sizeof(T);
        return v;
    }
    uint8_t u8() { return get<uint8_t>(); }
    uint16_t u16() { return get<uint16_t>(); }
    uint32_t u32() { return get<uint32_t>(); }
    uint64_t u64() { return get<uint64_t>(); }
    int32_t i32() { return get<int32_t>(); }

    const uint8_t* take(size_t k) {
        need(k);
        const uint8_t* q = p_ + at_;
        at_ += k;
        return q;
    }
    std::string str() {
        const uint32_t k = u32();
        const uint8_t* q = take(k);
        return std::string(reinterpret_cast<const char*>(q), k);
    }
    std::string_view str_view() {
        const uint32_t k = u32();
        const uint8_t* q = take(k);
        return std::string_view(reinterpret_cast<const char*>(q), k);
    }
    void magic(const char (&m)[5]) {
        need(4);
        if (std::memcmp(p_ + at_, m, 4) != 0) {
            raise(err_, std::string("bad magic, expected '") + m + "'");
        }
        at_ += 4;
    }

    size_t pos() const { return at_; }
    size_t left() const { return n_ - at_; }
    bool at_end() const { return at_ == n_; }
    Errc error_code() const { return err_; }

private:
    void need(size_t k) const {
        if (k > n_ - at_) raise(err_, "truncated input");
    }

    const uint8_t* p_;
    size_t n_;
    size_t at_ = 0;
    Errc err_;
};

class Sink {
public:
    template <typename T>
    void put(T v) {
        const size_t at = buf_.size();
        buf_.resize(at + sizeof(T));
        std::memcpy(buf_.data() + at, &v, sizeof(T));
    }
    void u8(uint8_t v) { buf_.push_back(v); }
    void u16(uint16_t v) { put(v); }
    void u32(uint32_t v) { put(v); }
    void u64(uint64_t v) { put(v); }
    void i32(int32_t v) { put(v); }
    void raw(const void* p, size_t k) {
        const auto* b = static_cast<const uint8_t*>(p);
        buf_.insert(buf_.end(), b, b + k);
    }
    void raw(std::span<const uint8_t> s) { raw(s.data(), s.size()); }
    void str(std::string_view s) {
        u32(static_cast<uint32_t>(s.size()));
        raw(s.data(), s.size());
    }
    void zeros(size_t k) { buf_.resize(buf_.size() + k, 0); }
    void align(size_t a) { buf_.resize((buf_.size() + a - 1) / a * a, 0); }
    template <typename T>
    void poke(size_t at, T v) {
        std::memcpy(buf_.data() + at, &v, sizeof(T));
    }

    size_t size() const { return buf_.size(); }
    const std::vector<uint8_t>& bytes() const { return buf_; }
    std::vector<uint8_t> release() { return std::move(buf_); }
    void reserve(size_t k) { buf_.reserve(k); }

private:
    std::vector<uint8_t> buf_;
};

std::vector<uint8_t> slurp(const std::filesystem::path& path);
void spit(const std::filesystem::path& path, std::span<const uint8_t> data);
void spit(const std::filesystem::path& path, std::string_view text);

}  // namespace foundry
