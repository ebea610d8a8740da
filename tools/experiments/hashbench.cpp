#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>
#include "foundry/hash.hpp"
using namespace foundry;
int main(int argc, char** argv) {
    const char* path = argv[1];
    int T = atoi(argv[2]);
    struct stat st; stat(path, &st);
    size_t n = st.st_size, piece = 2 << 20;
    size_t np = (n + piece - 1) / piece;
    for (int mode = 0; mode < 3; ++mode) for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::atomic<size_t> next{0};
        std::vector<uint64_t> out(np);
        int fd = open(path, O_RDONLY);
        const uint8_t* map = nullptr;
        if (mode == 1) { map = (const uint8_t*)mmap(nullptr, n, PROT_READ, MAP_SHARED, fd, 0); madvise((void*)map, n, MADV_SEQUENTIAL); }
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back([&] {
            std::unique_ptr<uint8_t[]> buf(new uint8_t[1 << 20]);
            for (size_t i; (i = next.fetch_add(1)) < np;) {
                size_t off = i * piece, len = std::min(piece, n - off);
                if (mode == 2) {
                    for (size_t d = 0; d < len;) { ssize_t r = pread(fd, buf.get(), std::min<size_t>(1 << 20, len - d), off + d); d += r; }
                } else if (mode == 0) {
                    Crc64 c;
                    for (size_t d = 0; d < len;) { ssize_t r = pread(fd, buf.get(), std::min<size_t>(1 << 20, len - d), off + d); c.update(buf.get(), r); d += r; }
                    out[i] = c.value();
                } else out[i] = crc64(map + off, len);
            }
        });
        for (auto& x : th) x.join();
        if (map) munmap((void*)map, n);
        close(fd);
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        printf("%s threads %d: %.3f ms  %.1f GB/s\n", mode == 2 ? "pread only" : mode ? "mmap " : "pread+crc", T, ms, n / ms / 1e6);
    }
}
