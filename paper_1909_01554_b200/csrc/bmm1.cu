// bmm1.cu -- BMM1 files straight between disk and caller storage (host code only).
//
// Format and acceptance rules are the reference's (bitmatrix.cpp:187-233): "BMM1",
// rows and cols as little-endian u64, then rows * ceil(cols/64) little-endian words;
// the same checks, in the same order, with the same messages.  What changes is the
// data path: the payload is read / written with positioned I/O (pread / pwrite) by
// several threads, each on its own contiguous byte range, directly into the caller's
// buffer -- page-locked memory from bmmgpu_host_alloc for the matrices the out-of-core
// drivers stream (configs[4]: 128 GiB per operand), so a file goes to the GPU without
// a staging copy.  The reference instead reads into a byte vector and converts word by
// word.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bmmgpu.h"
#include "common.cuh"

namespace bmmgpu {
namespace {

constexpr int kEformat = BMMGPU_EFORMAT;

uint64_t get_le(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}
void put_le(unsigned char* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

int header(int fd, const std::string& path, uint64_t* rows, uint64_t* cols) {
    unsigned char h[20];
    size_t got = 0;
    while (got < sizeof h) {
        const ssize_t r = pread(fd, h + got, sizeof h - got, off_t(got));
        if (r <= 0) break;
        got += size_t(r);
    }
    if (got != sizeof h) {
        set_error(path + ": truncated header");
        return kEformat;
    }
    if (std::memcmp(h, "BMM1", 4) != 0) {
        set_error(path + ": bad magic");
        return kEformat;
    }
    *rows = get_le(h + 4);
    *cols = get_le(h + 12);
    if (*rows == 0 || *cols == 0 || *rows > (uint64_t(1) << 30) || *cols > (uint64_t(1) << 30)) {
        set_error(path + ": unreasonable dimensions");
        return kEformat;
    }
    return kOk;
}

unsigned io_threads(int32_t requested, uint64_t bytes) {
    unsigned t = requested > 0 ? unsigned(requested) : std::max(1u, std::thread::hardware_concurrency());
    // at least 64 MiB per thread
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(t, bytes >> 26)));
}

// Run body(begin, end) over [0, bytes) split into `threads` contiguous ranges; false if
// any range failed.
template <class F>
bool parallel_ranges(uint64_t bytes, unsigned threads, F body) {
    std::atomic<bool> ok{true};
    std::vector<std::thread> th;
    const uint64_t step = (bytes + threads - 1) / threads;
    for (unsigned i = 0; i < threads; ++i) {
        const uint64_t b = std::min(bytes, i * step), e = std::min(bytes, (i + 1) * step);
        th.emplace_back([&, b, e] {
            if (!body(b, e)) ok = false;
        });
    }
    for (auto& t : th) t.join();
    return ok;
}

}  // namespace
}  // namespace bmmgpu

using namespace bmmgpu;

extern "C" {

int bmmgpu_bmm1_info(const char* path, uint64_t* rows, uint64_t* cols) {
    if (!path || !rows || !cols) {
        set_error("bmmgpu_bmm1_info: null argument");
        return kEinval;
    }
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) {
        set_error(std::string("cannot open ") + path);
        return kEformat;
    }
    return header(f.fd, path, rows, cols);
}

int bmmgpu_bmm1_read(const char* path, uint64_t* words, uint64_t n_words, int32_t threads) {
    if (!path || (!words && n_words)) {
        set_error("bmmgpu_bmm1_read: null argument");
        return kEinval;
    }
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) {
        set_error(std::string("cannot open ") + path);
        return kEformat;
    }
    uint64_t rows = 0, cols = 0;
    if (int st = header(f.fd, path, &rows, &cols)) return st;
    const uint64_t wpr = (cols + 63) / 64, total_words = rows * wpr;
    if (n_words != total_words) {
        set_error(std::string(path) + ": destination holds " + std::to_string(n_words) + " words, the matrix " +
                  std::to_string(total_words));
        return kEinval;
    }
    struct stat sb {};
    if (fstat(f.fd, &sb) != 0) {
        set_error(std::string(path) + ": truncated payload");
        return kEformat;
    }
    const uint64_t bytes = total_words * 8, size = uint64_t(sb.st_size);
    if (size < 20 + bytes) {
        set_error(std::string(path) + ": truncated payload");
        return kEformat;
    }
    if (size > 20 + bytes) {
        set_error(std::string(path) + ": trailing bytes");
        return kEformat;
    }
    auto* dst = reinterpret_cast<unsigned char*>(words);
    const bool ok = parallel_ranges(bytes, io_threads(threads, bytes), [&](uint64_t b, uint64_t e) {
        while (b < e) {
            const ssize_t r = pread(f.fd, dst + b, size_t(std::min<uint64_t>(e - b, uint64_t(1) << 30)), off_t(20 + b));
            if (r <= 0) return false;
            b += uint64_t(r);
        }
        return true;
    });
    if (!ok) {
        set_error(std::string(path) + ": truncated payload");
        return kEformat;
    }
    // little-endian host: the words are already in place (x86-64, aarch64 here)
    if (const unsigned tail = unsigned(cols % 64)) {
        const uint64_t pad = ~((uint64_t(1) << tail) - 1);
        std::atomic<bool> clean{true};
        parallel_ranges(rows, std::max(1u, std::min<unsigned>(16, unsigned(rows >> 16))), [&](uint64_t b, uint64_t e) {
            for (uint64_t i = b; i < e; ++i)
                if (words[i * wpr + wpr - 1] & pad) {
                    clean = false;
                    return false;
                }
            return true;
        });
        if (!clean) {
            set_error(std::string(path) + ": nonzero padding bits");
            return kEformat;
        }
    }
    return kOk;
}

int bmmgpu_bmm1_write(const char* path, uint64_t rows, uint64_t cols, const uint64_t* words, int32_t threads) {
    if (!path || (!words && rows && cols)) {
        set_error("bmmgpu_bmm1_write: null argument");
        return kEinval;
    }
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) {
        set_error(std::string("cannot open ") + path + " for writing");
        return kEformat;
    }
    unsigned char h[20];
    std::memcpy(h, "BMM1", 4);
    put_le(h + 4, rows);
    put_le(h + 12, cols);
    const uint64_t bytes = rows * ((cols + 63) / 64) * 8;
    bool ok = pwrite(f.fd, h, sizeof h, 0) == ssize_t(sizeof h) && ftruncate(f.fd, off_t(20 + bytes)) == 0;
    const auto* src = reinterpret_cast<const unsigned char*>(words);
    ok = ok && parallel_ranges(bytes, io_threads(threads, bytes), [&](uint64_t b, uint64_t e) {
             while (b < e) {
                 const ssize_t r =
                     pwrite(f.fd, src + b, size_t(std::min<uint64_t>(e - b, uint64_t(1) << 30)), off_t(20 + b));
                 if (r <= 0) return false;
                 b += uint64_t(r);
             }
             return true;
         });
    if (!ok) {
        set_error(std::string("write failed for ") + path);
        return kEformat;
    }
    return kOk;
}

}  // extern "C"
