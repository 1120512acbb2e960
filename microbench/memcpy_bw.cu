// Host memcpy bandwidth on the GPU box: pageable -> page-locked (the staging direction of
// uploads) and page-locked -> pageable (downloads), 1..16 threads, 512 MiB (dev helper).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double run(char* dst, const char* src, size_t bytes, int thr) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    const size_t step = bytes / thr;
    for (int i = 0; i < thr; ++i) ts.emplace_back([=] { std::memcpy(dst + i * step, src + i * step, step); });
    for (auto& t : ts) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
    const size_t bytes = size_t(512) << 20;
    char* page = static_cast<char*>(malloc(bytes));
    char* page2 = static_cast<char*>(malloc(bytes));
    memset(page, 1, bytes);
    memset(page2, 2, bytes);
    char *pin = nullptr, *pinwc = nullptr;
    cudaHostAlloc(&pin, bytes, cudaHostAllocPortable);
    cudaHostAlloc(&pinwc, bytes, cudaHostAllocPortable | cudaHostAllocWriteCombined);
    memset(pin, 3, bytes);
    memset(pinwc, 3, bytes);
    for (int thr : {1, 2, 4, 8, 16}) {
        double up = 1e9, down = 1e9, pp = 1e9, upwc = 1e9;
        for (int r = 0; r < 3; ++r) {
            up = std::min(up, run(pin, page, bytes, thr));
            down = std::min(down, run(page2, pin, bytes, thr));
            pp = std::min(pp, run(page2, page, bytes, thr));
            upwc = std::min(upwc, run(pinwc, page, bytes, thr));
        }
        printf("{\"threads\": %d, \"pageable_to_pinned_GBps\": %.1f, \"pinned_to_pageable_GBps\": %.1f, "
               "\"pageable_to_pageable_GBps\": %.1f, \"pageable_to_pinned_wc_GBps\": %.1f}\n",
               thr, bytes / up / 1e9, bytes / down / 1e9, bytes / pp / 1e9, bytes / upwc / 1e9);
    }
    return 0;
}
