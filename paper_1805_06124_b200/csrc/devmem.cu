#include <cstdlib>
// devmem.cu -- every device allocation of the library, with optional canaries.
//
// compute-sanitizer is closed on this GPU pool, so out-of-bounds WRITES are caught the cheap
// way: with canaries on (rbg_debug_set_canary), each allocation gets a 256-byte tail filled
// with 0xA5, checked when the buffer is freed and by rbg_debug_canary_violations() for every
// live buffer.  With canaries off, dmalloc / dfree are cudaMalloc / cudaFree.
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "kernels.h"

namespace rbg {
namespace {

constexpr size_t kCanary = 256;
constexpr unsigned char kByte = 0xA5;

struct Registry {
    std::mutex mu;
    std::unordered_map<void *, size_t> live;  // canaried allocations -> user bytes
    bool on = false;
    long long violations = 0;
    std::string first;
};

Registry &reg() {
    static Registry r;
    return r;
}

// true if the tail of p (user size `bytes`) still holds the pattern; syncs the device
bool intact(void *p, size_t bytes) {
    cudaPointerAttributes at;
    int dev0 = 0;
    cudaGetDevice(&dev0);
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice) cudaSetDevice(at.device);
    cudaDeviceSynchronize();
    unsigned char buf[kCanary];
    const bool ok = cudaMemcpy(buf, static_cast<unsigned char *>(p) + bytes, kCanary, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaSetDevice(dev0);
    if (!ok) return false;
    for (size_t i = 0; i < kCanary; i++)
        if (buf[i] != kByte) return false;
    return true;
}

void note(Registry &r, void *p, size_t bytes) {
    if (r.violations++ == 0) {
        char m[160];
        snprintf(m, sizeof m, "write past the end of a %zu-byte device buffer at %p", bytes, p);
        r.first = m;
    }
}

}  // namespace

cudaError_t dmalloc(void **p, size_t bytes) {
    Registry &r = reg();
    std::lock_guard<std::mutex> g(r.mu);
    if (!r.on) return cudaMalloc(p, bytes);
    cudaError_t e = cudaMalloc(p, bytes + kCanary);
    if (e != cudaSuccess) return e;
    e = cudaMemset(static_cast<unsigned char *>(*p) + bytes, kByte, kCanary);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(*p);
        *p = nullptr;
        return e;
    }
    r.live[*p] = bytes;
    return cudaSuccess;
}

cudaError_t dfree(void *p) {
    if (!p) return cudaSuccess;
    Registry &r = reg();
    std::lock_guard<std::mutex> g(r.mu);
    auto it = r.live.find(p);
    if (it != r.live.end()) {
        if (!intact(p, it->second)) note(r, p, it->second);
        r.live.erase(it);
    }
    return cudaFree(p);
}

void debug_set_canary(bool on) {
    Registry &r = reg();
    std::lock_guard<std::mutex> g(r.mu);
    r.on = on;
}

long long debug_canary_violations(std::string *msg) {
    Registry &r = reg();
    std::lock_guard<std::mutex> g(r.mu);
    for (auto &kv : r.live)
        if (!intact(kv.first, kv.second)) note(r, kv.first, kv.second);
    if (msg) *msg = r.first;
    return r.violations;
}

bool scratch_disabled() {
    static const bool off = getenv("RBG_NO_SCRATCH") != nullptr;
    return off;
}

cudaError_t ScratchPool::get(int slot, size_t n, void **out) {
    if (slot < 0 || slot >= kSlots) return cudaErrorInvalidValue;
    if (n == 0) n = 1;
    if (bytes[slot] < n) {
        dfree(p[slot]);
        p[slot] = nullptr;
        bytes[slot] = 0;
        const cudaError_t e = dmalloc(&p[slot], n);
        if (e != cudaSuccess) {
            p[slot] = nullptr;
            *out = nullptr;
            return e;
        }
        bytes[slot] = n;
    }
    *out = p[slot];
    return cudaSuccess;
}

void ScratchPool::release() {
    for (int i = 0; i < kSlots; i++) {
        dfree(p[i]);
        p[i] = nullptr;
        bytes[i] = 0;
    }
}

}  // namespace rbg
