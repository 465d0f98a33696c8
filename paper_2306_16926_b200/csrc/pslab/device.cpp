// Caching device allocator of the pslab façade (see device.hpp).
#include "device.hpp"

#include <mutex>
#include <unordered_map>

namespace pslab_b200 {

namespace {

struct Pool {
    std::mutex mu;
    std::unordered_map<size_t, std::vector<void*>> free;  // size class -> blocks
};

Pool& pool() {
    static Pool* p = new Pool();  // never destroyed: blocks live until process exit
    return *p;
}

// Size classes: powers of two up to 2 MiB, then multiples of 2 MiB (whole-model
// vectors of the same layout always land in the same class).
size_t size_class(size_t bytes) {
    constexpr size_t kBig = size_t(2) << 20;
    if (bytes >= kBig) return (bytes + kBig - 1) / kBig * kBig;
    size_t c = 256;
    while (c < bytes) c <<= 1;
    return c;
}

}  // namespace

void* pool_alloc(size_t bytes, size_t* cls) {
    const size_t c = size_class(bytes);
    *cls = c;
    Pool& p = pool();
    {
        std::lock_guard<std::mutex> lk(p.mu);
        auto it = p.free.find(c);
        if (it != p.free.end() && !it->second.empty()) {
            void* b = it->second.back();
            it->second.pop_back();
            return b;
        }
    }
    void* b = nullptr;
    osp_status s = osp_device_alloc(c, &b);
    if (s != OSP_OK) {
        // out of memory with cached blocks around: give them back and retry once
        std::vector<void*> drop;
        {
            std::lock_guard<std::mutex> lk(p.mu);
            for (auto& kv : p.free) drop.insert(drop.end(), kv.second.begin(), kv.second.end());
            p.free.clear();
        }
        for (void* q : drop) osp_device_free(q);
        check(osp_device_alloc(c, &b));
    }
    return b;
}

void pool_free(void* b, size_t cls) {
    if (!b) return;
    Pool& p = pool();
    std::lock_guard<std::mutex> lk(p.mu);
    p.free[cls].push_back(b);
}

}  // namespace pslab_b200
