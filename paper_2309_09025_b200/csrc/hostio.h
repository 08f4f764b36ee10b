// hostio.h — the int64 host boundary of the C ABI.
//
// The reference's API moves ciphertexts as numpy int64 arrays (masks A
// (count, n), bodies b (count,); lwe.py:75-96, network.py:372-390).  Copying
// those to the device as int64 from pageable memory costs twice the PCIe bytes
// of the uint32 row format and runs at pageable-copy speed.  Instead the rows
// are packed on the host (mod q, [a_0..a_{n-1}, b, pad]) by a small persistent
// thread pool straight into page-locked staging slots, and each slot is DMA'd
// while the pool packs the next one; the way back is the mirror image (DMA
// into a slot, unpack the previous slot meanwhile).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <sched.h>

namespace fdsnn {

// Fixed pool of worker threads; parallel_for(n, fn) runs fn(i) for i < n and
// returns when all are done.  Calls are serialised (one job at a time).  Idle
// workers spin briefly before sleeping, so the back-to-back jobs of one
// transfer (one per staging slot) do not pay a wake-up each.  Each job is a
// shared object: a worker that picks up a job late only finds its items all
// claimed (it never touches the caller's function after the caller returned).
class HostPool {
  public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    int size() const { return (int)workers_.size() + 1; }

    void parallel_for(int64_t n, const std::function<void(int64_t)>& fn) {
        if (n <= 0) return;
        if (n == 1 || workers_.empty()) {
            for (int64_t i = 0; i < n; ++i) fn(i);
            return;
        }
        std::lock_guard<std::mutex> serial(job_mu_);
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->total = n;
        {
            std::lock_guard<std::mutex> lk(mu_);
            current_ = job;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        run(*job);  // the caller works too
        while (job->done.load(std::memory_order_acquire) != n) std::this_thread::yield();
    }

    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

  private:
    struct Job {
        const std::function<void(int64_t)>* fn = nullptr;
        int64_t total = 0;
        std::atomic<int64_t> next{0}, done{0};
    };

    HostPool() {
        cpu_set_t set;
        int cores = 1;
        if (sched_getaffinity(0, sizeof set, &set) == 0) cores = CPU_COUNT(&set);
        const int nthreads = std::max(1, std::min(cores, 16)) - 1;
        for (int i = 0; i < nthreads; ++i) workers_.emplace_back([this] { loop(); });
    }

    static void run(Job& job) {
        for (int64_t i; (i = job.next.fetch_add(1, std::memory_order_relaxed)) < job.total;) {
            (*job.fn)(i);
            job.done.fetch_add(1, std::memory_order_release);
        }
    }

    void loop() {
        uint64_t seen = 0;
        for (;;) {
            for (int spin = 0; gen_.load(std::memory_order_acquire) == seen && spin < 20000; ++spin)
                std::this_thread::yield();
            std::shared_ptr<Job> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                seen = gen_.load(std::memory_order_acquire);
                if (stop_) return;
                job = current_;
            }
            if (job) run(*job);
        }
    }

    std::vector<std::thread> workers_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_;
    std::shared_ptr<Job> current_;
    std::atomic<uint64_t> gen_{0};
    bool stop_ = false;
};

// Page-locked staging: a ring of NSLOT slots, each guarded by an event
// recorded after the DMA that last used it (so up to NSLOT-1 DMAs are in
// flight while the pool packs / unpacks the next slot).
struct PinnedSlots {
    static constexpr int NSLOT = 4;
    static constexpr size_t SLOT_BYTES = 2u << 20;
    void* slot[NSLOT] = {};
    cudaEvent_t ev[NSLOT] = {};

    cudaError_t ensure() {
        for (int s = 0; s < NSLOT; ++s) {
            if (!slot[s]) {
                cudaError_t e = cudaHostAlloc(&slot[s], SLOT_BYTES, cudaHostAllocPortable);
                if (e != cudaSuccess) return e;
            }
            if (!ev[s]) {
                cudaError_t e = cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming);
                if (e != cudaSuccess) return e;
            }
        }
        return cudaSuccess;
    }
    void release() {
        for (int s = 0; s < NSLOT; ++s) {
            if (ev[s]) cudaEventSynchronize(ev[s]), cudaEventDestroy(ev[s]);
            if (slot[s]) cudaFreeHost(slot[s]);
            ev[s] = nullptr;
            slot[s] = nullptr;
        }
    }
};

// rows [r0, r1) of the int64 (A, b) arrays -> uint32 rows at dst (row r0 first)
inline void pack_rows_host(const int64_t* A, const int64_t* b, int64_t r0, int64_t r1, int n, int stride,
                           uint32_t qmask, uint32_t* dst) {
    HostPool& pool = HostPool::get();
    const int64_t rows = r1 - r0;
    const int64_t per = std::max<int64_t>(64, (rows + pool.size() - 1) / pool.size());
    pool.parallel_for((rows + per - 1) / per, [&](int64_t part) {
        const int64_t lo = r0 + part * per, hi = std::min(r1, lo + per);
        for (int64_t r = lo; r < hi; ++r) {
            const int64_t* a = A + r * n;
            uint32_t* o = dst + (r - r0) * stride;
            for (int c = 0; c < n; ++c) o[c] = (uint32_t)a[c] & qmask;
            o[n] = (uint32_t)b[r] & qmask;
            for (int c = n + 1; c < stride; ++c) o[c] = 0u;
        }
    });
}

// uint32 rows at src (row r0 first) -> int64 (A, b) rows [r0, r1)
inline void unpack_rows_host(const uint32_t* src, int64_t r0, int64_t r1, int n, int stride, int64_t* A,
                             int64_t* b) {
    HostPool& pool = HostPool::get();
    const int64_t rows = r1 - r0;
    const int64_t per = std::max<int64_t>(64, (rows + pool.size() - 1) / pool.size());
    pool.parallel_for((rows + per - 1) / per, [&](int64_t part) {
        const int64_t lo = r0 + part * per, hi = std::min(r1, lo + per);
        for (int64_t r = lo; r < hi; ++r) {
            const uint32_t* s = src + (r - r0) * stride;
            int64_t* a = A + r * n;
            for (int c = 0; c < n; ++c) a[c] = (int64_t)s[c];
            b[r] = (int64_t)s[n];
        }
    });
}

// One host-side source of ciphertexts: `count` rows of int64 (A, b).
struct HostPart {
    const int64_t* A;
    const int64_t* b;
    int64_t count;
};

// int64 host parts (stacked in order) -> device uint32 rows, through the
// pinned slots.  Returns the first CUDA error.  The caller's arrays may be
// reused when it returns (every slot was packed from them before the return).
inline cudaError_t upload_parts(PinnedSlots& ps, const HostPart* parts, int nparts, int n, int stride,
                                uint32_t qmask, uint32_t* d_rows, cudaStream_t s) {
    cudaError_t e = ps.ensure();
    if (e != cudaSuccess) return e;
    const int64_t chunk = std::max<int64_t>(1, (int64_t)(PinnedSlots::SLOT_BYTES / (4 * (size_t)stride)));
    int k = 0;
    int64_t dst_row = 0;
    for (int p = 0; p < nparts; ++p) {
        const HostPart& hp = parts[p];
        for (int64_t r0 = 0; r0 < hp.count; r0 += chunk, k = (k + 1) % PinnedSlots::NSLOT) {
            const int64_t r1 = std::min(hp.count, r0 + chunk);
            if ((e = cudaEventSynchronize(ps.ev[k])) != cudaSuccess) return e;  // slot's last DMA done
            uint32_t* slot = static_cast<uint32_t*>(ps.slot[k]);
            pack_rows_host(hp.A, hp.b, r0, r1, n, stride, qmask, slot);
            if ((e = cudaMemcpyAsync(d_rows + (dst_row + r0) * stride, slot, (size_t)(r1 - r0) * stride * 4,
                                     cudaMemcpyHostToDevice, s)) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(ps.ev[k], s)) != cudaSuccess) return e;
        }
        dst_row += hp.count;
    }
    return cudaSuccess;
}

inline cudaError_t upload_rows(PinnedSlots& ps, const int64_t* A, const int64_t* b, int64_t count, int n,
                               int stride, uint32_t qmask, uint32_t* d_rows, cudaStream_t s) {
    const HostPart part{A, b, count};
    return upload_parts(ps, &part, 1, n, stride, qmask, d_rows, s);
}

// device uint32 rows -> int64 host (A, b); returns after the host arrays are
// complete (the stream's earlier work included).
inline cudaError_t download_rows(PinnedSlots& ps, const uint32_t* d_rows, int64_t count, int n, int stride,
                                 int64_t* A, int64_t* b, cudaStream_t s) {
    cudaError_t e = ps.ensure();
    if (e != cudaSuccess) return e;
    constexpr int NS = PinnedSlots::NSLOT;
    const int64_t chunk = std::max<int64_t>(1, (int64_t)(PinnedSlots::SLOT_BYTES / (4 * (size_t)stride)));
    const int64_t nchunks = (count + chunk - 1) / chunk;
    auto issue = [&](int64_t c) -> cudaError_t {
        const int k = (int)(c % NS);
        const int64_t r0 = c * chunk, r1 = std::min(count, r0 + chunk);
        cudaError_t e2 = cudaEventSynchronize(ps.ev[k]);
        if (e2 != cudaSuccess) return e2;
        e2 = cudaMemcpyAsync(ps.slot[k], d_rows + r0 * stride, (size_t)(r1 - r0) * stride * 4,
                             cudaMemcpyDeviceToHost, s);
        if (e2 != cudaSuccess) return e2;
        return cudaEventRecord(ps.ev[k], s);
    };
    // keep NS-1 chunks in flight ahead of the one being unpacked
    for (int64_t c = 0; c < std::min<int64_t>(nchunks, NS - 1); ++c)
        if ((e = issue(c)) != cudaSuccess) return e;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int k = (int)(c % NS);
        if ((e = cudaEventSynchronize(ps.ev[k])) != cudaSuccess) return e;
        if (c + NS - 1 < nchunks && (e = issue(c + NS - 1)) != cudaSuccess) return e;
        const int64_t r0 = c * chunk, r1 = std::min(count, r0 + chunk);
        unpack_rows_host(static_cast<const uint32_t*>(ps.slot[k]), r0, r1, n, stride, A, b);
    }
    return cudaSuccess;
}

}  // namespace fdsnn
