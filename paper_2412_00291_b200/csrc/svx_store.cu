// K7 and the block store: VMM-backed pools, hash maintenance, batched lookup,
// observed-voxel count, dirty-block compaction (voxel_store.cpp:9-80).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <string>

#include <chrono>

#include "svx_map.hpp"

namespace svx {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(SVX_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

namespace {

// Driver entry points fetched through the runtime, so the library does not
// link libcuda (it loads on hosts without a driver; the GPU box has one).
struct Drv {
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) gran = nullptr;
};

const Drv& drv() {
    static Drv d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            SVX_CUDA(cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q));
            if (q != cudaDriverEntryPointSuccess)
                throw Error(SVX_CUDA, std::string("driver entry point missing: ") + name);
        };
        get("cuMemAddressReserve", reinterpret_cast<void**>(&d.reserve));
        get("cuMemAddressFree", reinterpret_cast<void**>(&d.addr_free));
        get("cuMemCreate", reinterpret_cast<void**>(&d.create));
        get("cuMemRelease", reinterpret_cast<void**>(&d.release));
        get("cuMemMap", reinterpret_cast<void**>(&d.map));
        get("cuMemUnmap", reinterpret_cast<void**>(&d.unmap));
        get("cuMemSetAccess", reinterpret_cast<void**>(&d.set_access));
        get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&d.gran));
    });
    return d;
}

void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw Error(SVX_CUDA, std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")");
}

CUmemAllocationProp prop_for(int device) {
    CUmemAllocationProp p{};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    return p;
}

}  // namespace

void VmmArray::reserve(int device, size_t max_bytes) {
    device_ = device;
    const CUmemAllocationProp p = prop_for(device);
    cu_check(drv().gran(&gran_, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    reserved_ = ((max_bytes + gran_ - 1) / gran_) * gran_;
    if (reserved_ == 0) reserved_ = gran_;
    cu_check(drv().reserve(&base_, reserved_, gran_, 0, 0), "cuMemAddressReserve");
}

// Maps [mapped_, >= bytes) in chunks of at most kVmmChunk, publishing each chunk
// as soon as it is mapped (a waiting ensure() can proceed early).
static constexpr size_t kVmmChunk = size_t(256) << 20;

void VmmArray::grow(size_t bytes) {
    size_t cur = mapped_.load(std::memory_order_relaxed);
    if (bytes <= cur) return;
    if (bytes > reserved_) throw Error(SVX_CAPACITY, "device pool reservation exceeded");
    // grow by >= 1/4 of the mapped size: keeps the number of mappings logarithmic
    size_t want = std::max(bytes, cur + cur / 4);
    want = ((want + gran_ - 1) / gran_) * gran_;
    if (want > reserved_) want = reserved_;
    const CUmemAllocationProp p = prop_for(device_);
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device_;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    while (cur < want) {
        const size_t add = std::min(want - cur, std::max(kVmmChunk, gran_));
        CUmemGenericAllocationHandle h;
        cu_check(drv().create(&h, add, &p, 0), "cuMemCreate");
        cu_check(drv().map(base_ + cur, add, 0, h, 0), "cuMemMap");
        cu_check(drv().set_access(base_ + cur, add, &acc, 1), "cuMemSetAccess");
        chunks_.push_back({h, add});
        cur += add;
        mapped_.store(cur, std::memory_order_release);
    }
}

void VmmArray::join() {
    if (worker_.joinable()) worker_.join();
    if (worker_err_) {
        std::exception_ptr e = worker_err_;
        worker_err_ = nullptr;
        std::rethrow_exception(e);
    }
}

void VmmArray::ensure(size_t bytes) {
    if (bytes <= mapped()) return;
    // a background growth may already cover it: wait for its chunks, not its end
    while (worker_.joinable() && !worker_done_.load(std::memory_order_acquire) && mapped() < bytes)
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    if (bytes <= mapped()) return;
    join();
    grow(bytes);
}

void VmmArray::prefetch(size_t bytes) {
    if (bytes > reserved_) bytes = reserved_;
    if (worker_.joinable()) {
        if (!worker_done_.load(std::memory_order_acquire)) return;  // still mapping
        join();
    }
    if (bytes <= mapped()) return;
    worker_done_.store(false, std::memory_order_relaxed);
    worker_ = std::thread([this, bytes] {
        try {
            cudaSetDevice(device_);  // primary context current on this thread
            grow(bytes);
        } catch (...) {
            worker_err_ = std::current_exception();
        }
        worker_done_.store(true, std::memory_order_release);
    });
}

VmmArray::~VmmArray() {
    if (worker_.joinable()) worker_.join();
    if (!base_) return;
    cudaDeviceSynchronize();
    size_t off = 0;
    for (auto& [h, sz] : chunks_) {
        drv().unmap(base_ + off, sz);
        drv().release(h);
        off += sz;
    }
    drv().addr_free(base_, reserved_);
}

// Maps TSDF pool and visit-mask memory (svx_tsdf.cu) for `blocks` blocks now and `ahead`
// more in the background. C_MAPPED (what kernels may allocate into) counts blocks whose
// pool and zero-filled masks are both mapped; the mask zero-fill is stream-ordered before
// the new count is published.
void ensure_blocks(svx_map* m, uint64_t blocks, uint64_t ahead) {
    if (blocks > m->cfg.max_blocks) blocks = m->cfg.max_blocks;
    const uint64_t mask_bytes = 4ull * kMaskWords;
    if (blocks * m->block_bytes > m->tsdf_pool.mapped() || blocks * mask_bytes > m->mask_pool.mapped()) {
        const auto t0 = std::chrono::steady_clock::now();
        m->tsdf_pool.ensure(blocks * m->block_bytes);
        m->mask_pool.ensure(blocks * mask_bytes);
        m->prof_acc.host_map_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    // keep the next growth off the critical path: map ahead in the background
    const uint64_t target = std::min<uint64_t>(m->cfg.max_blocks, blocks + ahead);
    m->tsdf_pool.prefetch(target * m->block_bytes);
    m->mask_pool.prefetch(target * mask_bytes);
    // a map with semantic layers needs a layer for every block a label pass may reach (the
    // label passes map up to the mapped block count): keep the layers' mapping in step, in
    // the background too
    if (m->n_layers) m->sem_pool.prefetch(target * m->layer_bytes);
    const uint64_t mapped = std::min<uint64_t>(
        std::min<uint64_t>(m->tsdf_pool.mapped() / m->block_bytes, m->mask_pool.mapped() / mask_bytes),
        m->cfg.max_blocks);
    if (mapped > m->mask_zeroed) {
        SVX_CUDA(cudaMemsetAsync(mask_base(m) + m->mask_zeroed * kMaskWords, 0,
                                 (mapped - m->mask_zeroed) * mask_bytes, m->stream));
        m->mask_zeroed = mapped;
    }
    if (mapped != m->mapped_blocks) {
        m->mapped_blocks = mapped;
        m->h_ctr[C_MAPPED] = uint32_t(mapped);
        SVX_CUDA(cudaMemcpyAsync(m->d_ctr + C_MAPPED, &m->h_ctr[C_MAPPED], 4,
                                 cudaMemcpyHostToDevice, m->stream));
    }
}

void push_block_counters(svx_map* m) {
    m->h_ctr[C_BLOCKS] = m->h_ctr[C_BLOCKS_BEFORE] = uint32_t(m->n_blocks);
    m->h_ctr[C_SEM] = uint32_t(m->n_layers);
    m->h_ctr[C_MAPPED] = uint32_t(m->mapped_blocks);
    for (int c : {C_BLOCKS, C_SEM, C_BLOCKS_BEFORE, C_MAPPED})
        SVX_CUDA(cudaMemcpyAsync(m->d_ctr + c, &m->h_ctr[c], 4, cudaMemcpyHostToDevice, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
}

void ensure_layers(svx_map* m, uint64_t layers) {
    if (layers > m->cfg.max_blocks) layers = m->cfg.max_blocks;
    if (layers * m->layer_bytes > m->sem_pool.mapped()) {
        const auto t0 = std::chrono::steady_clock::now();
        m->sem_pool.ensure(layers * m->layer_bytes);
        m->prof_acc.host_map_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    m->sem_pool.prefetch(std::min<uint64_t>(m->cfg.max_blocks, layers + layers / 2) * m->layer_bytes);
}

void sync_counters(svx_map* m) {
    SVX_CUDA(cudaMemcpyAsync(m->h_ctr, m->d_ctr, sizeof(uint32_t) * kNumCounters,
                             cudaMemcpyDeviceToHost, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    if (m->prof) prof_resolve(m);
}

namespace {
cudaEvent_t take_event(svx_map* m) {
    if (!m->prof_free.empty()) {
        cudaEvent_t e = m->prof_free.back();
        m->prof_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    SVX_CUDA(cudaEventCreate(&e));
    return e;
}
}  // namespace

ProfMark::ProfMark(svx_map* map, int k, int n_launches) : m(map), kid(k), launches(n_launches) {
    if (!m->prof || !((m->prof_mask >> k) & 1u)) return;
    a = take_event(m);
    SVX_CUDA(cudaEventRecord(a, m->stream));
}

ProfMark::~ProfMark() {
    if (!a) return;
    cudaEvent_t b = take_event(m);
    cudaEventRecord(b, m->stream);
    m->prof_pending.push_back({kid, a, b});
    m->prof_acc.launches[kid] += uint64_t(launches);
}

void prof_resolve(svx_map* m) {
    for (auto& p : m->prof_pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.b);
        cudaEventElapsedTime(&ms, p.a, p.b);
        m->prof_acc.ms[p.kid] += ms;
        m->prof_free.push_back(p.a);
        m->prof_free.push_back(p.b);
    }
    m->prof_pending.clear();
}

namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(uint64_t n) { return unsigned((n + kThreads - 1) / kThreads); }

__global__ void k_rebuild(HashView h, const uint64_t* __restrict__ block_keys, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int ins = 0;
    const uint32_t s = hash_insert(h, block_keys[i], &ins);
    if (s != kInvalid) h.vals[s] = i;
}

__global__ void k_count_observed(const svx_tsdf_voxel* __restrict__ pool, uint64_t n_vox,
                                 unsigned long long* __restrict__ out) {
    uint32_t c = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_vox;
         i += uint64_t(gridDim.x) * blockDim.x)
        c += pool[i].weight > 0.f ? 1u : 0u;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, static_cast<unsigned long long>(c));
}

__global__ void k_find(HashView h, const uint64_t* __restrict__ q, uint32_t n,
                       uint32_t* __restrict__ idx) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = hash_find(h, q[i]);
    idx[i] = s == kInvalid ? kInvalid : h.vals[s];
}

__global__ void k_insert_one(HashView h, uint64_t key, uint64_t* __restrict__ block_keys,
                             uint32_t* __restrict__ ctr, uint32_t* __restrict__ out) {
    int ins = 0;
    const uint32_t s = hash_insert(h, key, &ins);
    if (s == kInvalid) {
        *out = kInvalid;
        return;
    }
    if (ins) {
        const uint32_t idx = ctr[C_BLOCKS]++;
        h.vals[s] = idx;
        block_keys[idx] = key;
    }
    *out = h.vals[s];
}

__global__ void k_lookup(HashView h, const int32_t* __restrict__ v, uint64_t n,
                         const svx_tsdf_voxel* __restrict__ pool, const float* __restrict__ sem,
                         const uint32_t* __restrict__ sem_idx, int K,
                         svx_tsdf_voxel* __restrict__ out, float* __restrict__ probs,
                         uint8_t* __restrict__ found) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t x = v[3 * i], y = v[3 * i + 1], z = v[3 * i + 2];
    const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
    uint32_t s = kInvalid;
    if (key_in_range(bx) && key_in_range(by) && key_in_range(bz)) s = hash_find(h, pack_key(bx, by, bz));
    if (s == kInvalid) {
        found[i] = 0;
        return;
    }
    found[i] = 1;
    const uint32_t idx = h.vals[s];
    const int lin = local_linear(x, y, z);
    out[i] = pool[uint64_t(idx) * kBlockVoxels + lin];
    if (probs) {
        const uint32_t sid = sem_idx[idx];
        for (int k = 0; k < K; ++k)
            probs[i * K + k] = sid == kInvalid ? 1.f / float(K)
                                               : sem[(uint64_t(sid) * kBlockVoxels + lin) * K + k];
    }
}

__global__ void k_fill_layer(float* __restrict__ layer, uint64_t n, float v) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        layer[i] = v;
}

// One CTA per requested block: 16-byte copies of the TSDF body (10240 B) and,
// when the block has a semantic layer, of its 512*K floats.
__global__ void k_gather_blocks(const uint4* __restrict__ pool, const float* __restrict__ sem_pool,
                                const uint32_t* __restrict__ sem_idx,
                                const uint32_t* __restrict__ idx, uint64_t n, int K,
                                uint4* __restrict__ out, float* __restrict__ sem_out,
                                uint8_t* __restrict__ has_sem) {
    constexpr int kVec = kBlockVoxels * int(sizeof(svx_tsdf_voxel)) / 16;  // 640
    for (uint64_t b = blockIdx.x; b < n; b += gridDim.x) {
        const uint32_t i = idx[b];
        const uint4* src = pool + uint64_t(i) * kVec;
        uint4* dst = out + b * kVec;
        for (int t = threadIdx.x; t < kVec; t += blockDim.x) dst[t] = src[t];
        if (!sem_out) continue;
        const uint32_t s = sem_idx[i];
        if (threadIdx.x == 0) has_sem[b] = s != kInvalid;
        if (s == kInvalid) continue;
        const uint64_t nf = uint64_t(kBlockVoxels) * K;
        const float* ss = sem_pool + uint64_t(s) * nf;
        float* sd = sem_out + b * nf;
        for (uint64_t t = threadIdx.x; t < nf; t += blockDim.x) sd[t] = ss[t];
    }
}

}  // namespace

void gather_blocks(svx_map* m, const uint32_t* d_idx, uint64_t n, svx_tsdf_voxel* d_out,
                   float* d_sem, uint8_t* d_has_sem) {
    if (!n) return;
    k_gather_blocks<<<unsigned(std::min<uint64_t>(n, 148 * 8)), kThreads, 0, m->stream>>>(
        reinterpret_cast<const uint4*>(tsdf_base(m)), sem_base(m), m->sem_idx, d_idx, n,
        m->cfg.num_labels, reinterpret_cast<uint4*>(d_out), d_sem, d_has_sem);
    count_launch();
    SVX_CUDA(cudaGetLastError());
}

void rebuild_hash(svx_map* m) {
    SVX_CUDA(cudaMemsetAsync(m->keys, 0xFF, sizeof(uint64_t) * m->cap, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->vals, 0xFF, sizeof(uint32_t) * m->cap, m->stream));
    if (m->n_blocks)
        k_rebuild<<<grid_for(m->n_blocks), kThreads, 0, m->stream>>>(hash_view(m), m->block_keys,
                                                                     uint32_t(m->n_blocks));
    count_launch();
    SVX_CUDA(cudaGetLastError());
}

void launch_zero_blocks(svx_map* m, uint64_t first, uint64_t count) {
    if (!count) return;
    SVX_CUDA(cudaMemsetAsync(tsdf_base(m) + first * kBlockVoxels, 0, count * m->block_bytes,
                             m->stream));
}

uint64_t count_observed(svx_map* m) {
    DevBuf<unsigned long long> acc;
    acc.alloc(1);
    SVX_CUDA(cudaMemsetAsync(acc.p, 0, 8, m->stream));
    const uint64_t nv = m->n_blocks * kBlockVoxels;
    if (nv)
        k_count_observed<<<std::min<unsigned>(grid_for(nv), 148 * 16), kThreads, 0, m->stream>>>(
            tsdf_base(m), nv, acc.p);
    count_launch();
    unsigned long long h = 0;
    SVX_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    acc.release();
    return h;
}

// Pool indices of the given packed keys (kInvalid when absent).
void find_blocks(svx_map* m, const uint64_t* h_keys, uint32_t n, uint32_t* h_idx) {
    if (!n) return;
    m->q_keys.alloc(std::max<uint32_t>(n, 64));
    m->q_idx.alloc(std::max<uint32_t>(n, 64));
    SVX_CUDA(cudaMemcpyAsync(m->q_keys.p, h_keys, 8ull * n, cudaMemcpyHostToDevice, m->stream));
    k_find<<<grid_for(n), kThreads, 0, m->stream>>>(hash_view(m), m->q_keys.p, n, m->q_idx.p);
    count_launch();
    SVX_CUDA(cudaMemcpyAsync(h_idx, m->q_idx.p, 4ull * n, cudaMemcpyDeviceToHost, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
}

// get_or_allocate_block (voxel_store.cpp:9-23). Returns the pool index.
uint32_t get_or_alloc_block(svx_map* m, uint64_t key, bool* was_new) {
    uint32_t idx = kInvalid;
    find_blocks(m, &key, 1, &idx);
    if (was_new) *was_new = false;
    if (idx != kInvalid) return idx;
    if (m->n_blocks >= m->cfg.max_blocks)
        throw Error(SVX_CAPACITY,
                    "block budget exhausted (max_blocks = " + std::to_string(m->cfg.max_blocks) + ")");
    ensure_blocks(m, m->n_blocks + 1);
    m->q_idx.alloc(64);
    k_insert_one<<<1, 1, 0, m->stream>>>(hash_view(m), key, m->block_keys, m->d_ctr, m->q_idx.p);
    count_launch();
    SVX_CUDA(cudaMemcpyAsync(&idx, m->q_idx.p, 4, cudaMemcpyDeviceToHost, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    if (idx == kInvalid) throw Error(SVX_CAPACITY, "block hash table full");
    launch_zero_blocks(m, idx, 1);
    m->n_blocks = uint64_t(idx) + 1;
    push_block_counters(m);
    if (was_new) *was_new = true;
    return idx;
}

// Ensures a semantic layer exists for pool block idx (VoxelBlock::ensure_semantics).
uint32_t ensure_layer(svx_map* m, uint32_t idx) {
    uint32_t sid = kInvalid;
    SVX_CUDA(cudaMemcpyAsync(&sid, m->sem_idx + idx, 4, cudaMemcpyDeviceToHost, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    if (sid != kInvalid) return sid;
    sid = uint32_t(m->n_layers);
    ensure_layers(m, m->n_layers + 1);
    const int K = m->cfg.num_labels;
    const uint64_t nf = uint64_t(kBlockVoxels) * K;
    k_fill_layer<<<64, kThreads, 0, m->stream>>>(sem_base(m) + uint64_t(sid) * nf, nf, 1.f / float(K));
    count_launch();
    SVX_CUDA(cudaMemcpyAsync(m->sem_idx + idx, &sid, 4, cudaMemcpyHostToDevice, m->stream));
    m->n_layers++;
    m->h_ctr[C_SEM] = uint32_t(m->n_layers);
    SVX_CUDA(cudaMemcpyAsync(m->d_ctr + C_SEM, &m->h_ctr[C_SEM], 4, cudaMemcpyHostToDevice, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    return sid;
}

void lookup_voxels(svx_map* m, const int32_t* d_v, uint64_t n, svx_tsdf_voxel* d_out,
                   float* d_probs, uint8_t* d_found) {
    if (!n) return;
    k_lookup<<<grid_for(n), kThreads, 0, m->stream>>>(hash_view(m), d_v, n, tsdf_base(m),
                                                      sem_base(m), m->sem_idx, m->cfg.num_labels,
                                                      d_out, d_probs, d_found);
    count_launch();
    SVX_CUDA(cudaGetLastError());
}

}  // namespace svx
