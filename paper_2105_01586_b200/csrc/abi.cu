// abi.cu -- the extern "C" boundary of libfemi (include/femi.h). Argument checking, handle
// life cycle, uploads; every compute step is one of the kernels in the other .cu files.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "device.cuh"

namespace femi {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }

femi_status cuda_fail(cudaError_t e, const char* what) {
    set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? FEMI_E_OOM : FEMI_E_CUDA;
}

namespace {

// Device memory of a system: arrays up to 2 MB are carved (256-byte aligned) from 8 MB arena
// chunks, larger ones get their own allocation; all of it from the stream-ordered pool on the
// assembling stream (S->ast), released with cudaFreeAsync -- no device-wide synchronisation
// per allocation or free.
constexpr size_t kArenaChunk = 8u << 20, kArenaMax = 2u << 20;
femi_status dev_alloc(femi_system_s* S, void** p, size_t bytes) {
    bytes = (std::max<size_t>(bytes, 1) + 255) & ~(size_t)255;
    if (bytes > kArenaMax) {
        FEMI_CUDA(cudaMallocAsync(p, bytes, S->ast));
        S->allocs.push_back(*p);
        return FEMI_OK;
    }
    if (S->arena_left < bytes) {
        void* c = nullptr;
        FEMI_CUDA(cudaMallocAsync(&c, kArenaChunk, S->ast));
        S->arena_chunks.push_back(c);  // never in allocs: carved temporaries are not freed early
        S->arena_cur = (char*)c;
        S->arena_left = kArenaChunk;
    }
    *p = S->arena_cur;
    S->arena_cur += bytes;
    S->arena_left -= bytes;
    return FEMI_OK;
}

// Pinned staging of the assemble uploads: a host array is copied into one pinned buffer and
// sent with an asynchronous copy; a pageable cudaMemcpyAsync stages and waits on its own
// (tens of us per call, ~25 calls per assemble -- a C3 densification step's tables are small).
// One assemble at a time holds the buffer (others, and arrays that do not fit, go pageable);
// the holder synchronises its stream before releasing it.
struct PinnedStage {
    std::mutex m;
    char* buf = nullptr;
    size_t cap = 0, used = 0;
};
PinnedStage g_stage;
thread_local PinnedStage* t_stage = nullptr;
constexpr size_t kStageBytes = 32u << 20;

struct StageHold {
    std::unique_lock<std::mutex> lk;
    cudaStream_t st;
    explicit StageHold(cudaStream_t s) : lk(g_stage.m, std::try_to_lock), st(s) {
        if (!lk.owns_lock()) return;
        if (!g_stage.buf) {
            void* b = nullptr;
            if (cudaHostAlloc(&b, kStageBytes, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
            g_stage.buf = (char*)b;
            g_stage.cap = kStageBytes;
        }
        g_stage.used = 0;
        t_stage = &g_stage;
    }
    ~StageHold() {
        if (t_stage) cudaStreamSynchronize(st);  // the copies have read the buffer
        t_stage = nullptr;
    }
};

femi_status h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return FEMI_OK;
    if (t_stage && bytes <= t_stage->cap - t_stage->used) {
        char* h = t_stage->buf + t_stage->used;
        std::memcpy(h, src, bytes);
        t_stage->used += (bytes + 255) & ~(size_t)255;
        FEMI_CUDA(cudaMemcpyAsync(dst, h, bytes, cudaMemcpyHostToDevice, st));
        return FEMI_OK;
    }
    FEMI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return FEMI_OK;
}

template <class T>
femi_status upload(femi_system_s* S, T** dst, const std::vector<T>& src, cudaStream_t st, size_t extra = 0) {
    size_t n = src.size() + extra;
    void* p = nullptr;
    femi_status s = dev_alloc(S, &p, sizeof(T) * std::max<size_t>(n, 1));
    if (s) return s;
    if ((s = h2d(p, src.data(), sizeof(T) * src.size(), st))) return s;
    *dst = (T*)p;
    return FEMI_OK;
}

template <class T>
femi_status alloc(femi_system_s* S, T** dst, size_t n) {
    void* p = nullptr;
    femi_status s = dev_alloc(S, &p, sizeof(T) * std::max<size_t>(n, 1));
    if (s) return s;
    *dst = (T*)p;
    return FEMI_OK;
}

femi_status check_device() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    static int checked_dev = -1;  // cudaGetDeviceProperties is slow (ms): query two attributes once
    if (checked_dev == dev) return FEMI_OK;
    int major = 0, minor = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    if (major != 10 || minor != 0) {
        set_error("libfemi is built for sm_100a (B200); current device is sm_" + std::to_string(major) +
                  std::to_string(minor));
        return FEMI_E_CUDA;
    }
    checked_dev = dev;
    static bool pool_set = false;
    if (!pool_set) {  // keep stream-ordered scratch cached between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_set = true;
    }
    return FEMI_OK;
}

}  // namespace
}  // namespace femi

using namespace femi;

namespace femi {
namespace {
// A femi_system may be shared across host threads and streams. Calls that use it are
// serialised: host side by the system's mutex (systems locked in address order, a system
// repeated in a batch once), device side by the system's event -- the call's stream waits for
// the work of the previous call on the system when that ran on another stream, and the event is
// recorded after this call's work. The cached scratch of a system (graph caches, halo tables,
// solve workspace) is therefore never used by two calls at once.
class SysGuard {
  public:
    SysGuard(femi_system_s* const* S, int B, cudaStream_t st) : st_(st) {
        for (int b = 0; b < B; ++b)
            if (S[b]) v_.push_back(S[b]);
        std::sort(v_.begin(), v_.end());
        v_.erase(std::unique(v_.begin(), v_.end()), v_.end());
        for (femi_system_s* s : v_) s->mu.lock();
        for (femi_system_s* s : v_)
            if (s->ev && s->ev_stream != st_) cudaStreamWaitEvent(st_, s->ev, 0);
    }
    ~SysGuard() {
        for (femi_system_s* s : v_) {
            if (!s->ev) cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming);
            if (s->ev) cudaEventRecord(s->ev, st_);
            s->ev_stream = st_;
        }
        for (auto it = v_.rbegin(); it != v_.rend(); ++it) (*it)->mu.unlock();
    }
    SysGuard(const SysGuard&) = delete;
    SysGuard& operator=(const SysGuard&) = delete;

  private:
    cudaStream_t st_;
    std::vector<femi_system_s*> v_;
};
}  // namespace
}  // namespace femi
using femi::SysGuard;

extern "C" {

const char* femi_last_error(void) { return g_last_error.c_str(); }

const char* femi_version(void) { return "femi-b200 0.1 (sm_100a)"; }

int64_t femi_kernel_launches(void) { return g_launches.load(); }

femi_status femi_mesh_build(int32_t W, int32_t H, const int32_t* mask_px, int64_t m, const int32_t* unknown_px,
                            int64_t p, femi_mesh* out) {
    if (!out) {
        set_error("mesh_build: out is NULL");
        return FEMI_E_ARG;
    }
    *out = nullptr;
    femi_mesh_s* h = new (std::nothrow) femi_mesh_s();
    if (!h) return FEMI_E_OOM;
    femi_status s;
    try {
        s = build_mesh(W, H, mask_px, m, unknown_px, p, h->mesh);
    } catch (const std::bad_alloc&) {
        set_error("mesh_build: host allocation failed");
        s = FEMI_E_OOM;
    } catch (...) {
        set_error("mesh_build: internal error");
        s = FEMI_E_ARG;
    }
    if (s != FEMI_OK) {
        delete h;
        return s;
    }
    *out = h;
    return FEMI_OK;
}

femi_status femi_mesh_insert(femi_mesh prev, const int32_t* new_mask_px, int64_t b, femi_mesh* out) {
    if (!prev || !out) {
        set_error("mesh_insert: NULL argument");
        return FEMI_E_ARG;
    }
    *out = nullptr;
    femi_mesh_s* h = new (std::nothrow) femi_mesh_s();
    if (!h) return FEMI_E_OOM;
    femi_status s;
    try {
        s = insert_mesh(prev->mesh, new_mask_px, b, h->mesh);
    } catch (const std::bad_alloc&) {
        set_error("mesh_insert: host allocation failed");
        s = FEMI_E_OOM;
    } catch (...) {
        set_error("mesh_insert: internal error");
        s = FEMI_E_ARG;
    }
    if (s != FEMI_OK) {
        delete h;
        return s;
    }
    *out = h;
    return FEMI_OK;
}

femi_status femi_mesh_info_get(femi_mesh mesh, femi_mesh_info* info) {
    if (!mesh || !info) {
        set_error("mesh_info_get: NULL argument");
        return FEMI_E_ARG;
    }
    const Mesh& M = mesh->mesh;
    info->width = M.W;
    info->height = M.H;
    info->n_vert = M.nv;
    info->n_unknown = M.n_u;
    info->n_mask = M.m;
    info->n_tri = M.T;
    info->nnz_uu = (int64_t)M.uu_col.size();
    info->nnz_uk = (int64_t)M.uk_col.size();
    return FEMI_OK;
}

femi_status femi_mesh_export(femi_mesh mesh, int32_t* vert_px, int32_t* tri_vert, int32_t* uu_rowptr, int32_t* uu_col,
                             int32_t* uk_rowptr, int32_t* uk_col) {
    if (!mesh) {
        set_error("mesh_export: NULL mesh");
        return FEMI_E_ARG;
    }
    const Mesh& M = mesh->mesh;
    auto cp = [](int32_t* dst, const std::vector<int32_t>& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(int32_t) * v.size());
    };
    cp(vert_px, M.vpix);
    cp(tri_vert, M.tri);
    cp(uu_rowptr, M.uu_rowptr);
    cp(uu_col, M.uu_col);
    cp(uk_rowptr, M.uk_rowptr);
    cp(uk_col, M.uk_col);
    return FEMI_OK;
}

femi_status femi_mesh_timing(femi_mesh mesh, double* seconds, int32_t* threads) {
    if (!mesh) return FEMI_E_ARG;
    if (seconds) *seconds = mesh->mesh.build_seconds;
    if (threads) *threads = mesh->mesh.threads;
    return FEMI_OK;
}

void femi_mesh_free(femi_mesh mesh) { delete mesh; }

void femi_system_free(femi_system sys) {
    if (!sys) return;
    cudaDeviceSynchronize();  // no work of any stream may still read the system
    pcg_cache_free(sys);
    if (sys->ev) cudaEventDestroy(sys->ev);
    for (void* p : sys->allocs) cudaFreeAsync(p, nullptr);
    for (void* p : sys->arena_chunks) cudaFreeAsync(p, nullptr);
    delete sys;
}

femi_status femi_assemble(femi_mesh mesh, femi_stream stream, femi_system* out) {
    if (!mesh || !out) {
        set_error("assemble: NULL argument");
        return FEMI_E_ARG;
    }
    *out = nullptr;
    femi_status s = check_device();
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const Mesh& M = mesh->mesh;
    // FEMI_ASM_PROF=1: stage stamps after a stream synchronisation (host + device time);
    // FEMI_ASM_PROF=2: without it (host time of each stage only)
    const char* prof_env = std::getenv("FEMI_ASM_PROF");
    const bool prof = prof_env != nullptr, prof_sync = prof && std::atoi(prof_env) != 2;
    const auto t_start = std::chrono::steady_clock::now();
    auto stamp = [&](const char* what) {
        if (!prof) return;
        if (prof_sync) cudaStreamSynchronize(st);
        std::fprintf(stderr, "assemble %-10s %.3f ms\n", what,
                     1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
    };
    StageHold stage_hold(st);
    femi_system_s* S = new (std::nothrow) femi_system_s();
    if (!S) return FEMI_E_OOM;
    S->ast = st;
    S->W = M.W;
    S->H = M.H;
    S->n_u = M.n_u;
    S->m = M.m;
    S->nv = M.nv;
    S->T = M.T;
    S->nnz_uu = (int64_t)M.uu_col.size();
    S->nnz_uk = (int64_t)M.uk_col.size();
    int32_t* d_tri = nullptr;
    uint32_t* d_flags = nullptr;
#define U(x)                              \
    do {                                  \
        s = (x);                          \
        if (s != FEMI_OK) goto fail;      \
    } while (0)
    U(upload(S, &S->vpix, M.vpix, st));
    U(upload(S, &d_tri, M.tri, st));
    U(upload(S, &d_flags, M.flags, st));
    U(alloc(S, &S->tri, (size_t)M.T));
    U(upload(S, &S->vt_ptr, M.vt_ptr, st));
    U(upload(S, &S->vt_idx, M.vt_idx, st));
    U(upload(S, &S->uu_rowptr, M.uu_rowptr, st));
    U(upload(S, &S->uu_col, M.uu_col, st));
    U(upload(S, &S->uu_opp, M.uu_opp, st));
    U(alloc(S, &S->uu_val, M.uu_col.size()));
    U(upload(S, &S->uk_rowptr, M.uk_rowptr, st));
    U(upload(S, &S->uk_col, M.uk_col, st));
    U(upload(S, &S->uk_opp, M.uk_opp, st));
    U(alloc(S, &S->uk_val, M.uk_col.size()));
    U(upload(S, &S->ku_rowptr, M.ku_rowptr, st));
    U(upload(S, &S->ku_src, M.ku_src, st));
    U(upload(S, &S->ku_row, M.ku_row, st));
    U(alloc(S, &S->o_rowptr, (size_t)M.n_u + 1));
    U(alloc(S, &S->o_col, M.uu_col.size() - M.n_u));
    U(alloc(S, &S->o_val, M.uu_col.size() - M.n_u));
    U(alloc(S, &S->s, (size_t)M.n_u));
    stamp("uploads");
    {
        // Solver numbering + SELL-32-sigma layout of the off-diagonal pattern (values are
        // filled on the device after assembly). Internal order: unknowns sorted by
        // (y / kBand, x, y) -- 32 consecutive internal rows form a compact 2-D blob, so
        // row data is contiguous and gathered neighbours sit in few cache lines -- then
        // rows sorted by length (descending, stable) inside windows of kSellSigma.
        const int64_t n = M.n_u;
        const int SIG = kSellSigma;
        S->nwin = (int32_t)((n + SIG - 1) / SIG);
        const int32_t* rp = M.uu_rowptr.data();
        const int32_t* uc = M.uu_col.data();
        auto rl = [rp](int32_t i) { return rp[i + 1] - rp[i] - 1; };
        // position of the diagonal inside each row: the k-th off-diagonal entry of a row is
        // rp[row] + k + (k >= dpos[row])
        std::vector<int32_t> dpos(n);
        parallel_ranges(n, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) {
                int32_t e = rp[i];
                while (uc[e] != (int32_t)i) ++e;
                dpos[i] = e - rp[i];
            }
        });
        stamp("order.dpos");
        auto kth = [&](int32_t row, int32_t k) { return rp[row] + k + (k >= dpos[row] ? 1 : 0); };
        std::vector<int32_t> pi(n), pos(n);
        stamp("order.alloc");
        {
            // unknowns are numbered in ascending pix (row-major) order, so every band of
            // image rows is a contiguous run of them; inside a band sort by (x, y)
            // graph-mode (JDS) systems use taller bands: a 512-row tile is then ~64 x 400 px and
            // ~3/4 of its neighbour gathers hit the tile's own r slice in shared memory
            // (measured at C5: band 32 -> 64 with in-tile gathers, solve 3.95 -> 3.92 ms)
            int64_t band = S->nnz_uu > kGraphNnz ? kBandJds : kBand;
            if (const char* e = std::getenv("FEMI_BAND")) band = std::max(1, std::atoi(e));
            const int64_t nb = (M.H + band - 1) / band;
            std::vector<int64_t> bs(nb + 1);
            for (int64_t q = 0; q <= nb; ++q)
                bs[q] = std::lower_bound(M.vpix.begin(), M.vpix.begin() + n, std::min<int64_t>(q * band, M.H) * M.W) -
                        M.vpix.begin();
            const int32_t* vp = M.vpix.data();
            const int64_t W = M.W;
            // (x, y) order inside a band = a stable counting sort by x of the band's unknowns
            // (they are in ascending pix order, i.e. ascending y within one x): O(n + W) per
            // band, no comparison sort (a comparison sort of random keys costs ~5 ns per
            // mispredicted comparison: ~1 ms per C3-size assemble)
            // x without a division per element (a 64-bit divide is ~40-90 cycles on the host):
            // the band's unknowns ascend in pix, so the row start advances monotonically
            parallel_ranges(nb, [&](int64_t lo, int64_t hi) {
                std::vector<int32_t> cnt(W + 1), xs;
                for (int64_t q = lo; q < hi; ++q) {
                    std::fill(cnt.begin(), cnt.end(), 0);
                    xs.resize(bs[q + 1] - bs[q]);
                    int64_t row0 = std::min<int64_t>(q * band, M.H) * W;
                    for (int64_t i = bs[q]; i < bs[q + 1]; ++i) {
                        while (vp[i] >= row0 + W) row0 += W;
                        const int32_t x = (int32_t)(vp[i] - row0);
                        xs[i - bs[q]] = x;
                        ++cnt[x + 1];
                    }
                    for (int64_t x = 0; x < W; ++x) cnt[x + 1] += cnt[x];
                    for (int64_t i = bs[q]; i < bs[q + 1]; ++i) pi[bs[q] + cnt[xs[i - bs[q]]]++] = (int32_t)i;
                }
            }, n > 65536 ? 1 : (int64_t)nb);
        }
        stamp("order");
        // rows by length, descending and stable, inside each window: a counting sort on the
        // (small) row lengths
        parallel_ranges(S->nwin, [&](int64_t lo, int64_t hi) {
            int32_t tmp[SIG];
            std::vector<int32_t> cnt;
            for (int64_t w = lo; w < hi; ++w) {
                const int64_t a = w * SIG, b = std::min<int64_t>(n, (w + 1) * SIG);
                int32_t L = 0;
                for (int64_t i = a; i < b; ++i) L = std::max(L, rl(pi[i]));
                cnt.assign(L + 2, 0);
                for (int64_t i = a; i < b; ++i) ++cnt[L - rl(pi[i]) + 1];
                for (int32_t k = 0; k <= L; ++k) cnt[k + 1] += cnt[k];
                for (int64_t i = a; i < b; ++i) tmp[cnt[L - rl(pi[i])]++] = pi[i];
                std::copy(tmp, tmp + (b - a), pi.begin() + a);
            }
        }, 256);
        parallel_ranges(n, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) pos[pi[i]] = (int32_t)i;
        });
        // The layouts below are built on the device for systems under graph-mode size (the
        // per-densification-step path; FEMI_SELL_HOST=1 keeps the host construction): same arrays,
        // entry for entry (assemble.cu sell_layout_device).
        static const bool sell_host = std::getenv("FEMI_SELL_HOST") != nullptr;
        if (!sell_host && S->nnz_uu <= kGraphNnz && n > 0) {
            U(upload(S, &S->sell_inv, pi, st));
            int32_t nsl_d = 0;
            int64_t ent_d = 0;
            bool f16_d = true;
            U(sell_layout_device(S, n, S->sell_inv, st,
                                 [&](void** p, size_t bytes) { return dev_alloc(S, p, bytes); }, &nsl_d, &ent_d,
                                 &f16_d));
            S->nslices = nsl_d;
            S->sell_nnz = ent_d;
            stamp("sell_host");
            U(alloc(S, &S->sell_val, (size_t)std::max<int64_t>(ent_d, 1)));
            U(alloc(S, &S->s_int, (size_t)std::max<int64_t>((n + kJdsRows - 1) / kJdsRows * kJdsRows, 1)));
            U(alloc(S, &S->q_int, (size_t)std::max<int64_t>((n + kJdsRows - 1) / kJdsRows * kJdsRows, 1)));
        } else {
            // SELL-32: slice lengths, offsets, then the entries slice by slice
            const int32_t nsl = (int32_t)((n + 31) / 32);
            std::vector<int32_t> len(nsl), base(nsl);
            parallel_ranges(nsl, [&](int64_t lo, int64_t hi) {
                for (int64_t sl = lo; sl < hi; ++sl) {
                    int32_t L = 0;
                    for (int l = 0; l < 32 && 32 * sl + l < n; ++l) L = std::max(L, rl(pi[32 * sl + l]));
                    len[sl] = L;
                }
            }, 512);
            int64_t ent = 0;
            for (int32_t sl = 0; sl < nsl; ++sl) {
                base[sl] = (int32_t)ent;
                ent += 32 * (int64_t)len[sl];
            }
            std::vector<int32_t> src(ent), c32(ent);
            std::atomic<bool> fits16{true};
            parallel_ranges(nsl, [&](int64_t lo, int64_t hi) {
                bool f16 = true;
                for (int64_t sl = lo; sl < hi; ++sl) {
                    const int32_t wbase = (int32_t)((32 * sl / SIG) * SIG);
                    int64_t q = base[sl];
                    for (int32_t k = 0; k < len[sl]; ++k)
                        for (int l = 0; l < 32; ++l, ++q) {
                            const int64_t ri = 32 * sl + l;
                            int32_t col = (int32_t)std::min<int64_t>(ri, n - 1), sidx = -1;
                            if (ri < n && k < rl(pi[ri])) {
                                const int32_t row = pi[ri];
                                col = pos[uc[kth(row, k)]];
                                sidx = (rp[row] - row) + k;  // index into o_val (natural CSR)
                            }
                            src[q] = sidx;
                            c32[q] = col;
                            const int32_t d = col - wbase;
                            if (d < -32768 || d > 32767) f16 = false;
                        }
                }
                if (!f16) fits16 = false;
            }, 512);
            S->nslices = nsl;
            S->sell_nnz = ent;
            stamp("sell_host");
            U(upload(S, &S->sell_len, len, st));
            U(upload(S, &S->sell_base, base, st));
            S->sell_base_h = base;
            S->sell_base_h.push_back((int32_t)ent);  // [nslices] = total entries
            U(upload(S, &S->sell_inv, pi, st));
            {
                // internal-order CSR copies of A_uk and A_uu (with their natural-CSR sources)
                std::vector<int32_t> ukr(n + 1, 0), uur(n + 1, 0);
                for (int64_t i = 0; i < n; ++i) {
                    const int32_t nat = pi[i];
                    ukr[i + 1] = ukr[i] + (M.uk_rowptr[nat + 1] - M.uk_rowptr[nat]);
                    uur[i + 1] = uur[i] + (rp[nat + 1] - rp[nat]);
                }
                std::vector<int32_t> ukc(ukr[n]), uks(ukr[n]), uuc(uur[n]), uus(uur[n]);
                parallel_ranges(n, [&](int64_t lo, int64_t hi) {
                    for (int64_t i = lo; i < hi; ++i) {
                        const int32_t nat = pi[i];
                        int32_t o = ukr[i];
                        for (int32_t e = M.uk_rowptr[nat]; e < M.uk_rowptr[nat + 1]; ++e, ++o) {
                            ukc[o] = M.uk_col[e];
                            uks[o] = e;
                        }
                        o = uur[i];
                        for (int32_t e = rp[nat]; e < rp[nat + 1]; ++e, ++o) {
                            uuc[o] = uc[e];
                            uus[o] = e;
                        }
                    }
                });
                U(upload(S, &S->ukI_rowptr, ukr, st));
                U(upload(S, &S->uuI_rowptr, uur, st));
                if (!ukc.empty()) {
                    U(upload(S, &S->ukI_col, ukc, st));
                    U(upload(S, &S->ukI_src_tmp, uks, st));
                    U(alloc(S, &S->ukI_val, ukc.size()));
                }
                if (!uuc.empty()) {
                    U(upload(S, &S->uuI_col, uuc, st));
                    U(upload(S, &S->uuI_src_tmp, uus, st));
                    U(alloc(S, &S->uuI_val, uuc.size()));
                }
            }
            U(alloc(S, &S->sell_val, (size_t)std::max<int64_t>(ent, 1)));
            // padded to whole JDS tiles: the TMA tiles read s_int in kJdsRows blocks
            U(alloc(S, &S->s_int, (size_t)std::max<int64_t>((n + kJdsRows - 1) / kJdsRows * kJdsRows, 1)));
            U(alloc(S, &S->q_int, (size_t)std::max<int64_t>((n + kJdsRows - 1) / kJdsRows * kJdsRows, 1)));
            if (fits16) {
                std::vector<int16_t> c16(c32.size());
                parallel_ranges(nsl, [&](int64_t lo, int64_t hi) {
                    for (int64_t sl = lo; sl < hi; ++sl) {
                        const int32_t wbase = (int32_t)((32 * sl / SIG) * SIG);
                        for (int64_t q = base[sl]; q < base[sl] + 32 * (int64_t)len[sl]; ++q)
                            c16[q] = (int16_t)(c32[q] - wbase);
                    }
                }, 512);
                U(upload(S, &S->sell_c16, c16, st));
            } else {
                U(upload(S, &S->sell_c32, c32, st));
            }
            int32_t* d_src = nullptr;
            U(upload(S, &d_src, src, st));
            S->sell_src_tmp = d_src;
        }
        stamp("sell");
        if (S->nnz_uu > kGraphNnz) {
            // tiled jagged-diagonal layout (device.cuh) of the same internal order: per tile,
            // a size pass (entries padded to 16 bytes, int16 or int32 columns, format checks),
            // offsets, then a fill pass -- tiles in parallel
            const int32_t ntile = (int32_t)((n + kJdsRows - 1) / kJdsRows);
            int32_t kmax = 1;
            for (int64_t i = 0; i < n; ++i) kmax = std::max(kmax, rl((int32_t)i));
            const int32_t meta_bytes = (kJdsRows + 2 * (kJdsRows / 32) * kmax + 15) / 16 * 16;
            std::vector<int32_t> tent(ntile), eb(ntile + 1), cbo(ntile + 1);
            std::vector<uint8_t> twide(ntile);
            std::atomic<bool> okA{kmax <= kJdsMaxK};
            auto row_len = [&](int64_t ri) { return ri < n ? rl(pi[ri]) : 0; };
            if (okA) {
                parallel_ranges(ntile, [&](int64_t lo, int64_t hi) {
                    bool ok = true;
                    for (int64_t t = lo; t < hi; ++t) {
                        const int64_t r0 = t * kJdsRows;
                        int64_t cnt = 0;
                        bool wide = false;
                        for (int w = 0; w < kJdsRows / 32; ++w) {
                            int32_t L = 0;
                            for (int l = 0; l < 32; ++l) {
                                const int32_t rlen = row_len(r0 + 32 * w + l);
                                if (rlen > 255 || (l > 0 && rlen > row_len(r0 + 32 * w + l - 1))) ok = false;
                                L = std::max(L, rlen);
                            }
                            for (int32_t k = 0; k < L; ++k) {
                                if (cnt > 65535) ok = false;
                                for (int l = 0; l < 32; ++l) {
                                    const int64_t ri = r0 + 32 * w + l;
                                    if (row_len(ri) <= k) continue;
                                    const int64_t d = (int64_t)pos[uc[kth(pi[ri], k)]] - r0;
                                    wide |= d < -32768 || d > 32767;
                                    ++cnt;
                                }
                            }
                        }
                        tent[t] = (int32_t)((cnt + 7) / 8 * 8);  // 16-byte aligned tile blocks
                        twide[t] = wide;
                    }
                    if (!ok) okA = false;
                }, 16);
            }
            bool ok = okA;
            int32_t maxe = 0, nwide = 0;
            for (int32_t t = 0; t < ntile && ok; ++t) {
                eb[t + 1] = eb[t] + tent[t];
                cbo[t + 1] = cbo[t] + tent[t] * (twide[t] ? 4 : 2);
                maxe = std::max(maxe, tent[t]);
                nwide += twide[t];
            }
            if (std::getenv("FEMI_DEBUG"))
                std::fprintf(stderr, "[femi] jds layout: ok %d tiles %d (int32 columns: %d) entries %d maxe %d kmax %d\n",
                             (int)ok, ntile, nwide, ok ? eb[ntile] : -1, maxe, kmax);
            if (ok) {
                std::vector<uint8_t> meta((size_t)ntile * meta_bytes, 0), jcolb(cbo[ntile]);
                std::vector<int32_t> jsrc(eb[ntile], -1);
                parallel_ranges(ntile, [&](int64_t lo, int64_t hi) {
                    for (int64_t t = lo; t < hi; ++t) {
                        const int64_t r0 = t * kJdsRows;
                        uint8_t* mt = meta.data() + (size_t)t * meta_bytes;
                        uint16_t* doff = (uint16_t*)(mt + kJdsRows);
                        int16_t* c16 = (int16_t*)(jcolb.data() + cbo[t]);
                        int32_t* c32w = (int32_t*)(jcolb.data() + cbo[t]);
                        int64_t q = 0;
                        for (int w = 0; w < kJdsRows / 32; ++w) {
                            int32_t L = 0;
                            for (int l = 0; l < 32; ++l) {
                                const int32_t rlen = row_len(r0 + 32 * w + l);
                                mt[32 * w + l] = (uint8_t)rlen;
                                L = std::max(L, rlen);
                            }
                            for (int32_t k = 0; k < L; ++k) {
                                doff[w * kmax + k] = (uint16_t)q;
                                for (int l = 0; l < 32; ++l) {
                                    const int64_t ri = r0 + 32 * w + l;
                                    if (row_len(ri) <= k) continue;
                                    const int32_t row = pi[ri];
                                    const int64_t d = (int64_t)pos[uc[kth(row, k)]] - r0;
                                    if (twide[t]) c32w[q] = (int32_t)d;
                                    else c16[q] = (int16_t)d;
                                    jsrc[eb[t] + q] = (rp[row] - row) + k;
                                    ++q;
                                }
                            }
                        }
                        for (; q < tent[t]; ++q) {  // padding entries: column 0, no source
                            if (twide[t]) c32w[q] = 0;
                            else c16[q] = 0;
                        }
                    }
                }, 16);
                S->jds_ntile = ntile;
                S->jds_maxe = maxe;
                S->jds_kmax = kmax;
                S->jds_meta_bytes = meta_bytes;
                S->jds_nnz = (int64_t)eb[ntile];
                U(upload(S, &S->jds_eb, eb, st));
                U(upload(S, &S->jds_cb, cbo, st));
                {
                    // values | columns | metadata in ONE allocation: the SpMV's matrix stream is one
                    // address range (an L2 access-policy window can cover it)
                    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
                    const size_t bv = al(sizeof(double) * (size_t)std::max<int64_t>(S->jds_nnz, 1));
                    const size_t bc = al(std::max<size_t>(jcolb.size(), 1));
                    const size_t bm = al(std::max<size_t>(meta.size(), 1));
                    void* blk = nullptr;
                    const cudaError_t e = cudaMallocAsync(&blk, bv + bc + bm, st);
                    if (e != cudaSuccess) {
                        s = cuda_fail(e, "assemble: matrix stream block");
                        goto fail;
                    }
                    S->allocs.push_back(blk);
                    S->jds_val = (double*)blk;
                    S->jds_col = (uint8_t*)blk + bv;
                    S->jds_meta = (uint8_t*)blk + bv + bc;
                    S->jds_block_bytes = bv + bc + bm;
                    U(h2d(S->jds_col, jcolb.data(), jcolb.size(), st));
                    U(h2d(S->jds_meta, meta.data(), meta.size(), st));
                }
                int32_t* d_js = nullptr;
                U(upload(S, &d_js, jsrc, st));
                S->jds_src_tmp = d_js;
            }
        }
    }
    stamp("jds");
    U(launch_tri_records(S, d_tri, d_flags, st));
    stamp("trirec");
    U(alloc(S, &S->tp_ptr, (size_t)M.T + 1));
    U(alloc(S, &S->tp_pix, (size_t)M.W * M.H));
    U(build_owner_tables(S, st));
    stamp("owner");
    U(launch_assemble_values(S, st));
    stamp("values");
    U(launch_sell_values(S, S->sell_src_tmp, st));
    // the int32 triangle table and flags are folded into TriRec; drop them once done
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        s = cuda_fail(cudaGetLastError(), "assemble: sync");
        goto fail;
    }
    for (auto it = S->allocs.begin(); it != S->allocs.end();) {
        if (*it == (void*)d_tri || *it == (void*)d_flags || *it == (void*)S->sell_src_tmp ||
            (S->jds_src_tmp && *it == (void*)S->jds_src_tmp) || (S->ukI_src_tmp && *it == (void*)S->ukI_src_tmp) ||
            (S->uuI_src_tmp && *it == (void*)S->uuI_src_tmp)) {
            cudaFreeAsync(*it, st);
            it = S->allocs.erase(it);
        } else {
            ++it;
        }
    }
    stamp("done");
#undef U
    *out = S;
    return FEMI_OK;
fail:
    femi_system_free(S);
    return s;
}

femi_status femi_system_info_get(femi_system sys, femi_mesh_info* info) {
    if (!sys || !info) return FEMI_E_ARG;
    info->width = sys->W;
    info->height = sys->H;
    info->n_vert = sys->nv;
    info->n_unknown = sys->n_u;
    info->n_mask = sys->m;
    info->n_tri = sys->T;
    info->nnz_uu = sys->nnz_uu;
    info->nnz_uk = sys->nnz_uk;
    return FEMI_OK;
}

femi_status femi_system_export(femi_system sys, double* uu_val, double* uk_val, femi_stream stream) {
    if (!sys || sys->raster_only) {
        set_error("system_export: NULL system");
        return FEMI_E_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (uu_val && sys->nnz_uu)
        FEMI_CUDA(cudaMemcpyAsync(uu_val, sys->uu_val, sizeof(double) * sys->nnz_uu, cudaMemcpyDeviceToHost, st));
    if (uk_val && sys->nnz_uk)
        FEMI_CUDA(cudaMemcpyAsync(uk_val, sys->uk_val, sizeof(double) * sys->nnz_uk, cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaStreamSynchronize(st));
    return FEMI_OK;
}

femi_status femi_inpaint_solve_batched(int32_t B, const femi_system* sys, const double* const* g,
                                       double* const* u_vert, const femi_cg_opts* opts, int32_t* iters,
                                       double* relres, femi_stream stream) {
    if (B < 0 || (B > 0 && (!sys || !g || !u_vert || !opts))) {
        set_error("inpaint_solve_batched: NULL argument or B < 0");
        return FEMI_E_ARG;
    }
    if (B == 0) return FEMI_OK;
    if (!(opts->rtol > 0.0) || opts->max_iter <= 0 || opts->precond != 1 || opts->x0 < 0 || opts->x0 > 3 ||
        opts->check_every != 0) {
        set_error("inpaint_solve_batched: invalid options (rtol > 0, max_iter > 0, precond 1, x0 0..3, check_every 0)");
        return FEMI_E_ARG;
    }
    for (int b = 0; b < B; ++b)
        if (!sys[b] || !g[b] || !u_vert[b] || sys[b]->raster_only) {
            set_error("inpaint_solve_batched: NULL entry or a raster-only (band) system");
            return FEMI_E_ARG;
        }
    femi_status s = check_device();
    if (s) return s;
    std::vector<femi_system_s*> Sv(sys, sys + B);
    SysGuard guard(Sv.data(), B, (cudaStream_t)stream);
    return pcg_solve(B, Sv.data(), g, nullptr, u_vert, *opts, iters, relres, (cudaStream_t)stream, nullptr);
}

femi_status femi_rasterise_error_batched(int32_t B, const femi_system* sys, const double* const* u_vert,
                                         const double* const* f, double* const* u_px, double* const* e_px,
                                         double* const* tri_err, int32_t* const* tri_best_px, double* const* sse,
                                         femi_stream stream) {
    if (B < 0 || (B > 0 && (!sys || !u_vert || !f || !sse))) {
        set_error("rasterise_error: NULL argument");
        return FEMI_E_ARG;
    }
    for (int b = 0; b < B; ++b)
        if (!sys[b] || !u_vert[b] || !f[b] || !sse[b]) {
            set_error("rasterise_error: NULL entry");
            return FEMI_E_ARG;
        }
    std::vector<femi_system_s*> Sv(sys, sys + B);
    SysGuard guard(Sv.data(), B, (cudaStream_t)stream);
    return launch_raster(B, Sv.data(), u_vert, f, u_px, e_px, tri_err, tri_best_px, sse, (cudaStream_t)stream);
}

femi_status femi_rasterise_error(femi_system sys, const double* u_vert, const double* f, double* u_px, double* e_px,
                                 double* tri_err, int32_t* tri_best_px, double* sse, femi_stream stream) {
    femi_system sv[1] = {sys};
    const double* uv[1] = {u_vert};
    const double* fv[1] = {f};
    double* up[1] = {u_px};
    double* ep[1] = {e_px};
    double* te[1] = {tri_err};
    int32_t* bp[1] = {tri_best_px};
    double* sp[1] = {sse};
    return femi_rasterise_error_batched(1, sv, uv, fv, up, ep, te, bp, sp, stream);
}

femi_status femi_densify_step(femi_system sys, const double* f, const double* u_vert, int64_t b,
                              int32_t* new_mask_px, int64_t* n_added, femi_stream stream) {
    if (!sys || !f || !u_vert || !n_added || b < 0 || (b > 0 && !new_mask_px) || sys->raster_only) {
        set_error("densify_step: NULL argument, b < 0 or a raster-only (band) system");
        return FEMI_E_ARG;
    }
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return densify_select(sys, 1, &f, &u_vert, b, new_mask_px, n_added, (cudaStream_t)stream);
}

femi_status femi_rasterise_error_channels(femi_system sys, int32_t C, const double* const* u_vert,
                                          const double* const* f, double* const* u_px, double* e_px, double* tri_err,
                                          int32_t* tri_best_px, double* sse, femi_stream stream) {
    if (!sys || C < 1 || C > 4 || !u_vert) {
        set_error("rasterise_error_channels: NULL system/u_vert or C outside 1..4");
        return FEMI_E_ARG;
    }
    for (int c = 0; c < C; ++c)
        if (!u_vert[c] || (f && !f[c])) {
            set_error("rasterise_error_channels: NULL channel pointer");
            return FEMI_E_ARG;
        }
    if (!f && (e_px || tri_err || tri_best_px || sse)) {
        set_error("rasterise_error_channels: error outputs need f");
        return FEMI_E_ARG;
    }
    femi_status s = check_device();
    if (s) return s;
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return launch_raster_channels(sys, C, u_vert, f, u_px, e_px, tri_err, tri_best_px, sse, (cudaStream_t)stream);
}

femi_status femi_densify_step_channels(femi_system sys, int32_t C, const double* const* f,
                                       const double* const* u_vert, int64_t b, int32_t* new_mask_px,
                                       int64_t* n_added, femi_stream stream) {
    if (!sys || sys->raster_only || C < 1 || C > 4 || !f || !u_vert || !n_added || b < 0 || (b > 0 && !new_mask_px)) {
        set_error("densify_step_channels: NULL argument, C outside 1..4 or b < 0");
        return FEMI_E_ARG;
    }
    for (int c = 0; c < C; ++c)
        if (!f[c] || !u_vert[c]) {
            set_error("densify_step_channels: NULL channel pointer");
            return FEMI_E_ARG;
        }
    femi_status s = check_device();
    if (s) return s;
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return densify_select(sys, C, f, u_vert, b, new_mask_px, n_added, (cudaStream_t)stream);
}

femi_status femi_tonal_optimise_l1(femi_system sys, const double* f, double* g, const femi_tonal_opts* opts,
                                   int32_t irls, double eps, femi_tonal_l1_report* report, femi_stream stream) {
    if (!sys || sys->raster_only || !f || !g || !opts || !report || irls < 0 || !(eps > 0.0)) {
        set_error("tonal_optimise_l1: NULL argument, irls < 0 or eps <= 0");
        return FEMI_E_ARG;
    }
    if (!(opts->outer_rtol > 0.0) || opts->outer_max < 0 || !(opts->inner.rtol > 0.0) || opts->inner.max_iter <= 0 ||
        opts->inner.precond != 1 || opts->inner.check_every != 0 || opts->warm_start != 0) {
        set_error("tonal_optimise_l1: invalid options");
        return FEMI_E_ARG;
    }
    femi_status s = check_device();
    if (s) return s;
    if (sys->n_u == 0 || sys->m == 0) {
        *report = femi_tonal_l1_report{};
        return FEMI_OK;
    }
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return tonal_irls(sys, f, g, *opts, irls, eps, report, (cudaStream_t)stream);
}

int64_t femi_device_check_failures(int64_t* first_site) {
    int64_t site = 0;
    int64_t n = 0;
    for (auto fn : {dcheck_abi, dcheck_assemble, dcheck_pcg, dcheck_raster, dcheck_select, dcheck_tonal, dcheck_band}) {
        const int64_t k = fn(&site);
        if (k < 0) return -1;
        n += k;
    }
    if (first_site) *first_site = site;
    return n;
}

femi_status femi_system_solver_path(femi_system sys, int32_t* path) {
    if (!sys || !path) return FEMI_E_ARG;
    *path = sys->last_path;
    return FEMI_OK;
}

static femi_status apply_common(const char* what, femi_system sys, const double* in, double* out,
                                const femi_cg_opts* opts) {
    if (!sys || sys->raster_only || !in || !out || !opts) {
        set_error(std::string(what) + ": NULL argument");
        return FEMI_E_ARG;
    }
    if (!(opts->rtol > 0.0) || opts->max_iter <= 0 || opts->precond != 1 || opts->check_every != 0) {
        set_error(std::string(what) + ": invalid options (rtol > 0, max_iter > 0, precond 1, check_every 0)");
        return FEMI_E_ARG;
    }
    return check_device();
}

femi_status femi_apply_B(femi_system sys, const double* g, double* u_px, const femi_cg_opts* opts, femi_stream stream) {
    femi_status s = apply_common("apply_B", sys, g, u_px, opts);
    if (s) return s;
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return tonal_apply(sys, 0, g, u_px, *opts, (cudaStream_t)stream);
}

femi_status femi_apply_BT(femi_system sys, const double* r, double* s_out, const femi_cg_opts* opts,
                          femi_stream stream) {
    femi_status s = apply_common("apply_BT", sys, r, s_out, opts);
    if (s) return s;
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return tonal_apply(sys, 1, r, s_out, *opts, (cudaStream_t)stream);
}

femi_status femi_tonal_optimise_channels(femi_system sys, int32_t C, const double* const* f, double* const* g,
                                         const femi_tonal_opts* opts, femi_tonal_report* reports, femi_stream stream) {
    if (!sys || sys->raster_only || C < 1 || C > 4 || !f || !g || !opts || !reports) {
        set_error("tonal_optimise_channels: NULL argument or C outside 1..4");
        return FEMI_E_ARG;
    }
    for (int c = 0; c < C; ++c)
        if (!f[c] || !g[c]) {
            set_error("tonal_optimise_channels: NULL channel pointer");
            return FEMI_E_ARG;
        }
    if (!(opts->outer_rtol > 0.0) || opts->outer_max < 0 || !(opts->inner.rtol > 0.0) || opts->inner.max_iter <= 0 ||
        opts->inner.precond != 1 || opts->inner.check_every != 0 || opts->warm_start != 0) {
        set_error("tonal_optimise_channels: invalid options");
        return FEMI_E_ARG;
    }
    femi_status s = check_device();
    if (s) return s;
    std::memset(reports, 0, sizeof(femi_tonal_report) * C);
    if (sys->n_u == 0) return FEMI_OK;
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return tonal_cgls_channels(sys, C, f, g, *opts, reports, (cudaStream_t)stream);
}

femi_status femi_tonal_optimise(femi_system sys, const double* f, double* g, const femi_tonal_opts* opts,
                                femi_tonal_report* report, femi_stream stream) {
    if (!sys || sys->raster_only || !f || !g || !opts || !report) {
        set_error("tonal_optimise: NULL argument");
        return FEMI_E_ARG;
    }
    if (!(opts->outer_rtol > 0.0) || opts->outer_max < 0 || !(opts->inner.rtol > 0.0) || opts->inner.max_iter <= 0 ||
        opts->inner.precond != 1 || opts->inner.check_every != 0 || opts->warm_start != 0) {
        set_error("tonal_optimise: invalid options");
        return FEMI_E_ARG;
    }
    femi_status s = check_device();
    if (s) return s;
    std::memset(report, 0, sizeof(*report));
    SysGuard guard(&sys, 1, (cudaStream_t)stream);
    return tonal_cgls(sys, f, g, *opts, report, (cudaStream_t)stream);
}

}  // extern "C"

FEMI_DCHECK_READER(dcheck_abi)
