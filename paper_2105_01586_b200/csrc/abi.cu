// abi.cu -- the extern "C" boundary of libfemi (include/femi.h). Argument checking, handle
// life cycle, uploads; every compute step is one of the kernels in the other .cu files.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

template <class T>
femi_status upload(femi_system_s* S, T** dst, const std::vector<T>& src, cudaStream_t st, size_t extra = 0) {
    size_t n = src.size() + extra;
    void* p = nullptr;
    FEMI_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
    S->allocs.push_back(p);
    if (!src.empty()) FEMI_CUDA(cudaMemcpyAsync(p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, st));
    *dst = (T*)p;
    return FEMI_OK;
}

template <class T>
femi_status alloc(femi_system_s* S, T** dst, size_t n) {
    void* p = nullptr;
    FEMI_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
    S->allocs.push_back(p);
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

// row chunks for the PCG kernels: <= kRowsPerChunk rows and <= kChunkNnzCap off-diagonals
std::vector<Chunk> make_chunks(const std::vector<int32_t>& uu_rowptr, int64_t n_u) {
    std::vector<Chunk> ch;
    int64_t i = 0;
    int32_t local = 0;
    while (i < n_u) {
        int64_t j = i;
        int64_t nnz = 0;
        while (j < n_u && j - i < kRowsPerChunk) {
            int64_t rn = (uu_rowptr[j + 1] - uu_rowptr[j]) - 1;
            if (j > i && nnz + rn > kChunkNnzCap) break;
            nnz += rn;
            ++j;
        }
        ch.push_back({0, (int32_t)i, (int32_t)j, local++});
        i = j;
    }
    return ch;
}

}  // namespace
}  // namespace femi

using namespace femi;

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
    cudaDeviceSynchronize();
    pcg_cache_free(sys);
    for (void* p : sys->allocs) cudaFree(p);
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
    femi_system_s* S = new (std::nothrow) femi_system_s();
    if (!S) return FEMI_E_OOM;
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
    S->chunks_h = make_chunks(M.uu_rowptr, M.n_u);
    U(upload(S, &S->chunks_d, S->chunks_h, st));
    {
        // chunk row table and int16 column offsets (relative to the chunk's first row)
        std::vector<int32_t> row0(S->chunks_h.size() + 1);
        for (size_t c = 0; c < S->chunks_h.size(); ++c) row0[c] = S->chunks_h[c].row0;
        row0.back() = (int32_t)M.n_u;
        S->nchunks = (int32_t)S->chunks_h.size();
        U(upload(S, &S->chunk_row0, row0, st));
        std::vector<int16_t> cd(M.uu_col.size() - M.n_u);
        bool fits = true;
        size_t o = 0;
        for (size_t c = 0; c < S->chunks_h.size() && fits; ++c) {
            const int32_t r0 = S->chunks_h[c].row0;
            for (int32_t i = r0; i < S->chunks_h[c].row1 && fits; ++i)
                for (int32_t e = M.uu_rowptr[i]; e < M.uu_rowptr[i + 1]; ++e) {
                    const int32_t j = M.uu_col[e];
                    if (j == i) continue;
                    const int32_t d = j - r0;
                    if (d < -32768 || d > 32767) {
                        fits = false;
                        break;
                    }
                    cd[o++] = (int16_t)d;
                }
        }
        if (fits && !cd.empty()) U(upload(S, &S->o_cd, cd, st));
    }
    {
        // Solver numbering + SELL-32-sigma layout of the off-diagonal pattern (values are
        // filled on the device after assembly). Internal order: unknowns sorted by
        // (y / kBand, x, y) -- 32 consecutive internal rows form a compact 2-D blob, so
        // row data is contiguous and gathered neighbours sit in few cache lines -- then
        // rows sorted by length (descending, stable) inside windows of kSellSigma.
        const int64_t n = M.n_u;
        const int SIG = kSellSigma;
        S->nwin = (int32_t)((n + SIG - 1) / SIG);
        auto rl = [&](int32_t i) { return M.uu_rowptr[i + 1] - M.uu_rowptr[i] - 1; };
        std::vector<int32_t> pi(n), pos(n);
        {
            std::vector<std::pair<uint64_t, int32_t>> key(n);
            uint64_t band = kBand;
            if (const char* e = std::getenv("FEMI_BAND")) band = (uint64_t)std::max(1, std::atoi(e));
            for (int64_t i = 0; i < n; ++i) {
                const uint64_t x = (uint64_t)(M.vpix[i] % M.W), y = (uint64_t)(M.vpix[i] / M.W);
                key[i] = {((y / band) << 40) | (x << 20) | y, (int32_t)i};
            }
            std::sort(key.begin(), key.end());
            for (int64_t i = 0; i < n; ++i) pi[i] = key[i].second;
        }
        for (int64_t w0 = 0; w0 < n; w0 += SIG)
            std::stable_sort(pi.begin() + w0, pi.begin() + std::min<int64_t>(n, w0 + SIG),
                             [&](int32_t a, int32_t b) { return rl(a) > rl(b); });
        for (int64_t i = 0; i < n; ++i) pos[pi[i]] = (int32_t)i;
        const int32_t nsl = (int32_t)((n + 31) / 32);
        std::vector<int32_t> len(nsl), base(nsl), src, c32;
        std::vector<int16_t> c16;
        bool fits16 = true;
        int64_t ent = 0;
        for (int32_t sl = 0; sl < nsl; ++sl) {
            int32_t L = 0;
            for (int l = 0; l < 32 && 32 * sl + l < n; ++l) L = std::max(L, rl(pi[32 * sl + l]));
            len[sl] = L;
            base[sl] = (int32_t)ent;
            const int32_t wbase = (32 * sl / SIG) * SIG;
            for (int32_t k = 0; k < L; ++k)
                for (int l = 0; l < 32; ++l) {
                    const int64_t ri = 32 * (int64_t)sl + l;
                    int32_t col = (int32_t)std::min<int64_t>(ri, n - 1), sidx = -1;
                    if (ri < n && k < rl(pi[ri])) {
                        const int32_t row = pi[ri];
                        int32_t e = M.uu_rowptr[row], q = 0;  // k-th off-diagonal entry of row
                        for (; e < M.uu_rowptr[row + 1]; ++e) {
                            if (M.uu_col[e] == row) continue;
                            if (q == k) break;
                            ++q;
                        }
                        col = pos[M.uu_col[e]];
                        sidx = (M.uu_rowptr[row] - row) + k;  // index into o_val (natural CSR)
                    }
                    src.push_back(sidx);
                    c32.push_back(col);
                    const int32_t d = col - wbase;
                    if (d < -32768 || d > 32767) fits16 = false;
                    ++ent;
                }
        }
        S->nslices = nsl;
        S->sell_nnz = ent;
        U(upload(S, &S->sell_len, len, st));
        U(upload(S, &S->sell_base, base, st));
        S->sell_base_h = base;
        S->sell_base_h.push_back((int32_t)ent);  // [nslices] = total entries
        U(upload(S, &S->sell_inv, pi, st));
        {
            std::vector<int32_t> ukr(n + 1), ukc, uks, uur(n + 1), uuc, uus;
            ukc.reserve(M.uk_col.size());
            uks.reserve(M.uk_col.size());
            uuc.reserve(M.uu_col.size());
            uus.reserve(M.uu_col.size());
            for (int64_t i = 0; i < n; ++i) {
                const int32_t nat = pi[i];
                ukr[i] = (int32_t)ukc.size();
                for (int32_t e = M.uk_rowptr[nat]; e < M.uk_rowptr[nat + 1]; ++e) {
                    ukc.push_back(M.uk_col[e]);
                    uks.push_back(e);
                }
                uur[i] = (int32_t)uuc.size();
                for (int32_t e = M.uu_rowptr[nat]; e < M.uu_rowptr[nat + 1]; ++e) {
                    uuc.push_back(M.uu_col[e]);
                    uus.push_back(e);
                }
            }
            ukr[n] = (int32_t)ukc.size();
            uur[n] = (int32_t)uuc.size();
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
            c16.resize(c32.size());
            for (int32_t sl = 0, q = 0; sl < nsl; ++sl) {
                const int32_t wbase = (32 * sl / SIG) * SIG;
                for (int32_t k = 0; k < len[sl] * 32; ++k, ++q) c16[q] = (int16_t)(c32[q] - wbase);
            }
            U(upload(S, &S->sell_c16, c16, st));
        } else {
            U(upload(S, &S->sell_c32, c32, st));
        }
        int32_t* d_src = nullptr;
        U(upload(S, &d_src, src, st));
        S->sell_src_tmp = d_src;
        if (S->nnz_uu > kGraphNnz) {
            // tiled jagged-diagonal layout (device.cuh) of the same internal order
            const int32_t ntile = (int32_t)((n + kJdsRows - 1) / kJdsRows);
            std::vector<int32_t> eb(ntile + 1), cbo(ntile + 1), jsrc;
            std::vector<uint8_t> jcolb;  // per tile: int16 columns, or int32 when a column is out of range
            // kmax = longest row; meta per tile: lengths + [slice][kmax] uint16 diagonal offsets
            int32_t kmax = 1;
            for (int64_t i = 0; i < n; ++i) kmax = std::max(kmax, rl((int32_t)i));
            const int32_t meta_bytes = (kJdsRows + 2 * (kJdsRows / 32) * kmax + 15) / 16 * 16;
            std::vector<uint8_t> meta((size_t)ntile * meta_bytes, 0);
            bool ok = kmax <= kJdsMaxK;
            int32_t maxe = 0, nwide = 0;
            auto kth = [&](int32_t row, int32_t k) {  // k-th off-diagonal of a row (natural CSR)
                int32_t e = M.uu_rowptr[row], q = 0;
                for (; e < M.uu_rowptr[row + 1]; ++e) {
                    if (M.uu_col[e] == row) continue;
                    if (q == k) break;
                    ++q;
                }
                return e;
            };
            std::vector<int64_t> tcol;
            for (int32_t t = 0; t < ntile && ok; ++t) {
                eb[t] = (int32_t)jsrc.size();
                cbo[t] = (int32_t)jcolb.size();
                tcol.clear();
                const int64_t r0 = (int64_t)t * kJdsRows;
                uint8_t* mt = meta.data() + (size_t)t * meta_bytes;
                uint16_t* doff = (uint16_t*)(mt + kJdsRows);
                for (int w = 0; w < kJdsRows / 32; ++w) {
                    int32_t L = 0;
                    for (int l = 0; l < 32; ++l) {
                        const int64_t ri = r0 + 32 * w + l;
                        const int32_t len = ri < n ? rl(pi[ri]) : 0;
                        if (len > 255) ok = false;
                        if (l > 0 && len > mt[32 * w + l - 1]) ok = false;  // descending inside the slice
                        mt[32 * w + l] = (uint8_t)len;
                        L = std::max(L, len);
                    }
                    for (int32_t k = 0; k < L; ++k) {
                        const int64_t off = (int64_t)jsrc.size() - eb[t];
                        if (off > 65535) ok = false;
                        doff[w * kmax + k] = (uint16_t)off;
                        for (int l = 0; l < 32; ++l) {
                            const int64_t ri = r0 + 32 * w + l;
                            if (ri >= n || rl(pi[ri]) <= k) continue;
                            const int32_t row = pi[ri];
                            const int32_t e = kth(row, k);
                            tcol.push_back((int64_t)pos[M.uu_col[e]] - r0);
                            jsrc.push_back((M.uu_rowptr[row] - row) + k);
                        }
                    }
                }
                while (jsrc.size() % 8) {  // 16-byte aligned tile blocks for the bulk copies
                    tcol.push_back(0);
                    jsrc.push_back(-1);
                }
                bool wide = false;
                for (int64_t d : tcol) wide |= d < -32768 || d > 32767;
                nwide += wide;
                for (int64_t d : tcol) {
                    if (wide) {
                        const int32_t v = (int32_t)d;
                        const uint8_t* b = (const uint8_t*)&v;
                        jcolb.insert(jcolb.end(), b, b + 4);
                    } else {
                        const int16_t v = (int16_t)d;
                        const uint8_t* b = (const uint8_t*)&v;
                        jcolb.insert(jcolb.end(), b, b + 2);
                    }
                }
                maxe = std::max(maxe, (int32_t)jsrc.size() - eb[t]);
            }
            eb[ntile] = (int32_t)jsrc.size();
            cbo[ntile] = (int32_t)jcolb.size();
            if (std::getenv("FEMI_DEBUG"))
                std::fprintf(stderr, "[femi] jds layout: ok %d tiles %d (int32 columns: %d) entries %zu maxe %d kmax %d\n",
                             (int)ok, ntile, nwide, jsrc.size(), maxe, kmax);
            if (ok) {
                S->jds_ntile = ntile;
                S->jds_maxe = maxe;
                S->jds_kmax = kmax;
                S->jds_meta_bytes = meta_bytes;
                S->jds_nnz = (int64_t)jsrc.size();
                U(upload(S, &S->jds_eb, eb, st));
                U(upload(S, &S->jds_cb, cbo, st));
                U(upload(S, &S->jds_meta, meta, st));
                U(upload(S, &S->jds_col, jcolb, st));
                U(alloc(S, &S->jds_val, (size_t)std::max<int64_t>(S->jds_nnz, 1)));
                int32_t* d_js = nullptr;
                U(upload(S, &d_js, jsrc, st));
                S->jds_src_tmp = d_js;
            }
        }
    }
    U(launch_tri_records(S, d_tri, d_flags, st));
    U(alloc(S, &S->tp_ptr, (size_t)M.T + 1));
    U(alloc(S, &S->tp_pix, (size_t)M.W * M.H));
    U(build_owner_tables(S, st));
    U(launch_assemble_values(S, st));
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
            cudaFree(*it);
            it = S->allocs.erase(it);
        } else {
            ++it;
        }
    }
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
    if (!sys) {
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
    if (!(opts->rtol > 0.0) || opts->max_iter <= 0 || opts->precond < 0 || opts->precond > 1 || opts->x0 < 0 ||
        opts->x0 > 2 || opts->check_every < 0) {
        set_error("inpaint_solve_batched: invalid options");
        return FEMI_E_ARG;
    }
    for (int b = 0; b < B; ++b)
        if (!sys[b] || !g[b] || !u_vert[b]) {
            set_error("inpaint_solve_batched: NULL entry");
            return FEMI_E_ARG;
        }
    femi_status s = check_device();
    if (s) return s;
    std::vector<femi_system_s*> Sv(sys, sys + B);
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
    if (!sys || !f || !u_vert || !n_added || b < 0 || (b > 0 && !new_mask_px)) {
        set_error("densify_step: NULL argument or b < 0");
        return FEMI_E_ARG;
    }
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
    return launch_raster_channels(sys, C, u_vert, f, u_px, e_px, tri_err, tri_best_px, sse, (cudaStream_t)stream);
}

femi_status femi_densify_step_channels(femi_system sys, int32_t C, const double* const* f,
                                       const double* const* u_vert, int64_t b, int32_t* new_mask_px,
                                       int64_t* n_added, femi_stream stream) {
    if (!sys || C < 1 || C > 4 || !f || !u_vert || !n_added || b < 0 || (b > 0 && !new_mask_px)) {
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
    return densify_select(sys, C, f, u_vert, b, new_mask_px, n_added, (cudaStream_t)stream);
}

femi_status femi_tonal_optimise_l1(femi_system sys, const double* f, double* g, const femi_tonal_opts* opts,
                                   int32_t irls, double eps, femi_tonal_l1_report* report, femi_stream stream) {
    if (!sys || !f || !g || !opts || !report || irls < 0 || !(eps > 0.0)) {
        set_error("tonal_optimise_l1: NULL argument, irls < 0 or eps <= 0");
        return FEMI_E_ARG;
    }
    if (!(opts->outer_rtol > 0.0) || opts->outer_max < 0 || !(opts->inner.rtol > 0.0) || opts->inner.max_iter <= 0 ||
        opts->warm_start != 0) {
        set_error("tonal_optimise_l1: invalid options");
        return FEMI_E_ARG;
    }
    femi_status s = check_device();
    if (s) return s;
    if (sys->n_u == 0 || sys->m == 0) {
        *report = femi_tonal_l1_report{};
        return FEMI_OK;
    }
    return tonal_irls(sys, f, g, *opts, irls, eps, report, (cudaStream_t)stream);
}

femi_status femi_tonal_optimise(femi_system sys, const double* f, double* g, const femi_tonal_opts* opts,
                                femi_tonal_report* report, femi_stream stream) {
    if (!sys || !f || !g || !opts || !report) {
        set_error("tonal_optimise: NULL argument");
        return FEMI_E_ARG;
    }
    if (!(opts->outer_rtol > 0.0) || opts->outer_max < 0 || !(opts->inner.rtol > 0.0) || opts->inner.max_iter <= 0 ||
        opts->warm_start != 0) {
        set_error("tonal_optimise: invalid options");
        return FEMI_E_ARG;
    }
    femi_status s = check_device();
    if (s) return s;
    std::memset(report, 0, sizeof(*report));
    return tonal_cgls(sys, f, g, *opts, report, (cudaStream_t)stream);
}

}  // extern "C"
