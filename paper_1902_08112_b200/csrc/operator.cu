// C ABI of the fused matrix-free operator: argument checking and dispatch to
// the per-dimension kernel instantiations (op2d.cu, op3d.cu; kernels in
// op_kernels.cuh).  Replaces reference model.py:368-413 and the vector
// updates of mgsolve.py:82-113 / 227 (fused epilogues).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "op_launch.cuh"

namespace pffmg {

template <int MODE, int EPI>
static int launch(const OpArgs& A, cudaStream_t s, const char* what) {
    const Lat& L = A.L;
    const bool iso = L.hx == L.hy && (L.dim == 2 || L.hz == L.hx);
    if (L.order == 2)
        launch2q<MODE, EPI>(A, s);
    else if (L.dim == 2)
        launch2d<MODE, EPI>(A, iso, s);
    else
        launch3d<MODE, EPI>(A, iso, s);
    return check_launch(what);
}

static int fill_args(const pffmg_lattice* lat, const pffmg_state* st, OpArgs* A) {
    PFFMG_REQUIRE(lat && st, "null lattice/state");
    *A = OpArgs{};
    int rc = make_lat(lat, &A->L);
    if (rc) return rc;
    rc = make_consts(lat, st, &A->K);
    if (rc) return rc;
    A->I = make_iso_host(A->K);
    if (st->split != 0 && st->split != 1) {
        set_error("unknown split kind %d (0 NoSplit, 1 Miehe)", st->split);
        return PFFMG_ERR_ARG;
    }
    PFFMG_REQUIRE(st->split_band >= 0.0 && std::isfinite(st->split_band), "split_band must be finite and >= 0");
    A->split = st->split;
    PFFMG_REQUIRE(st->flags, "state.flags is NULL");
    A->U = st->U;
    A->pt = st->phi_tilde;
    A->rho = st->rho;
    A->flags = st->flags;
    // the a_phiphi table serves the phi block of isotropic NoSplit Q1 lattices
    // (3D phi block; 2D block-diagonal smoother)
    const bool iso = A->L.order == 1 && A->L.hx == A->L.hy && (A->L.dim == 2 || A->L.hz == A->L.hx);
    A->ptab = (st->phi_coef && (iso || A->L.order == 2) && st->split == 0) ? st->phi_coef : nullptr;
    A->premasked = (st->hints & PFFMG_HINT_PREMASKED) ? 1 : 0;
    A->ends = (st->hints & PFFMG_HINT_ENDS) ? 1 : 0;
    if (A->ends) {
        PFFMG_REQUIRE(A->L.own_hi - A->L.own_lo >= 2 && A->L.order == 1,
                      "PFFMG_HINT_ENDS needs >= 2 owned planes of a Q1 lattice");
    }
    return PFFMG_OK;
}

template <int EPI>
static int dispatch_which(const OpArgs& A, int which, cudaStream_t s, const char* what) {
    if (which == PFFMG_FULL) {
        PFFMG_REQUIRE(A.U && A.pt, "%s: full operator needs U and phi_tilde", what);
        return launch<M_FULL, EPI>(A, s, what);
    }
    if (which == PFFMG_UBLOCK) {
        PFFMG_REQUIRE(A.pt, "%s: u block needs phi_tilde", what);
        return launch<M_UBLK, EPI>(A, s, what);
    }
    if (which == PFFMG_PBLOCK) {
        PFFMG_REQUIRE(A.U, "%s: phi block needs U", what);
        return launch<M_PBLK, EPI>(A, s, what);
    }
    if (which == PFFMG_BLOCKDIAG) {
        PFFMG_REQUIRE(A.U && A.pt, "%s: block-diagonal operator needs U and phi_tilde", what);
        OpArgs B = A;
        B.nocoup = 1;
        return launch<M_FULL, EPI>(B, s, what);
    }
    set_error("%s: which must be -1, 0, 1 or 2 (got %d)", what, which);
    return PFFMG_ERR_ARG;
}

}  // namespace pffmg

using namespace pffmg;

extern "C" int pffmg_phi_coef(const pffmg_lattice* lat, const pffmg_state* st, double* out, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(out && A.U, "pffmg_phi_coef: needs U and out");
    PFFMG_REQUIRE(A.split == 0 && (A.L.order == 2 || (A.L.hx == A.L.hy && (A.L.dim == 2 || A.L.hz == A.L.hx))),
                  "pffmg_phi_coef: NoSplit Q2 or isotropic Q1 lattices only");
    PFFMG_REQUIRE(out != st->phi_coef, "pffmg_phi_coef: out aliases state.phi_coef");
    if (A.L.order == 2)
        launch_phi_coefq(A, out, as_stream(stream));
    else if (A.L.dim == 3)
        launch_phi_coef3(A, out, as_stream(stream));
    else
        launch_phi_coef2(A, out, as_stream(stream));
    return check_launch("pffmg_phi_coef");
}

extern "C" int pffmg_apply(const pffmg_lattice* lat, const pffmg_state* st, int which,
                           const double* v, double* out, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(v && out && v != out, "pffmg_apply: bad v/out");
    A.v = v;
    A.out = out;
    return dispatch_which<E_STORE>(A, which, as_stream(stream), "pffmg_apply");
}

// Host-buffer form of pffmg_apply: the H2D copy of v, the stencil and the D2H
// copy of the result are overlapped plane strip by plane strip (strip i's
// kernel needs planes [P_i - 1, P_{i+1}] of v, so it waits for the copies of
// strips i and i+1; its output strip goes back while strip i+1 computes).
namespace pffmg {
namespace {
struct PipeRes {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev[3 * 64 + 2] = {};
    bool ok = false;
    // page-locked staging of pffmg_apply_pageable (grown on demand, kept)
    double* stage_in = nullptr;
    double* stage_out = nullptr;
    size_t stage_cap = 0;
};
PipeRes& pipe_res() {
    static thread_local PipeRes R;
    if (!R.ok) {
        bool good = cudaStreamCreateWithFlags(&R.h2d, cudaStreamNonBlocking) == cudaSuccess &&
                    cudaStreamCreateWithFlags(&R.d2h, cudaStreamNonBlocking) == cudaSuccess;
        for (auto& e : R.ev) good = good && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
        R.ok = good;
    }
    return R;
}
}  // namespace
}  // namespace pffmg

extern "C" int pffmg_apply_host(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                const double* h_v, double* h_out, double* d_v, double* d_out,
                                const int64_t* h_plane_off, int n_strips, void* stream) {
    PFFMG_REQUIRE(lat && st && h_v && h_out && d_v && d_out && d_v != d_out, "pffmg_apply_host: bad pointers");
    PFFMG_REQUIRE(which == PFFMG_FULL || which == PFFMG_UBLOCK || which == PFFMG_PBLOCK,
                  "pffmg_apply_host: bad which %d", which);
    const bool q2 = lat->order == 2;
    const int nplanes = q2 ? 2 * lat->ny + 1 : (lat->dim == 3 ? lat->nz : lat->ny) + 1;
    PFFMG_REQUIRE(lat->own_lo == 0 && (lat->own_hi == 0 || lat->own_hi == nplanes),
                  "pffmg_apply_host: needs a whole (non-slab) lattice");
    PFFMG_REQUIRE(lat->vrow_off == nullptr || h_plane_off != nullptr,
                  "pffmg_apply_host: non-box lattices need host plane offsets");
    if (n_strips == 0) {   // zero-copy: the stencil reads v from / writes out to mapped host memory
        void *dv = nullptr, *dout = nullptr;
        if (cudaHostGetDevicePointer(&dv, const_cast<double*>(h_v), 0) != cudaSuccess ||
            cudaHostGetDevicePointer(&dout, h_out, 0) != cudaSuccess) {
            cudaGetLastError();
            set_error("pffmg_apply_host: zero-copy needs page-locked (pinned) host buffers");
            return PFFMG_ERR_ARG;
        }
        return pffmg_apply(lat, st, which, static_cast<const double*>(dv), static_cast<double*>(dout), stream);
    }
    int K = n_strips < 1 ? 1 : (n_strips > 64 ? 64 : n_strips);
    if (K > nplanes) K = nplanes;
    if (lat->order == 2) K = 1;       // Q2: one strip (the kernel does not take node-row ranges)
    PipeRes& R = pipe_res();
    if (!R.ok) {
        set_error("pffmg_apply_host: could not create copy streams/events");
        return PFFMG_ERR_CUDA;
    }
    const cudaStream_t s = as_stream(stream);
    const int64_t V = lat->n_vertices;
    const int nc = which == PFFMG_FULL ? lat->dim + 1 : (which == PFFMG_UBLOCK ? lat->dim : 1);
    const int64_t per_plane = q2 ? (int64_t)(2 * lat->nx + 1)
                                 : (lat->dim == 3 ? (int64_t)(lat->nx + 1) * (lat->ny + 1) : (int64_t)(lat->nx + 1));
    auto off = [&](int p) -> int64_t { return h_plane_off ? h_plane_off[p] : (int64_t)p * per_plane; };
    // Strip i's kernel finalises planes [bound(i), bound(i+1)) and reads one plane
    // more on either side, so copy-in chunk i carries planes up to bound(i+1) + 1
    // (hbound): the kernel then waits for its own chunk only and the copy out of
    // strip i starts one chunk earlier.  The copy out of the last strip runs
    // alone: small strips at both ends shorten the exposed head and tail
    // (triangular weights 1, 2, .., 2, 1).
    static const int tri = [] {
        const char* e = getenv("PFFMG_PIPE_TRI");
        return e ? atoi(e) : 1;
    }();
    int wsum = 0, wcum[65] = {0};
    for (int i = 0; i < K; ++i) {
        const int w = tri ? min(i + 1, K - i) : 1;
        wsum += w;
        wcum[i + 1] = wsum;
    }
    auto bound = [&](int i) -> int { return (int)(((int64_t)nplanes * wcum[i]) / wsum); };
    auto hbound = [&](int i) -> int { return i == 0 ? 0 : (i == K ? nplanes : min(bound(i) + 1, nplanes)); };
    const size_t pitch = (size_t)V * sizeof(double);
    cudaEvent_t* ein = R.ev;          // [K]
    cudaEvent_t* ek = R.ev + 64;      // [K]
    cudaEvent_t e0 = R.ev[192], edone = R.ev[193];
    cudaEventRecord(e0, s);           // d_v / d_out free once prior work on `stream` is done
    cudaStreamWaitEvent(R.h2d, e0, 0);
    cudaStreamWaitEvent(R.d2h, e0, 0);
    // (copies of a few MiB: much smaller ones serialise the two directions on this link)
    auto copy_in = [&](int i) {
        const int64_t a = off(hbound(i)), b = off(hbound(i + 1));
        if (b > a)
            cudaMemcpy2DAsync(d_v + a, pitch, h_v + a, pitch, (size_t)(b - a) * sizeof(double), nc,
                              cudaMemcpyHostToDevice, R.h2d);
        cudaEventRecord(ein[i], R.h2d);
    };
    pffmg_lattice sub = *lat;
    // enqueue order: the copy engine stays one chunk ahead of the stencils, and
    // the first stencil is submitted before the later chunks' API calls
    copy_in(0);
    for (int i = 0; i < K; ++i) {
        if (i + 1 < K) copy_in(i + 1);
        cudaStreamWaitEvent(s, ein[i], 0);
        if (lat->order != 2) {
            sub.own_lo = bound(i);
            sub.own_hi = bound(i + 1);
        }
        if (q2 || sub.own_hi > sub.own_lo) {
            const int rc = pffmg_apply(&sub, st, which, d_v, d_out, stream);
            if (rc) return rc;
        }
        cudaEventRecord(ek[i], s);
        cudaStreamWaitEvent(R.d2h, ek[i], 0);
        const int64_t a = off(bound(i)), b = off(bound(i + 1));
        if (b > a)
            cudaMemcpy2DAsync(h_out + a, pitch, d_out + a, pitch, (size_t)(b - a) * sizeof(double), nc,
                              cudaMemcpyDeviceToHost, R.d2h);
    }
    cudaEventRecord(edone, R.d2h);
    cudaStreamWaitEvent(s, edone, 0);  // the caller's stream orders after the last copy
    return check_launch("pffmg_apply_host");
}

namespace pffmg {
namespace {
int copy_threads() {
    static const int t = [] {
        const char* e = getenv("PFFMG_COPY_THREADS");
        int n = e ? atoi(e) : (int)(std::thread::hardware_concurrency() / 2);
        return n < 1 ? 1 : (n > 16 ? 16 : n);
    }();
    return t;
}

// The host threads of the pageable paths: created once and parked on a
// condition variable between calls (creating a thread in a process with a
// CUDA context costs ~150 us, more than a 4 MiB chunk's copy).  Never
// destroyed: the threads would outlive a static object at exit.  A job owns
// its state (shared_ptr captured by value) and tracks its own completion, so
// nobody waits for a thread that wakes late; it just finds nothing to do.
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool(copy_threads());
        return *p;
    }
    std::mutex exclusive;                  // one job at a time: held by the caller for the whole call
    void start(std::function<void(int)> fn) {
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = std::move(fn);
            ++gen_;
        }
        cv_.notify_all();
    }

  private:
    explicit CopyPool(int n) {
        for (int t = 0; t < n; ++t) std::thread([this, t] { loop(t); }).detach();
    }
    void loop(int t) {
        unsigned long long seen = 0;
        for (;;) {
            std::function<void(int)> job;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                job = job_;
            }
            job(t);
        }
    }
    std::mutex m_;
    std::condition_variable cv_;
    std::function<void(int)> job_;
    unsigned long long gen_ = 0;
};
}  // namespace
}  // namespace pffmg

namespace pffmg {
namespace {
// Shared state of the host copies of one pffmg_apply_pageable call (see
// CopyJob below for why it is shared with the pool threads): pieces of at most
// PIECE doubles, claimed in order -- every chunk's copy-in pieces, then every
// strip's copy-out pieces (which wait for the strip to land).
struct StripJob {
    struct Piece { int strip; int64_t off; int64_t len; };       // off: element offset incl. the component
    static constexpr int64_t PIECE = 64 << 10;
    const double* h_v = nullptr;
    double* h_out = nullptr;
    double* pin = nullptr;
    double* pout = nullptr;
    int K = 0;
    std::vector<Piece> in_pieces, out_pieces;    // claimed in this order: all copy-in, then all copy-out
    int in_cnt[64] = {0};
    std::atomic<int> in_done[64], out_ready[64];
    std::atomic<long long> next{0}, out_done{0};
    std::atomic<int> inflight{0};

    void run_piece(long long q) {                // q already claimed
        const long long PI = (long long)in_pieces.size();
        if (q < PI) {
            const Piece& pc = in_pieces[(size_t)q];
            memcpy(pin + pc.off, h_v + pc.off, (size_t)pc.len * sizeof(double));
            in_done[pc.strip].fetch_add(1, std::memory_order_release);
        } else {
            const Piece& pc = out_pieces[(size_t)(q - PI)];
            int r;
            while ((r = out_ready[pc.strip].load(std::memory_order_acquire)) == 0) std::this_thread::yield();
            if (r > 0) {
                memcpy(h_out + pc.off, pout + pc.off, (size_t)pc.len * sizeof(double));
                out_done.fetch_add(1, std::memory_order_release);
            }
        }
        inflight.fetch_sub(1, std::memory_order_release);
    }
    void work() {
        const long long total = (long long)(in_pieces.size() + out_pieces.size());
        for (;;) {
            inflight.fetch_add(1, std::memory_order_acquire);
            const long long q = next.fetch_add(1, std::memory_order_relaxed);
            if (q >= total) {
                inflight.fetch_sub(1, std::memory_order_release);
                return;
            }
            run_piece(q);
        }
    }
    bool help() {                                // the caller: one piece that cannot block
        const long long PI = (long long)in_pieces.size();
        long long q = next.load(std::memory_order_relaxed);
        if (q >= PI + (long long)out_pieces.size()) return false;
        if (q >= PI && out_ready[out_pieces[(size_t)(q - PI)].strip].load(std::memory_order_acquire) == 0)
            return false;
        inflight.fetch_add(1, std::memory_order_acquire);
        if (next.compare_exchange_strong(q, q + 1, std::memory_order_relaxed))
            run_piece(q);
        else
            inflight.fetch_sub(1, std::memory_order_release);
        return true;
    }
};
}  // namespace
}  // namespace pffmg

// Host-buffer apply for ORDINARY (pageable) memory -- what a numpy caller
// (the reference's drivers) hands over.  A pageable cudaMemcpy is staged by
// the driver on one thread; here copy_threads() host threads move the strips
// of v into a page-locked staging buffer (kept between calls) while earlier
// strips are already on the link, and move finished output strips out of the
// second staging buffer while later strips are still being computed.  The
// stencil launches are those of pffmg_apply_host.  Synchronous: h_out is
// complete when the call returns.
extern "C" int pffmg_apply_pageable(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                    const double* h_v, double* h_out, double* d_v, double* d_out,
                                    const int64_t* h_plane_off, int n_strips, void* stream) {
    PFFMG_REQUIRE(lat && st && h_v && h_out && d_v && d_out && d_v != d_out, "pffmg_apply_pageable: bad pointers");
    PFFMG_REQUIRE(which == PFFMG_FULL || which == PFFMG_UBLOCK || which == PFFMG_PBLOCK,
                  "pffmg_apply_pageable: bad which %d", which);
    const bool q2 = lat->order == 2;
    const int nplanes = q2 ? 2 * lat->ny + 1 : (lat->dim == 3 ? lat->nz : lat->ny) + 1;
    PFFMG_REQUIRE(lat->own_lo == 0 && (lat->own_hi == 0 || lat->own_hi == nplanes),
                  "pffmg_apply_pageable: needs a whole (non-slab) lattice");
    PFFMG_REQUIRE(lat->vrow_off == nullptr || h_plane_off != nullptr,
                  "pffmg_apply_pageable: non-box lattices need host plane offsets");
    int K = n_strips < 1 ? 1 : (n_strips > 64 ? 64 : n_strips);
    if (K > nplanes) K = nplanes;
    if (q2) K = 1;
    PipeRes& R = pipe_res();
    PFFMG_REQUIRE(R.ok, "pffmg_apply_pageable: could not create copy streams/events");
    const cudaStream_t s = as_stream(stream);
    const int64_t V = lat->n_vertices;
    const int nc = which == PFFMG_FULL ? lat->dim + 1 : (which == PFFMG_UBLOCK ? lat->dim : 1);
    const size_t need = (size_t)nc * (size_t)V;
    if (R.stage_cap < need) {
        if (R.stage_in) cudaFreeHost(R.stage_in);
        if (R.stage_out) cudaFreeHost(R.stage_out);
        R.stage_in = R.stage_out = nullptr;
        R.stage_cap = 0;
        if (cudaHostAlloc((void**)&R.stage_in, need * sizeof(double), cudaHostAllocDefault) != cudaSuccess ||
            cudaHostAlloc((void**)&R.stage_out, need * sizeof(double), cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            set_error("pffmg_apply_pageable: could not allocate %zu bytes of page-locked staging",
                      2 * need * sizeof(double));
            return PFFMG_ERR_CUDA;
        }
        R.stage_cap = need;
    }
    double* const pin = R.stage_in;
    double* const pout = R.stage_out;
    const int64_t per_plane = q2 ? (int64_t)(2 * lat->nx + 1)
                                 : (lat->dim == 3 ? (int64_t)(lat->nx + 1) * (lat->ny + 1) : (int64_t)(lat->nx + 1));
    auto off = [&](int p) -> int64_t { return h_plane_off ? h_plane_off[p] : (int64_t)p * per_plane; };
    int wsum = 0, wcum[65] = {0};
    for (int i = 0; i < K; ++i) {
        wsum += min(i + 1, K - i);
        wcum[i + 1] = wsum;
    }
    int64_t lo[65], hlo[65];                     // strip bounds (elements): copy-out / stencil, copy-in
    int pb[65];
    for (int i = 0; i <= K; ++i) {
        pb[i] = (int)(((int64_t)nplanes * wcum[i]) / wsum);
        lo[i] = off(pb[i]);
        // copy-in chunk i carries one plane more than strip i finalises (see pffmg_apply_host)
        hlo[i] = i == 0 ? 0 : off(i == K ? nplanes : min(pb[i] + 1, nplanes));
    }
    CopyPool& pool = CopyPool::get();
    std::lock_guard<std::mutex> pool_guard(pool.exclusive);
    auto J = std::make_shared<StripJob>();
    J->h_v = h_v;
    J->h_out = h_out;
    J->pin = pin;
    J->pout = pout;
    J->K = K;
    for (int i = 0; i < K; ++i) {
        J->in_done[i].store(0, std::memory_order_relaxed);
        J->out_ready[i].store(0, std::memory_order_relaxed);
        for (int c = 0; c < nc; ++c)
            for (int64_t a = hlo[i]; a < hlo[i + 1]; a += StripJob::PIECE) {
                J->in_pieces.push_back({i, (int64_t)c * V + a, std::min<int64_t>(StripJob::PIECE, hlo[i + 1] - a)});
                ++J->in_cnt[i];
            }
        for (int c = 0; c < nc; ++c)
            for (int64_t a = lo[i]; a < lo[i + 1]; a += StripJob::PIECE)
                J->out_pieces.push_back({i, (int64_t)c * V + a, std::min<int64_t>(StripJob::PIECE, lo[i + 1] - a)});
    }
    const long long P = (long long)J->out_pieces.size();
    pool.start([J](int) { J->work(); });         // the calling thread orchestrates the device side and helps
    const size_t pitch = (size_t)V * sizeof(double);
    cudaEvent_t* ein = R.ev;
    cudaEvent_t* ek = R.ev + 64;
    cudaEvent_t* eo = R.ev + 128;
    cudaEvent_t e0 = R.ev[192];
    cudaEventRecord(e0, s);
    cudaStreamWaitEvent(R.h2d, e0, 0);
    cudaStreamWaitEvent(R.d2h, e0, 0);
    pffmg_lattice sub = *lat;
    int rc = PFFMG_OK;
    auto stencil = [&](int i) {                      // strip i: needs copy-in chunks 0..i
        cudaStreamWaitEvent(s, ein[i], 0);
        if (!q2) {
            sub.own_lo = pb[i];
            sub.own_hi = pb[i + 1];
        }
        if (rc == PFFMG_OK && (q2 || sub.own_hi > sub.own_lo)) rc = pffmg_apply(&sub, st, which, d_v, d_out, stream);
        cudaEventRecord(ek[i], s);
        cudaStreamWaitEvent(R.d2h, ek[i], 0);
        if (lo[i + 1] > lo[i])
            cudaMemcpy2DAsync(pout + lo[i], pitch, d_out + lo[i], pitch, (size_t)(lo[i + 1] - lo[i]) * sizeof(double),
                              nc, cudaMemcpyDeviceToHost, R.d2h);
        cudaEventRecord(eo[i], R.d2h);
    };
    for (int i = 0; i < K; ++i) {
        while (J->in_done[i].load(std::memory_order_acquire) < J->in_cnt[i])
            if (!J->help()) std::this_thread::yield();
        if (hlo[i + 1] > hlo[i])
            cudaMemcpy2DAsync(d_v + hlo[i], pitch, pin + hlo[i], pitch, (size_t)(hlo[i + 1] - hlo[i]) * sizeof(double),
                              nc, cudaMemcpyHostToDevice, R.h2d);
        cudaEventRecord(ein[i], R.h2d);
        stencil(i);
    }
    for (int i = 0; i < K; ++i) {
        const bool good = cudaEventSynchronize(eo[i]) == cudaSuccess && rc == PFFMG_OK;
        J->out_ready[i].store(good ? 1 : -1, std::memory_order_release);
        if (!good) {
            for (int k = i + 1; k < K; ++k) J->out_ready[k].store(-1, std::memory_order_release);
            if (rc == PFFMG_OK) {
                set_error("pffmg_apply_pageable: copy-out failed: %s", cudaGetErrorString(cudaGetLastError()));
                rc = PFFMG_ERR_CUDA;
            }
            break;
        }
        J->help();
    }
    while (rc == PFFMG_OK && J->out_done.load(std::memory_order_acquire) < P)   // drain with the pool
        if (!J->help()) std::this_thread::yield();
    // no thread may still be inside a memcpy on the caller's buffers
    while (J->inflight.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    cudaEventRecord(R.ev[193], R.d2h);
    cudaStreamWaitEvent(s, R.ev[193], 0);
    if (rc) return rc;
    return check_launch("pffmg_apply_pageable");
}

// Pageable host <-> device copies for the numpy-facing twins (states, masks,
// right-hand sides and results of a Newton step driven by the reference's own
// Python loop): COPY_CH-byte chunks through a ring of page-locked slots, host
// threads filling / draining the slots while earlier chunks are on the link.
// Synchronous.  dir = 0: host -> device, 1: device -> host.
namespace pffmg {
namespace {
constexpr size_t COPY_CH = (size_t)4 << 20;
constexpr int COPY_SLOTS = 8;

// Shared state of one threaded copy: owned jointly by the caller and by every
// pool thread that picked the job up, so a thread that wakes after the copy
// has finished (a parked thread of a virtualised host can take ~1 ms to wake)
// finds no piece left and touches nothing else -- the caller never waits for it.
struct CopyJob {
    int dir = 0;
    const char* src = nullptr;
    char* dst = nullptr;
    char* ring = nullptr;
    size_t bytes = 0;
    int n = 0;                                   // chunks
    long long total = 0;                         // pieces
    std::atomic<long long> next{0}, done{0};
    std::atomic<int> inflight{0};
    // go[k]: chunk k's slot may be touched (h2d: free; d2h: landed); -1 aborts
    // filled[k]: pieces of chunk k done (h2d: slot written; d2h: slot drained)
    std::unique_ptr<std::atomic<int>[]> go, filled;
    static constexpr size_t PIECE = (size_t)512 << 10;
    static constexpr int PPC = (int)(COPY_CH / PIECE);          // pieces per full chunk

    size_t chunk_len(int k) const { return k + 1 < n ? COPY_CH : bytes - (size_t)k * COPY_CH; }
    int pieces_of(int k) const { return (int)((chunk_len(k) + PIECE - 1) / PIECE); }
    // copy piece q (already claimed); waits for its chunk to become touchable
    void copy_piece(long long q) {
        const int k = (int)(q / PPC), pi = (int)(q % PPC);
        int g;
        while ((g = go[k].load(std::memory_order_acquire)) == 0) std::this_thread::yield();
        if (g > 0) {
            const size_t len = chunk_len(k);
            const size_t a = (size_t)pi * PIECE, b = a + PIECE < len ? a + PIECE : len;
            char* slot = ring + (size_t)(k % COPY_SLOTS) * COPY_CH;
            if (dir == 0)
                memcpy(slot + a, src + (size_t)k * COPY_CH + a, b - a);
            else
                memcpy(dst + (size_t)k * COPY_CH + a, slot + a, b - a);
            filled[k].fetch_add(1, std::memory_order_release);
            done.fetch_add(1, std::memory_order_release);
        }
        inflight.fetch_sub(1, std::memory_order_release);
    }
    void work() {                                // pool threads: pieces in order until none is left
        for (;;) {
            inflight.fetch_add(1, std::memory_order_acquire);
            const long long q = next.fetch_add(1, std::memory_order_relaxed);
            if (q >= total) {
                inflight.fetch_sub(1, std::memory_order_release);
                return;
            }
            copy_piece(q);
            if (go[(int)(q / PPC)].load(std::memory_order_relaxed) < 0) return;
        }
    }
    bool help() {                                // the caller: one piece, only if its chunk is touchable now
        long long q = next.load(std::memory_order_relaxed);
        if (q >= total || go[(int)(q / PPC)].load(std::memory_order_acquire) <= 0) return false;
        inflight.fetch_add(1, std::memory_order_acquire);
        if (next.compare_exchange_strong(q, q + 1, std::memory_order_relaxed))
            copy_piece(q);
        else
            inflight.fetch_sub(1, std::memory_order_release);
        return true;
    }
};

int threaded_copy(int dir, const void* src, void* dst, size_t bytes, cudaStream_t s, const char* what) {
    PFFMG_REQUIRE(src && dst, "%s: null pointer", what);
    if (bytes == 0) return PFFMG_OK;
    PipeRes& R = pipe_res();
    PFFMG_REQUIRE(R.ok, "%s: could not create copy streams/events", what);
    const size_t need = COPY_SLOTS * COPY_CH / sizeof(double);
    if (R.stage_cap < need) {
        if (R.stage_in) cudaFreeHost(R.stage_in);
        if (R.stage_out) cudaFreeHost(R.stage_out);
        R.stage_in = R.stage_out = nullptr;
        R.stage_cap = 0;
        if (cudaHostAlloc((void**)&R.stage_in, need * sizeof(double), cudaHostAllocDefault) != cudaSuccess ||
            cudaHostAlloc((void**)&R.stage_out, need * sizeof(double), cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            set_error("%s: could not allocate page-locked staging", what);
            return PFFMG_ERR_CUDA;
        }
        R.stage_cap = need;
    }
    CopyPool& pool = CopyPool::get();
    std::lock_guard<std::mutex> pool_guard(pool.exclusive);
    auto J = std::make_shared<CopyJob>();
    J->dir = dir;
    J->src = static_cast<const char*>(src);
    J->dst = static_cast<char*>(dst);
    J->ring = reinterpret_cast<char*>(dir == 0 ? R.stage_in : R.stage_out);
    J->bytes = bytes;
    const int n = J->n = (int)((bytes + COPY_CH - 1) / COPY_CH);
    J->total = (long long)(n - 1) * CopyJob::PPC + J->pieces_of(n - 1);
    J->go.reset(new std::atomic<int>[n]);
    J->filled.reset(new std::atomic<int>[n]);
    for (int k = 0; k < n; ++k) {
        J->filled[k].store(0, std::memory_order_relaxed);
        J->go[k].store(dir == 0 && k < COPY_SLOTS ? 1 : 0, std::memory_order_relaxed);
    }
    pool.start([J](int) { J->work(); });
    const cudaStream_t cs = dir == 0 ? R.h2d : R.d2h;
    cudaEvent_t* ev = R.ev;                       // [COPY_SLOTS] of the ring
    cudaEvent_t e0 = R.ev[192];
    cudaEventRecord(e0, s);                       // the device buffer is ready / free on `stream`
    cudaStreamWaitEvent(cs, e0, 0);
    bool good = true;
    auto abort_all = [&]() {
        good = false;
        for (int k = 0; k < n; ++k) J->go[k].store(-1, std::memory_order_release);
    };
    auto await_chunk = [&](int k) {               // all pieces of chunk k done; the caller helps meanwhile
        while (J->filled[k].load(std::memory_order_acquire) < J->pieces_of(k))
            if (!J->help()) std::this_thread::yield();
    };
    if (dir == 0) {
        constexpr int AHEAD = COPY_SLOTS - 2;     // link copies in flight before a slot is recycled
        for (int k = 0; k < n && good; ++k) {
            await_chunk(k);
            cudaMemcpyAsync(J->dst + (size_t)k * COPY_CH, J->ring + (size_t)(k % COPY_SLOTS) * COPY_CH,
                            J->chunk_len(k), cudaMemcpyHostToDevice, cs);
            cudaEventRecord(ev[k % COPY_SLOTS], cs);
            const int j = k - AHEAD;              // chunk j's copy done -> its slot serves chunk j + SLOTS
            if (j >= 0 && j + COPY_SLOTS < n) {
                if (cudaEventSynchronize(ev[j % COPY_SLOTS]) != cudaSuccess) abort_all();
                else J->go[j + COPY_SLOTS].store(1, std::memory_order_release);
            }
        }
        if (good && cudaStreamSynchronize(cs) != cudaSuccess) abort_all();
    } else {
        for (int k = 0; k <= n && good; ++k) {
            if (k < n) {
                if (k >= COPY_SLOTS) await_chunk(k - COPY_SLOTS);   // the slot's previous chunk has been drained
                cudaMemcpyAsync(J->ring + (size_t)(k % COPY_SLOTS) * COPY_CH, J->src + (size_t)k * COPY_CH,
                                J->chunk_len(k), cudaMemcpyDeviceToHost, cs);
                cudaEventRecord(ev[k % COPY_SLOTS], cs);
            }
            const int j = k - 1;
            if (j >= 0) {
                if (cudaEventSynchronize(ev[j % COPY_SLOTS]) != cudaSuccess) abort_all();
                else J->go[j].store(1, std::memory_order_release);
            }
        }
        while (good && J->done.load(std::memory_order_acquire) < J->total)   // drain with the pool
            if (!J->help()) std::this_thread::yield();
    }
    // no thread may still be inside a memcpy on the caller's buffers
    while (J->inflight.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    if (!good) {
        set_error("%s: copy failed: %s", what, cudaGetErrorString(cudaGetLastError()));
        return PFFMG_ERR_CUDA;
    }
    return PFFMG_OK;
}
}  // namespace
}  // namespace pffmg

extern "C" int pffmg_copy_h2d(const void* host, void* device, size_t bytes, void* stream) {
    return threaded_copy(0, host, device, bytes, as_stream(stream), "pffmg_copy_h2d");
}

extern "C" int pffmg_copy_d2h(const void* device, void* host, size_t bytes, void* stream) {
    return threaded_copy(1, device, host, bytes, as_stream(stream), "pffmg_copy_d2h");
}

extern "C" int pffmg_residual(const pffmg_lattice* lat, const pffmg_state* st, int which,
                              const double* x, const double* b, double* out, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && out && x != out, "pffmg_residual: bad x/b/out");
    A.v = x;
    A.b = b;
    A.out = out;
    return dispatch_which<E_RESID>(A, which, as_stream(stream), "pffmg_residual");
}

extern "C" int pffmg_semilinear_residual(const pffmg_lattice* lat, const pffmg_state* st, double* out,
                                         void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(out && A.U && A.pt, "pffmg_semilinear_residual: needs out, U and phi_tilde");
    A.out = out;
    A.v = A.U;   // unused (no v fields in residual mode)
    return launch<M_RES, E_RESZ>(A, as_stream(stream), "pffmg_semilinear_residual");
}

extern "C" int pffmg_diagonal(const pffmg_lattice* lat, const pffmg_state* st, double* out,
                              void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(out && A.U && A.pt, "pffmg_diagonal: needs out, U and phi_tilde");
    A.out = out;
    return launch<M_DIAG, E_DIAG>(A, as_stream(stream), "pffmg_diagonal");
}

extern "C" int pffmg_cheb_step(const pffmg_lattice* lat, const pffmg_state* st, int which,
                               const double* d_in, double* d_out, double* r, double* x,
                               const double* invdiag, double c_dd, double c_dr, int x_add_din,
                               void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && d_out && r && x && invdiag && d_in != d_out && x != d_in,
                  "pffmg_cheb_step: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.c1 = c_dd;
    A.c2 = c_dr;
    A.x_add_din = x_add_din;
    return dispatch_which<E_CHEB>(A, which, as_stream(stream), "pffmg_cheb_step");
}

extern "C" int pffmg_cheb_step_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                  const double* d_in, double* d_out, double* r, double* x,
                                  const double* invdiag, const double* coef, int x_add_din, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && d_out && r && x && invdiag && coef && d_in != d_out && x != d_in,
                  "pffmg_cheb_step_dc: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.coef = coef;
    A.x_add_din = x_add_din;
    return dispatch_which<E_CHEB>(A, which, as_stream(stream), "pffmg_cheb_step_dc");
}

extern "C" int pffmg_cheb_init_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                  const double* x, const double* b, double* r, double* d,
                                  const double* invdiag, const double* theta, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && r && d && invdiag && theta && d != x && r != x, "pffmg_cheb_init_dc: bad pointers");
    A.v = x;
    A.b = b;
    A.r = r;
    A.dout = d;
    A.inv = invdiag;
    A.coef = theta;
    return dispatch_which<E_CHEB0>(A, which, as_stream(stream), "pffmg_cheb_init_dc");
}

extern "C" int pffmg_cheb_step_bd(const pffmg_lattice* lat, const pffmg_state* st, const double* d_in,
                                  double* d_out, double* r, double* x, const double* invdiag,
                                  const double* coef_u, const double* coef_p, int x_add_din, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && d_out && r && x && invdiag && coef_u && coef_p && d_in != d_out && x != d_in,
                  "pffmg_cheb_step_bd: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.coef = coef_u;
    A.coef2 = coef_p;
    A.x_add_din = x_add_din;
    return dispatch_which<E_CHEB>(A, PFFMG_BLOCKDIAG, as_stream(stream), "pffmg_cheb_step_bd");
}

// First Chebyshev step after the x = 0 start (mgsolve.py:95, 103-111 with
// x = 0): the start's residual is the right-hand side itself and its iterate
// is d_in, so the step reads r from `rhs`, never reads x, and writes r, d_out
// and x -- the init then stores d only (r / x = NULL in the *_init_zero* /
// *_init_bd entry points).  Bit-identical to init + pffmg_cheb_step_*.
extern "C" int pffmg_cheb_first_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                   const double* d_in, const double* rhs, double* d_out, double* r, double* x,
                                   const double* invdiag, const double* coef, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && rhs && d_out && r && x && invdiag && coef && d_in != d_out && x != d_in && r != rhs,
                  "pffmg_cheb_first_dc: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r_in = rhs;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.coef = coef;
    A.x_add_din = 2;
    return dispatch_which<E_CHEB>(A, which, as_stream(stream), "pffmg_cheb_first_dc");
}

extern "C" int pffmg_cheb_first_bd(const pffmg_lattice* lat, const pffmg_state* st, const double* d_in,
                                   const double* rhs, double* d_out, double* r, double* x, const double* invdiag,
                                   const double* coef_u, const double* coef_p, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && rhs && d_out && r && x && invdiag && coef_u && coef_p && d_in != d_out && x != d_in &&
                      r != rhs,
                  "pffmg_cheb_first_bd: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r_in = rhs;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.coef = coef_u;
    A.coef2 = coef_p;
    A.x_add_din = 2;
    return dispatch_which<E_CHEB>(A, PFFMG_BLOCKDIAG, as_stream(stream), "pffmg_cheb_first_bd");
}

extern "C" int pffmg_cheb_init_bd(const pffmg_lattice* lat, const pffmg_state* st, const double* x,
                                  const double* b, double* r, double* d, const double* invdiag,
                                  const double* theta_u, const double* theta_p, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && r && d && invdiag && theta_u && theta_p && d != x && r != x,
                  "pffmg_cheb_init_bd: bad pointers");
    A.v = x;
    A.b = b;
    A.r = r;
    A.dout = d;
    A.inv = invdiag;
    A.coef = theta_u;
    A.coef2 = theta_p;
    return dispatch_which<E_CHEB0>(A, PFFMG_BLOCKDIAG, as_stream(stream), "pffmg_cheb_init_bd");
}

extern "C" int pffmg_cheb_init(const pffmg_lattice* lat, const pffmg_state* st, int which,
                               const double* x, const double* b, double* r, double* d,
                               const double* invdiag, double theta, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && r && d && invdiag && d != x && r != x, "pffmg_cheb_init: bad pointers");
    A.v = x;
    A.b = b;
    A.r = r;
    A.dout = d;
    A.inv = invdiag;
    A.c1 = theta;
    return dispatch_which<E_CHEB0>(A, which, as_stream(stream), "pffmg_cheb_init");
}
