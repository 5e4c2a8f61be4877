// capi.cpp — the extern "C" boundary (include/hjmsv_b200.h): solver handles,
// device memory, the step loop (direct launches or one captured CUDA graph per
// full march), status conversion back to the reference's error messages, and
// the multi-GPU batch driver (caplet_ladder's fan-out, instruments.cpp:238-266).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "device_types.hpp"
#include "hjmsv_b200.h"
#include "host_math.hpp"
#include "lowering.hpp"

using namespace hjmsv_b200;

namespace {

thread_local std::string g_err;

struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Failure(HJMSV_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class F>
int32_t guarded(F&& f) {
    try {
        f();
        // surface any asynchronous/unchecked CUDA error at the call that caused it
        const cudaError_t pending = cudaGetLastError();
        if (pending != cudaSuccess && pending != cudaErrorNoDevice &&
            pending != cudaErrorInsufficientDriver) {
            g_err = std::string("CUDA error pending after call: ") + cudaGetErrorString(pending);
            return HJMSV_CUDA_ERROR;
        }
        return HJMSV_OK;
    } catch (const Failure& e) {
        g_err = e.what();
        cudaGetLastError();  // do not leak a sticky error into the next call
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return HJMSV_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return HJMSV_DOMAIN;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return HJMSV_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HJMSV_INVALID_ARGUMENT;
    }
}

// Stage entry points (apply_operator, douglas_step, thomas_batch) run on the
// calling thread's current device, the CUDA runtime convention.
int current_device() {
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    return d;
}

// Device buffers come from the current device's stream-ordered memory pool with
// an unbounded release threshold: a handle's arrays go back to the pool on
// destroy and are reused by the next handle without returning memory to the
// driver (create/destroy per pricing call stays cheap).
void keep_pool() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

template <class T>
T* dalloc(size_t n) {
    keep_pool();
    void* p = nullptr;
    CK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), nullptr));
    CK(cudaStreamSynchronize(nullptr));
    return static_cast<T*>(p);
}

void dfree(void* p) {
    if (p) cudaFreeAsync(p, nullptr);
}

// Process-wide pinned host staging buffers (grow-only, reused across handles):
// descriptor uploads and large grid readouts go through them at full DMA rate
// instead of the driver's pageable path.
struct PinnedBuf {
    void* p = nullptr;
    size_t n = 0;
    bool busy = false;
};
std::mutex g_pin_mu;
std::list<PinnedBuf>& pinned_bufs() {
    static auto* l = new std::list<PinnedBuf>();  // process lifetime (no exit-time cudaFreeHost)
    return *l;
}

class PinnedLease {
  public:
    explicit PinnedLease(size_t bytes) {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto& l = pinned_bufs();
        for (auto& x : l)
            if (!x.busy && x.n >= bytes) { b_ = &x; break; }
        if (!b_)
            for (auto& x : l)
                if (!x.busy) { b_ = &x; break; }
        if (!b_) {
            l.emplace_back();
            b_ = &l.back();
        }
        if (b_->n < bytes) {
            if (b_->p) cudaFreeHost(b_->p);
            b_->p = nullptr;
            b_->n = 0;
            const size_t want = ((bytes + (16u << 20) - 1) >> 24) << 24;  // 16 MiB granules
            CK(cudaMallocHost(&b_->p, want));
            b_->n = want;
        }
        b_->busy = true;
    }
    ~PinnedLease() {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        b_->busy = false;
    }
    PinnedLease(const PinnedLease&) = delete;
    PinnedLease& operator=(const PinnedLease&) = delete;
    template <class T>
    T* as(size_t offset_bytes = 0) const {
        return reinterpret_cast<T*>(static_cast<char*>(b_->p) + offset_bytes);
    }

  private:
    PinnedBuf* b_ = nullptr;
};

// run f(p) for p in [0, count) on up to `workers` host threads
template <class F>
void parallel_for(int count, int workers, F f) {
    workers = std::max(1, std::min(workers, count));
    if (workers == 1) {
        for (int p = 0; p < count; ++p) f(p);
        return;
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w)
        pool.emplace_back([&, w] {
            for (int p = w; p < count; p += workers) f(p);
        });
    for (auto& t : pool) t.join();
}

int host_workers() { return static_cast<int>(std::max(1u, std::thread::hardware_concurrency())); }

// device -> (pageable) host copy of a large readout through pinned staging:
// the DMA of chunk k+1 overlaps the host threads' copy of chunk k
void d2h_staged(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    constexpr size_t CH = 16u << 20;
    if (bytes < 2 * CH) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return;
    }
    PinnedLease lease(2 * CH);
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    const size_t nch = (bytes + CH - 1) / CH;
    auto issue = [&](size_t k) {
        const size_t off = k * CH, n = std::min(CH, bytes - off);
        CK(cudaMemcpyAsync(lease.as<char>((k & 1) * CH), static_cast<const char*>(src) + off, n,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ev[k & 1], st));
    };
    const int nth = std::min(8, host_workers());
    issue(0);
    for (size_t k = 0; k < nch; ++k) {
        if (k + 1 < nch) issue(k + 1);  // its buffer's previous chunk (k-1) is already copied out
        CK(cudaEventSynchronize(ev[k & 1]));
        const size_t off = k * CH, n = std::min(CH, bytes - off);
        const size_t per = (n / nth + 63) & ~size_t(63);
        parallel_for(nth, nth, [&](int t) {
            const size_t a = std::min(n, t * per), e = std::min(n, a + per);
            if (e > a) std::memcpy(static_cast<char*>(dst) + off + a, lease.as<char>((k & 1) * CH) + a, e - a);
        });
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
}

}  // namespace

struct hjmsv_solver {
    int device = 0;
    int mode = HJMSV_MODE_STRICT;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int P = 0, nr = 0, nv = 0, ny = 0, S = 0;
    long long N = 0;
    std::vector<double> maturity, spot_w_host;
    std::vector<long long> spot_idx_host;
    std::vector<std::vector<double>> term_steps;  // per problem: t_next per step
    std::vector<double> bound;
    // device
    double *U = nullptr, *D = nullptr, *C = nullptr, *U0 = nullptr;
    double *axes = nullptr, *steps = nullptr, *fast = nullptr, *fb = nullptr;
    double* ab = nullptr;      // per-step a_i, b_i (model functions of t only)
    double* ylu = nullptr;     // y-line pivot table of pass B (constant models, two-pass shapes)
    ProblemConst* pc = nullptr;
    DevStatus* st = nullptr;
    long long* spot_idx = nullptr;
    double *spot_w = nullptr, *spot_out = nullptr;
    BatchView view{};
    int step = 0;
    double last_ms = 0.0;
    long long last_launches = 0;
    double wall_seconds = 0.0;
    cudaGraphExec_t graph = nullptr;
    long long graph_launches = 0;
    int full_marches = 0;      // full marches launched on this handle
    std::vector<hjmsv_report> reports;
    std::vector<std::string> messages;
    std::vector<Lowered> low;  // host tables (init freed) for readouts
    bool stage = false;        // single-step stage handle: messages unprefixed

    ~hjmsv_solver() {
        if (device >= 0) cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);  // buffers return to the pool only when idle
        if (graph) cudaGraphExecDestroy(graph);
        for (void* p : {(void*)U, (void*)D, (void*)C, (void*)U0, (void*)axes, (void*)steps,
                        (void*)fast, (void*)fb, (void*)ab, (void*)ylu, (void*)pc, (void*)st, (void*)spot_idx, (void*)spot_w,
                        (void*)spot_out})
            dfree(p);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

void enqueue_steps(hjmsv_solver* h, int from, int count, long long* launches) {
    for (int s = from; s < from + count; ++s) {
        const int flags = (s == from ? STEP_FIRST : 0) | (s == from + count - 1 ? STEP_LAST : 0);
        if (h->mode == HJMSV_MODE_FAST)
            fast_step(h->view, s, h->stream, launches, nullptr, flags);
        else
            strict_step(h->view, s, h->stream, launches);
    }
}

std::string status_message(hjmsv_solver* h, int p, const DevStatus& ds, int* code,
                           int* row) {
    const std::string prefix =
        h->stage ? std::string()
                 : "step " + std::to_string(ds.fail_step) + "/" + std::to_string(h->S) + ": ";
    *row = -1;
    // a singular pivot of the failing step wins over a guard hit of the same
    // step: the reference's sweeps all run before guard_finite (solver.cpp:121-176)
    if (ds.pivot_key != ~0ull) {
        *code = HJMSV_SINGULAR_PIVOT;
        *row = static_cast<int>(ds.pivot_key & 0xFFFFFull);
        return prefix + "thomas_solve: singular pivot at row " + std::to_string(*row);
    }
    if (ds.nonfinite_first < ds.diverge_first) {
        *code = HJMSV_NONFINITE;
        return prefix + "solution left the finite range (NaN/Inf)";
    }
    *code = HJMSV_DIVERGED;
    return prefix + "solution exceeded the divergence bound " + std::to_string(h->bound[p]);
}

int collect(hjmsv_solver* h) {
    CK(cudaStreamSynchronize(h->stream));
    std::vector<DevStatus> ds(h->P);
    CK(cudaMemcpy(ds.data(), h->st, sizeof(DevStatus) * h->P, cudaMemcpyDeviceToHost));
    int first = HJMSV_OK;
    for (int p = 0; p < h->P; ++p) {
        hjmsv_report& r = h->reports[p];
        r.n_steps = h->S;
        r.wall_seconds = h->wall_seconds;
        if (ds[p].fail_step) {
            int code = 0, row = -1;
            h->messages[p] = status_message(h, p, ds[p], &code, &row);
            r.status = code;
            r.failed_step = ds[p].fail_step;
            r.failed_row = row;
            r.nan_guard_ok = 0;
            r.steps_done = ds[p].fail_step - 1;
            if (first == HJMSV_OK) {
                first = code;
                g_err = h->messages[p];
            }
        } else {
            r.status = HJMSV_OK;
            r.failed_step = 0;
            r.failed_row = -1;
            r.nan_guard_ok = 1;
            r.steps_done = h->step;
            double md;
            const unsigned long long bits = ds[p].maxdelta_bits;
            std::memcpy(&md, &bits, sizeof(md));
            if (h->step > 0) r.last_max_delta = md;
            // run() lands exactly on t = 0 after the march (solver.cpp:253)
            r.time = h->step >= h->S ? 0.0
                     : h->step == 0  ? h->maturity[p]
                                     : h->term_steps[p][h->step - 1];
        }
    }
    return first;
}

struct StageOverride {
    double t_from = 0.0, dt = 0.0, dt_mult = 0.0;
    bool faces = true, apply_only = false;
};

// HJMSV_TIMING=1: phase times of hjmsv_solver_create on stderr (diagnostic)
struct PhaseTimer {
    bool on;
    std::chrono::steady_clock::time_point t0;
    PhaseTimer() : on(std::getenv("HJMSV_TIMING") != nullptr), t0(std::chrono::steady_clock::now()) {}
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[hjmsv create] %-22s %8.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

hjmsv_solver* create_handle(const hjmsv_problem* problems, int count,
                            const hjmsv_solver_config& cfg, int device, int mode,
                            const StageOverride* ov = nullptr) {
    PhaseTimer pt;
    if (!problems || count < 1) throw std::invalid_argument("no problems given");
    if (mode != HJMSV_MODE_STRICT && mode != HJMSV_MODE_FAST)
        throw std::invalid_argument("unknown arithmetic mode");
    std::vector<Lowered> L(count);
    // FAST marches build the terminal level on the device;
    // STRICT keeps the host restatement, bit-identical to smooth_terminal
    const int init_mode = (mode == HJMSV_MODE_FAST && !ov) ? INIT_DEVICE : INIT_HOST;
    {
        // lower the problems on all host cores (each lowering is independent)
        std::vector<std::exception_ptr> errs(count);
        auto one = [&](int p) {
            try {
                L[p] = lower_problem(problems[p], cfg, init_mode);
            } catch (...) {
                errs[p] = std::current_exception();
            }
        };
        const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        const int workers = init_mode == INIT_DEVICE ? std::min(hw, count) : 1;
        if (workers <= 1) {
            for (int p = 0; p < count; ++p) one(p);
        } else {
            std::vector<std::thread> pool;
            for (int w = 0; w < workers; ++w)
                pool.emplace_back([&, w] {
                    for (int p = w; p < count; p += workers) one(p);
                });
            for (auto& t : pool) t.join();
        }
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);  // the first problem's error, in input order
    }
    pt.mark("lower");
    for (int p = 0; p < count; ++p) {
        if (ov) {  // one explicit level (t_from, dt): the douglas_step / apply_operator stages
            L[p].n_steps = 1;
            L[p].dt = ov->dt;
            L[p].pc.dt = ov->dt_mult;
            L[p].pc.theta_dt = cfg.theta_cn * ov->dt;
            build_step_table(L[p], {ov->t_from}, ov->dt, ov->faces);
            build_model_steps(L[p]);
        }
        if (L[p].nr != L[0].nr || L[p].nv != L[0].nv || L[p].ny != L[0].ny ||
            L[p].n_steps != L[0].n_steps)
            throw std::invalid_argument("batched problems must share grid dims and step count");
    }
    // model functions of t anywhere in the batch: every problem gets per-step
    // coefficient tables (a constant model's are its constants, step by step)
    bool timedep = false;
    for (int p = 0; p < count; ++p) timedep = timedep || L[p].timedep;
    if (timedep)
        for (int p = 0; p < count; ++p)
            if (!L[p].timedep) {
                L[p].timedep = true;
                build_model_steps(L[p]);
            }
    if (mode == HJMSV_MODE_FAST && !fast_supported(L[0].nr, L[0].nv, L[0].ny))
        throw Failure(HJMSV_UNSUPPORTED, "FAST kernels do not support this grid shape");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw std::invalid_argument("no such CUDA device");
    auto h = std::make_unique<hjmsv_solver>();
    h->device = device;
    CK(cudaSetDevice(device));
    h->mode = mode;
    h->P = count;
    h->nr = L[0].nr;
    h->nv = L[0].nv;
    h->ny = L[0].ny;
    h->S = L[0].n_steps;
    h->N = static_cast<long long>(h->nr) * h->nv * h->ny;
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    const size_t PN = static_cast<size_t>(count) * h->N;
    const int astride = axes_stride(h->nr, h->nv, h->ny);
    h->U = dalloc<double>(PN);
    h->D = dalloc<double>(PN);
    h->U0 = dalloc<double>(PN);
    // the Thomas c' scratch of the STRICT sweeps; FAST allocates it on the first
    // readout that needs a second grid-sized buffer (Greeks / surface)
    if (mode == HJMSV_MODE_STRICT) h->C = dalloc<double>(PN);
    h->axes = dalloc<double>(static_cast<size_t>(count) * astride);
    h->steps = dalloc<double>(static_cast<size_t>(count) * h->S * kStepStride);
    h->pc = dalloc<ProblemConst>(count);
    h->st = dalloc<DevStatus>(count);
    h->spot_idx = dalloc<long long>(static_cast<size_t>(count) * 8);
    h->spot_w = dalloc<double>(static_cast<size_t>(count) * 8);
    h->spot_out = dalloc<double>(count);
    pt.mark("alloc");
    std::vector<ProblemConst> pcs(count);
    h->spot_idx_host.resize(static_cast<size_t>(count) * 8);
    h->spot_w_host.resize(static_cast<size_t>(count) * 8);
    h->term_steps.resize(count);
    // per-problem axes and per-step tables packed into pinned staging, in parallel
    const size_t steps_n = static_cast<size_t>(count) * h->S * kStepStride;
    const size_t axes_n = static_cast<size_t>(count) * astride;
    PinnedLease stage(sizeof(double) * (steps_n + axes_n));
    double* steps_h = stage.as<double>();
    double* axes_h = steps_h + steps_n;
    parallel_for(count, count >= 64 ? host_workers() : 1, [&](int p) {
        const Lowered& l = L[p];
        std::copy(l.axes.begin(), l.axes.end(), axes_h + static_cast<size_t>(p) * astride);
        std::copy(l.steps.begin(), l.steps.end(), steps_h + static_cast<size_t>(p) * h->S * kStepStride);
    });
    std::vector<TermParam> term_h(count);
    std::vector<int> term_kind(count);
    for (int p = 0; p < count; ++p) h->term_steps[p].reserve(h->S);
    for (int p = 0; p < count; ++p) {
        const Lowered& l = L[p];
        term_h[p] = l.term;
        term_kind[p] = l.term.kind;
        if (l.term.kind == TERM_HOST)
            CK(cudaMemcpy(h->U0 + static_cast<size_t>(p) * h->N, l.init.data(),
                          sizeof(double) * h->N, cudaMemcpyHostToDevice));
        pcs[p] = l.pc;
        std::copy(l.spot_idx, l.spot_idx + 8, h->spot_idx_host.begin() + p * 8);
        std::copy(l.spot_w, l.spot_w + 8, h->spot_w_host.begin() + p * 8);
        h->maturity.push_back(l.maturity);
        h->bound.push_back(l.pc.bound);
        for (int s = 0; s < h->S; ++s)
            h->term_steps[p].push_back(l.steps[static_cast<size_t>(s) * kStepStride + ST_TNEXT]);
    }
    CK(cudaMemcpyAsync(h->axes, axes_h, sizeof(double) * axes_n, cudaMemcpyHostToDevice, h->stream));
    if (timedep) {  // [P][S][2 nr] a_i, b_i of every step's prepare(t_mid)
        const size_t ab_n = 2 * static_cast<size_t>(h->nr) * h->S;
        h->ab = dalloc<double>(static_cast<size_t>(count) * ab_n);
        for (int p = 0; p < count; ++p)
            CK(cudaMemcpy(h->ab + static_cast<size_t>(p) * ab_n, L[p].ab_steps.data(), sizeof(double) * ab_n,
                          cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpyAsync(h->steps, steps_h, sizeof(double) * steps_n, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));  // the staging buffer is released with this scope
    CK(cudaMemcpy(h->pc, pcs.data(), sizeof(ProblemConst) * count, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->spot_idx, h->spot_idx_host.data(), sizeof(long long) * 8 * count,
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->spot_w, h->spot_w_host.data(), sizeof(double) * 8 * count,
                  cudaMemcpyHostToDevice));
    pt.mark("pack + H2D tables");
    BatchView& v = h->view;
    v.P = count;
    v.nr = h->nr;
    v.nv = h->nv;
    v.ny = h->ny;
    v.N = h->N;
    v.S = h->S;
    v.y_order = cfg.y_boundary_order;
    v.r_order = cfg.r_boundary_order;
    v.dxr = L[0].r.dx();
    v.dxv = L[0].v.dx();
    v.dxy = L[0].y.dx();
    v.U = h->U;
    v.D = h->D;
    v.C = h->C;
    v.axes = h->axes;
    v.axes_stride = astride;
    v.pc = h->pc;
    v.steps = h->steps;
    v.ab = h->ab;
    v.fast_step = 0;
    v.st = h->st;
    v.apply_only = ov && ov->apply_only ? 1 : 0;
    v.dmask = 0;
    for (int f = 0; f < 6; ++f) {
        const bool dir = pcs[0].rule[f] == RULE_DIRICHLET;
        for (int p = 1; p < count; ++p)
            if ((pcs[p].rule[f] == RULE_DIRICHLET) != dir)
                throw std::invalid_argument("batched problems must share face rules");
        // is_dirichlet / dirichlet_value ignore the faces of a singleton axis
        // (discretization.cpp:153-192: r_.n > 1, v_.n > 1, y_.n > 1)
        const int n_axis = f < 2 ? h->nr : (f < 4 ? h->nv : h->ny);
        if (dir && n_axis > 1) v.dmask |= 1 << f;
    }
    h->stage = ov != nullptr;
    if (mode == HJMSV_MODE_FAST) {
        // one table per problem, or one per (problem, step) with model functions of t
        const int tab = fast_stride(h->nr, h->nv, h->ny);
        const int nsteps_tab = timedep ? h->S : 1;
        v.fast_step = timedep ? tab : 0;
        v.fast_stride = tab * nsteps_tab;
        h->fast = dalloc<double>(static_cast<size_t>(count) * v.fast_stride);
        v.fast = h->fast;
        v.fb_stride = 2 * h->ny + 2 * h->nr + 2 * h->nr * h->ny;
        h->fb = dalloc<double>(2 * static_cast<size_t>(count) * v.fb_stride);  // two step parities
        v.fb = h->fb;
        const size_t fast_n = static_cast<size_t>(count) * v.fast_stride;
        PinnedLease fstage(sizeof(double) * fast_n);
        double* fast_h = fstage.as<double>();
        parallel_for(count, count >= 64 ? host_workers() : 1, [&](int p) {
            for (int st = 0; st < nsteps_tab; ++st) {
                const std::vector<double> ft = build_fast_tables(L[p], cfg, L[p].pc.theta_dt, timedep ? st : -1);
                std::copy(ft.begin(), ft.end(),
                          fast_h + static_cast<size_t>(p) * v.fast_stride + static_cast<size_t>(st) * tab);
            }
        });
        CK(cudaMemcpyAsync(h->fast, fast_h, sizeof(double) * fast_n, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        pt.mark("fast tables");
        // constant models: the y-line matrices are the same at every step, so their
        // pivots (the reference's Thomas order) are computed once; a vanishing or
        // non-finite pivot keeps the handle on the partition method, which reports it
        if (fast_ylu_supported(v)) {
            h->ylu = dalloc<double>(PN);
            int* flag = dalloc<int>(count);
            CK(cudaMemsetAsync(flag, 0, sizeof(int) * count, h->stream));
            fast_ylu_build(v, h->ylu, flag, h->stream);
            std::vector<int> fl(count);
            CK(cudaMemcpyAsync(fl.data(), flag, sizeof(int) * count, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            dfree(flag);
            bool ok = true;
            for (int f : fl) ok = ok && f == 0;
            if (ok) {
                v.ylu = h->ylu;
            } else {
                dfree(h->ylu);
                h->ylu = nullptr;
            }
            pt.mark("y-line pivots");
        }
    }
    if (init_mode == INIT_DEVICE) {
        TermParam* tp = dalloc<TermParam>(count);
        CK(cudaMemcpy(tp, term_h.data(), sizeof(TermParam) * count, cudaMemcpyHostToDevice));
        device_terminal(v, tp, term_kind.data(), h->U0, h->stream);
        CK(cudaStreamSynchronize(h->stream));
        dfree(tp);
        pt.mark("device terminal");
    }
    h->reports.assign(count, hjmsv_report{});
    h->messages.assign(count, std::string());
    for (auto& r : h->reports) r.failed_row = -1;
    CK(cudaMemcpyAsync(h->U, h->U0, sizeof(double) * PN, cudaMemcpyDeviceToDevice, h->stream));
    reset_status(v, h->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    for (auto& l : L) {
        l.init.clear();
        l.init.shrink_to_fit();
        l.steps.clear();
        l.steps.shrink_to_fit();
        l.ab_steps.clear();
        l.ab_steps.shrink_to_fit();
    }
    h->low = std::move(L);
    pt.mark("U0 -> U, status");
    return h.release();
}

struct ProfCtx {
    std::vector<std::string>* names;  // by kernel slot
    std::vector<double>* bytes;
};

void prof_after(void* vctx, int idx, const char* name, double b) {
    auto* c = static_cast<ProfCtx*>(vctx);
    if (idx >= static_cast<int>(c->names->size())) {
        c->names->resize(idx + 1);
        c->bytes->resize(idx + 1, 0.0);
    }
    (*c->names)[idx] = name;
    (*c->bytes)[idx] = b;
}

}  // namespace

namespace {
// one problem's second grid-sized readout buffer (FAST handles allocate it on demand)
void ensure_scratch(hjmsv_solver* h) {
    if (!h->C) {
        h->C = dalloc<double>(static_cast<size_t>(h->N));
        h->view.C = h->C;
    }
}
}  // namespace

extern "C" {

// Per-kernel durations inside a march launched exactly as the first march of a
// handle (direct launches, programmatic dependent launch between the passes):
// every block of every FAST kernel records its start (after the programmatic
// wait) and end on %globaltimer into a per-(step, kernel) min/max pair, so a
// kernel's duration is the span of its own blocks and the durations of one
// step add up to at most the step (no host events between the launches).
int32_t hjmsv_solver_kernel_timeline(hjmsv_solver* h, int32_t steps, int32_t max_kernels,
                                     double* avg_ms, double* alg_bytes, int64_t* launches_out,
                                     int32_t* n_kernels, char* names, int32_t name_len,
                                     double* march_ms) {
    return guarded([&] {
        if (!h || !avg_ms || !alg_bytes || !n_kernels) throw std::invalid_argument("null argument");
        if (h->mode != HJMSV_MODE_FAST) throw Failure(HJMSV_UNSUPPORTED, "kernel timeline: FAST mode only");
        CK(cudaSetDevice(h->device));
        const int count = std::min(steps, h->S - h->step);
        if (count < 1) throw std::invalid_argument("no steps left to profile (reset first)");
        std::vector<std::string> nm;
        std::vector<double> by;
        ProfCtx ctx{&nm, &by};
        LaunchHook hook;
        hook.after = prof_after;
        hook.ctx = &ctx;
        const size_t n_tl = static_cast<size_t>(count) * kTlSlots;
        std::vector<unsigned long long> tl(2 * n_tl);
        for (size_t q = 0; q < n_tl; ++q) {
            tl[2 * q] = ~0ull;
            tl[2 * q + 1] = 0ull;
        }
        unsigned long long* dtl = nullptr;
        CK(cudaMalloc(&dtl, sizeof(unsigned long long) * tl.size()));
        CK(cudaMemcpy(dtl, tl.data(), sizeof(unsigned long long) * tl.size(), cudaMemcpyHostToDevice));
        BatchView v = h->view;
        // step s of the march writes entry s - h->step
        v.tl = dtl - 2 * static_cast<size_t>(h->step) * kTlSlots;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, h->stream));
        long long n = 0;
        for (int s = h->step; s < h->step + count; ++s) {
            const int flags = (s == h->step ? STEP_FIRST : 0) | (s == h->step + count - 1 ? STEP_LAST : 0);
            fast_step(v, s, h->stream, &n, &hook, flags);
        }
        CK(cudaEventRecord(e1, h->stream));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
        float total = 0.f;
        CK(cudaEventElapsedTime(&total, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        CK(cudaMemcpy(tl.data(), dtl, sizeof(unsigned long long) * tl.size(), cudaMemcpyDeviceToHost));
        cudaFree(dtl);
        h->step += count;
        const int K = std::min<int>(max_kernels, static_cast<int>(std::min<size_t>(nm.size(), kTlSlots)));
        for (int q = 0; q < K; ++q) {
            double sum_ns = 0.0;
            int calls = 0;
            for (int s = 0; s < count; ++s) {
                const unsigned long long a = tl[2 * (static_cast<size_t>(s) * kTlSlots + q)];
                const unsigned long long b = tl[2 * (static_cast<size_t>(s) * kTlSlots + q) + 1];
                if (a != ~0ull && b > a) {
                    sum_ns += static_cast<double>(b - a);
                    ++calls;
                }
            }
            avg_ms[q] = calls ? 1e-6 * sum_ns / calls : 0.0;
            alg_bytes[q] = by[q] * static_cast<double>(h->N) * h->P;
            if (names && name_len > 0) {
                std::strncpy(names + static_cast<size_t>(q) * name_len, nm[q].c_str(), name_len - 1);
                names[static_cast<size_t>(q) * name_len + name_len - 1] = 0;
            }
        }
        *n_kernels = K;
        if (launches_out) *launches_out = n;
        if (march_ms) *march_ms = total;
    });
}

int32_t hjmsv_solver_kernel_profile(hjmsv_solver* h, int32_t steps, int32_t max_kernels,
                                    double* avg_ms, double* alg_bytes, int64_t* launches_out,
                                    int32_t* n_kernels, char* names, int32_t name_len) {
    return hjmsv_solver_kernel_timeline(h, steps, max_kernels, avg_ms, alg_bytes, launches_out,
                                        n_kernels, names, name_len, nullptr);
}

void hjmsv_default_solver_config(hjmsv_solver_config* cfg) {
    if (cfg) *cfg = default_config();
}

const char* hjmsv_last_error(void) { return g_err.c_str(); }
int32_t hjmsv_abi_version(void) { return HJMSV_ABI_VERSION; }

int32_t hjmsv_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int32_t hjmsv_uniform_axis(double z0, double z_inf, int32_t n, double* z, double* j1, double* j2) {
    return guarded([&] {
        Axis a = make_uniform_axis(z0, z_inf, n);
        std::copy(a.z.begin(), a.z.end(), z);
        std::copy(a.j1.begin(), a.j1.end(), j1);
        std::copy(a.j2.begin(), a.j2.end(), j2);
    });
}

int32_t hjmsv_sinh_axis(double center, double alpha, double z0, double z_inf, int32_t n,
                        double* z, double* j1, double* j2, double* c1c2) {
    return guarded([&] {
        Axis a = make_sinh_axis(center, alpha, z0, z_inf, n);
        std::copy(a.z.begin(), a.z.end(), z);
        std::copy(a.j1.begin(), a.j1.end(), j1);
        std::copy(a.j2.begin(), a.j2.end(), j2);
        if (c1c2) {
            c1c2[0] = a.c1;
            c1c2[1] = a.c2;
        }
    });
}

int32_t hjmsv_curve_eval(const hjmsv_curve* c, int32_t what, int32_t count, const double* t,
                         double* out) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("curve must be given");
        hjmsv_problem tmp{};
        Curve curve = c->kind == HJMSV_CURVE_FLAT
                          ? Curve::flat(c->flat_base)
                          : [&] {
                                std::vector<std::pair<double, double>> nodes;
                                for (int i = 0; i < c->n_nodes; ++i)
                                    nodes.emplace_back(c->maturities[i], c->discounts[i]);
                                return Curve::from_nodes(std::move(nodes));
                            }();
        (void)tmp;
        for (int q = 0; q < count; ++q)
            out[q] = what == 0   ? curve.discount(t[q])
                     : what == 1 ? curve.forward(t[q])
                                 : curve.forward_slope(t[q]);
    });
}

int32_t hjmsv_zcb_closed_form(const hjmsv_curve* c, double kappa, double t, double maturity,
                              double x, double y, double* out) {
    return guarded([&] {
        Curve curve = c->kind == HJMSV_CURVE_FLAT
                          ? Curve::flat(c->flat_base)
                          : [&] {
                                std::vector<std::pair<double, double>> nodes;
                                for (int i = 0; i < c->n_nodes; ++i)
                                    nodes.emplace_back(c->maturities[i], c->discounts[i]);
                                return Curve::from_nodes(std::move(nodes));
                            }();
        *out = zcb_closed_form(t, maturity, x, y, curve, kappa);
    });
}

int32_t hjmsv_solver_create(const hjmsv_problem* problems, int32_t count,
                            const hjmsv_solver_config* cfg, int32_t device, int32_t mode,
                            hjmsv_solver** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("output handle pointer is null");
        *out = nullptr;
        *out = create_handle(problems, count, cfg ? *cfg : default_config(), device, mode);
    });
}

void hjmsv_solver_destroy(hjmsv_solver* h) { delete h; }

int32_t hjmsv_solver_reset(hjmsv_solver* h) {
    return guarded([&] {
        if (!h) throw std::invalid_argument("null handle");
        CK(cudaSetDevice(h->device));
        CK(cudaMemcpyAsync(h->U, h->U0, sizeof(double) * h->P * h->N, cudaMemcpyDeviceToDevice,
                           h->stream));
        reset_status(h->view, h->stream);
        CK(cudaGetLastError());
        h->step = 0;
        for (auto& r : h->reports) {
            r = hjmsv_report{};
            r.failed_row = -1;
        }
    });
}

int32_t hjmsv_solver_step_async(hjmsv_solver* h, int32_t steps) {
    return guarded([&] {
        if (!h) throw std::invalid_argument("null handle");
        if (steps < 0) throw std::invalid_argument("step count must be nonnegative");
        CK(cudaSetDevice(h->device));
        const int count = std::min(steps, h->S - h->step);
        h->last_launches = 0;
        CK(cudaEventRecord(h->ev0, h->stream));
        if (count > 0 && h->step == 0 && count == h->S && h->full_marches++ > 0) {
            // a repeated full march (reset + run on the same handle): one captured
            // graph, instantiated once per handle. The first march of a handle is
            // launched directly: its launches overlap the kernels, while capture
            // and instantiation (several ms for 2000 launches) would delay them all
            if (!h->graph) {
                cudaGraph_t g = nullptr;
                CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
                long long n = 0;
                enqueue_steps(h, 0, h->S, &n);
                CK(cudaStreamEndCapture(h->stream, &g));
                CK(cudaGraphInstantiate(&h->graph, g, 0));
                cudaGraphDestroy(g);
                h->graph_launches = n;
            }
            CK(cudaGraphLaunch(h->graph, h->stream));
            h->last_launches = h->graph_launches;
        } else if (count > 0) {
            enqueue_steps(h, h->step, count, &h->last_launches);
        }
        CK(cudaEventRecord(h->ev1, h->stream));
        CK(cudaGetLastError());
        h->step += count;
    });
}

int32_t hjmsv_solver_synchronize(hjmsv_solver* h) {
    int32_t first = HJMSV_OK;
    int32_t code = guarded([&] {
        if (!h) throw std::invalid_argument("null handle");
        CK(cudaSetDevice(h->device));
        first = collect(h);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        h->last_ms = ms;
    });
    return code != HJMSV_OK ? code : first;
}

int32_t hjmsv_solver_step(hjmsv_solver* h, int32_t steps) {
    const auto t0 = std::chrono::steady_clock::now();
    int32_t code = hjmsv_solver_step_async(h, steps);
    if (code != HJMSV_OK) return code;
    code = hjmsv_solver_synchronize(h);
    if (h) {
        h->wall_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& r : h->reports) r.wall_seconds = h->wall_seconds;
    }
    return code;
}

int32_t hjmsv_solver_run(hjmsv_solver* h) {
    if (!h) {
        g_err = "null handle";
        return HJMSV_INVALID_ARGUMENT;
    }
    return hjmsv_solver_step(h, h->S - h->step);
}

int32_t hjmsv_solver_report(hjmsv_solver* h, int32_t problem, hjmsv_report* out) {
    return guarded([&] {
        if (!h || !out) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        *out = h->reports[problem];
    });
}

int32_t hjmsv_solver_dims(hjmsv_solver* h, int32_t* nr, int32_t* nv, int32_t* ny,
                          int32_t* count, int32_t* n_steps) {
    return guarded([&] {
        if (!h) throw std::invalid_argument("null handle");
        if (nr) *nr = h->nr;
        if (nv) *nv = h->nv;
        if (ny) *ny = h->ny;
        if (count) *count = h->P;
        if (n_steps) *n_steps = h->S;
    });
}

int32_t hjmsv_solver_get_grid(hjmsv_solver* h, int32_t problem, double* host_out) {
    return guarded([&] {
        if (!h || !host_out) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        CK(cudaSetDevice(h->device));
        d2h_staged(host_out, h->U + static_cast<size_t>(problem) * h->N, sizeof(double) * h->N, h->stream);
    });
}

int32_t hjmsv_solver_greeks(hjmsv_solver* h, int32_t problem, int32_t scale_rate, double* rho,
                            double* vega) {
    return guarded([&] {
        if (!h) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        if (h->nr == 2 || h->nv == 2)
            throw Failure(HJMSV_UNSUPPORTED, "extract_greeks needs 1 or >= 3 nodes per axis");
        CK(cudaSetDevice(h->device));
        ensure_scratch(h);
        // D / C are step workspaces, free between steps
        greeks(h->view, problem, scale_rate ? 1 : 0, h->low[problem].r0, h->D, h->C, h->stream);
        CK(cudaGetLastError());
        if (rho)
            CK(cudaMemcpyAsync(rho, h->D, sizeof(double) * h->N, cudaMemcpyDeviceToHost, h->stream));
        if (vega)
            CK(cudaMemcpyAsync(vega, h->C, sizeof(double) * h->N, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int32_t hjmsv_solver_surface(hjmsv_solver* h, int32_t problem, int32_t k, double* out) {
    return guarded([&] {
        if (!h || !out) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        if (k < 0 || k >= h->ny) throw std::invalid_argument("slice index out of range");
        if (h->nr == 2 || h->nv == 2)
            throw Failure(HJMSV_UNSUPPORTED, "extract_greeks needs 1 or >= 3 nodes per axis");
        CK(cudaSetDevice(h->device));
        ensure_scratch(h);
        const double r0 = h->low[problem].r0;
        greeks(h->view, problem, 1, r0, h->D, h->C, h->stream);
        const size_t rows = static_cast<size_t>(h->nr) * h->nv;
        double* dev = dalloc<double>(rows * 5);
        surface(h->view, problem, k, r0, h->D, h->C, dev, h->stream);
        CK(cudaGetLastError());
        const cudaError_t e = cudaMemcpyAsync(out, dev, sizeof(double) * rows * 5,
                                              cudaMemcpyDeviceToHost, h->stream);
        const cudaError_t e2 = e == cudaSuccess ? cudaStreamSynchronize(h->stream) : e;
        dfree(dev);
        CK(e2);
    });
}

void hjmsv_default_mc_config(hjmsv_mc_config* cfg) {
    if (!cfg) return;
    cfg->n_paths = 200000;  // McConfig defaults, montecarlo.hpp:15-24
    cfg->steps_per_year = 96;
    cfg->seed = 20070423ull;
    cfg->full_truncation = 1;
}

int32_t hjmsv_mc_price(const hjmsv_problem* problem, const hjmsv_mc_config* cfg, int32_t device,
                       double* mean, double* std_error, int64_t* n_paths) {
    return guarded([&] {
        if (!problem || !cfg || !mean || !std_error || !n_paths) throw std::invalid_argument("null argument");
        const McSetup m = lower_mc(*problem, *cfg);
        *n_paths = cfg->n_paths;
        if (m.horizon == 0.0) {  // simulate(): horizon 0 returns payout(0, 0, 1), montecarlo.cpp:92
            *mean = 1.0;
            *std_error = 0.0;
            return;
        }
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw std::invalid_argument("no such CUDA device");
        CK(cudaSetDevice(device));
        McParams mp{};
        mp.n_paths = cfg->n_paths;
        mp.n_steps = m.n_steps;
        mp.full_truncation = cfg->full_truncation ? 1 : 0;
        mp.seed = cfg->seed;
        mp.dt = m.dt;
        mp.sqrt_dt = m.sqrt_dt;
        mp.decay_y = m.decay_y;
        mp.decay_h = m.decay_h;
        mp.f0 = m.f0;
        const hjmsv_model& md = problem->model;
        mp.kappa = md.kappa;
        mp.theta = md.theta;
        mp.rho = md.rho;
        mp.sq1mr2 = std::sqrt(1.0 - md.rho * md.rho);
        mp.caplet = m.caplet;
        mp.accrual = m.accrual;
        mp.ratio = m.ratio;
        mp.g = m.g;
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const long long want = (cfg->n_paths + 255) / 256;
        const int blocks = static_cast<int>(std::min<long long>(want, 8LL * sms));
        double* f = dalloc<double>(m.steps.size());
        double* part = dalloc<double>(2 * static_cast<size_t>(blocks));
        std::vector<double> ph(2 * static_cast<size_t>(blocks));
        cudaError_t e = cudaMemcpy(f, m.steps.data(), sizeof(double) * m.steps.size(),
                                   cudaMemcpyHostToDevice);
        if (e == cudaSuccess) {
            mc_simulate(mp, f, part, blocks, nullptr);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess)
            e = cudaMemcpy(ph.data(), part, sizeof(double) * ph.size(), cudaMemcpyDeviceToHost);
        dfree(f);
        dfree(part);
        CK(e);
        double sum = 0.0, sum_sq = 0.0;  // block order: independent of scheduling
        for (int b = 0; b < blocks; ++b) {
            sum += ph[2 * b];
            sum_sq += ph[2 * b + 1];
        }
        const double n = static_cast<double>(cfg->n_paths);
        const double mu = sum / n;  // simulate(), montecarlo.cpp:130-137
        const double var = cfg->n_paths > 1 ? std::max(0.0, (sum_sq - n * mu * mu) / (n - 1)) : 0.0;
        *mean = mu;
        *std_error = std::sqrt(var / n);
    });
}

int32_t hjmsv_solver_get_grids(hjmsv_solver* h, double* host_out) {
    return guarded([&] {
        if (!h || !host_out) throw std::invalid_argument("null argument");
        CK(cudaSetDevice(h->device));
        d2h_staged(host_out, h->U, sizeof(double) * h->N * h->P, h->stream);
    });
}

int32_t hjmsv_solver_set_grid(hjmsv_solver* h, int32_t problem, const double* host_in,
                              int32_t step_index) {
    return guarded([&] {
        if (!h || !host_in) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        if (step_index < 0 || step_index > h->S) throw std::invalid_argument("step index out of range");
        CK(cudaSetDevice(h->device));
        CK(cudaMemcpyAsync(h->U + static_cast<size_t>(problem) * h->N, host_in,
                           sizeof(double) * h->N, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->step = step_index;
    });
}

int32_t hjmsv_solver_price(hjmsv_solver* h, int32_t problem, double zr, double zv, double zy,
                           double* out) {
    return guarded([&] {
        if (!h || !out) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        long long idx[8];
        double w[8];
        locate_point(h->low[problem], zr, zv, zy, idx, w);
        CK(cudaSetDevice(h->device));
        double val[8];
        const double* U = h->U + static_cast<size_t>(problem) * h->N;
        for (int c = 0; c < 8; ++c)
            CK(cudaMemcpyAsync(&val[c], U + idx[c], sizeof(double), cudaMemcpyDeviceToHost,
                               h->stream));
        CK(cudaStreamSynchronize(h->stream));
        double acc = 0.0;  // interpolate_at accumulation order (instruments.cpp:77-87)
        for (int c = 0; c < 8; ++c) {
            if (w[c] == 0.0) continue;
            acc += w[c] * val[c];
        }
        *out = acc;
    });
}

int32_t hjmsv_solver_spot_prices(hjmsv_solver* h, double* out) {
    return guarded([&] {
        if (!h || !out) throw std::invalid_argument("null argument");
        CK(cudaSetDevice(h->device));
        gather_spot(h->view, h->spot_idx, h->spot_w, h->spot_out, h->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, h->spot_out, sizeof(double) * h->P, cudaMemcpyDeviceToHost,
                           h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int32_t hjmsv_solver_device_grid(hjmsv_solver* h, int32_t problem, double** dev_ptr) {
    return guarded([&] {
        if (!h || !dev_ptr) throw std::invalid_argument("null argument");
        if (problem < 0 || problem >= h->P) throw std::invalid_argument("problem index out of range");
        *dev_ptr = h->U + static_cast<size_t>(problem) * h->N;
    });
}

int32_t hjmsv_solver_last_device_ms(hjmsv_solver* h, double* ms) {
    return guarded([&] {
        if (!h || !ms) throw std::invalid_argument("null argument");
        *ms = h->last_ms;
    });
}

int32_t hjmsv_solver_last_launches(hjmsv_solver* h, int64_t* launches) {
    return guarded([&] {
        if (!h || !launches) throw std::invalid_argument("null argument");
        *launches = h->last_launches;
    });
}

int32_t hjmsv_apply_operator(const hjmsv_problem* p, const hjmsv_solver_config* cfg, double t,
                             const double* u, double* out, int32_t mode) {
    return guarded([&] {
        if (!p || !u || !out) throw std::invalid_argument("null argument");
        hjmsv_problem q = *p;
        q.initial_grid = u;
        q.n_steps = 1;
        StageOverride ov;
        ov.t_from = t;  // dt = 0: t_mid = t exactly
        ov.dt = 0.0;
        ov.dt_mult = 1.0;
        ov.faces = false;
        ov.apply_only = true;
        const hjmsv_solver_config c = cfg ? *cfg : default_config();
        std::unique_ptr<hjmsv_solver> h(create_handle(&q, 1, c, current_device(), mode, &ov));
        if (mode == HJMSV_MODE_FAST)
            fast_explicit(h->view, 0, h->stream);
        else
            strict_explicit(h->view, 0, h->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, h->D, sizeof(double) * h->N, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int32_t hjmsv_douglas_step(const hjmsv_problem* p, const hjmsv_solver_config* cfg,
                           const double* u_in, double t_from, double dt, double* u_out,
                           double* max_delta, int32_t mode) {
    int32_t status = HJMSV_OK;
    int32_t code = guarded([&] {
        if (!p || !u_in || !u_out) throw std::invalid_argument("null argument");
        hjmsv_problem q = *p;
        q.initial_grid = u_in;
        q.n_steps = 1;
        StageOverride ov;
        ov.t_from = t_from;
        ov.dt = dt;
        ov.dt_mult = dt;
        const hjmsv_solver_config c = cfg ? *cfg : default_config();
        std::unique_ptr<hjmsv_solver> h(create_handle(&q, 1, c, current_device(), mode, &ov));
        status = hjmsv_solver_step(h.get(), 1);
        CK(cudaMemcpyAsync(u_out, h->U, sizeof(double) * h->N, cudaMemcpyDeviceToHost,
                           h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (max_delta) *max_delta = h->reports[0].last_max_delta;
        if (status != HJMSV_OK) throw Failure(status, h->messages[0]);
    });
    return code;
}

int32_t hjmsv_thomas_batch(int32_t n, int32_t count, const double* lower, const double* diag,
                           const double* upper, const double* super2, double* rhs,
                           int32_t mode) {
    return guarded([&] {
        if (n < 0 || count < 0) throw std::invalid_argument("negative size");
        if (n == 0 || count == 0) return;
        if (!lower || !diag || !upper || !super2 || !rhs) throw std::invalid_argument("null argument");
        if (mode < HJMSV_MODE_STRICT || mode > HJMSV_THOMAS_FAST_TWISTED)
            throw std::invalid_argument("unknown arithmetic mode");
        if (mode != HJMSV_MODE_STRICT && n > 512)
            throw Failure(HJMSV_UNSUPPORTED, "FAST lines hold at most 32 segments of 16 rows (n <= 512)");
        // the calling thread's current device (cudaSetDevice), as every stage entry point
        const size_t m = static_cast<size_t>(n) * count;
        double *dl = dalloc<double>(m), *dd = dalloc<double>(m), *du = dalloc<double>(m);
        double *ds2 = dalloc<double>(count), *dr = dalloc<double>(m), *dsc = dalloc<double>(m);
        int* dfail = dalloc<int>(count);
        auto cleanup = [&] {  // idempotent: pointers are cleared once freed
            dfree(dl); dfree(dd); dfree(du); dfree(ds2); dfree(dr); dfree(dsc); dfree(dfail);
            dl = dd = du = ds2 = dr = dsc = nullptr;
            dfail = nullptr;
        };
        try {
            CK(cudaMemcpy(dl, lower, m * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dd, diag, m * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(du, upper, m * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(ds2, super2, static_cast<size_t>(count) * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dr, rhs, m * 8, cudaMemcpyHostToDevice));
            thomas_batch(n, count, dl, dd, du, ds2, dr, dsc, dfail, mode, nullptr);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            std::vector<int> fail(count);
            CK(cudaMemcpy(fail.data(), dfail, sizeof(int) * count, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(rhs, dr, m * 8, cudaMemcpyDeviceToHost));
            cleanup();
            for (int q = 0; q < count; ++q)
                if (fail[q] >= 0)
                    throw Failure(HJMSV_SINGULAR_PIVOT,
                                  "thomas_solve: singular pivot at row " + std::to_string(fail[q]));
        } catch (...) {
            cleanup();
            throw;
        }
    });
}

int32_t hjmsv_batch_run(const hjmsv_problem* problems, int32_t count,
                        const hjmsv_solver_config* cfg, const int32_t* devices,
                        int32_t n_devices, int32_t mode, double* prices_out,
                        hjmsv_report* reports_out, double* grids_out) {
    return guarded([&] {
        if (!problems || count < 1) throw std::invalid_argument("no problems given");
        std::vector<int> devs;
        if (devices && n_devices > 0)
            devs.assign(devices, devices + n_devices);
        else
            devs.push_back(0);
        const int G = static_cast<int>(std::min<size_t>(devs.size(), static_cast<size_t>(count)));
        const hjmsv_solver_config c = cfg ? *cfg : default_config();
        // contiguous shards of ceil(count/G) problems
        const int per = (count + G - 1) / G;
        // grids_out holds the problems' grids back to back in input order; each
        // problem's offset is the prefix sum of nr*nv*ny (dims may differ between shards)
        std::vector<size_t> goff(static_cast<size_t>(count) + 1, 0);
        for (int q = 0; q < count; ++q) {
            const hjmsv_problem& pq = problems[q];
            if (pq.r.n < 1 || pq.v.n < 1 || pq.y.n < 1)
                throw std::invalid_argument("axis sizes must be positive");
            goff[q + 1] = goff[q] + static_cast<size_t>(pq.r.n) * pq.v.n * pq.y.n;
        }
        std::vector<std::thread> pool;
        std::vector<int> codes(G, HJMSV_OK);
        std::vector<std::string> errs(G);
        for (int g = 0; g < G; ++g) {
            const int lo = g * per, hi = std::min(count, lo + per);
            if (lo >= hi) continue;
            pool.emplace_back([&, g, lo, hi] {
                hjmsv_solver* h = nullptr;
                int code = hjmsv_solver_create(problems + lo, hi - lo, &c, devs[g], mode, &h);
                if (code == HJMSV_OK) code = hjmsv_solver_run(h);
                if (h) {
                    const int run_code = code;
                    std::vector<double> pr(hi - lo);
                    // readout failures are reported too, after the march's own status
                    int read_code = hjmsv_solver_spot_prices(h, pr.data());
                    auto keep = [&](int c2) {
                        if (read_code == HJMSV_OK) read_code = c2;
                    };
                    for (int q = lo; q < hi; ++q) {
                        hjmsv_report r{};
                        keep(hjmsv_solver_report(h, q - lo, &r));
                        if (prices_out)
                            prices_out[q] = r.status == HJMSV_OK ? pr[q - lo] : std::nan("");
                        if (reports_out) reports_out[q] = r;
                        if (grids_out) keep(hjmsv_solver_get_grid(h, q - lo, grids_out + goff[q]));
                    }
                    code = run_code != HJMSV_OK ? run_code : read_code;
                    hjmsv_solver_destroy(h);
                }
                codes[g] = code;
                errs[g] = g_err;
            });
        }
        for (auto& t : pool) t.join();
        for (int g = 0; g < G; ++g)
            if (codes[g] != HJMSV_OK) throw Failure(codes[g], errs[g]);
    });
}

}  // extern "C"
