// gate_jit.cu -- pass-specialised gate kernels, generated from a pass's op
// program and compiled at run time with NVRTC for sm_100a (SURVEY 8(f)
// NEXT-4).
//
// What it computes: exactly what the op-program interpreter
// (gate_tile_kernel_p / gate_tile_kernel, gate_kernels.cuh) computes for the
// same program -- every op is emitted as a call of the SAME device function
// the interpreter dispatches to (gate_apply<I, K>, apply_linphase, the DIAGT
// factor loop, relayout<L, from, to>), in program order, so results are
// bitwise identical (tests/test_gates_gpu.py).
//
// Why: the interpreter pays per op for uniform loads of 16 coefficients and 5
// metadata words, a switch over (target register bit x matrix shape) and
// predicate set-up -- ncu of the QFT's first pass: 9526 instructions per
// warp-tile, of them 1634 MOV, 925 LOP3, 613 ISETP, 522 BRA next to 2860
// FFMA2/FMUL2, 52 % issue-active (profiles/r1_gate_ncu.json).  With the
// program known at compile time the target bit, shape, masks and layout
// changes are constants and the dispatch disappears.
//
// How: host code generation (one straight-line kernel per distinct program,
// coefficients as exact float bit patterns), NVRTC -> cubin ->
// cudaLibraryLoadData, cached per process by source text.  complex64, one
// GPU / no fused exchange store; other passes keep the interpreter.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gate_kernels.cuh"

namespace sv {

namespace {

#define SV_STR2(x) #x
#define SV_STR(x) SV_STR2(x)

std::string csrc_dir() {
    if (const char *e = getenv("SV_JIT_INCLUDE")) return e;
    Dl_info info{};
    if (dladdr(reinterpret_cast<void *>(&csrc_dir), &info) && info.dli_fname) {
        std::string lib(info.dli_fname);
        const size_t slash = lib.rfind('/');
        return (slash == std::string::npos ? std::string(".") : lib.substr(0, slash)) + "/csrc";
    }
    return "csrc";
}

std::string hexf(float v) {
    unsigned int u;
    memcpy(&u, &v, 4);
    char b[48];
    snprintf(b, sizeof b, "__int_as_float(0x%08xu)", u);
    return b;
}

std::string u32(unsigned int v) { return std::to_string(v) + "u"; }

// Straight-line kernel of one pass program (the interpreter's run_gate_ops,
// unrolled at code-generation time).  glb: the program is read from global
// memory (else it is a __grid_constant__ parameter) -- only merged phase runs
// read it, with the same GLB flavour as the interpreter would use.
std::string generate(const GOp<float> *ops, uint64_t nops, bool lin, bool glb) {
    std::string b;
    b += "#include \"gate_kernels.cuh\"\nusing namespace sv;\n";
    // co-resident CTAs per SM the kernel is compiled for (SV_GATE_JIT_MINB, A/B; default 2 -- the
    // interpreter's; 3 caps registers at 85)
    static const int minb = [] {
        const char *e = getenv("SV_GATE_JIT_MINB");
        return e ? atoi(e) : 2;
    }();
    b += "extern \"C\" __global__ void __launch_bounds__(256, " + std::to_string(minb) + ") sv_gate_jit(const KParams p, ";
    if (lin && !glb) b += "const __grid_constant__ GProg<float> prog, int nops) {\n    const GOp<float> *ops = prog.op;\n";
    else b += "const GOp<float> *__restrict__ ops, int nops) {\n";
    b += "    (void)ops; (void)nops;\n"
         "    using L = Layout<float2, " + std::to_string(kGateTileBitsC64) + ", " + std::to_string(kRegBitsC64) + ">;\n"
         "    extern __shared__ __align__(16) unsigned char smem_raw[];\n"
         "    float2 *sm = reinterpret_cast<float2 *>(smem_raw);\n"
         "    const int tid = threadIdx.x;\n"
         "    const unsigned long long base = tile_base(blockIdx.x, p);\n"
         "    (void)base;\n"
         "    float2 x[L::NR];\n"
         "    global_load<L, 0>(x, reinterpret_cast<const float2 *>(p.in) + base, p, tid);\n";
    unsigned int cur = 0;
    for (uint64_t k = 0; k < nops; ++k) {
        const GOp<float> &o = ops[k];
        const unsigned int kind = o.ph >> 8, ph = o.ph & 0xffu;
        if (ph != cur) {
            b += "    relayout<L, " + std::to_string(cur) + ", " + std::to_string(ph) + ">(x, sm, tid);\n";
            cur = ph;
        }
        const std::string et = "L::ethr(" + std::to_string(cur) + ", (unsigned int)tid)";
        if (kind == GK_LINPHASE) {
            b += "    apply_linphase<L, " + std::string(glb ? "true" : "false") + ">(x, ops + " + std::to_string(k + 1) +
                 ", " + u32(o.tm) + ", " + u32(o.ri) + ", " + u32(o.jm) + ", " + et + ", base, " +
                 u32((unsigned int)o.fm) + ");\n";
            k += o.tm;
            continue;
        }
        std::string cond;
        if (o.tm) cond += "((" + et + " & " + u32(o.tm) + ") == " + u32(o.tm) + ")";
        if (o.fm) {
            if (!cond.empty()) cond += " && ";
            cond += "((base & " + std::to_string(o.fm) + "ull) == " + std::to_string(o.fm) + "ull)";
        }
        b += "    " + (cond.empty() ? std::string("{") : "if (" + cond + ") {") + "  // op " + std::to_string(k) + "\n";
        if (kind == GK_DIAGT) {  // the interpreter's DIAGT branch with constant coefficients
            b += "        const bool one = (" + et + " >> " + u32(o.ri) + ") & 1u;\n"
                 "        const float fr = one ? " + hexf(o.m[6]) + " : " + hexf(o.m[0]) + ";\n"
                 "        const float fi = one ? " + hexf(o.m[7]) + " : " + hexf(o.m[1]) + ";\n"
                 "        if (!(fr == 1.0f && fi == 0.0f)) {\n";
#if SV_GATE_PACKED
            b += "            const float2 pr = make_float2(fr, fr), pi = make_float2(-fi, fi);\n"
                 "#pragma unroll\n"
                 "            for (int j = 0; j < L::NR; ++j)\n"
                 "                if (((unsigned int)j & " + u32(o.jm) + ") == " + u32(o.jm) + ")\n"
                 "                    x[j] = __ffma2_rn(pi, make_float2(x[j].y, x[j].x), __fmul2_rn(pr, x[j]));\n";
#else
            b += "#pragma unroll\n"
                 "            for (int j = 0; j < L::NR; ++j)\n"
                 "                if (((unsigned int)j & " + u32(o.jm) + ") == " + u32(o.jm) + ") cmul_by(x[j], fr, fi);\n";
#endif
            b += "        }\n    }\n";
            continue;
        }
        b += "        const float m[16] = {";
        for (int e = 0; e < 16; ++e) b += hexf(o.m[e]) + (e < 15 ? ", " : "");
        b += "};\n";
        // the interpreter's gate_dispatch: target register index, then shape
        const unsigned int kk = (kind == GK_DIAG || kind == GK_PHASE || kind == GK_ANTI || kind == GK_SWAP) ? kind : GK_GENERAL;
        b += "        gate_apply<" + std::to_string(o.ri) + ", " + u32(kk) + ">(x, m, " + u32(o.jm) + ");\n    }\n";
    }
    b += "    pass_store<L, " + std::to_string(cur) + ", false>(x, reinterpret_cast<float2 *>(p.out) + base, base, p, tid, "
         "static_cast<float2 *const *>(nullptr));\n}\n";
    return b;
}

// One cache entry per distinct kernel source.  The automatic mode compiles in
// the background (one worker thread) and keeps launching the interpreter
// until the cubin is ready -- tiered, never blocking a call on NVRTC; the
// library is loaded on the launching thread at first use.
struct Entry {
    enum State { QUEUED, READY, FAILED } state = QUEUED;
    int device = 0;              // the device of the first request (the worker loads the module there)
    std::vector<char> cubin;
    std::string err;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
};

// Process-lifetime state, deliberately never destroyed: the detached worker
// may still hold it while static destructors run at exit.
struct JitState {
    std::mutex mu;
    std::condition_variable cv;        // worker wake-up / queue drained
    std::map<std::string, Entry> cache;
    std::deque<std::string> queue;     // sources waiting for the worker
    bool busy = false;
    bool stop = false;                 // exit: the worker finishes its current job and returns
    std::thread worker;                // joined at exit (no thread left running during teardown)
    uint64_t compiles = 0;             // kernels loaded for launches
    double compile_s = 0.0;            // NVRTC seconds (worker + synchronous)
};
JitState &J() {
    static JitState *j = new JitState;
    return *j;
}
#define g_mu (J().mu)
#define g_cv (J().cv)
#define g_cache (J().cache)
#define g_queue (J().queue)
#define g_busy (J().busy)
#define g_compiles (J().compiles)
#define g_compile_s (J().compile_s)

// At exit: drop queued work, let a running compile finish and JOIN the
// worker, so no thread of ours is alive while the CUDA runtime and NVRTC are
// torn down (a parked detached worker crashed the process at exit).
void drain_at_exit() {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_queue.clear();
        J().stop = true;
    }
    g_cv.notify_all();
    if (J().worker.joinable()) J().worker.join();
}

std::vector<char> compile_cubin(const std::string &src) {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "sv_gate_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        throw Error{SV_ECUDA, "nvrtcCreateProgram failed"};
    const std::string inc = "-I" + csrc_dir();
    const std::string d1 = "-DSV_GATE_TILE_BITS_C64=" + std::to_string(kGateTileBitsC64);
    const std::string d2 = "-DSV_TILE_BITS_C64=" + std::to_string(kTileBitsC64);
    const std::string d3 = std::string("-DSV_GATE_PACKED=") + SV_STR(SV_GATE_PACKED);
    const std::string d4 = std::string("-DSV_GATE_KINDS=") + SV_STR(SV_GATE_KINDS);
    const std::string d5 = std::string("-DSV_LD_MODE=") + SV_STR(SV_LD_MODE);
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", inc.c_str(), d1.c_str(), d2.c_str(),
                          d3.c_str(), d4.c_str(), d5.c_str()};
    const nvrtcResult r = nvrtcCompileProgram(prog, (int)(sizeof opts / sizeof opts[0]), opts);
    if (r != NVRTC_SUCCESS) {
        size_t ls = 0;
        nvrtcGetProgramLogSize(prog, &ls);
        std::string log(ls, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        nvrtcDestroyProgram(&prog);
        throw Error{SV_ECUDA, std::string("NVRTC: ") + nvrtcGetErrorString(r) + "\n" + log.substr(0, 2000)};
    }
    size_t cs = 0;
    nvrtcGetCUBINSize(prog, &cs);
    std::vector<char> cubin(cs);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    if (const char *dir = getenv("SV_JIT_DUMP")) {  // inspection: source + cubin (cuobjdump -sass)
        const std::string stem = std::string(dir) + "/sv_gate_jit_" + std::to_string(std::hash<std::string>{}(src));
        if (FILE *f = fopen((stem + ".cu").c_str(), "w")) {
            fwrite(src.data(), 1, src.size(), f);
            fclose(f);
        }
        if (FILE *f = fopen((stem + ".cubin").c_str(), "wb")) {
            fwrite(cubin.data(), 1, cubin.size(), f);
            fclose(f);
        }
    }
    return cubin;
}

std::vector<char> timed_compile(const std::string &src) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<char> cubin = compile_cubin(src);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::lock_guard<std::mutex> lk(g_mu);
    g_compile_s += dt;
    return cubin;
}

void load_kernel(const std::vector<char> &cubin, cudaLibrary_t *lib, cudaKernel_t *kern) {
    SV_CUDA(cudaLibraryLoadData(lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    SV_CUDA(cudaLibraryGetKernel(kern, *lib, "sv_gate_jit"));
    SV_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void *>(*kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (1 << kGateTileBitsC64) * (int)sizeof(float2)));
    cudaFuncAttributes fa{};  // forces the module into the current context now
    SV_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void *>(*kern)));
}

void worker_main() {
    std::unique_lock<std::mutex> lk(g_mu);
    for (;;) {
        g_cv.wait(lk, [] { return !g_queue.empty() || J().stop; });
        if (J().stop) return;
        const std::string src = g_queue.front();  // (moved out before the lock is released)
        g_queue.pop_front();
        g_busy = true;
        const int device = g_cache[src].device;
        lk.unlock();
        std::vector<char> cubin;
        std::string err;
        (void)device;
        try {
            cubin = timed_compile(src);  // NVRTC only: the worker makes no CUDA calls
        } catch (const Error &e) {
            err = e.msg;
        }
        lk.lock();
        Entry &e = g_cache[src];
        if (err.empty()) {
            e.cubin.swap(cubin);
            e.state = Entry::READY;
        } else {
            e.err = err;
            e.state = Entry::FAILED;
        }
        g_busy = false;
        g_cv.notify_all();
    }
}


void enqueue_locked(const std::string &src, int device) {
    static std::once_flag once;
    std::call_once(once, [] {
        std::atexit(drain_at_exit);
        J().worker = std::thread(worker_main);
    });
    g_cache[src].device = device;  // QUEUED
    g_queue.push_back(src);
    g_cv.notify_all();
}

// Load a READY entry's cubin on this thread (forced mode).  Caller holds g_mu.
void load_locked(Entry &e) {
    load_kernel(e.cubin, &e.lib, &e.kern);
    ++g_compiles;
}

}  // namespace

// SV_GATE_JIT: "0" never, "1" every complex64 one-GPU pass, compiled before
// its first launch (errors propagate), unset = passes of >= 2^11 tiles (states
// of >= 2^24 amplitudes), compiled in the background on first sight while the
// interpreter runs them (a one-shot circuit never waits for NVRTC; a repeated
// one switches to the specialised kernel once it is ready); a compile failure
// in the automatic mode leaves the pass on the interpreter.
int gate_jit_mode() {
    const char *e = getenv("SV_GATE_JIT");
    if (!e) return 2;
    return strcmp(e, "0") == 0 ? 0 : 1;
}

std::string gate_jit_source(const void *host_ops, uint64_t nops, bool lin, bool glb) {
    return generate(reinterpret_cast<const GOp<float> *>(host_ops), nops, lin, glb);
}

bool launch_gate_jit(const KParams &kp, const void *dev_ops, const void *host_ops, uint64_t nops, bool lin,
                     bool param, unsigned long long ntiles, cudaStream_t s) {
    const int mode = gate_jit_mode();
    if (mode == 0 || host_ops == nullptr) return false;
    if (mode == 2 && ntiles < (1ull << 11)) return false;
    const std::string src = generate(reinterpret_cast<const GOp<float> *>(host_ops), nops, lin, !param);
    cudaKernel_t kern = nullptr;
    {
        std::unique_lock<std::mutex> lk(g_mu);
        auto it = g_cache.find(src);
        if (mode == 1) {  // forced: compile now, errors propagate
            if (it == g_cache.end() || it->second.state == Entry::FAILED) {
                lk.unlock();
                std::vector<char> cubin = timed_compile(src);
                lk.lock();
                Entry &e = g_cache[src];
                if (e.state != Entry::READY) {
                    e.cubin.swap(cubin);
                    e.state = Entry::READY;
                }
                it = g_cache.find(src);
            } else if (it->second.state == Entry::QUEUED) {
                g_cv.wait(lk, [&] { return it->second.state != Entry::QUEUED; });
                if (it->second.state == Entry::FAILED) throw Error{SV_ECUDA, it->second.err};
            }
        } else {  // automatic: queue it and run the interpreter until it is ready
            if (it == g_cache.end()) {
                int dev = 0;
                SV_CUDA(cudaGetDevice(&dev));
                enqueue_locked(src, dev);
                return false;
            }
            if (it->second.state != Entry::READY) {
                if (it->second.state == Entry::FAILED) {
                    static bool warned = false;
                    if (!warned) {
                        fprintf(stderr, "libsv: gate JIT unavailable, using the interpreter kernel: %s\n",
                                it->second.err.c_str());
                        warned = true;
                    }
                }
                return false;
            }
        }
        Entry &e = it->second;
        if (e.kern == nullptr) load_locked(e);
        kern = e.kern;
    }
    KParams p = kp;
    int n = (int)nops;
    const int smem = (1 << kGateTileBitsC64) * (int)sizeof(float2);
    if (lin && param) {
        auto prog = std::make_unique<GProg<float>>();
        memcpy(prog->op, host_ops, nops * sizeof(GOp<float>));
        void *args[] = {&p, prog.get(), &n};
        SV_CUDA(cudaLaunchKernel(reinterpret_cast<const void *>(kern), dim3((unsigned int)ntiles), dim3(256), args,
                                 smem, s));
    } else {
        const void *ops = dev_ops;
        void *args[] = {&p, &ops, &n};
        SV_CUDA(cudaLaunchKernel(reinterpret_cast<const void *>(kern), dim3((unsigned int)ntiles), dim3(256), args,
                                 smem, s));
    }
    return true;
}

// Load every compiled-but-unloaded kernel on the calling thread (run_gates
// calls this before its first launch, outside the launches' profiling events:
// with CUDA's lazy module loading a first launch would otherwise pay the
// module load inside the pass it times).  The background worker itself makes
// no CUDA calls (a worker thread with CUDA state crashed the process at exit).
void gate_jit_load_ready() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &kv : g_cache) {
        Entry &e = kv.second;
        if (e.state == Entry::READY && e.kern == nullptr) load_locked(e);
    }
}

// NVRTC only (no device): the cubin size of the pass kernel, for host tests.
size_t gate_jit_compile_only(const void *host_ops, uint64_t nops, bool lin, bool glb) {
    return compile_cubin(generate(reinterpret_cast<const GOp<float> *>(host_ops), nops, lin, glb)).size();
}

void gate_jit_stats(uint64_t *compiles, double *seconds, bool wait) {
    std::unique_lock<std::mutex> lk(g_mu);
    if (wait) g_cv.wait(lk, [] { return g_queue.empty() && !g_busy; });
    if (compiles) *compiles = g_compiles;
    if (seconds) *seconds = g_compile_s;
}

}  // namespace sv
