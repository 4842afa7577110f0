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
#include <map>
#include <memory>
#include <mutex>
#include <string>
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
std::string generate(const GOp<float> *ops, uint64_t nops, bool lin, bool glb, bool l2) {
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
         "    using L = " + (l2 ? "Layout2<" + std::to_string(kGateTileBitsC64) + ", " + std::to_string(kRegBitsC64) + ">"
                          : "Layout<float2, " + std::to_string(kGateTileBitsC64) + ", " + std::to_string(kRegBitsC64) + ">") + ";\n"
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

// One cache entry per distinct kernel source.  Tiering without a thread: the
// automatic mode leaves a program's first call on the interpreter (a one-shot
// circuit never waits for NVRTC) and compiles it, synchronously, when a
// later call meets it again.  (A background compiler thread was tried: NVRTC's
// lazily-constructed statics are destroyed by exit() while a compile can still
// be running on it, which crashed processes at exit.)
struct Entry {
    enum State { SEEN, READY, FAILED } state = SEEN;
    uint64_t call = 0;           // the run_gates call that first saw it (SEEN)
    std::vector<char> cubin;     // kept alive for the library's lifetime
    std::string err;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
};

// Process-lifetime state, deliberately never destroyed (no teardown order
// against the CUDA runtime at exit).
struct JitState {
    std::mutex mu;
    std::map<std::string, Entry> cache;
    uint64_t compiles = 0;             // kernels compiled and loaded for launches
    double compile_s = 0.0;            // NVRTC seconds
};
JitState &J() {
    static JitState *j = new JitState;
    return *j;
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

// Compile and load one entry on the calling thread.  Caller holds J().mu.
void compile_load_locked(const std::string &src, Entry &e) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<char> cubin = compile_cubin(src);
    J().compile_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    e.cubin.swap(cubin);
    SV_CUDA(cudaLibraryLoadData(&e.lib, e.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    SV_CUDA(cudaLibraryGetKernel(&e.kern, e.lib, "sv_gate_jit"));
    SV_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void *>(e.kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (1 << kGateTileBitsC64) * (int)sizeof(float2)));
    cudaFuncAttributes fa{};  // forces the module into the current context now, not at the first launch
    SV_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void *>(e.kern)));
    e.state = Entry::READY;
    ++J().compiles;
}

}  // namespace

// SV_GATE_JIT: "0" never, "1" every complex64 one-GPU pass, compiled before
// its first launch (errors propagate), unset = passes of >= 2^11 tiles (states
// of >= 2^24 amplitudes) from the second call that runs the same program on
// (the first runs the interpreter); a compile failure in the automatic mode
// leaves the pass on the interpreter.
int gate_jit_mode() {
    const char *e = getenv("SV_GATE_JIT");
    if (!e) return 2;
    return strcmp(e, "0") == 0 ? 0 : 1;
}

std::string gate_jit_source(const void *host_ops, uint64_t nops, bool lin, bool glb, bool l2) {
    return generate(reinterpret_cast<const GOp<float> *>(host_ops), nops, lin, glb, l2);
}

// Before a run_gates call launches anything (host work only; module loads
// stay out of the passes' profiling events): decide and, where due, compile
// this pass's kernel.  Returns the kernel to launch, or nullptr for the
// interpreter.  `call` numbers the run_gates calls (>= 1).
void *gate_jit_prepare(const void *host_ops, uint64_t nops, bool lin, bool param, bool l2, unsigned long long ntiles,
                       uint64_t call) {
    const int mode = gate_jit_mode();
    if (mode == 0 || host_ops == nullptr) return nullptr;
    if (mode == 2 && ntiles < (1ull << 11)) return nullptr;
    const std::string src = generate(reinterpret_cast<const GOp<float> *>(host_ops), nops, lin, !param, l2);
    std::lock_guard<std::mutex> lk(J().mu);
    auto it = J().cache.find(src);
    if (it == J().cache.end()) {
        Entry &e = J().cache[src];
        e.call = call;
        if (mode == 2) return nullptr;  // first sight: the interpreter
        compile_load_locked(src, e);    // forced: errors propagate
        return e.kern;
    }
    Entry &e = it->second;
    if (e.state == Entry::READY) return e.kern;
    if (e.state == Entry::SEEN && mode == 2 && e.call == call) return nullptr;  // again within the first call
    if (e.state == Entry::FAILED && mode == 2) return nullptr;
    if (mode == 1) {
        compile_load_locked(src, e);
        return e.kern;
    }
    try {  // automatic, second call: compile now; a failure keeps the interpreter
        compile_load_locked(src, e);
        return e.kern;
    } catch (const Error &err) {
        e.state = Entry::FAILED;
        e.err = err.msg;
        fprintf(stderr, "libsv: gate JIT unavailable, using the interpreter kernel: %s\n", e.err.c_str());
        return nullptr;
    }
}

void launch_gate_jit(void *kern, const KParams &kp, const void *dev_ops, const void *host_ops, uint64_t nops,
                     bool lin, bool param, unsigned long long ntiles, cudaStream_t s) {
    KParams p = kp;
    int n = (int)nops;
    const int smem = (1 << kGateTileBitsC64) * (int)sizeof(float2);
    if (lin && param) {
        auto prog = std::make_unique<GProg<float>>();
        memcpy(prog->op, host_ops, nops * sizeof(GOp<float>));
        void *args[] = {&p, prog.get(), &n};
        SV_CUDA(cudaLaunchKernel(kern, dim3((unsigned int)ntiles), dim3(256), args, smem, s));
    } else {
        const void *ops = dev_ops;
        void *args[] = {&p, &ops, &n};
        SV_CUDA(cudaLaunchKernel(kern, dim3((unsigned int)ntiles), dim3(256), args, smem, s));
    }
}

// NVRTC only (no device): the cubin size of the pass kernel, for host tests.
size_t gate_jit_compile_only(const void *host_ops, uint64_t nops, bool lin, bool glb, bool l2) {
    return compile_cubin(generate(reinterpret_cast<const GOp<float> *>(host_ops), nops, lin, glb, l2)).size();
}

void gate_jit_stats(uint64_t *compiles, double *seconds) {
    std::lock_guard<std::mutex> lk(J().mu);
    if (compiles) *compiles = J().compiles;
    if (seconds) *seconds = J().compile_s;
}

}  // namespace sv
