// plan.cpp -- host-side schedule of the WHT diffusion (no device code).
//
// A transform applies the butterfly (x, y) -> (x + y, x - y) on every qubit,
// i.e. "a sequence of V/2 independent 2x2 transformations" per bit (section
// 2.1; Fig. 3 with w = x = y = 1, z = -1).  Stages on different
// qubits commute, so a transform may visit the qubits in any grouping; each
// group is one HBM pass of a tile kernel that runs all of the group's stages
// on-chip.
//
// Sharding (section 3.1): with P = 2^g ranks the top g qubits
// are the parallel bits.  "All of the processors can run in parallel
// operating only on local data as long as they do not use any of the QU-bits
// in the set N.  When the computation needs to operate on one of the bits in
// N, a new set is picked and the simulator redistributes the data"
// (P:4108-4111).  Our new set is always the top g LOCAL slots U, so the
// redistribution (Fig. 8) is one all-to-all of contiguous
// chunks; a second one restores the natural layout.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "sv_internal.h"

namespace sv {

static uint64_t range_mask(int lo, int hi) {  // slots [lo, hi)
    uint64_t m = 0;
    for (int s = lo; s < hi; ++s) m |= 1ull << s;
    return m;
}

// Tile of a group: its processed slots plus the lowest unprocessed slots up
// to T (the unprocessed low slots give contiguous runs of >= 64 B).
static Group make_group(uint64_t proc, int T, int nl) {
    Group gr;
    gr.proc = proc;
    gr.tile = proc;
    int have = __builtin_popcountll(proc);
    for (int s = 0; s < nl && have < T; ++s)
        if (!((gr.tile >> s) & 1)) { gr.tile |= 1ull << s; ++have; }
    return gr;
}

// Split an ascending slot list into m near-equal ascending chunks.
static std::vector<uint64_t> chunk(const std::vector<int> &slots, int cap) {
    std::vector<uint64_t> out;
    if (slots.empty()) return out;
    int len = (int)slots.size();
    int m = (len + cap - 1) / cap;
    int base = len / m, extra = len % m, pos = 0;
    for (int i = 0; i < m; ++i) {
        int sz = base + (i < extra ? 1 : 0);
        uint64_t mask = 0;
        for (int j = 0; j < sz; ++j) mask |= 1ull << slots[pos++];
        out.push_back(mask);
    }
    return out;
}

// Test-only override of the one-GPU group split (SV_PLAN_CHUNKS, read at
// sv_init / sv_plan_wht): comma-separated processed-slot counts of the
// strided groups in ascending slot order, each optionally tagged `o` (hosts
// the oracle O) or `f` (hosts F0), e.g. "10o,1f" at n = 24 gives the n = 32
// O-group's shape (10 processed slots, 3 carry slots, U = 3) at a size the
// oracle runs in seconds.  Untagged roles follow the default rule.  Any
// split is a valid schedule: stages on different qubits commute (G18).
struct ChunkOverride {
    std::vector<int> len;
    int og = -1, f0g = -1;  // index into len, -1 = default rule
};

static bool chunk_override(int nstrided, int Rs, ChunkOverride &ov) {
    const char *env = getenv("SV_PLAN_CHUNKS");
    if (!env || !*env) return false;
    std::string s(env);
    size_t pos = 0;
    int sum = 0;
    while (pos < s.size()) {
        size_t end = s.find(',', pos);
        if (end == std::string::npos) end = s.size();
        std::string tok = s.substr(pos, end - pos);
        pos = end + 1;
        SV_CHECK(!tok.empty(), SV_EINVAL, "SV_PLAN_CHUNKS: empty entry");
        char role = 0;
        if (tok.back() == 'o' || tok.back() == 'f') {
            role = tok.back();
            tok.pop_back();
        }
        SV_CHECK(!tok.empty() && tok.find_first_not_of("0123456789") == std::string::npos, SV_EINVAL,
                 "SV_PLAN_CHUNKS: entries are <count>[o|f]");
        const int v = std::stoi(tok);
        SV_CHECK(v >= 1 && v <= Rs, SV_EINVAL, "SV_PLAN_CHUNKS: a group holds 1.." + std::to_string(Rs) + " slots");
        if (role == 'o') {
            SV_CHECK(ov.og < 0, SV_EINVAL, "SV_PLAN_CHUNKS: two O groups");
            ov.og = (int)ov.len.size();
        }
        if (role == 'f') {
            SV_CHECK(ov.f0g < 0, SV_EINVAL, "SV_PLAN_CHUNKS: two F0 groups");
            ov.f0g = (int)ov.len.size();
        }
        ov.len.push_back(v);
        sum += v;
    }
    SV_CHECK(sum == nstrided, SV_EINVAL,
             "SV_PLAN_CHUNKS: counts must add up to the " + std::to_string(nstrided) + " strided slots");
    return true;
}

Plan make_plan(int n, int g, sv_dtype dtype) {
    SV_CHECK(n >= 1 && n <= 40, SV_EINVAL, "n must be in [1, 40]");
    SV_CHECK(dtype == SV_C64 || dtype == SV_C128, SV_EINVAL, "dtype must be SV_C64 or SV_C128");
    SV_CHECK(g >= 0 && g <= 6, SV_EINVAL, "world must be 2^g with g in [0, 6]");
    Plan p;
    p.g = g;
    p.nl = n - g;
    p.T = tile_bits(dtype);
    const int T = p.T, nl = p.nl;
    const int Rs = T - carry_bits(dtype);  // processed slots per strided tile
    if (g == 0 && nl <= T) {                // the whole state is one tile
        p.whole = true;
        return p;
    }
    SV_CHECK(nl - g >= T, SV_EINVAL,
             "shard too small for the sharded WHT: need n - 2*log2(world) >= " + std::to_string(T));
    p.groups.push_back(make_group(range_mask(0, T), T, nl));  // G1: contiguous
    // Which groups host the elementwise ops.  The O- and F0-groups are visited
    // once per iteration with both stage sets fused around the op; the others
    // twice.  Fusing doubles a pass's on-chip work (stages + shared-memory
    // relayouts), so the fused roles go to the groups with the FEWEST
    // processed slots and the contiguous 13-slot G1 -- the cheapest pass to
    // run unfused -- is visited twice.
    auto nproc = [&](int i) { return __builtin_popcountll(p.groups[i].proc); };
    if (g == 0) {
        std::vector<int> rest;
        for (int s = T; s < nl; ++s) rest.push_back(s);
        ChunkOverride ov;
        const bool overridden = chunk_override((int)rest.size(), Rs, ov);
        // Supertile plan (complex64, one GPU): G1 hosts O (fused, visited once
        // per iteration), all remaining R = nl - T slots form ONE group run as
        // an L2-staged supertile pass with F0 -- 2 HBM passes per iteration,
        // the lower bound (each transform must read and write the state once).
        // Level A = 11 slots (tiles of 2 carry + 11 processed slots), level B =
        // the other R - 11 (>= 1).  The supertile (2 + R slots) must leave
        // room in the 126 MB L2 for the sub-passes in flight: 2 + R <=
        // SV_SUPER_MAX_BITS (default 21 = 16 MiB).
        const int R = nl - T;
        static const int super_max = [] {
            const char *e = getenv("SV_SUPER_MAX_BITS");
            return e ? atoi(e) : 21;
        }();
        // measured slower than the plain schedule on the B200 (DESIGN.md
        // "Supertile pass: tried"), so opt-in: SV_SUPER=1
        const char *se = getenv("SV_SUPER");
        const bool super_on = se && strcmp(se, "1") == 0;
        // test-only SV_SUPER_A: level A's slot count (default 11); a small
        // state then gets a large one's level-B tile (e.g. a = 4 at n = 25:
        // level B of 8 slots, n = 32's shape)
        int a = 11;
        if (const char *e = getenv("SV_SUPER_A")) a = atoi(e);
        const int cA = T - a, uB = T - (R - a);
        const bool fits = a >= 1 && a <= 11 && R - a >= 1 && cA + R <= super_max && super_pair_supported(cA, uB);
        if (getenv("SV_SUPER_A") && super_on && dtype == SV_C64 && !overridden)
            SV_CHECK(fits, SV_EINVAL, "SV_SUPER_A: no supertile kernel for this level split");
        if (!overridden && super_on && dtype == SV_C64 && T == 13 && R >= 12 && fits) {
            p.super = true;
            SuperSpec &sp = p.sup;
            sp.procA = range_mask(T, T + a);
            sp.tileA = range_mask(0, cA) | sp.procA;
            sp.procB = range_mask(T + a, nl);
            sp.uB = uB;
            sp.st = range_mask(0, cA) | range_mask(T, nl);
            // level B tiles: its processed slots + the lowest uB other supertile slots
            sp.tileB = sp.procB;
            for (int sl = 0, have = 0; sl < nl && have < uB; ++sl)
                if (((sp.st & ~sp.procB) >> sl) & 1) { sp.tileB |= 1ull << sl; ++have; }
            Group sg;
            sg.proc = range_mask(T, nl);
            sg.tile = sp.st;
            p.groups.push_back(sg);
            sp.group = 1;
            p.fwd = {0, 1};  // O on G1, F0 on the supertile group
            return p;
        }
        if (overridden) {
            size_t pos = 0;
            for (int len : ov.len) {
                uint64_t mask = 0;
                for (int j = 0; j < len; ++j) mask |= 1ull << rest[pos++];
                p.groups.push_back(make_group(mask, T, nl));
            }
        } else {
            // one processed slot more per strided group (2 carry slots, 32-B
            // runs) when that saves a group -- two HBM passes per iteration --
            // e.g. n = 34: 13 | 10 | 11 instead of 13 | 7 | 7 | 7 (SV_WIDE=1;
            // measured in DESIGN.md "Wide strided groups")
            const char *we = getenv("SV_WIDE");
            const bool wide = we && strcmp(we, "1") == 0 && dtype == SV_C64 &&
                              chunk(rest, Rs + 1).size() < chunk(rest, Rs).size();
            for (uint64_t m : chunk(rest, wide ? Rs + 1 : Rs)) p.groups.push_back(make_group(m, T, nl));
        }
        const int ng = (int)p.groups.size();
        std::vector<int> order;
        for (int i = 1; i < ng; ++i)
            if (i - 1 != ov.og && i - 1 != ov.f0g) order.push_back(i);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return nproc(a) < nproc(b); });
        // smallest strided group -> F0; the next one (or G1) -> O; tagged
        // groups of the override take their role first
        size_t next = 0;
        const int f0g = ov.f0g >= 0 ? ov.f0g + 1 : (next < order.size() ? order[next++] : 0);
        const int og = ov.og >= 0 ? ov.og + 1 : (next < order.size() ? order[next++] : 0);
        SV_CHECK(og != f0g, SV_EINVAL, "SV_PLAN_CHUNKS: O and F0 need different groups");
        p.fwd.push_back(og);
        for (int i = 0; i < ng; ++i)
            if (i != og && i != f0g) p.fwd.push_back(i);
        p.fwd.push_back(f0g);
        return p;
    }
    // P > 1: U = top g local slots, processed once before the swap (they hold
    // logical qubits nl-g..nl-1) and once after it (logical nl..n-1).
    std::vector<int> rest;
    for (int s = T; s < nl - g; ++s) rest.push_back(s);
    int take = std::min<int>(Rs - g, (int)rest.size());
    // test-only (SV_PLAN_L1): the post-swap group's processed-slot count,
    // g .. g + take, so small states reproduce the large configs' shapes
    if (const char *env = getenv("SV_PLAN_L1")) {
        const int l1n = atoi(env);
        SV_CHECK(l1n >= g && l1n - g <= take, SV_EINVAL,
                 "SV_PLAN_L1 must be in [" + std::to_string(g) + ", " + std::to_string(g + take) + "]");
        take = l1n - g;
    }
    uint64_t l1 = range_mask(nl - g, nl);
    for (int j = 0; j < take; ++j) l1 |= 1ull << rest[rest.size() - 1 - j];
    rest.resize(rest.size() - take);
    std::vector<int> l0 = rest;
    for (int s = nl - g; s < nl; ++s) l0.push_back(s);
    for (uint64_t m : chunk(l0, Rs)) p.groups.push_back(make_group(m, T, nl));
    // O must run in the natural layout (before the swap): smallest L0 group
    int og = 0;
    for (int i = 1; i < (int)p.groups.size(); ++i)
        if (og == 0 || nproc(i) < nproc(og)) og = i;
    p.fwd.push_back(og);
    for (int i = 0; i < (int)p.groups.size(); ++i)
        if (i != og) p.fwd.push_back(i);
    p.fwd.push_back(-1);  // reorganisation (qubit swap)
    p.groups.push_back(make_group(l1, T, nl));
    p.fwd.push_back((int)p.groups.size() - 1);
    return p;
}

namespace {
enum ItemKind { VISIT, OP, SWAP };
struct Item {
    ItemKind kind;
    int arg;      // group index or MidOp
    int tr = -1;  // VISIT: transform index within the call (2 x iteration + w)
};
}  // namespace

std::vector<Step> schedule_wht(const Plan &plan, int k, bool with_oracle) {
    std::vector<Step> steps;
    if (plan.whole) {
        if (!with_oracle || k > 0) {
            Step s;
            s.kind = STEP_WHOLE;
            steps.push_back(s);
        }
        return steps;
    }
    std::vector<Item> items;
    auto transform = [&](bool forward, int tr) {
        if (forward)
            for (int gi : plan.fwd) items.push_back(gi < 0 ? Item{SWAP, 0} : Item{VISIT, gi, tr});
        else
            for (auto it = plan.fwd.rbegin(); it != plan.fwd.rend(); ++it)
                items.push_back(*it < 0 ? Item{SWAP, 0} : Item{VISIT, *it, tr});
    };
    int reps = with_oracle ? k : 1;
    for (int it = 0; it < reps; ++it) {
        if (with_oracle) items.push_back({OP, MID_ORACLE});
        transform(true, 2 * it);
        items.push_back({OP, MID_F0});
        transform(false, 2 * it + 1);
    }
    // Fuse: visit(G) op visit(G) -> one pass; op visit(G) / visit(G) op at the
    // ends -> one pass; everything else one pass per visit.
    bool after_swap = false;
    int layout = 0;
    size_t i = 0, L = items.size();
    while (i < L) {
        Step s;
        const Item &a = items[i];
        if (a.kind == SWAP) {
            s.kind = STEP_SWAP;
            steps.push_back(s);
            after_swap = true;
            layout ^= 1;
            ++i;
            continue;
        }
        s.kind = STEP_PASS;
        s.in_recv = after_swap ? 1 : 0;
        s.layout = layout;
        after_swap = false;
        if (a.kind == VISIT) {
            s.group = a.arg;
            s.pre = 1;
            s.tr_pre = a.tr;
            if (i + 2 < L && items[i + 1].kind == OP && items[i + 2].kind == VISIT &&
                items[i + 2].arg == a.arg) {
                s.mid = items[i + 1].arg;
                s.post = 1;
                s.tr_post = items[i + 2].tr;
                i += 3;
            } else if (i + 1 < L && items[i + 1].kind == OP &&
                       (i + 2 == L || items[i + 2].kind != VISIT)) {
                s.mid = items[i + 1].arg;
                i += 2;
            } else {
                i += 1;
            }
        } else {  // OP
            if (i + 1 < L && items[i + 1].kind == VISIT) {
                s.group = items[i + 1].arg;
                s.mid = a.arg;
                s.post = 1;
                s.tr_post = items[i + 1].tr;
                i += 2;
            } else {
                s.kind = STEP_SCATTER;
                s.mid = a.arg;
                i += 1;
            }
        }
        // the oracle's per-tile marked lookup (sv_api.cu) is built for the
        // O-group only; by construction O only meets plan.fwd[0]
        if (s.kind == STEP_PASS && s.mid == MID_ORACLE)
            SV_CHECK(s.group == plan.fwd[0], SV_EINVAL, "internal: oracle fused into a non-O group");
        steps.push_back(s);
    }
    for (size_t j = 0; j + 1 < steps.size(); ++j)
        if (steps[j].kind == STEP_PASS && steps[j + 1].kind == STEP_SWAP) steps[j].pre_swap = 1;
    return steps;
}

}  // namespace sv
