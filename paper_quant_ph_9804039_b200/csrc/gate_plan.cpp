// gate_plan.cpp -- host-side schedule of a gate circuit (
// no device code).
//
// A gate is Fig. 3's 2x2 on one qubit, replicated over the V/2 pairs
// (section 2.1), optionally controlled (G23).  On
// the B200 a gate costs one HBM read + write of the state if run alone; the
// planner packs runs of gates whose targets fit one tile (<= T physical
// slots, the tile also holding the low "carry" slots so each tile row is a
// >= 64 B contiguous run) into ONE tile pass that applies them all on-chip.
//
// Order: gates are taken greedily left to right.  A later gate may join the
// current pass ahead of gates it skips only if it commutes with every skipped
// gate (CommuteSet: sufficient conditions), so the result is the circuit's
// product exactly (up to rounding order).
//
// Sharding (section 3.1): "All of the processors can run in
// parallel operating only on local data as long as they do not use any of
// the QU-bits in the set N.  When the computation needs to operate on one of
// the bits in N, a new set is picked and the simulator redistributes the data"
// (Fig. 8).  Our new set is always the top g local slots, so a
// swap is one all-to-all of contiguous chunks and the layout is either
// natural or swapped; a pass that cannot take any pending gate means the next
// gate targets a rank bit -> swap.  Controls need no locality: a control on a
// rank bit is decided per rank, on a slot outside the tile per tile.
#include <algorithm>

#include "sv_internal.h"

namespace sv {

static void validate_gate(int n, const sv_gate &g, uint64_t j) {
    const uint64_t all = (n >= 64) ? ~0ull : ((1ull << n) - 1ull);
    SV_CHECK(g.target >= 0 && g.target < n, SV_EINVAL,
             "gate " + std::to_string(j) + ": target " + std::to_string(g.target) + " not in [0, n)");
    SV_CHECK(g.reserved == 0, SV_EINVAL, "gate " + std::to_string(j) + ": reserved field must be 0");
    SV_CHECK((g.controls & ~all) == 0, SV_EINVAL, "gate " + std::to_string(j) + ": control qubit >= n");
    SV_CHECK(((g.controls >> g.target) & 1ull) == 0, SV_EINVAL,
             "gate " + std::to_string(j) + ": a gate cannot control its own target");
}

// Ops a pass runs after the host merging of gates.cu (build_tile_ops):
//  * a phase gate diag(1, z) with at most one control joins an earlier run
//    on the same target when only commuting gates lie between; runs of >= 4
//    become one phase-polynomial op (*lin counts them), shorter runs stay
//    one op per gate;
//  * any other gate with the same target and controls as an earlier op, with
//    only commuting ops in between, is multiplied into it.
static bool phase1_gate(const sv_gate &g) {
    return g.m[0] == 1.0 && g.m[1] == 0.0 && gate_diag(g) && __builtin_popcountll(g.controls) <= 1;
}

uint64_t fused_op_count(const sv_gate *gates, const uint64_t *order, uint64_t count, uint64_t *lin) {
    struct Op {
        const sv_gate *g;
        sv_gate proxy;   // merged phase run: target + union of controls, diagonal
        uint64_t run;    // > 0: a phase run of this many gates
    };
    std::vector<Op> ops;
    for (uint64_t k = 0; k < count; ++k) {
        const sv_gate &g = gates[order[k]];
        bool done = false;
        CommuteSet between;
        for (size_t i = ops.size(); i-- > 0;) {
            const sv_gate &e = ops[i].run ? ops[i].proxy : *ops[i].g;
            if (phase1_gate(g) && ops[i].run && e.target == g.target && between.commutes(g)) {
                ops[i].run += 1;
                ops[i].proxy.controls |= g.controls;
                done = true;
                break;
            }
            if (!phase1_gate(g) && !ops[i].run && e.target == g.target && e.controls == g.controls &&
                between.commutes(g)) {
                done = true;
                break;
            }
            between.add(e);
            if (!between.commutes(g)) break;
        }
        if (done) continue;
        Op o{&g, g, phase1_gate(g) ? 1u : 0u};
        if (o.run) { o.proxy.m[6] = 1.0; o.proxy.m[7] = 0.0; }
        ops.push_back(o);
    }
    uint64_t n = 0, nl = 0;
    for (const Op &o : ops) {
        if (o.run >= 4) { ++n; ++nl; }
        else n += o.run ? o.run : 1;
    }
    if (lin) *lin = nl;
    return n;
}

GatePlan plan_gates(int n, int g, sv_dtype dtype, const sv_gate *gates, uint64_t count) {
    SV_CHECK(n >= 1 && n <= 40, SV_EINVAL, "n must be in [1, 40]");
    SV_CHECK(dtype == SV_C64 || dtype == SV_C128, SV_EINVAL, "dtype must be SV_C64 or SV_C128");
    SV_CHECK(g >= 0 && g <= 6, SV_EINVAL, "world must be 2^g with g in [0, 6]");
    SV_CHECK(count == 0 || gates != nullptr, SV_EINVAL, "gates is NULL");
    for (uint64_t j = 0; j < count; ++j) validate_gate(n, gates[j], j);
    GatePlan p;
    p.n = n;
    p.g = g;
    p.nl = n - g;
    p.T = gate_tile_bits(dtype);
    if (count == 0) return p;
    if (g == 0 && n <= p.T) {  // the whole state is one CTA's shared-memory tile
        GateStep s;
        s.kind = GSTEP_WHOLE;
        s.first = 0;
        s.count = count;
        for (uint64_t j = 0; j < count; ++j) {
            p.order.push_back(j);
            s.proc |= 1ull << gates[j].target;
        }
        s.ops = count;  // the one-CTA kernel runs every gate as given
        s.tile = (n >= 64) ? ~0ull : ((1ull << n) - 1ull);
        p.steps.push_back(s);
        return p;
    }
    const int nl = p.nl, T = p.T, c = carry_bits(dtype);
    SV_CHECK(nl >= T && nl >= g, SV_EINVAL, "shard too small for gate tiles: need n - log2(world) >= T");
    const uint64_t carry = (1ull << c) - 1ull;
    // bounded lookahead: a pass scans at most this many pending gates
    const size_t kWindow = 4096;
    std::vector<uint64_t> pending(count), next;
    for (uint64_t j = 0; j < count; ++j) pending[j] = j;
    int swapped = 0;
    while (!pending.empty()) {
        GateStep s;
        s.kind = GSTEP_PASS;
        s.swapped = swapped;
        s.first = p.order.size();
        uint64_t proc = 0;
        CommuteSet skipped;  // gates left for a later pass (logical qubits)
        next.clear();
        for (size_t k = 0; k < pending.size(); ++k) {
            const uint64_t j = pending[k];
            if (k >= kWindow) {
                next.push_back(j);
                continue;
            }
            const sv_gate &gt = gates[j];
            const int pt = gate_phys(gt.target, nl, g, swapped);
            bool ok = pt < nl && skipped.commutes(gt);
            if (ok) {
                const uint64_t np = proc | (1ull << pt);
                ok = __builtin_popcountll(np | carry) <= T;
                if (ok) {
                    proc = np;
                    p.order.push_back(j);
                }
            }
            if (!ok) {
                next.push_back(j);
                skipped.add(gt);
            }
        }
        s.count = p.order.size() - s.first;
        if (s.count == 0) {
            // the first pending gate targets a rank qubit: reorganise
            SV_CHECK(g > 0, SV_EINVAL, "internal: gate planner made no progress");
            GateStep w;
            w.kind = GSTEP_SWAP;
            w.swapped = swapped;
            p.steps.push_back(w);
            swapped ^= 1;
            continue;
        }
        s.ops = fused_op_count(gates, p.order.data() + s.first, s.count, &s.lin_ops);
        // tile = processed slots + the lowest other slots (carry first) up to T
        s.proc = proc;
        s.tile = proc;
        int have = __builtin_popcountll(proc);
        for (int sl = 0; sl < nl && have < T; ++sl)
            if (!((s.tile >> sl) & 1)) {
                s.tile |= 1ull << sl;
                ++have;
            }
        p.steps.push_back(s);
        pending.swap(next);
    }
    if (swapped) {  // restore the natural layout before returning
        GateStep w;
        w.kind = GSTEP_SWAP;
        w.swapped = 1;
        p.steps.push_back(w);
    }
    return p;
}

}  // namespace sv
