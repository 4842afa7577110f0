import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_quant_ph_9804039_b200 as sv
for n, dt, k in ((16, sv.SV_C64, 200), (20, sv.SV_C64, 200), (22, sv.SV_C64, 100), (24, sv.SV_C64, 50)):
    st = torch.cuda.Stream()
    with sv.sv_init(n, 1, dt, sv.SV_INIT_UNIFORM, stream=st.cuda_stream) as c:
        sv.sv_set_marked(c, sv.sv_marked_from_seed(n, 4, 1))
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        e1.record(st)
        torch.cuda.synchronize()
        wall = e0.elapsed_time(e1)
        sv.sv_profile(c, True)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        ker = sum(ms for _, ms in sv.sv_profile_timeline(c))
        nl = len(sv.sv_profile_timeline(c))
        sv.sv_profile(c, False)
    print(f"n={n} k={k}: stream time {wall:.3f} ms, kernel sum {ker:.3f} ms over {nl} launches, gap {100*(wall-ker)/wall:.1f}%  per-iter {1e3*wall/k:.1f} us")
