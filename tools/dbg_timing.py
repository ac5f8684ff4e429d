import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2405_04237_b200 as t, synth
A, _, _ = synth.generate_np(65536, 256, 1e8, seed=0)
for graph in (True, False):
    p = t.Plan(65536, 256, 64, "mcqr2gs")
    p.set_graph(graph)
    p.set_timing(True)
    Ad = t.to_colmajor(A); R = t.colmajor_empty(256, 256)
    for i in range(3):
        Ad.copy_(torch.from_numpy(A)); p.factor(Ad, R)
    tm = p.timing()
    print("graph", graph, {k: (round(v["ms"], 3), v["launches"]) for k, v in tm.items()})
    L = t.load(); print(L.tsqr_last_error())
