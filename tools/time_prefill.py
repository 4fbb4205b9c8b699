"""Quick timing of sbvr_prefill vs cuBLAS fp16 (torch.matmul) at one shape over a ring of weight copies larger
than L2, CUDA graphs of `reps` calls, events on the replay stream.  Usage: python tools/time_prefill.py M N T..."""
import sys

import torch

import paper_2509_18172_b200 as sb
import synthetic


def main():
    M, N = int(sys.argv[1]), int(sys.argv[2])
    Ts = [int(t) for t in sys.argv[3:]] or [16]
    ring = max(2, int(160e6 // (M * N // 2)) + 1)
    ws_ = []
    for i in range(ring):
        pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=i)
        ws_.append(sb.pack_canonical(pc, s16, b16, ri, 16))
    Wf = [torch.randn(M, N, device="cuda", dtype=torch.float16) for _ in range(max(2, int(160e6 // (2 * M * N)) + 1))]
    stream = torch.cuda.Stream()
    for T in Ts:
        X = torch.randn(T, N, device="cuda", dtype=torch.float16)
        Y = torch.empty(T, M, device="cuda")
        wss = [sb.prefill_workspace(w, T) for w in ws_]
        reps = 4 * ring
        with torch.cuda.stream(stream):
            for i in range(ring):
                sb.prefill(ws_[i], X, Y, wss[i])
            for Wi in Wf:
                torch.mm(X, Wi.t())                      # cuBLAS handle + workspace before capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(reps):
                    sb.prefill(ws_[i % ring], X, Y, wss[i % ring])
            gc = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gc, stream=stream):
                for i in range(reps):
                    torch.mm(X, Wf[i % len(Wf)].t())
            res = {}
            for name, gg in (("sbvr", g), ("cublas", gc)):
                gg.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    gg.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                res[name] = e0.elapsed_time(e1) * 1e3 / (5 * reps)
        wbytes = M * N * 4 // 8 + 5 * M * N // 128
        print(f"M={M} N={N} T={T}: sbvr {res['sbvr']:.2f} us ({wbytes / res['sbvr'] / 1e3:.0f} GB/s weights, "
              f"{2 * M * N * T / res['sbvr'] / 1e6:.1f} TFLOP/s)  cublas fp16 {res['cublas']:.2f} us  "
              f"speedup {res['cublas'] / res['sbvr']:.2f}x", flush=True)


if __name__ == "__main__":
    main()
