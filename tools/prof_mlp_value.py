"""One tensor-core forward of the reference's default MLPValue (5x256) on
8192 rows, for an ncu capture (-k regex:mlp_tc_kernel -s 3 -c 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2502_08844_b200 import mlp as M
    from paper_2502_08844_b200 import rollout as R

    torch.manual_seed(0)
    kind = os.environ.get("MLP_KIND", "value")
    din = int(os.environ.get("MLP_DIN", "5"))
    net = (R.make_value(din) if kind == "value" else R.make_policy(din, 1)).cuda()
    tc = M.tc_value(net) if kind == "value" else M.tc_policy(net)
    x = torch.randn(int(os.environ.get("MLP_ROWS", "8192")), din, device="cuda")
    with torch.no_grad():
        for _ in range(5):
            tc(x)
        torch.cuda.synchronize()
        # 20 calls captured in a CUDA graph: device time per call, no host overhead
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            tc(x)
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            for _ in range(20):
                tc(x)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
    print(kind, "d_in", din, x.shape[0], "rows: %.1f us per call (graph)" % (e0.elapsed_time(e1) / 100 * 1e3))


if __name__ == "__main__":
    main()
