"""Time the tensor-core MLP forward against torch (cuBLAS float32) at 8192 rows
for the reference's default policy / value networks.  Not a bench line."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2502_08844_b200 import mlp as M
    from paper_2502_08844_b200 import rollout as R

    for kind, net in (("policy", R.make_policy(5, 1)), ("value", R.make_value(5))):
        net = net.cuda()
        x = torch.randn(8192, 5, device="cuda")
        tc = M.tc_policy(net) if kind == "policy" else M.tc_value(net)
        fns = {"tcgen05": lambda: tc(x), "cublas": lambda: net(x)}
        for name, fn in fns.items():
            with torch.no_grad():
                for _ in range(5):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(50):
                    fn()
                e1.record()
                torch.cuda.synchronize()
            print(kind, name, "%.1f us" % (e0.elapsed_time(e1) / 50 * 1e3), flush=True)


if __name__ == "__main__":
    main()
