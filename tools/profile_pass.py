"""Generate one day's message CSR at N agents and run the message pass alone
a few times (for ncu: -k regex:k_pass)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2110_04421_b200 import roofline
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    sim = roofline.prepare(n, warm_days=60)
    lam = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(4):
        roofline.gather(sim, lam)
    torch.cuda.synchronize()
    print("ok", float(lam.sum()))


if __name__ == "__main__":
    main()
