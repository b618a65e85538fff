"""One fused bintriple deal of 2^27 items (n = 3): the dealer's dominant kernel, for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200.preprocessing import Dealer, MaterialKey  # noqa: E402
d = Dealer(7, 3, 0, 3, "cuda")
d.generate(MaterialKey.from_name("bintriple"), 1 << 27)
torch.cuda.synchronize()
