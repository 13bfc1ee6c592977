"""Launch the benchmark-mask generator (fga_random_keep) for an ncu launch list."""
import sys, torch
sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib
st = torch.cuda.current_stream().cuda_stream
keep = torch.empty((3072, 32760), dtype=torch.uint8, device="cuda")
for _ in range(2):
    _lib.call("fga_random_keep", 3072, 32760, 14742, 77, keep.data_ptr(), st)
torch.cuda.synchronize()
