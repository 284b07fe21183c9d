"""Print the measured pipe / L2 rates (bvc_pipe_probe) per SM per clock."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2302_11825_b200 as B  # noqa: E402

p = B.pipe_probe()
sms = torch.cuda.get_device_properties(0).multi_processor_count
f = float(sys.argv[1]) * 1e6 if len(sys.argv) > 1 else 1965e6
print(json.dumps({k: {"per_s": v, "per_sm_clk": v / (sms * f)} for k, v in p.items()}, indent=1))
