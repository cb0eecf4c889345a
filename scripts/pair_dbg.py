import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_02367_b200 import sage_attention_cuda, synth
from oracle.oracle import Oracle, cosine_sim, relative_l1
orc = Oracle()
for n, causal in [(256, False), (512, False), (512, True), (1024, False), (1024, True), (2048, False)]:
    q, k, v = synth.qkv(2, n, 128, dtype=np.float32)
    qd, kd, vd = (torch.from_numpy(x.reshape(1, 2, n, 128)).cuda().half() for x in (q, k, v))
    try:
        o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32)
        torch.cuda.synchronize()
    except Exception as e:
        print(n, causal, "FAIL", e); break
    ref, _ = orc.sage_b(q, k, v, causal, pv_fp32=True)
    o = o.cpu().numpy().reshape(2, n, 128)
    print(n, causal, "cos", cosine_sim(o, ref), "rl", relative_l1(o, ref), flush=True)
