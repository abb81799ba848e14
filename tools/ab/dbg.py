import sys, torch
sys.path.insert(0, ".")
from paper_2012_08099_b200 import engine
v = engine.synth_noise(256, 12, 0, 16, 5)
torch.cuda.synchronize()
print("synth ok", flush=True)
try:
    imgs, prof = engine.project_profile(v, 3)
    print("call returned", flush=True)
    torch.cuda.synchronize()
    print("sync ok", flush=True)
except Exception as e:
    print("EXC", repr(e), flush=True)
    try:
        torch.cuda.synchronize()
    except Exception as e2:
        print("SYNC EXC", repr(e2), flush=True)
