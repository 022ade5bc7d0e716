import cProfile, pstats, sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import configs
dev = torch.device("cuda", 0)
dm = P.DeviceMatrix(configs.gen_device("C2", dev), 0)
P.set_omega_cache(True)
for _ in range(3): P.powerlu(dm, 200, 20, 4, 0)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(10): P.powerlu(dm, 200, 20, 4, 0)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
