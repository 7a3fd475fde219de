import cProfile, pstats, sys, time
sys.path.insert(0, '/root/repo')
from paper_2501_12151_b200.configs import WORKLOADS, build
build(WORKLOADS['C1'])  # warm-up (library load)
t0=time.perf_counter()
pr=cProfile.Profile(); pr.enable()
prob, x0, kw = build(WORKLOADS['C3'])
pr.disable()
print("C3 build", time.perf_counter()-t0)
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
