import sys, cProfile, pstats, time
sys.path.insert(0, '.')
sys.argv = ['bench.py', '--no-cpu-baseline', '--quick', '--no-parity', '--steps', '5', '--warmup', '3', '--e2e-steps', '200']
import bench
import paper_2605_24832_b200.native_step as ns
pr = cProfile.Profile()
orig = bench.run_e2e
def wrapped(*a, **k):
    pr.enable()
    r = orig(*a, **k)
    pr.disable()
    return r
bench.run_e2e = wrapped
bench.main()
st = pstats.Stats(pr); st.sort_stats('tottime').print_stats(25)
