import sys, time, gc
sys.path.insert(0, "/root/repo")
sys.argv = ["x", "0", "0"]
exec(open("/root/repo/tools/probe_recon_var.py").read().split("for mode in")[0])
import paper_2305_06482_b200.recon as R
for mode in (False, True):
    R.OUTER_GRAPH = mode
    for _ in range(3):
        cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg, **kw)
        t = time.perf_counter(); n = gc.collect(); dt = (time.perf_counter() - t) * 1e3
        print("graph" if mode else "eager", "gc.collect %.1f ms, %d unreachable; tracked objects %d" % (dt, n, len(gc.get_objects())))
gc.collect()
import collections
cnt = collections.Counter(type(o).__name__ for o in gc.get_objects())
print(cnt.most_common(12))
