import sys, time
sys.path.insert(0, "/root/repo")
sys.argv = ["x", "1", "0"]
src = open("/root/repo/tools/probe_recon_var.py").read().split("for mode in")[0]
exec(src)
for _ in range(3):
    cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg, **kw)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg, **kw)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
