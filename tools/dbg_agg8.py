"""Debug: production (k_agg8 FAST/EDGE/GENERAL/EMPTY) vs exporting instantiation vs
the k_agg build (FBS_LIB) on small frames; prints where the maps differ."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import stereo_synth as synth

def run(lib, W, H, dmin, dmax, rho, seed):
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import stereo_synth as synth, paper_1807_02044_b200 as fbs
L, R, _, _ = synth.layered({W}, {H}, {dmin}, {dmax}, {seed}, p_flat=0.3)
m = fbs.FBS({W}, {H}, {dmin}, {dmax}, {rho}, 4.0, 30.0)
Ld, Rd = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
vols, em = m.volumes(Ld, Rd, maps=True)
pm = m.maps(Ld, Rd)
np.savez(sys.argv[1], out=pm[0].cpu().numpy(), dl=pm[1].cpu().numpy(), dr=pm[2].cpu().numpy(),
         eout=em[0].cpu().numpy(), edl=em[1].cpu().numpy(), edr=em[2].cpu().numpy(),
         al=vols[2].cpu().numpy(), ar=vols[3].cpu().numpy())
"""
    env = dict(os.environ)
    if lib: env["FBS_LIB"] = lib
    f = f"/tmp/dbg_{os.path.basename(lib or 'new')}.npz"
    subprocess.run([sys.executable, "-c", code, f], env=env, check=True)
    return np.load(f)

for (W, H, dmin, dmax, rho, seed) in [(64, 48, 0, 15, 3, 7), (70, 36, 0, 23, 1, 41), (70, 36, 0, 23, 4, 44)]:
    a = run(None, W, H, dmin, dmax, rho, seed)
    b = run(os.environ.get("OLDLIB"), W, H, dmin, dmax, rho, seed)
    print(f"== {W}x{H} d{dmin}..{dmax} rho={rho}")
    for k in ("dl", "dr", "out"):
        d1 = np.argwhere(a[k] != a["e" + k]); d2 = np.argwhere(a[k] != b[k]); d3 = np.argwhere(a["e" + k] != b["e" + k])
        print(f"  {k}: prod!=export {len(d1)} {d1[:8].tolist()}  new!=old {len(d2)} {d2[:8].tolist()}  exp new!=old {len(d3)}")
    for k in ("al", "ar"):
        x = a[k]; y = b[k]
        bad = np.argwhere(~np.isclose(x, y, atol=1e-5))
        print(f"  {k}: new vs old volume mismatches {len(bad)} {bad[:6].tolist()}")
