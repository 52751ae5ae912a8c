import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2211_00645_b200.deskew import deskew_device
from paper_2211_00645_b200.geometry import SheetGeometry, view_transform, output_extent
from paper_2211_00645_b200.pipeline import warp_projection_device
n,h,w=512,2048,2048
g=SheetGeometry(30.0,0.115,0.115,n,w,h)
raw=torch.randint(0,4096,(n,h,w),dtype=torch.int32,device="cuda").to(torch.uint16)
for a in (0.0,15.0,30.0,45.0):
    vt=view_transform(g, view_angle_deg=a)
    _,rows=output_extent(g, vt.shear_px)
    for rep in range(3):
        torch.cuda.synchronize(); t0=time.perf_counter()
        res=deskew_device(raw, vt.shear_px, "linear", canvas_rows=rows, projection_axes=(0,), write_volume=False)
        torch.cuda.synchronize(); t1=time.perf_counter()
        img=warp_projection_device(res.projections[0], vt.warp_scale)
        torch.cuda.synchronize(); t2=time.perf_counter()
    print(a, "shear", round(vt.shear_px,4), "warp", round(vt.warp_scale,4), "rows", rows, "deskew ms", round((t1-t0)*1e3,3), "warp ms", round((t2-t1)*1e3,3))
