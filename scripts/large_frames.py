"""Robustness at large images: 8K and 16K x 16K frames of the C3 scene (eager vs graph
identical, no tile errors) with their frame time."""
import sys, numpy as np, time
sys.path.insert(0,'.')
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
for (w,h) in [(7680,4320),(16384,16384)]:
    s=Scene.build("C3",0,w,h); rd=Renderer(0); rd.upload(s); cfg=RenderConfig(); cam=s.device_camera
    rd.render_frame(cam,cfg,exact=False,graph=False); g1=rd.download_gbuffer()
    rd.render_frame(cam,cfg,exact=False,graph=True); rd.render_frame(cam,cfg,exact=False,graph=True); g2=rd.download_gbuffer()
    t=time.perf_counter(); 
    for _ in range(3): rd.render_frame(cam,cfg,exact=False,graph=True)
    rd.sync(); dt=(time.perf_counter()-t)/3
    st=rd.stats()
    print(w,h,"hits",int(g1.hit.sum()),"graph==eager",g1.depth.tobytes()==g2.depth.tobytes(),"tileErrors",int(g1.tileError.sum()),f"{dt*1e3:.2f} ms/frame", f"{w*h/dt/1e6:.0f} Mrays/s")
    rd.close(); s.close()
