import sys, numpy as np
sys.path.insert(0,'.')
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
for name in ["C1","C3","C2","C5"]:
    s=Scene.build(name); rd=Renderer(0); rd.upload(s); cfg=RenderConfig()
    rd.render_frame(s.device_camera,cfg,exact=False,graph=False)
    g=rd.download_gbuffer()
    ev=g.evalCount.reshape(s.height,s.width)
    H,W=ev.shape; ty,tx=(H+7)//8,(W+7)//8
    pad=np.zeros((ty*8,tx*8),np.int64); pad[:H,:W]=ev
    t=pad.reshape(ty,8,tx,8).transpose(0,2,1,3).reshape(ty*tx,64)
    tmax=t.max(1); tsum=t.sum(1)
    nz=tmax[tmax>0]
    print(name, "pix evals max", ev.max(), "p99.9", np.percentile(ev,99.9), "tile max-evals p50/p99/p99.9/max", np.percentile(nz,[50,99,99.9]).round(), nz.max(),
          "sum top10 tiles", np.sort(tsum)[-10:].sum(), "total", tsum.sum())
    rd.close()
