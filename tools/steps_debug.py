import sys, time; sys.path.insert(0,'/root/repo')
import torch, paper_1906_12211_b200 as pfg, synth
c=synth.CONFIGS[2]; dev=torch.device('cuda:0')
data,q=synth.config_data(2); X=torch.from_numpy(data).to(dev); Q=torch.from_numpy(q).to(dev)
idx=pfg.Index(X,c['budget'],'fht_cp',seed=1)
for s in range(25):
    torch.cuda.synchronize(); t=time.perf_counter()
    idx.search(Q,10,0.9,timing=True)
    torch.cuda.synchronize(); el=time.perf_counter()-t
    print(s, ['%.3f'%v for v in idx.last_timing()[:3]], '%.3f ms wall'%(el*1e3))
