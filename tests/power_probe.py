import subprocess, time, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2511_23113_b200 as D
from paper_2511_23113_b200.attention import AttentionSchedule
H,S,d=40,32768,128
m=D.generate_mask_set(D.GeneratorSpec(H,S//64,S//64,64,"clustered",.15,.45,1.0,1))
q,k,v=(torch.randn(S,H,d,device="cuda",dtype=torch.bfloat16) for _ in range(3))
for fl in (1, 9):
    sc=AttentionSchedule().build(m,kv_tokens_global=S,flags=fl); sc.upload()
    out=torch.empty_like(q)
    for _ in range(20): sc.launch(q,k,v,out)
    torch.cuda.synchronize()
    p=subprocess.Popen(["nvidia-smi","--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active","--format=csv,noheader","-lms","100"],stdout=subprocess.PIPE,text=True)
    t=time.time()
    while time.time()-t<3:
        for _ in range(50): sc.launch(q,k,v,out)
        torch.cuda.synchronize()
    p.terminate(); outp=p.communicate()[0]
    print("flags",fl); print("\n".join(outp.strip().splitlines()[-12:]))
