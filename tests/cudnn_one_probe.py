import torch, sys
from torch.nn.attention import SDPBackend, sdpa_kernel
S,H,d=32768,40,128
q,k,v=(torch.randn(1,H,S,d,device='cuda',dtype=torch.bfloat16) for _ in range(3))
with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
    for _ in range(3): o=torch.nn.functional.scaled_dot_product_attention(q,k,v)
torch.cuda.synchronize()
