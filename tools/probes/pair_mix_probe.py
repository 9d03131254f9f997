"""Run tools/probes/pair_mix_probe.cu on a GPU: mixed cta_group::2 / ::1 MMAs."""
import ctypes, os, sys, json
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_pair_mix_probe.so"))
torch.manual_seed(0)
A = torch.randn(256, 128, device="cuda").bfloat16()
B = torch.randn(128, 128, device="cuda").bfloat16()
C = torch.randn(256, 128, device="cuda").bfloat16()
Dp = torch.zeros(256, 128, device="cuda")
Do = torch.zeros(256, 128, device="cuda")
rc = lib.pair_mix_probe(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                        ctypes.c_void_p(Dp.data_ptr()), ctypes.c_void_p(Do.data_ptr()))
refp = A.float() @ B.float().T
refo = torch.cat([A[:128].float() @ C[:128].float().T, A[128:].float() @ C[128:].float().T])
print(json.dumps({"rc": rc, "pair_max_err": float((Dp - refp).abs().max()), "own_max_err": float((Do - refo).abs().max()),
                  "scale": float(refp.abs().max())}))
