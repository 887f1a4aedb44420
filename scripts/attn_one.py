import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
import test_gpu_kernels as T
args = [int(a) for a in sys.argv[1:]]
try:
    T.test_attention(*args)
    print("OK", args)
except Exception as e:
    print("FAIL", args, str(e)[:200])
