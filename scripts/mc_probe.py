"""Does this box support CUDA multicast objects (NVLS through NVSwitch)?"""
import ctypes
import os

import torch

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
n = torch.cuda.device_count()
for d in range(n):
    dv = ctypes.c_int()
    cu.cuDeviceGet(ctypes.byref(dv), d)
    v = ctypes.c_int(-1)
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), 132, dv)  # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
    f = ctypes.c_int(-1)
    r2 = cu.cuDeviceGetAttribute(ctypes.byref(f), 128, dv)  # HANDLE_TYPE_FABRIC_SUPPORTED
    print(f"dev {d}: multicast_supported={v.value} (rc {r}) fabric_handles={f.value} (rc {r2})")
