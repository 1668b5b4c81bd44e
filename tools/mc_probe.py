import os, torch
from cuda.bindings import driver as cu
cu.cuInit(0)
for d in range(torch.cuda.device_count()):
    err, dev = cu.cuDeviceGet(d)
    err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    err2, f = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    print("device", d, "multicast_supported", v, err, "fabric", f)
