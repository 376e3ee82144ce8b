"""Probe: does this box support NVLS multicast objects (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED)?"""
from cuda.bindings import driver as cu

cu.cuInit(0)
_, n = cu.cuDeviceGetCount()
for d in range(n):
    _, dev = cu.cuDeviceGet(d)
    _, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    _, fab = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    _, fd = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev)
    print(f"device {d}: multicast={mc} fabric_handle={fab} posix_fd={fd}")
