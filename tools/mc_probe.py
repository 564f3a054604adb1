import ctypes, torch
torch.cuda.init(); torch.zeros(1, device="cuda")
cu = ctypes.CDLL("libcuda.so.1")
v = ctypes.c_int(-1)
print("multicast_supported", cu.cuDeviceGetAttribute(ctypes.byref(v), 132, 0), v.value)
class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong), ("flags", ctypes.c_ulonglong)]
p = Prop(1, 2 << 20, 1, 0)  # POSIX FD handle type = 1
gran = ctypes.c_size_t(0)
print("gran", cu.cuMulticastGetGranularity(ctypes.byref(gran), ctypes.byref(p), 0), gran.value)
p.size = max(gran.value, 2 << 20)
h = ctypes.c_ulonglong(0)
print("create", cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p)))
print("adddev", cu.cuMulticastAddDevice(h, 0))
