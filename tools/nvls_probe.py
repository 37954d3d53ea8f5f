"""Probe cuMulticastCreate on this box (development aid for the N4 multicast gather): which
(numDevices, handleTypes) combinations the driver accepts."""
import ctypes

cu = ctypes.CDLL("libcuda.so.1")
print("cuInit", cu.cuInit(0))
dev = ctypes.c_int()
print("cuDeviceGet", cu.cuDeviceGet(ctypes.byref(dev), 0))
for attr, name in ((132, "MULTICAST_SUPPORTED"), (128, "HANDLE_TYPE_FABRIC_SUPPORTED"), (102, "VMM_SUPPORTED")):
    v = ctypes.c_int()
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, r, v.value)
ctx = ctypes.c_void_p()
print("cuDevicePrimaryCtxRetain", cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev), "setCurrent", cu.cuCtxSetCurrent(ctx))


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


for nd in (1, 2):
    for ht, hn in ((0, "NONE"), (1, "POSIX_FD"), (8, "FABRIC")):
        p = Prop(nd, 1 << 21, ht, 0)
        g = ctypes.c_size_t()
        rg = cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
        p.size = max(g.value, 1 << 21)
        h = ctypes.c_ulonglong()
        rc = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        print(f"numDevices={nd} handle={hn}: granularity rc={rg} g={g.value} create rc={rc}", flush=True)
        if rc == 0:
            ra = cu.cuMulticastAddDevice(h, dev)
            print("   addDevice rc", ra, flush=True)
            cu.cuMemRelease(h)
