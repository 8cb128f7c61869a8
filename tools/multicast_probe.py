#!/usr/bin/env python
"""Probe the driver's NVLS multicast object creation on this box (ctypes on
libcuda): granularities and cuMulticastCreate results per handle type/size."""
import ctypes as C


class Prop(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                ("flags", C.c_ulonglong)]


def main():
    cu = C.CDLL("libcuda.so.1")
    print("cuInit", cu.cuInit(0))
    dev = C.c_int()
    print("cuDeviceGet", cu.cuDeviceGet(C.byref(dev), 0), dev.value)
    v = C.c_int()
    print("cuDriverGetVersion", cu.cuDriverGetVersion(C.byref(v)), v.value)
    for attr, name in ((132, "MULTICAST_SUPPORTED"), (129, "? 129"), (130, "? 130"), (131, "? 131")):
        x = C.c_int()
        print(name, cu.cuDeviceGetAttribute(C.byref(x), attr, dev), x.value)
    ctx = C.c_void_p()
    print("cuDevicePrimaryCtxRetain", cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev))
    print("cuCtxSetCurrent", cu.cuCtxSetCurrent(ctx))
    for ht in (0, 1, 8):
        for size in (2 << 20, 64 << 20, 512 << 20):
            p = Prop(1, size, ht, 0)
            g0, g1 = C.c_size_t(), C.c_size_t()
            r0 = cu.cuMulticastGetGranularity(C.byref(g0), C.byref(p), 0)
            r1 = cu.cuMulticastGetGranularity(C.byref(g1), C.byref(p), 1)
            h = C.c_ulonglong()
            r = cu.cuMulticastCreate(C.byref(h), C.byref(p))
            print(f"handleTypes={ht} size={size >> 20}MB gran min={g0.value} ({r0}) rec={g1.value} ({r1}) "
                  f"create={r}")
            if r == 0:
                print("  addDevice", cu.cuMulticastAddDevice(h, dev))
                cu.cuMemRelease(h)


if __name__ == "__main__":
    main()
