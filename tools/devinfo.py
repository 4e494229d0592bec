"""Device attributes that size the L2 policies (experiment tool)."""
import ctypes as C

rt = C.CDLL("libcudart.so.12")


def attr(a):
    v = C.c_int()
    rt.cudaDeviceGetAttribute(C.byref(v), a, 0)
    return v.value


# driver_types.h: L2CacheSize 38, MultiProcessorCount 16, MaxSharedMemoryPerBlockOptin 97,
# MaxPersistingL2CacheSize 108, MaxAccessPolicyWindowSize 109
print({"l2_bytes": attr(38), "max_persisting_l2": attr(108), "sms": attr(16),
       "max_smem_per_block_optin": attr(97), "max_access_policy_window": attr(109)})
