"""Print the L2-related device attributes (persisting carve-out limits) of cuda:0."""
from cuda.bindings import runtime as rt

names = ["cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize",
         "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrMultiProcessorCount",
         "cudaDevAttrMaxSharedMemoryPerBlockOptin", "cudaDevAttrMaxSharedMemoryPerMultiprocessor"]
for nm in names:
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, nm), 0)
    print(nm, int(v), err)
