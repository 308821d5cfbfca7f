import os, torch
from cuda.bindings import driver as cu
print("torch", torch.__version__)
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"]:
    a = getattr(cu.CUdevice_attribute, name, None)
    print(name, cu.cuDeviceGetAttribute(a, dev) if a is not None else "n/a")
# try a 1-device multicast object
torch.cuda.init()
prop = cu.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
err, gran = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
print("gran", err, gran)
err, mc = cu.cuMulticastCreate(prop)
print("create", err)
if err == cu.CUresult.CUDA_SUCCESS:
    print("adddev", cu.cuMulticastAddDevice(mc, dev))
# torch symmetric memory, world size 1
try:
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    t = symm.empty(1 << 20, device="cuda:0", dtype=torch.float32)
    h = symm.rendezvous(t, dist.group.WORLD)
    print("symm ok; multicast_ptr", h.multicast_ptr, "buffer_ptrs", h.buffer_ptrs)
except Exception as e:
    print("symm failed", type(e).__name__, e)
