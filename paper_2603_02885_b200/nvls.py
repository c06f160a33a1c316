"""NVLink SHARP (NVLS) buffers for the in-switch reduce-scatter / all-gather of
libmux (include/mux.h mux_nvls_*; csrc/nvls.cu; NEXT-1).

`NvlsBuffer(group, rows_per_rank, cols)` gives every rank one copy of a
[world * rows_per_rank, cols] bf16 buffer plus a flag block, all bound to one
CUDA multicast object (cuMulticastCreate / cuMulticastBindMem), and maps both
the rank's own copy (unicast, `uc`) and the multicast address (`mc`).  The
multicast handle is created on rank 0 and shared as a POSIX file descriptor
(pidfd_getfd), every rank adds its device and binds its own physical memory.
Plumbing only (device memory and mappings, like torch symmetric memory); the
reduction and broadcast run in libmux's kernels.  Nothing here falls back:
without multicast support the constructor raises.
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import mux

_SYS_pidfd_getfd = 438


def _ck(res):
    err = res[0] if isinstance(res, tuple) else res
    from cuda.bindings import driver as drv
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver call failed: {err}")
    if isinstance(res, tuple):
        return res[1] if len(res) == 2 else res[1:]
    return None


class NvlsUnavailable(RuntimeError):
    """The driver refused to create a multicast object (no NVSwitch fabric access in this process:
    e.g. a container without the fabric manager's IMEX channels)."""


class _Cai:
    """__cuda_array_interface__ wrapper: lets torch view a raw mapping (no copy, no ownership)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _fd_from(pid: int, fd: int) -> int:
    """Duplicate file descriptor `fd` of process `pid` into this process (Linux >= 5.6)."""
    pidfd = os.pidfd_open(pid)
    try:
        libc = ctypes.CDLL(None, use_errno=True)
        r = libc.syscall(_SYS_pidfd_getfd, pidfd, fd, 0)
        if r < 0:
            raise OSError(ctypes.get_errno(), "pidfd_getfd failed")
        return r
    finally:
        os.close(pidfd)


class NvlsBuffer:
    FLAG_BYTES = 256

    def __init__(self, group, rows_per_rank: int, cols: int, device=None):
        from cuda.bindings import driver as drv
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows, self.cols = rows_per_rank, cols
        dev_idx = torch.cuda.current_device() if device is None else torch.device(device).index
        _ck(drv.cuInit(0))
        dev = _ck(drv.cuDeviceGet(dev_idx))
        if _ck(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)) != 1:
            raise RuntimeError("device has no multicast (NVLS) support")
        torch.cuda.synchronize()
        data = self.world * rows_per_rank * cols * 2
        fd_type = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = self.world
        prop.handleTypes = fd_type if self.world > 1 else 0
        prop.size = data + self.FLAG_BYTES
        gran = _ck(drv.cuMulticastGetGranularity(
            prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = -(-(data + self.FLAG_BYTES) // gran) * gran
        prop.size = size
        self.size = size
        # multicast object: rank 0 creates it, the others import it by file descriptor
        if self.rank == 0:
            err, mc = drv.cuMulticastCreate(prop)
            if err != drv.CUresult.CUDA_SUCCESS:
                raise NvlsUnavailable(f"cuMulticastCreate failed ({err}): no NVLS multicast in this process")
            fd = _ck(drv.cuMemExportToShareableHandle(mc, fd_type, 0)) if self.world > 1 else -1
            info = [(os.getpid(), int(fd))]
        else:
            info = [None]
        if self.world > 1:
            dist.broadcast_object_list(info, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            if self.rank != 0:
                fd = _fd_from(*info[0])
                mc = _ck(drv.cuMemImportFromShareableHandle(fd, fd_type))
                os.close(fd)
        _ck(drv.cuMulticastAddDevice(mc, dev))
        if self.world > 1:
            dist.barrier(group)             # every device is added before any memory is bound
        aprop = drv.CUmemAllocationProp()
        aprop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = dev_idx
        mem = _ck(drv.cuMemCreate(size, aprop, 0))
        _ck(drv.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
        if self.world > 1:
            dist.barrier(group)
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev_idx
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self._maps = []
        ptrs = []
        for handle in (mem, mc):
            va = _ck(drv.cuMemAddressReserve(size, gran, 0, 0))
            _ck(drv.cuMemMap(va, size, 0, handle, 0))
            _ck(drv.cuMemSetAccess(va, size, [acc], 1))
            self._maps.append(va)
            ptrs.append(int(va))
        self.uc_ptr, self.mc_ptr = ptrs
        self._mem, self._mc = mem, mc
        self.uc = torch.as_tensor(_Cai(self.uc_ptr, (self.world * rows_per_rank, cols), "<i2"),
                                  device=f"cuda:{dev_idx}").view(torch.bfloat16)
        self.uc_flags_ptr = self.uc_ptr + data
        self.mc_flags_ptr = self.mc_ptr + data
        flags = torch.as_tensor(_Cai(self.uc_flags_ptr, (self.FLAG_BYTES // 8,), "<i8"), device=f"cuda:{dev_idx}")
        flags.zero_()
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group)
        self.seq = 0

    def desc(self):
        """mux_nvls descriptor for the next call (seq + 1)."""
        self.seq += 1
        return mux.make_nvls(self.world, self.rank, self.rows, self.seq, self.uc_ptr, self.mc_ptr,
                             self.uc_flags_ptr, self.mc_flags_ptr)

    def reduce_scatter(self, out: torch.Tensor, ctas: int = 0, stream=None) -> torch.Tensor:
        """out [rows_per_rank, cols] = sum over ranks of their copies' rows of this rank (uc must hold
        this rank's partial, written earlier in stream order)."""
        mux.nvls_reduce_scatter(self.desc(), out, ctas, stream)
        return out

    def all_gather(self, rows: torch.Tensor, ctas: int = 0, stream=None) -> torch.Tensor:
        """every rank's `rows` [rows_per_rank, cols] -> self.uc [world * rows_per_rank, cols] on every rank."""
        d = self.desc()
        self._last_ag = d
        mux.nvls_all_gather(d, rows, ctas, stream)
        return self.uc

    def release(self, stream=None):
        """this rank has finished reading the last all-gather's uc."""
        mux.nvls_release(self._last_ag, stream)
