"""Guard-paged device buffers (tests only): a stand-in for compute-sanitizer,
which is closed on this GPU pool.

`guarded(nbytes, where)` reserves virtual address space for the buffer plus
a guard region, maps physical memory only under the buffer, and places the
buffer's bytes flush against the unmapped guard -- after it (`where="tail"`,
catches reads / writes past the end) or before it (`where="head"`, catches
negative offsets).  Any access into the guard faults (illegal address), so an
operator that over- or under-reads its operands fails its test instead of
silently reading a neighbouring allocation.  Built on the CUDA driver's
virtual memory management API (cuMemAddressReserve / cuMemCreate / cuMemMap),
exposed to torch through __cuda_array_interface__.
"""
from __future__ import annotations

import torch

_KEEP = []  # mappings live for the test session (unmapping mid-run is not needed)


def _check(res):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class _Buf:
    def __init__(self, ptr, shape, dtype):
        typestr = {torch.float64: "<f8", torch.float32: "<f4"}[dtype]
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def guarded_empty(shape, dtype=torch.float64, where: str = "tail") -> torch.Tensor:
    """A device tensor of `shape` whose storage ends (tail) or starts (head)
    exactly at an unmapped guard region of at least one granule."""
    from cuda.bindings import driver as d

    torch.cuda.init()
    dev = torch.cuda.current_device()
    esize = torch.empty((), dtype=dtype).element_size()
    nbytes = esize
    for s in shape:
        nbytes *= int(s)
    prop = d.CUmemAllocationProp()
    prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = dev
    gran = _check(d.cuMemGetAllocationGranularity(
        prop, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
    mapped = max(gran, (nbytes + gran - 1) // gran * gran)
    total = mapped + 2 * gran  # a guard granule on both sides
    base = int(_check(d.cuMemAddressReserve(total, 0, 0, 0)))
    handle = _check(d.cuMemCreate(mapped, prop, 0))
    _check(d.cuMemMap(base + gran, mapped, 0, handle, 0))
    acc = d.CUmemAccessDesc()
    acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = dev
    acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    _check(d.cuMemSetAccess(base + gran, mapped, [acc], 1))
    ptr = base + gran + (mapped - nbytes if where == "tail" else 0)
    _KEEP.append((base, handle))
    t = torch.as_tensor(_Buf(ptr, shape, dtype), device=f"cuda:{dev}")
    t.fill_(float("nan"))  # untrusted cells (corners, padding lanes) start as NaN
    return t


def guarded_like(x: torch.Tensor, where: str = "tail", copy: bool = True) -> torch.Tensor:
    t = guarded_empty(tuple(x.shape), x.dtype, where)
    if copy:
        t.copy_(x)
    return t
