"""torch-tensor ensembles over the libboris C ABI (marshalling only).

PyTorch provides device / pinned-host memory and streams; every push step runs
in libboris's CUDA kernels.  Layouts follow include/libboris.h:

* SoA: one tensor per component (x, y, z, px, py, pz, weight, gamma, type),
  per-particle fields Ex..Bz.
* AoS: an (n, 9) FP tensor = n records of 36 B (fp32) / 72 B (fp64), the paper's
  ``Particle {FP3 position; FP3 momentum; FP weight; FP gamma; short type;}``
  (L200-222); the int16 type sits in the first two bytes of column 8.  Fields are
  an (n, 6) FP tensor = n records {E[3], B[3]}.
"""
from __future__ import annotations

import torch

from . import (BORIS_FP32, BORIS_FP64, BORIS_LAYOUT_AOS, BORIS_LAYOUT_SOA, BORIS_MEMORY_DEVICE,
               BORIS_MEMORY_HOST, boris_ensemble_destroy, boris_ensemble_wrap_aos,
               boris_ensemble_wrap_soa, boris_field_create_arrays_aos,
               boris_field_create_arrays_soa, boris_field_destroy)

SOA_STATE = ("x", "y", "z", "px", "py", "pz")
FIELD_COMPONENTS = ("Ex", "Ey", "Ez", "Bx", "By", "Bz")


def torch_dtype(precision):
    return torch.float32 if precision == BORIS_FP32 else torch.float64


class SoaEnsemble:
    """An SoA ensemble whose arrays are torch tensors, wrapped by libboris."""

    def __init__(self, n, precision, types, light_velocity, device=0, host=False,
                 with_fields=True, pin=True):
        self.n = n
        self.precision = precision
        self.types = list(types)
        self.c = light_velocity
        self.host = host
        dt = torch_dtype(precision)
        if host:
            dev = "cpu"
            kw = dict(pin_memory=pin)
        else:
            dev = torch.device("cuda", device)
            kw = {}
        self.t = {k: torch.zeros(n, dtype=dt, device=dev, **kw) for k in SOA_STATE}
        self.t["weight"] = torch.ones(n, dtype=dt, device=dev, **kw)
        self.t["gamma"] = torch.ones(n, dtype=dt, device=dev, **kw)
        self.t["type"] = (torch.zeros(n, dtype=torch.int16, device=dev, **kw)
                          if len(self.types) > 1 else None)
        if with_fields:
            for k in FIELD_COMPONENTS:
                self.t[k] = torch.zeros(n, dtype=dt, device=dev, **kw)
        self.device = device
        self.memory = BORIS_MEMORY_HOST if host else BORIS_MEMORY_DEVICE
        self.handle = None
        self.field = None
        self.with_fields = with_fields

    def ptr(self, k):
        v = self.t.get(k)
        return v.data_ptr() if v is not None and v.numel() else None

    def wrap(self):
        """Create the libboris handles (validates types synchronously)."""
        self.close()
        t = self.t
        self.handle = boris_ensemble_wrap_soa(
            self.device, self.memory, self.precision, self.n, *(self.ptr(k) for k in SOA_STATE),
            self.ptr("weight"), self.ptr("gamma"), self.ptr("type"), self.types, self.c)
        if self.with_fields:
            self.field = boris_field_create_arrays_soa(self.handle,
                                                       *(self.ptr(k) for k in FIELD_COMPONENTS))
        return self

    def fill(self, d, first=0):
        """Copy (and cast) a dict of tensors (synth.Workload.generate output) in."""
        cnt = None
        for k, v in d.items():
            if k in self.t and self.t[k] is not None:
                dst = self.t[k][first:first + v.numel()]
                dst.copy_(v.to(dst.device) if v.device != dst.device else v)
                cnt = v.numel()
        return cnt

    def state(self):
        """float64 CPU copies of r, p, gamma, weight, type (test readback)."""
        out = {k: self.t[k].detach().to("cpu", torch.float64) for k in SOA_STATE + ("gamma",
                                                                                   "weight")}
        out["type"] = (self.t["type"].cpu() if self.t["type"] is not None
                       else torch.zeros(self.n, dtype=torch.int16))
        return out

    def close(self):
        if self.field is not None:
            boris_field_destroy(self.field)
            self.field = None
        if self.handle is not None:
            boris_ensemble_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AosEnsemble:
    """An AoS ensemble: (n, 9) FP tensor of records + (n, 6) FP field records."""

    def __init__(self, n, precision, types, light_velocity, device=0, host=False,
                 with_fields=True, pin=True):
        self.n = n
        self.precision = precision
        self.types = list(types)
        self.c = light_velocity
        dt = torch_dtype(precision)
        dev = "cpu" if host else torch.device("cuda", device)
        kw = dict(pin_memory=pin) if host else {}
        self.rec = torch.zeros((n, 9), dtype=dt, device=dev, **kw)
        self.rec[:, 6] = 1.0
        self.rec[:, 7] = 1.0
        self.fld = torch.zeros((n, 6), dtype=dt, device=dev, **kw) if with_fields else None
        self.device = device
        self.memory = BORIS_MEMORY_HOST if host else BORIS_MEMORY_DEVICE
        self.handle = None
        self.field = None

    @property
    def type_view(self):
        """The int16 type of every record (a strided view into the records)."""
        per = 2 if self.precision == BORIS_FP32 else 4   # int16 slots per FP element
        return self.rec.view(torch.int16)[:, 8 * per]

    def wrap(self):
        self.close()
        self.handle = boris_ensemble_wrap_aos(self.device, self.memory, self.precision, self.n,
                                              self.rec.data_ptr() if self.n else None,
                                              self.types, self.c)
        if self.fld is not None:
            self.field = boris_field_create_arrays_aos(self.handle,
                                                       self.fld.data_ptr() if self.n else None)
        return self

    def fill(self, d, first=0):
        sl = slice(first, first + d["x"].numel())
        dev = self.rec.device
        for j, k in enumerate(SOA_STATE):
            self.rec[sl, j] = d[k].to(dev)
        if "weight" in d:
            self.rec[sl, 6] = d["weight"].to(dev)
        if "gamma" in d:
            self.rec[sl, 7] = d["gamma"].to(dev)
        if "type" in d:
            self.type_view[sl] = d["type"].to(dev)
        if self.fld is not None and "Ex" in d:
            for j, k in enumerate(FIELD_COMPONENTS):
                self.fld[sl, j] = d[k].to(dev)

    def state(self):
        r = self.rec.detach().to("cpu", torch.float64)
        out = {k: r[:, j].clone() for j, k in enumerate(SOA_STATE)}
        out["weight"] = r[:, 6].clone()
        out["gamma"] = r[:, 7].clone()
        out["type"] = self.type_view.cpu().clone()
        return out

    def close(self):
        if self.field is not None:
            boris_field_destroy(self.field)
            self.field = None
        if self.handle is not None:
            boris_ensemble_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_ensemble(layout, n, precision, types, light_velocity, device=0, host=False,
                  with_fields=True):
    cls = SoaEnsemble if layout == BORIS_LAYOUT_SOA else AosEnsemble
    return cls(n, precision, types, light_velocity, device=device, host=host,
               with_fields=with_fields)


__all__ = ["SoaEnsemble", "AosEnsemble", "make_ensemble", "torch_dtype", "BORIS_FP64",
           "BORIS_LAYOUT_AOS"]
