"""Repeated-apply driver: the mapping cycle of the
reference's iteration experiment, with the field resident in HBM.

`PointwiseCycle` mirrors `metrics._PointwiseCycle` (metrics.py:127-148): one
mesh -> vertices to centroids and back, or two meshes -> vertices of one to
vertices of the other and back, each leg a `PreparedTransfer`.  The
reference re-solves every target on every apply and copies the field through
host arrays each cycle (metrics.py:221-224); here both legs are operators
in HBM (or device patch CSRs for ElementPatch) and `iterate` keeps the field
on the device for all cycles.  The accuracy / conservation metrics recorded
per cycle by `run_iteration_experiment` (quadrature, conservative transfer)
are out of scope.
"""

import numpy as np
import torch

from .pointwise import PreparedTransfer


class PointwiseCycle:
    def __init__(self, mesh, fitspec, target_mesh=None, threads=1):
        self.threads = threads
        if target_mesh is None:
            # vertices -> centroids -> vertices on one mesh (metrics.py:130-137)
            cen = mesh.centroids()
            self.down = PreparedTransfer(mesh.coords, cen, fitspec, mesh=mesh,
                                         source_location="vertices")
            self.up = PreparedTransfer(cen, mesh.coords, fitspec, mesh=mesh,
                                       source_location="centroids")
        else:
            self.down = PreparedTransfer(mesh.coords, target_mesh.coords, fitspec, mesh=mesh,
                                         source_location="vertices")
            self.up = PreparedTransfer(target_mesh.coords, mesh.coords, fitspec,
                                       mesh=target_mesh, source_location="vertices")

    def cycle(self, values):
        """One down + up mapping (metrics.py:146-148).  numpy in -> numpy out;
        CUDA tensor in -> CUDA tensor out."""
        mid = self.down.apply(values, threads=self.threads)
        return self.up.apply(mid, threads=self.threads)

    def iterate(self, values, n_iters, keep_history=False):
        """`n_iters` cycles with the field on the device throughout (one H2D
        before, one D2H after when `values` is a host array).  Returns the
        final field, or (final, history (n_iters, n, ...)) with keep_history."""
        if n_iters < 1:
            raise ValueError("n_iters must be >= 1")
        host = not (isinstance(values, torch.Tensor) and values.is_cuda)
        v = values if not host else torch.as_tensor(np.ascontiguousarray(values,
                                                                         dtype=np.float64)).cuda()
        hist = []
        for _ in range(n_iters):
            v = self.cycle(v)
            if keep_history:
                hist.append(v)
        out = v.cpu().numpy() if host else v
        if not keep_history:
            return out
        h = torch.stack(hist)
        return out, (h.cpu().numpy() if host else h)
