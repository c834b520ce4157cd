"""Zero-copy device path: inputs already resident in HBM, outputs left there.

torch is plumbing only (allocation, the current CUDA stream); the compute is
one ``tbn_forward`` launch of libtabnet_b200.so per call.
"""
from __future__ import annotations

import torch

from . import _native as N
from .network import TabNetModel


class DeviceRunner:
    """Preallocated device outputs + workspace for repeated forwards of up to
    ``max_rows`` rows (bench.py and the device-path tests use this)."""

    def __init__(self, model: TabNetModel, max_rows: int, *, device: int | None = None,
                 outputs: tuple = ("logits", "probabilities", "masks", "importance",
                                   "predicted_class"), flags: int = 0):
        self.model = model
        dev = torch.cuda.current_device() if device is None else device
        self.engine = model.engine(device=dev)
        self.n_out = self.engine.n_out
        if self.n_out == 1 and getattr(model, "n_outputs", None) == 1:
            # regression head: the kernel writes the one output value only
            outputs = tuple(k for k in outputs if k not in ("probabilities", "predicted_class"))
        self.device = torch.device("cuda", dev)
        self.max_rows = max_rows
        self.flags = flags
        self.out_names = outputs
        self.ws_bytes = self.engine.workspace_bytes(max_rows, flags)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.outputs = self.alloc_outputs(max_rows)

    def alloc_outputs(self, rows: int) -> dict:
        cfg = self.model.config
        f, c, s = cfg.feature_count, self.n_out, cfg.n_steps
        shapes = dict(logits=(rows, c), probabilities=(rows, c), masks=(s, rows, f),
                      importance=(rows, f), predicted_class=(rows,))
        return {k: torch.empty(shapes[k], dtype=torch.int32 if k == "predicted_class" else torch.float32,
                               device=self.device) for k in self.out_names}

    def views(self, rows: int) -> dict:
        """Outputs for a ``rows``-row call carved from the preallocated buffers
        (masks keep the step-major (S, rows, F) layout of network.py:231)."""
        cfg = self.model.config
        f, c, s = cfg.feature_count, self.n_out, cfg.n_steps
        shapes = dict(logits=(rows, c), probabilities=(rows, c), masks=(s, rows, f),
                      importance=(rows, f), predicted_class=(rows,))
        out = {}
        for k, v in self.outputs.items():
            n = 1
            for d in shapes[k]:
                n *= d
            out[k] = v.view(-1)[:n].view(shapes[k])
        return out

    def run(self, x: torch.Tensor, outputs: dict | None = None, stream=None) -> dict:
        """One fused forward over ``x`` (float32, (rows, F), contiguous, on device)."""
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
        rows = x.shape[0]
        if outputs is None:
            if rows > self.max_rows:
                raise ValueError("rows > max_rows")
            outputs = self.views(rows)
        ptrs = {k: v.data_ptr() for k, v in outputs.items()}
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self.engine.forward_device(x.data_ptr(), rows, self.flags, ptrs, self.err.data_ptr(),
                                   self.ws.data_ptr(), self.ws_bytes, st)
        return outputs

    def check_finite(self) -> None:
        """Raise InvalidInputError if any forward since the last reset saw a
        non-finite feature (synchronizes)."""
        if int(self.err.item()) != 0:
            self.err.zero_()
            from .errors import InvalidInputError
            raise InvalidInputError("features must be finite")
