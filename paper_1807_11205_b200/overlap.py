"""Backward-overlap driver: the step fed by autograd as gradients arrive.

The reference enqueues every gradient into its FusionBuffer after the whole
backward pass (experiment.py:360-379); the paper's design enqueues them in
backward ARRIVAL order so a bucket's all-reduce overlaps the rest of the
backward pass.  `BackwardOverlap` does the
latter on top of `GradientPipeline`'s incremental step (begin / submit /
end):

  * a post-accumulate-grad hook on every parameter records its fp16 gradient;
    when the last gradient of a theta-bucket has arrived the bucket is packed
    into the wire, all-reduced (ordered NVLink kernel / NCCL / fused
    reduce-scatter) and run through LARS pass 1 on a side stream while the
    backward pass keeps computing on the compute stream;
  * `finish()` (after `loss.backward()`) closes the step: trust ratios and
    pass 2 on the compute stream, then the one flag read (LossScale update,
    experiment.py:403-413).

Bucket membership is the pipeline's, i.e. FusionBuffer's over the pipeline's
enqueue order (default: reversed registration, the usual backward order), so
the reduced buckets, the skip decision and the update are bit-identical to
`GradientPipeline.step()` on the same gradients; only the launch timing
changes.  With `bind_weights=True` the model's fp16 parameters become views
of the pipeline's binary16 working arena, so pass 2's working-copy refresh
(lars.py:180) IS the model-weight update — nothing is copied back.
"""

from __future__ import annotations

import torch

from .pipeline import GradientPipeline, ParamSpec

__all__ = ["BackwardOverlap", "specs_from_module", "param_kind"]


def param_kind(name: str, p: torch.Tensor, bn_names: set) -> str:
    """Kind map of SURVEY.md §8d (shapes.py): BN weight -> bn_gamma, BN bias ->
    bn_beta, any other tensor with dim > 1 -> weight, other 1-D -> bias."""
    owner, _, leaf = name.rpartition(".")
    if owner in bn_names:
        return "bn_gamma" if leaf == "weight" else "bn_beta"
    return "weight" if p.dim() > 1 else "bias"


def specs_from_module(module: torch.nn.Module) -> list[ParamSpec]:
    """ParamSpecs of a module's trainable parameters in registration order."""
    bn = {n for n, m in module.named_modules()
          if isinstance(m, torch.nn.modules.batchnorm._NormBase)}
    return [ParamSpec(n, tuple(p.shape), param_kind(n, p, bn))
            for n, p in module.named_parameters() if p.requires_grad]


class BackwardOverlap:
    """Hooks a module's parameters into a GradientPipeline.

    Args:
      module: the model; its trainable parameters, in registration order,
        must match `pipeline.specs` (names and sizes) and be float16.
      pipeline: the rank's GradientPipeline.
      bind_weights: make the parameters views of the pipeline's working
        arena (pass 2 then updates the model in place).

    Per step::

        drv.begin(step)                    # before backward
        (loss * drv.loss_scale).backward() # buckets launch from the hooks
        res = drv.finish()                 # trust + pass 2 + flag read
    """

    def __init__(self, module: torch.nn.Module, pipeline: GradientPipeline, *,
                 bind_weights: bool = True):
        self.pipe = pipeline
        named = [(n, p) for n, p in module.named_parameters() if p.requires_grad]
        if len(named) != len(pipeline.specs):
            raise ValueError(f"module has {len(named)} trainable parameters, pipeline "
                             f"{len(pipeline.specs)}")
        for (n, p), s in zip(named, pipeline.specs):
            if p.numel() != s.numel:
                raise ValueError(f"parameter {n!r}: {p.numel()} elements, spec {s.name!r} "
                                 f"has {s.numel}")
            if p.dtype != torch.float16 or p.device != pipeline.device:
                raise ValueError(f"parameter {n!r} must be float16 on {pipeline.device}")
        self.params = [p for _, p in named]
        self._bucket_of = {}
        for b, bk in enumerate(pipeline.buckets):
            for i in bk.params:
                self._bucket_of[i] = b
        self._left = None
        self._grads = None
        self._open = False
        if bind_weights:
            self.bind_weights()
        self._handles = [p.register_post_accumulate_grad_hook(self._hook(i))
                         for i, p in enumerate(self.params)]

    @classmethod
    def for_module(cls, module: torch.nn.Module, cfg, device=None, **pipeline_kw):
        """Build the pipeline from a module: its current (fp32) weights become
        the fp32 masters, the module is cast to float16 and its parameters are
        bound to the working arena."""
        specs = specs_from_module(module)
        named = [p for p in module.parameters() if p.requires_grad]
        device = device or named[0].device
        master = torch.cat([p.detach().to(device, torch.float32).reshape(-1) for p in named])
        module.to(device=device, dtype=torch.float16)
        pipe = GradientPipeline(specs, cfg, init_master=master, device=device, **pipeline_kw)
        return cls(module, pipe, bind_weights=True)

    @property
    def loss_scale(self) -> float:
        return self.pipe.loss_scale.scale

    def bind_weights(self) -> None:
        """Parameters -> views of the working arena (wire layout).  The
        arena must already hold the fp16 weights (load_master refreshes it)."""
        w16 = self.pipe.working
        with torch.no_grad():
            for i, p in enumerate(self.params):
                o, n = self.pipe.wire_off[i], self.pipe.sizes[i]
                p.data = w16[o:o + n].view(torch.float16).view(p.shape)

    def _hook(self, i: int):
        def hook(p: torch.Tensor) -> None:
            if not self._open:
                return
            g = p.grad
            if g is None:
                return
            if not g.is_contiguous():
                g = g.contiguous()
            self._grads[i] = g
            b = self._bucket_of[i]
            self._left[b] -= 1
            if self._left[b] == 0:
                bk = self.pipe.buckets[b]
                self.pipe.submit(b, [self._grads[j] for j in bk.params])
        return hook

    def begin(self, step: int) -> None:
        """Open the step (call before backward)."""
        self.pipe.begin(step)
        self._left = [len(bk.params) for bk in self.pipe.buckets]
        self._grads = [None] * len(self.params)
        self._open = True
        self._step = step

    def finish(self, set_grads_to_none: bool = True):
        """Close the step after backward; returns the pipeline's StepResult."""
        self._open = False
        pipe = self.pipe
        for b, left in enumerate(self._left):
            if left:
                missing = [pipe.specs[i].name for i in pipe.buckets[b].params
                           if self._grads[i] is None]
                raise RuntimeError(f"no gradient arrived for {missing[:4]} (bucket {b}); "
                                   "every trainable parameter must take part in the loss")
        pipe.end()
        if set_grads_to_none:
            for p in self.params:
                p.grad = None
        self._grads = None
        return pipe.finish()

    def remove(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []
