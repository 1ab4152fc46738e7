"""Building the codebooks on the GPU (reference codebook.py:175-340; CLI
``nsnkv build-codebook``, cli.py:63-96).

Same algorithm and the same random stream as the reference -- every draw
comes from the caller's numpy ``Generator`` in the reference's order
(training samples, the initial centroid choice, the evaluation set, one
fresh batch per fine-tune step) -- with the O(n x 256) passes on the GPU:

* ``kmeans_init``: Lloyd's iterations, the assignment and the fp64
  per-cluster sums in ``nsnkv_kmeans_assign``;
* ``finetune``: each step assigns the batch with the inference-time rule, the
  exact cosine match ``nsnkv_match_block`` (bit-identical to the reference's
  ``kernels.match_block``), and accumulates the per-entry statistics in
  ``nsnkv_finetune_stats``.

The per-cluster sums are accumulated with fp64 atomics (their order is not
the reference's ``np.add.at`` order) and the k-means gram products use fused
multiply-adds where numpy uses its BLAS, so a build tracks the reference's
trajectory closely but not bit for bit; the tests hold it to the reference's
held-out fidelity (test_acceptance.py floors).
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib
from .codebook import ENTRY_DIM, N_ENTRIES, BitMode, Codebook

DTYPE = np.float32


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _view(samples: np.ndarray, bit_mode: BitMode) -> np.ndarray:
    return np.abs(samples) if bit_mode.folded else samples


def kmeans_init(rng: np.random.Generator, bit_mode, n_samples: int = 1 << 17, n_iters: int = 50,
                seed: int = 0, device=None) -> Codebook:
    """Lloyd's algorithm over synthetic standard-normal 8-dim vectors
    (codebook.py:175-221); 2-bit clusters the folded |v|."""
    bm = BitMode.parse(bit_mode)
    if n_samples < N_ENTRIES:
        raise ValueError(f"need at least {N_ENTRIES} samples")
    if n_iters < 1:
        raise ValueError("n_iters must be >= 1")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    data = _view(rng.standard_normal((n_samples, ENTRY_DIM), dtype=DTYPE), bm)
    init_idx = rng.choice(n_samples, size=N_ENTRIES, replace=False)
    x = torch.from_numpy(np.ascontiguousarray(data)).to(dev)
    cent = torch.from_numpy(data[np.sort(init_idx)].astype(np.float64)).to(dev)
    assign = torch.empty(n_samples, dtype=torch.int32, device=dev)
    sums = torch.empty(N_ENTRIES, ENTRY_DIM, dtype=torch.float64, device=dev)
    counts = torch.empty(N_ENTRIES, dtype=torch.int32, device=dev)
    d2 = torch.empty(n_samples, dtype=torch.float64, device=dev)
    for _ in range(n_iters):
        sums.zero_()
        counts.zero_()
        _lib.check(_lib.lib.nsnkv_kmeans_assign(x.data_ptr(), n_samples, cent.data_ptr(),
                                                assign.data_ptr(), sums.data_ptr(), counts.data_ptr(),
                                                d2.data_ptr(), _stream()))
        nonempty = counts > 0
        cent = torch.where(nonempty[:, None], sums / counts.clamp(min=1)[:, None].double(), cent)
        n_empty = int((~nonempty).sum())
        if n_empty:  # reseed from the points farthest from their centroid
            far = torch.sort(-d2, stable=True).indices[:n_empty]
            cent[~nonempty] = x[far].double()
    entries = cent.float()
    if bm.folded:
        entries = entries.clamp(min=0.0)
    e = entries.cpu().numpy()
    bad = np.linalg.norm(e.astype(np.float64), axis=1) < 1e-12
    if bad.any():  # a zero centroid cannot take part in cosine matching
        x_sq = (data.astype(np.float64) ** 2).sum(axis=1)
        e[bad] = data[np.argsort(-x_sq, kind="stable")[: int(bad.sum())]]
    return Codebook(entries=e, bit_mode=bm, seed=seed, tuned=False)


def _match_idx(vecs: torch.Tensor, entries32: torch.Tensor, inv: torch.Tensor,
               out: torch.Tensor) -> torch.Tensor:
    _lib.check(_lib.lib.nsnkv_match_block(vecs.data_ptr(), vecs.shape[0], entries32.data_ptr(),
                                          inv.data_ptr(), 0, out.data_ptr(), None, None, None,
                                          _stream()))
    return out


def mean_cossim_gpu(cb: Codebook, vecs: np.ndarray, device=None) -> float:
    """codebook.mean_cossim (codebook.py:240-250) on the GPU: match,
    reconstruct, mean cosine over the non-zero vectors."""
    from .kernels import match_block_t

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    v = torch.from_numpy(np.ascontiguousarray(vecs, dtype=DTYPE)).to(dev)
    ent = torch.from_numpy(np.ascontiguousarray(cb.active_entries, dtype=np.float32)).to(dev)
    inv = torch.from_numpy(np.ascontiguousarray(cb.inv_norms, dtype=np.float64)).to(dev)
    idx, sg, zero = match_block_t(v, ent, inv, cb.bit_mode.folded, want_zero_mask=True)
    e = torch.from_numpy(cb.active_entries.astype(np.float64)).to(dev)[idx.long()]
    if cb.bit_mode.folded:
        bits = (sg.long()[:, None] >> torch.arange(8, device=dev)) & 1
        e = torch.where(bits.bool(), -e, e)
    vd = v.double()
    num = (vd * e).sum(1)
    den = vd.norm(dim=1) * e.norm(dim=1)
    ok = ~zero.bool()
    return float((num[ok] / den[ok]).mean())


def finetune(cb: Codebook, rng: np.random.Generator, n_samples: int = 8192, n_steps: int = 2000,
             lr: float = 0.2, device=None):
    """Gradient-tune entries on the mean cosine distance (codebook.py:260-340),
    one fresh batch per step from `rng`.  Returns (codebook, report dict)."""
    if n_steps < 0 or n_samples < 1:
        raise ValueError("n_steps must be >= 0 and n_samples >= 1")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    t0 = time.perf_counter()
    eval_vecs = rng.standard_normal((1 << 14, ENTRY_DIM), dtype=DTYPE)
    initial = mean_cossim_gpu(cb, eval_vecs, dev)
    entries = torch.from_numpy(cb.entries.astype(np.float64)).to(dev)
    folded = cb.bit_mode.folded
    idx = torch.empty(n_samples, dtype=torch.uint8, device=dev)
    idx32 = torch.empty(n_samples, dtype=torch.int32, device=dev)
    sum_unit = torch.empty(N_ENTRIES, ENTRY_DIM, dtype=torch.float64, device=dev)
    sum_cos = torch.empty(N_ENTRIES, dtype=torch.float64, device=dev)
    counts = torch.empty(N_ENTRIES, dtype=torch.int32, device=dev)
    cosdist = torch.empty(n_steps if n_steps else 1, dtype=torch.float64, device=dev)
    live = torch.empty(n_steps if n_steps else 1, dtype=torch.float64, device=dev)
    block = 64  # batches drawn (in the reference's order) and uploaded per 64 steps
    for s0 in range(0, n_steps, block):
        nb = min(block, n_steps - s0)
        host = np.stack([_view(rng.standard_normal((n_samples, ENTRY_DIM), dtype=DTYPE), cb.bit_mode)
                         for _ in range(nb)])
        batches = torch.from_numpy(host).to(dev)
        for j in range(nb):
            b = batches[j]
            f32 = entries.float().contiguous()
            inv = _inv_norms(f32)
            _match_idx(b, f32, inv, idx)
            idx32.copy_(idx)
            sum_unit.zero_()
            sum_cos.zero_()
            counts.zero_()
            step = s0 + j
            cosdist[step] = 0.0
            _lib.check(_lib.lib.nsnkv_finetune_stats(b.data_ptr(), n_samples, idx32.data_ptr(),
                                                     entries.data_ptr(), sum_unit.data_ptr(),
                                                     sum_cos.data_ptr(), counts.data_ptr(),
                                                     cosdist[step:step + 1].data_ptr(), _stream()))
            live[step] = counts.sum()
            e_norm = entries.norm(dim=1)
            hit = counts > 0
            cnt = counts.clamp(min=1).double()[:, None]
            grad = (sum_unit / e_norm[:, None] - sum_cos[:, None] * entries / (e_norm ** 2)[:, None]) / cnt
            new = entries + lr * torch.where(hit[:, None], grad, torch.zeros_like(grad))
            if folded:
                new = new.clamp(min=0.0)
            dead = new.norm(dim=1) < 1e-9  # keep any entry the projection would annihilate
            entries = torch.where(dead[:, None], entries, new)
    history = (cosdist / live.clamp(min=1)).cpu().numpy().tolist() if n_steps else []
    tuned = Codebook(entries=entries.float().cpu().numpy(), bit_mode=cb.bit_mode, seed=cb.seed,
                     tuned=n_steps > 0 or cb.tuned)
    final = mean_cossim_gpu(tuned, eval_vecs, dev)
    return tuned, {"iters": n_steps, "initial_mean_cossim": initial, "final_mean_cossim": final,
                   "wall_time": time.perf_counter() - t0, "batch_cosdist_history": history}


def _inv_norms(e32: torch.Tensor) -> torch.Tensor:
    """fp64 1/|e| with the squares accumulated in component order
    (kernels/__init__.py:44-51), on the device."""
    e = e32.double()
    acc = e[:, 0] * e[:, 0]
    for k in range(1, ENTRY_DIM):
        acc = acc + e[:, k] * e[:, k]
    return (1.0 / acc.sqrt()).contiguous()


def heldout_cossim(cb: Codebook, seed: int = 424242, n_samples: int = 1 << 14) -> float:
    """codebook.heldout_cossim (codebook.py:253-257) on the GPU."""
    vecs = np.random.Generator(np.random.PCG64(seed)).standard_normal((n_samples, ENTRY_DIM), dtype=DTYPE)
    return mean_cossim_gpu(cb, vecs)


def build_codebook(bit_mode, seed: int = 0, kmeans_samples: int = 1 << 17, kmeans_iters: int = 50,
                   tune_steps: int = 2000, tune_batch: int = 8192, tune_lr: float = 0.2,
                   finetune_entries: bool = True):
    """``nsnkv build-codebook`` (cli.py:71-96): make_rng(seed) -> kmeans_init
    -> finetune.  Returns (codebook, report)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cb = kmeans_init(rng, bit_mode, n_samples=kmeans_samples, n_iters=kmeans_iters, seed=seed)
    report = None
    if finetune_entries:
        cb, report = finetune(cb, rng, n_samples=tune_batch, n_steps=tune_steps, lr=tune_lr)
    return cb, report
