"""Expected weights of the asynchronous PS policy with fixed
per-rank batches: step s computes its gradient at W_max(s-1, 0) (one update
old), update s applies it to W_s. Gradients are taken from the synchronous
executor (lr = 0) at the given master weights, fed exactly as the
asynchronous step sees them: bf16 weights and bf16-rounded biases. Test
helper, not on the product path."""
import numpy as np
import torch


def grad_at(cfg, w, data_rank=0):
    from paper_1709_06622_b200.trainer import Trainer
    t = Trainer(dict(cfg, lr=0.0, data_rank=data_rank, cuda_graph=False, ps_async=False))
    t.step()  # materialise the arena
    wb = torch.from_numpy(np.ascontiguousarray(w)).cuda().bfloat16()
    t.tensor("param").copy_(wb.float())
    t.tensor("wcompute").copy_(wb)
    t.step()
    torch.cuda.synchronize()
    return t.tensor("grad").cpu().numpy()


def expected_async_weights(oracle, cfg, w0, steps, ranks=1):
    """W_steps of `steps` asynchronous updates over `ranks` workers (summed
    gradients, grad scale 1/ranks), from the host-side SGD restatement."""
    hist = [w0]
    v = np.zeros_like(w0)
    w = w0
    for s in range(steps):
        src = hist[max(s - 1, 0)]
        g = sum(grad_at(cfg, src, r).astype(np.float32) for r in range(ranks)) if ranks > 1 \
            else grad_at(cfg, src, 0)
        g = np.asarray(g, dtype=np.float32)
        w, v = oracle.sgd(w, g, v, cfg["lr"], cfg["momentum"], cfg["weight_decay"], 1.0 / ranks)
        hist.append(w)
    return w
