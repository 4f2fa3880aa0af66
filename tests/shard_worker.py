"""Worker of the multi-rank parity test (tests/test_gpu_shard.py): runs a few generations of
the device loop (harness._Stepper) on cuda:0 and writes the final population plus every
generation's ideal point.  Launched once plain (world 1) and once under torch.distributed.run
with the gloo backend (world 2/3, every rank on the same GPU), so the sharded offspring, HypE
column split and bitmap ND sort shards are checked bit-for-bit against the unsharded loop."""

import json
import os
import sys

import numpy as np


def main():
    cfg = json.loads(sys.argv[1])
    out = sys.argv[2]
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    predrawn = cfg.pop("predrawn", False)  # bench.py's loop: pre-drawn inputs, randomness overlap
    config = RunConfig(**cfg)
    config.validate()
    spec, R, n = _resolve(config)
    stepper = _Stepper(config, spec, R, n)
    assert (stepper.shard is not None) == (world > 1)
    gen = RngStream(config.seed).split(0).generator()
    st = stepper.init(gen)
    ideals = []
    pre = [None] * (config.generations + 2)
    if predrawn:
        pre = stepper.upload_host_inputs([stepper.draw_host_inputs(gen) for _ in range(config.generations)])
        pre += [None, None]
    for g in range(1, config.generations + 1):
        st, _ = stepper.step(st, g, gen, timed=False, pre=pre[g - 1], pre_next=pre[g])
        stepper.check()
        ideals.append(stepper.objectives(st).min(dim=0).values.cpu().numpy())
    X, F = stepper.population(st)
    np.savez(f"{out}.r{rank}.npz", X=X.cpu().numpy(), F=F.cpu().numpy(), ideals=np.asarray(ideals),
             tail=gen.random(4))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
