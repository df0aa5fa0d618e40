"""Multi-rank worker for tests/test_ddp.py (torchrun, one process per GPU).

Trains a small MLP under DistributedDataParallel with pact_hook as the comm
hook: two dense warm-up steps (no mask -> full_allreduce), then a global
magnitude prune of the flattened model (trainer.cpp:340-352) and packed steps
once the tracker is Stable. Every step the DDP gradients must equal, bit for
bit, the mean of the ranks' GSE-masked local gradients (computed on an
undistributed replica; for n = 2 the fp32 sum is order-free and 1/2 exact).
Exit code != 0 on any mismatch."""
import copy
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200.ddp import PactHookState, pact_hook  # noqa: E402


def flat_grads(m):
    return torch.cat([p.grad.reshape(-1) for p in m.parameters() if p.requires_grad])


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    failures = []

    def check(name, ok):
        if not ok:
            failures.append(name)
            print(f"[rank {rank}] FAIL {name}", flush=True)

    for transport in (pb.SyncPolicy.NCCL, pb.SyncPolicy.P2P, "auto-density"):
        auto = transport == "auto-density"
        if auto:
            transport = pb.SyncPolicy.AUTO
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 512), torch.nn.ReLU(), torch.nn.Linear(512, 384),
                                    torch.nn.ReLU(), torch.nn.Linear(384, 10)).to(dev)
        ref = copy.deepcopy(model)
        ddpm = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], bucket_cap_mb=0.25)
        state = PactHookState(model, stability_threshold=3, policy=pb.SyncPolicy(transport=transport),
                              auto_density=auto)
        ddpm.register_comm_hook(state, pact_hook)
        opt = torch.optim.SGD(model.parameters(), lr=0.05)
        modes = []
        for step in range(9):
            if step == 2:
                state.prune(0.8)
                check("pruned weights are zero", bool((state.flat_weights()[
                    ~_bits(state.mask, state.length)] == 0).all()))
            g = torch.Generator(device="cpu").manual_seed(1000 * rank + step)
            x = torch.randn(32, 64, generator=g).to(dev)
            y = torch.randint(0, 10, (32,), generator=g).to(dev)
            ref.load_state_dict(model.state_dict())
            ref.zero_grad()
            torch.nn.functional.cross_entropy(ref(x), y).backward()
            lg = flat_grads(ref)
            if state.mask is not None:
                lg = torch.where(_bits(state.mask, state.length), lg, torch.zeros_like(lg))
            allg = [torch.empty_like(lg) for _ in range(world)]
            dist.all_gather(allg, lg)
            want = allg[0]
            for r in range(1, world):
                want = want + allg[r]
            want = want * (1.0 / world)

            opt.zero_grad()
            torch.nn.functional.cross_entropy(ddpm(x), y).backward()
            got = flat_grads(model)
            tag = f"transport {transport} step {step}"
            if world == 2:
                check(f"{tag}: grads bit-exact", torch.equal(got, want))
            else:
                check(f"{tag}: grads", torch.allclose(got, want, rtol=1e-6, atol=1e-7))
            modes.append(sorted({int(s.mode_used) for s in state.last_stats.values()}))
            opt.step()
            state.enforce_weights()
        # dense warm-up (steps 0-1); the mask is observed from step 2 and the
        # tracker turns Stable on the 4th equal digest (sparsity.cpp:17-25,
        # K = 3): Full through step 4, Packed from step 5
        if not auto:
            check(f"transport {transport}: modes {modes}",
                  all(m == [0] for m in modes[:5]) and all(m == [1] for m in modes[5:]))
        else:  # packed or a density fallback (reason 3) per the measured crossover of each bucket length
            thr = state.density_thresholds
            check(f"auto density: thresholds {thr}", len(thr) >= 1 and all(0 < t <= 1 for t in thr.values()))
            check(f"auto density: modes {modes}", all(m == [0] for m in modes[:5]) and
                  all(st.mode_used == pb.SyncMode.PackedAllReduce or st.fallback_reason == 3
                      for st in state.last_stats.values()))
        w = state.flat_weights()
        ws = [torch.empty_like(w) for _ in range(world)]
        dist.all_gather(ws, w)
        check(f"transport {transport}: replicas identical", all(torch.equal(ws[0], v) for v in ws))
        dist.barrier()
        del ddpm
    dist.barrier()
    if failures:
        print(f"[rank {rank}] {len(failures)} failures", flush=True)
        sys.exit(1)
    print(f"[rank {rank}] ddp hook OK", flush=True)
    dist.destroy_process_group()


def _bits(mask, n):
    w = mask.words().view(torch.uint8)
    b = ((w.unsqueeze(1) >> torch.arange(8, device=w.device, dtype=torch.uint8)) & 1).reshape(-1)
    return b[:n].bool()


if __name__ == "__main__":
    main()
