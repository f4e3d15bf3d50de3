"""Measure the communication curves of a B200 MachineProfile over NCCL
(latency.hpp:45-67; fitted by fit_profile, latency.hpp:114-169; template
proj/profiles/a800x8.json) -- SURVEY.md §8(f) item 1.

  all2all[x](bytes)  all-to-all over x ranks (the Ulysses exchange), `bytes`
                     = the per-GPU payload, as predict_from_inputs prices it
                     (latency.hpp:242-248);
  p2p[y](bytes)      one ring step over y ranks: every rank sends `bytes` to
                     ring rank r-1 and receives from r+1 (latency.hpp:250-262).

Degrees 2/4/8 up to the world size; payloads 64 KiB .. 256 MiB (x4); CUDA
events, median of 10 after 3 warm-ups, max over ranks.  The dense-attention
samples of the existing profile (tests/measure_profile.py) are kept; the
result is written with "comm_source": "measured", which bench.py reports as
profile_comm.

    python tests/measure_comm.py --gpus 8 [--workload wan]      (self-launches torchrun)
    python tests/measure_comm.py --gpus 2 --dry-run             (gloo on CPU: checks the logic)
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def payloads(dry: bool):
    top = 1 << 20 if dry else 256 << 20
    b = 64 << 10
    out = []
    while b <= top:
        out.append(b)
        b *= 4
    return out


def measure(args):
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dry = args.dry_run
    if dry:
        dev = torch.device("cpu")
        dist.init_process_group("gloo")
    else:
        dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=dev)
    dist.barrier()
    degrees = [x for x in (2, 4, 8) if x <= world]
    groups = {}
    for x in degrees:  # contiguous groups of x ranks (every rank builds every group)
        for g0 in range(0, world - world % x, x):
            grp = dist.new_group(list(range(g0, g0 + x)))
            if g0 <= rank < g0 + x:
                groups[x] = (grp, g0)

    def clock(fn, reps):
        ts = []
        for i in range(3 + reps):
            if dry:
                t0 = time.perf_counter()
                fn()
                t = (time.perf_counter() - t0) * 1e3
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1)
            if i >= 3:
                ts.append(t)
        t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / 1e3

    out = {"all2all": [], "p2p": []}
    reps = 3 if dry else 10
    for x in degrees:
        if x not in groups:
            continue
        grp, g0 = groups[x]
        for b in payloads(dry):
            n = b // 2 // x * x  # bf16 elements, divisible by x
            src = torch.ones(n, dtype=torch.float32 if dry else torch.bfloat16, device=dev)
            dst = torch.empty_like(src)
            sec = clock(lambda: dist.all_to_all_single(dst, src, group=grp), reps)
            out["all2all"].append({"degree": x, "payload_bytes": float(n * 2), "seconds": sec})
            me = rank - g0
            prv, nxt = g0 + (me - 1) % x, g0 + (me + 1) % x

            def ring():
                ops = [dist.P2POp(dist.isend, src, prv, group=grp), dist.P2POp(dist.irecv, dst, nxt, group=grp)]
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            sec = clock(ring, reps)
            out["p2p"].append({"degree": x, "payload_bytes": float(n * 2), "seconds": sec})
    dist.barrier()
    dist.destroy_process_group()
    if rank != 0:
        return
    import paper_2511_23113_b200 as D
    base = ROOT / "paper_2511_23113_b200" / "profiles"
    src = base / f"b200_{args.workload}_measured.json"
    if not src.exists():
        src = base / "b200_nominal.json"
    j = json.loads(src.read_text())
    # fit_profile requires each curve monotone non-decreasing in payload, as the
    # reference does (latency.hpp:86-110).  Timing noise at latency-dominated
    # payloads can break that; the fitted curve is the running maximum over
    # increasing payload (the raw medians are kept in the JSON).
    raw = {p: [dict(e) for e in out[p]] for p in ("all2all", "p2p")}
    for p in ("all2all", "p2p"):
        for x in degrees:
            pts = sorted((e for e in out[p] if e["degree"] == x), key=lambda e: e["payload_bytes"])
            hi = 0.0
            for e in pts:
                hi = max(hi, e["seconds"])
                e["seconds"] = hi
    samples = [D.ProfileSample("dense", 1, e["density"], e["seconds"]) for e in j["dense"]]
    samples += [D.ProfileSample(p, e["degree"], e["payload_bytes"], e["seconds"]) for p in ("all2all", "p2p")
                for e in out[p]]
    prof = D.fit_profile(samples, D.FitOptions(j.get("exchange_overlap", 1.0), j.get("replan_seconds", 0.0),
                                               j.get("bytes_per_token_per_head", 256.0)))
    res = prof.to_json()
    res["dense"] = j["dense"]
    res["comm_source"] = "dry-run" if dry else "measured"
    res["comm_raw_medians"] = raw
    res["_comment"] = (f"B200 profile, {args.workload} shape: dense samples from {src.name}; all2all/p2p "
                       f"measured over {'gloo (dry run)' if dry else 'NCCL'} on {world} ranks by tests/measure_comm.py")
    dst = Path(args.out) if args.out else base / f"b200_{args.workload}_measured.json"
    dst.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps({"wrote": str(dst), "all2all_points": len(out["all2all"]), "p2p_points": len(out["p2p"]),
                      "degrees": degrees}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--workload", default="wan")
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())]
        sys.exit(subprocess.run(cmd + sys.argv[1:]).returncode)
    measure(args)


if __name__ == "__main__":
    main()
