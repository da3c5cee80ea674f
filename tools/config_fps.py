"""Per-config single-view frame rates (SURVEY §8(d) "Reporting"): one context on one
stream, the scene resident, 20 warm-up frames then 200 timed frames, each frame
(preprocess -> bin -> render) bracketed by CUDA events; median and p95, eager and as
a CUDA-graph replay.  Also the Fig.5a mirror: frame time with the
scene's meshes / frame time with the meshes removed (SPEC soft bound <= 2.0x).

python tools/config_fps.py [--configs nerf mip360 stress] [--frames 200] [--out profiles/round1_configs.json]
"""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_19233_b200 import renderer as R, scenes  # noqa: E402


def frame_times(sc, frames, warm, graph):
    cam = sc.cameras[0]
    r = R.renderer_for(sc, max_pairs=24 << 20)
    ds = R.to_device(sc)
    out = torch.empty((cam.height, cam.width, 4), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            r.render_view(ds, cam, out=out, stream=s)
    torch.cuda.synchronize()
    assert r.stats()["overflow"] == 0
    run = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            r.render_view(ds, cam, out=out, stream=s)
        torch.cuda.synchronize()
        run = g.replay
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(frames)]
    with torch.cuda.stream(s):
        for e0, e1 in ev:
            e0.record(s)
            if run is not None:
                run()
            else:
                r.render_view(ds, cam, out=out, stream=s)
            e1.record(s)
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    return ms, r.stats()


def summary(ms):
    med, p95 = float(np.median(ms)), float(np.percentile(ms, 95))
    return {"median_ms": med, "p95_ms": p95, "fps_median": 1000.0 / med, "fps_p95": 1000.0 / p95}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["nerf", "mip360", "stress"])
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"device": torch.cuda.get_device_name(0), "frames": a.frames, "warmup": a.warmup,
           "timing": "CUDA events around preprocess -> bin -> render of each frame, one stream", "configs": {}}
    for name in a.configs:
        sc = scenes.make_scene(name)
        ent = {}
        for graph in (False, True):
            ms, st = frame_times(sc, a.frames, a.warmup, graph)
            ent["graph" if graph else "eager"] = summary(ms)
        ent["pairs"] = st["num_pairs"]
        ent["visible_gaussians"] = st["visible_gaussians"]
        ent["visible_triangles"] = st["visible_triangles"]
        if name in ("mip360", "stress"):  # Fig.5a mirror: meshes removed
            bare = dataclasses.replace(sc, mesh=scenes.empty_mesh())
            ms0, _ = frame_times(bare, a.frames, a.warmup, True)
            ent["no_mesh_graph"] = summary(ms0)
            ent["mesh_over_no_mesh"] = ent["graph"]["median_ms"] / ent["no_mesh_graph"]["median_ms"]
        res["configs"][name] = ent
        print(name, json.dumps(ent), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
