"""Generate tests/golden/frontends_cases.json by running the REFERENCE's CLI
(`seriesaug.cli.main`) and JSON worker (`seriesaug.serve.handle_line`) here.

    python tests/golden/make_golden_frontends.py

augment cases store the input file text, the config, the flags and the
output file text; quality cases the two inputs and stdout; serve cases the
request line and the response line.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def rows_text(values, labels=None, headers=()):
    lines = list(headers)
    for r, row in enumerate(values):
        body = ",".join(repr(float(v)) for v in row)
        lines.append(body + (f":{labels[r]}" if labels is not None else ""))
    return "\n".join(lines) + "\n"


def main():
    sys.path.insert(0, REF)
    from seriesaug.cli import main as cli_main
    from seriesaug.serve import handle_line

    rng = np.random.default_rng(3)
    walk = np.cumsum(rng.normal(0, 1, (6, 40)), axis=1)
    csv_text = rows_text(walk)
    ts_text = rows_text(walk[:4, :24], labels=["a", "b", "a", "c"], headers=("@problemName w", "@data"))
    configs = {
        "jitter": {"stages": [{"kind": "jitter", "params": {"sigma": 0.3}}]},
        "exact_chain": {"master_seed": 7, "stages": [
            {"kind": "jitter", "params": {"sigma": 0.2}}, {"kind": "scale", "params": {"sigma_factor": 0.1}},
            {"kind": "time_warp", "params": {"n_knots": 4, "intensity": 0.5}, "probability": 0.5},
            {"kind": "reverse", "params": {}, "probability": 0.5},
            {"kind": "repeat", "params": {"r": 2}}]},
        "spectral": {"stages": [{"kind": "frequency_mask", "params": {"width": 3}},
                                {"kind": "reverse", "params": {}}]},
        "empty": {"stages": []},
    }
    augment = []
    with tempfile.TemporaryDirectory() as tmp:
        def run(argv):
            err = io.StringIO()
            out = io.StringIO()
            with contextlib.redirect_stderr(err), contextlib.redirect_stdout(out):
                rc = cli_main(argv)
            return rc, out.getvalue(), err.getvalue()

        for name, text in (("csv", csv_text), ("ts", ts_text)):
            src = os.path.join(tmp, f"in.{name}")
            with open(src, "w") as fh:
                fh.write(text)
            for cname, cfg in configs.items():
                for flags in ([], ["--seed", "9"], ["--seed", "9", "--mode", "per-sample"]):
                    if cname == "exact_chain" and "per-sample" in flags:
                        continue  # repeat requires standard mode (an error case below)
                    cpath = os.path.join(tmp, "c.json")
                    with open(cpath, "w") as fh:
                        json.dump(cfg, fh)
                    dst = os.path.join(tmp, "out")
                    rc, out, err = run(["augment", src, "-o", dst, "--config", cpath] + flags)
                    rec = {"input": text, "format_hint": name, "config": cfg, "flags": flags, "rc": rc}
                    if rc == 0:
                        rec["output"] = open(dst).read()
                    else:
                        rec["stderr"] = err
                    augment.append(rec)
            # the built-in default chain (no --config)
            dst = os.path.join(tmp, "out")
            rc, out, err = run(["augment", src, "-o", dst, "--seed", "3"])
            augment.append({"input": text, "format_hint": name, "config": None, "flags": ["--seed", "3"],
                            "rc": rc, "output": open(dst).read()})
        # errors
        bad = os.path.join(tmp, "bad.csv")
        with open(bad, "w") as fh:
            fh.write("1.0,2.0\n3.0\n")
        rc, out, err = run(["augment", bad, "-o", os.path.join(tmp, "o"), "--config", cpath])
        errors = [{"argv": ["augment", "BAD", "-o", "OUT"], "input": "1.0,2.0\n3.0\n", "rc": rc,
                   "stderr": err.replace(tmp, "TMP")}]
        quality = []
        a = os.path.join(tmp, "a.csv")
        b = os.path.join(tmp, "b.csv")
        with open(a, "w") as fh:
            fh.write(csv_text)
        for k, other in enumerate((walk, walk + 0.5, walk[:, ::-1] * 1.5)):
            with open(b, "w") as fh:
                fh.write(rows_text(other))
            rc, out, err = run(["quality", a, b])
            quality.append({"a": csv_text, "b": rows_text(other), "rc": rc, "stdout": out})
    vals = [[float(v) for v in row] for row in walk[:3, :16]]
    reqs = [
        {"id": 1, "op": "version"},
        {"id": 2, "op": "augment_batch", "stage": {"kind": "jitter", "params": {"sigma": 0.4}}, "seed": 11,
         "augmenter_index": 2, "values": vals},
        {"id": 3, "op": "augment_batch", "stage": {"kind": "time_warp", "params": {"n_knots": 3,
                                                                                   "intensity": 0.4}},
         "seed": 5, "values": vals},
        {"id": 4, "op": "augment_batch", "stage": {"kind": "jitter", "probability": 0.0,
                                                   "params": {"sigma": 9.0}}, "seed": 0, "values": vals},
        {"id": 5, "op": "augment_batch", "stage": {"kind": "repeat", "params": {"r": 3}}, "seed": 0,
         "values": vals},
        {"id": 6, "op": "dtw_distance", "a": vals[0], "b": vals[1]},
        {"id": 7, "op": "dtw_similarity", "a": vals[0], "b": vals[2]},
        {"id": 8, "op": "nope"},
        {"id": 9, "op": "augment_batch", "stage": {"kind": "jitter", "params": {"sigma": 0.4}}, "values": vals},
        {"id": 10, "op": "augment_batch", "stage": {"kind": "blur", "params": {}}, "seed": 1, "values": vals},
        {"id": 11, "op": "augment_batch", "stage": {"kind": "jitter", "params": {"sigma": -1.0}}, "seed": 1,
         "values": vals},
        {"id": 12, "op": "augment_batch", "stage": {"kind": "jitter", "params": {"sigma": 0.1}}, "seed": 1,
         "values": [[1.0, 2.0], [3.0]]},
        {"id": 13, "op": "roundtrip_check", "transform": "wavelet", "values": vals},
    ]
    lines = [json.dumps(r) for r in reqs] + ["{not json", "[1, 2]"]
    serve = [{"request": ln, "response": handle_line(ln)} for ln in lines]
    doc = {"generator": "tests/golden/make_golden_frontends.py", "augment": augment, "errors": errors,
           "quality": quality, "serve": serve}
    with open(os.path.join(HERE, "frontends_cases.json"), "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")
    print(len(augment), "augment,", len(quality), "quality,", len(serve), "serve cases")


if __name__ == "__main__":
    main()
