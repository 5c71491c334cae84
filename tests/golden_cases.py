"""TEST INFRASTRUCTURE: loads the reference-generated fixtures in tests/golden/."""
import json
import os

import numpy as np

from paper_2207_13901_b200.host import COMPRESSED, DENSE, Level, SparseTensor, level_grouping, parse_format

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(HERE, "index.json")) as f:
        index = json.load(f)
    data = np.load(os.path.join(HERE, "cases.npz"))
    return index, data


def tensor(data, key, spec):
    fmt = parse_format(spec["format"])
    dims = tuple(spec["dims"])
    levels = []
    for l, g in enumerate(level_grouping(fmt)):
        if fmt.kinds[g[0]] == DENSE:
            levels.append(Level(DENSE, dom=tuple(dims[fmt.mode_order[k]] for k in g)))
        else:
            levels.append(Level(COMPRESSED, pos=data[f"{key}/pos{l}"], crd=data[f"{key}/crd{l}"]))
    return SparseTensor.from_parts(dims, fmt, levels, data[f"{key}/vals"])


def case_tensors(data, entry):
    return {name: tensor(data, f"{entry['key']}/{name}", spec) for name, spec in entry["tensors"].items()}


def expected_out(data, entry):
    k = entry["key"]
    if entry["kernel"] == "spadd3":
        return (data[f"{k}/out_rowptr"], data[f"{k}/out_crd"], data[f"{k}/out_vals"])
    return data[f"{k}/out_vals"]
