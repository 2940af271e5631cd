"""PredictorBundle model-fit input (forest.hpp:217-251, bundle_from_json :379-391).

The bundle JSON written by the reference's cmd_train (commands.hpp:86-137) is
parsed into struct-of-arrays forests; only the throughput and power forests are
kept, because PredictorBundle::predict reads only those two (forest.hpp:227-235;
the efficiency forest serves feature importance only).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from ._lib import ConfigError, check
from .abi import Coeffs, ptr


@dataclass
class ForestSoA:
    """One Forest: nodes of all trees concatenated; children are tree-local."""

    tree_offset: np.ndarray  # int64 [n_trees + 1]
    feature: np.ndarray      # int32, -1 = leaf (forest.hpp:63)
    threshold: np.ndarray    # float64
    left: np.ndarray         # int32
    right: np.ndarray        # int32
    value: np.ndarray        # float64

    @property
    def n_trees(self) -> int:
        return len(self.tree_offset) - 1

    @staticmethod
    def from_json(j) -> "ForestSoA":
        """forest_from_json (forest.hpp:343-364): {"v": value} leaves, {"f","t","l","r"} splits."""
        sizes = [len(t) for t in j["trees"]]
        off = np.zeros(len(sizes) + 1, np.int64)
        off[1:] = np.cumsum(sizes)
        n = int(off[-1])
        f = np.full(n, -1, np.int32)
        thr = np.zeros(n)
        le = np.full(n, -1, np.int32)
        ri = np.full(n, -1, np.int32)
        val = np.zeros(n)
        i = 0
        for t in j["trees"]:
            for nd in t:
                if "v" in nd:
                    val[i] = float(nd["v"])
                else:
                    f[i] = int(nd["f"])
                    thr[i] = float(nd["t"])
                    le[i] = int(nd["l"])
                    ri[i] = int(nd["r"])
                i += 1
        return ForestSoA(off, f, thr, le, ri, val)


@dataclass
class Bundle:
    model_ids: list
    coeffs: Coeffs
    throughput: ForestSoA
    power: ForestSoA
    hyperparams: dict

    def model_index(self, model_id: str) -> int:
        """FeatureSchema::model_index (forest.hpp:34-39)."""
        try:
            return self.model_ids.index(model_id)
        except ValueError:
            raise ConfigError(2, "unknown model id in feature encoding: " + model_id) from None

    @staticmethod
    def load_json(path: str) -> "Bundle":
        with open(path) as f:
            j = json.load(f)
        k = j["system_power"]
        return Bundle(list(j["model_ids"]), Coeffs(float(k["alpha"]), float(k["beta_watts"])),
                      ForestSoA.from_json(j["throughput"]), ForestSoA.from_json(j["power"]),
                      dict(j["hyperparams"]))

    def to_json(self, path: str) -> None:
        """bundle_to_json layout (forest.hpp:366-377) so the reference can load it with
        bundle_from_json. The efficiency forest (importance only, never predicted)
        is not carried by this Bundle; the power forest stands in for it."""
        def forest_json(fs: ForestSoA):
            trees = []
            for t in range(fs.n_trees):
                a, b = int(fs.tree_offset[t]), int(fs.tree_offset[t + 1])
                nodes = []
                for i in range(a, b):
                    if fs.feature[i] < 0:
                        nodes.append({"v": float(fs.value[i])})
                    else:
                        nodes.append({"f": int(fs.feature[i]), "t": float(fs.threshold[i]),
                                      "l": int(fs.left[i]), "r": int(fs.right[i])})
                trees.append(nodes)
            return {"trees": trees, "impurity_gain": [0.0] * (5 + len(self.model_ids))}

        j = {"schema_version": 1, "model_ids": self.model_ids,
             "system_power": {"alpha": self.coeffs.alpha, "beta_watts": self.coeffs.beta_watts},
             "hyperparams": self.hyperparams, "seed": 0,
             "throughput": forest_json(self.throughput), "power": forest_json(self.power)}
        j["efficiency"] = j["power"]
        with open(path, "w") as f:
            json.dump(j, f)

    def save_npz(self, path: str) -> None:
        d = {"model_ids": np.array(self.model_ids),
             "coeffs": np.array([self.coeffs.alpha, self.coeffs.beta_watts]),
             "hp": np.array([self.hyperparams["n_trees"], self.hyperparams["max_depth"],
                             self.hyperparams["min_leaf"]])}
        for name, fs in (("T", self.throughput), ("P", self.power)):
            for fld in ("tree_offset", "feature", "threshold", "left", "right", "value"):
                d[f"{name}_{fld}"] = getattr(fs, fld)
        np.savez_compressed(path, **d)

    @staticmethod
    def load_npz(path: str) -> "Bundle":
        z = np.load(path)
        fs = []
        for name in ("T", "P"):
            fs.append(ForestSoA(*(z[f"{name}_{f}"] for f in ("tree_offset", "feature", "threshold",
                                                              "left", "right", "value"))))
        hp = z["hp"].tolist()
        return Bundle([str(s) for s in z["model_ids"]], Coeffs(*z["coeffs"].tolist()), fs[0],
                      fs[1], {"n_trees": hp[0], "max_depth": hp[1], "min_leaf": hp[2]})


def forest_args(fs: ForestSoA):
    return [fs.n_trees, ptr(fs.tree_offset), ptr(fs.feature), ptr(fs.threshold), ptr(fs.left),
            ptr(fs.right), ptr(fs.value)]


def make_forest_model(ctx, bundle: Bundle, model_id: str):
    """predictor_scorer(bundle, model_id) (controller.hpp:100-105) on the device."""
    from .wattserve import _Model

    mi = bundle.model_index(model_id)
    h = C.c_void_p()
    check(ctx.lib.pals_model_forest(ctx.h, len(bundle.model_ids), mi, C.byref(bundle.coeffs),
                                    *forest_args(bundle.throughput), *forest_args(bundle.power),
                                    C.byref(h)))
    m = _Model(ctx, h)
    m.kind = "forest"
    m.bundle = bundle
    m.model_id = model_id
    return m
