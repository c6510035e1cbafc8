"""Config dicts shared by the tests (mirror the reference defaults,
models.py:40-138 and the toy fixtures of tests/conftest.py:7-30)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

VOXEL = dict(grid_extent=16, in_channels=8, conv_filters_1=32, conv_filters_2=64,
             dense_nodes=128, residual_1=False, residual_2=True, batch_norm=False,
             kernel_1=5, kernel_2=3)
GRAPH = dict(c_elem=4, k_cov=6, k_noncov=3, gather_width_cov=24,
             gather_width_noncov=128, cov_thresh=2.24, noncov_thresh=5.22)
COHERENT = dict(mode="coherent", n_fusion_layers=4, model_specific_layers=False,
                residual_fusion=False, activation="selu", fusion_dense_nodes=64)
LATE = dict(COHERENT, mode="late")
MID = dict(mode="mid", n_fusion_layers=5, model_specific_layers=True,
           residual_fusion=True, activation="selu", fusion_dense_nodes=64)

TOY_VOXEL = dict(grid_extent=8, in_channels=2, conv_filters_1=2, conv_filters_2=2,
                 dense_nodes=8, residual_1=False, residual_2=True, batch_norm=False,
                 kernel_1=3, kernel_2=3)
TOY_GRAPH = dict(c_elem=1, k_cov=2, k_noncov=2, gather_width_cov=4,
                 gather_width_noncov=4, cov_thresh=2.24, noncov_thresh=5.22)
TOY_FUSION = dict(mode="coherent", n_fusion_layers=3, model_specific_layers=False,
                  residual_fusion=False, activation="selu", fusion_dense_nodes=6)


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def complexes_of(z):
    off = z["atom_off"]
    for p in range(len(off) - 1):
        s, e = off[p], off[p + 1]
        yield z["positions"][s:e], z["elements"][s:e], z["roles"][s:e]
