"""Shared helpers for the GPU parity tests (run on the B200 box)."""

import numpy as np

from oracle import tsg_oracle as O
from paper_1908_06094_b200 import PatchSpec, StructuredStepper


def stepper_for(rows, cols, levels, inp):
    st = StructuredStepper(PatchSpec(rows, cols, levels))
    st.set_geometry(inp["signs"], inp["dual"])
    st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
    return st


def fused_step(rows, cols, levels, inp, dt, pivbz, op="upwind"):
    st = stepper_for(rows, cols, levels, inp)
    st.step(dt, pivbz, op)
    return st.download()


def unfused_step(rows, cols, levels, inp, dt, pivbz, op="upwind"):
    st = stepper_for(rows, cols, levels, inp)
    st.step_unfused(dt, pivbz, op)
    return {"flux": st.fetch("flux"), "fluz": st.fetch("fluz"), "div": st.fetch("divvd"),
            "pd_out": st.fetch("pd_out")}


def golden_inputs(golden, key):
    return {n: golden[f"{key}_{n}"] for n in ("pd", "vn", "wn", "rho", "dual", "signs")}


def oracle_tables(rows, cols):
    return O.neighbor_table(rows, cols, "edges", "vertices"), O.neighbor_table(rows, cols, "vertices", "edges")
