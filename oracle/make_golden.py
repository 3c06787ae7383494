"""Generates tests/golden/reference_outputs.npz from the REFERENCE ITSELF
(oracle/_ref/libsf_ref.so, the reference's unmodified sources compiled in place).

Run in the build container (needs oracle/_ref, i.e. /root/reference at build time):
    python -m oracle.make_golden
The fixture holds outputs only; tests/golden_cases.py rebuilds the (deterministic) inputs.
"""
import os

import numpy as np

from oracle import ref
from tests import golden_cases as gc

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "reference_outputs.npz")


def main():
    out = {}
    for name, case in gc.CASES.items():
        c = case()
        rp = ref.Problem(c["shape"], c["spacing"], c["origin"], c["velocity"], c["nbl"], c["order"],
                         c["order"], c["src"], c["rec"], 0.0, c["tn"], c["dt"], c["f0"])
        fwd = rp.forward(backend=ref.EMITTED if ref.emit_available() else ref.INTERPRETER)
        out[f"{name}.nt"] = np.array(fwd["nt"])
        out[f"{name}.dt"] = np.array(c["dt"])
        out[f"{name}.rec"] = fwd["rec"]
        out[f"{name}.final_sub"] = fwd["final"][gc.SUB[len(c["shape"])]]
        adj = rp.adjoint(fwd["rec"])
        out[f"{name}.srca"] = adj["srca"]
        if c.get("gradient"):
            obs = fwd["rec"] * 0.6
            rp0 = ref.Problem(c["shape"], c["spacing"], c["origin"], c["velocity0"], c["nbl"],
                              c["order"], c["order"], c["src"], c["rec"], 0.0, c["tn"], c["dt"], c["f0"])
            phi, grad, _ = rp0.fwi_gradient(obs)
            out[f"{name}.phi"] = np.array(phi)
            out[f"{name}.grad"] = grad
        print(name, "nt", fwd["nt"], "max|rec|", np.abs(fwd["rec"]).max())
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
