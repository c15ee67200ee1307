"""Writes the "emu_fp16" section of tests/golden/softplus_hand_example.json: the hand-worked
softplus network under the tensor path's fp16 rounding points (R26, oracle step O8),
evaluated step by step in the order below with Python's math module and numpy's float64 ->
float16 conversion (round to nearest, ties to even).  It does NOT call oracle/ or the CUDA
path: it is the hand derivation written out, so the oracle's EMU_FP16 softplus mode can be
checked against it (tests/test_oracle_pins.py::test_softplus_emu_hand_worked).

The network is the hand-worked one of the same file with the output weight 4 replaced by
W7 = 1.313 (h6 . W7 stays f64, so any W7 is admissible): with the exact network's
dyadic output weight every delta e_l lands back on an fp16 grid point and a wrong sigma'
recovery would not show in the gradient.  W7 = 1.313 was picked (a scan of 1.000..1.999 in
steps of 0.001 finds four such values) so that each mutation listed
in MUTANTS changes f or the gradient (checked below; their values are stored with the golden).

Rounding points (R26): weights W2..W6 and W1 in the final backward GEMM rounded to fp16
(all of this network's weights are fp16-exact: 1, 1/2, -1, 2); the activations h1..h5 rounded
where they are the A operands of layers 2..6; the backward deltas e6..e1 rounded; layer 1's
forward, the biases and h6 . w7 unrounded; sigma' of layers 1..5 recovered from the rounded
activation as 1 - e^-h~, sigma' of layer 6 = sigmoid(z6) from the unrounded pre-activation.
"""
import json
import math
from pathlib import Path

import numpy as np

GOLD = Path(__file__).resolve().parent.parent / "tests" / "golden" / "softplus_hand_example.json"


def r16(x):
    return float(np.float16(x))


def sp(z):
    return math.log1p(math.exp(z)) if z < 30 else z + math.log1p(math.exp(-z))


W7 = 1.313
MUTANTS = {
    "M1 sigma'6 recovered from the rounded h6 (1 - e^-fp16(h6)) instead of sigmoid(z6)": "M1",
    "M2 sigma'1..5 = sigmoid(z) of the unrounded pre-activation instead of 1 - e^-h~": "M2",
    "M3 sigma'1..5 = 1 - e^-h from the unrounded activation": "M3",
    "M4 backward deltas e_l not rounded": "M4",
    "M5 h6 rounded before the output layer": "M5",
    "M6 forward activations h1..h5 not rounded": "M6",
}


def evaluate(mut=None, steps=None):
    log = steps.append if steps is not None else (lambda s: None)
    ln2, ln3 = math.log(2.0), math.log(3.0)
    b = [0.0, math.log(1.5), 0.0, -ln3, ln2 - ln3, math.log(27.0 / 16.0)]
    w = [None, 1.0, 0.5, 1.0, -1.0, 2.0]   # W2..W6 (fp16-exact)
    rh = (lambda x: x) if mut == "M6" else r16
    re = (lambda x: x) if mut == "M4" else r16
    z = [0.0] * 6
    h = [0.0] * 6
    ht = [0.0] * 6
    z[0] = 0.0                      # z1 = p'_x + theta / 2 = 0 for both cases (layer 1 unrounded)
    h[0] = sp(z[0])
    ht[0] = rh(h[0])
    log(f"z1 = 0, h1 = ln 2 = {h[0]!r}, h1~ = fp16(h1) = {ht[0]!r}")
    for l in range(1, 5):
        z[l] = w[l] * ht[l - 1] + b[l]
        h[l] = sp(z[l])
        ht[l] = rh(h[l])
        log(f"z{l + 1} = {w[l]} h{l}~ + b{l + 1} = {z[l]!r}, h{l + 1} = softplus = {h[l]!r}, h{l + 1}~ = {ht[l]!r}")
    z[5] = w[5] * ht[4] + b[5]
    h[5] = sp(z[5])
    log(f"z6 = 2 h5~ + ln(27/16) = {z[5]!r}, h6 = softplus = {h[5]!r} (not rounded)")
    f = W7 * (r16(h[5]) if mut == "M5" else h[5]) + 1.0
    log(f"f = 1.313 h6 + 1 = {f!r}")
    sig6 = -math.expm1(-r16(h[5])) if mut == "M1" else 1.0 / (1.0 + math.exp(-z[5]))
    e = re(W7 * sig6)
    log(f"sigma'6 = sigmoid(z6) = {sig6!r}; e6 = fp16(1.313 sigma'6) = {e!r}")
    gcur = w[5] * e
    for l in range(4, -1, -1):      # layers 5..1: sigma' = 1 - e^-h~, e = fp16(g sigma')
        if mut == "M2":
            sig = 1.0 / (1.0 + math.exp(-z[l]))
        elif mut == "M3":
            sig = -math.expm1(-h[l])
        else:
            sig = -math.expm1(-ht[l])
        e = re(gcur * sig)
        log(f"g{l + 1} = {gcur!r}; sigma'{l + 1} = 1 - e^-h{l + 1}~ = {sig!r}; e{l + 1} = fp16(g{l + 1} sigma'{l + 1}) = {e!r}")
        gcur = (w[l] if l > 0 else 1.0) * e
    grad = [-e, 0.0, 0.5 * e, 0, 0, 0, 0, 0, 0]
    log(f"dF/dp'_x = W1[0] e1 = {e!r}, dF/dtheta = W1[5] e1 = {0.5 * e!r}; "
        "grad_q f = [-dF/dp'_x, 0, dF/dtheta, 0 x 6]")
    return f, grad


def main():
    g = json.loads(GOLD.read_text())
    steps = []
    f, grad = evaluate(None, steps)
    mutants = {}
    for name, m in MUTANTS.items():
        fm, gm = evaluate(m)
        assert (fm, gm) != (f, grad), name   # the pin must see every mutation
        mutants[name] = {"f": fm, "grad0": gm[0]}
    layers = [dict(x) for x in g["layers"]]
    layers[6] = {"W": [[W7]], "b": [1]}
    g["emu_fp16"] = {"_what": "the hand-worked network with W7 = 1.313 under the oracle's EMU_FP16 mode (R26 "
                              "rounding points); written by tools/golden_softplus_emu.py (math + numpy float16, "
                              "no oracle).  Both cases of this file give z1 = 0, hence the same values.",
                     "_derivation": steps, "layers": layers, "f": f, "grad": grad,
                     "_mutants": mutants}
    GOLD.write_text(json.dumps(g, indent=1) + "\n")
    print("\n".join(steps))
    for k, v in mutants.items():
        print(k, v)


if __name__ == "__main__":
    main()
