"""Writes hand_2x2.json: Eq.3 expanded by hand for a 2x2 case.

Q = K = I_2, V = [[1,2],[3,4]], d_k = 2 so every score is a = 1/sqrt(2) on the
diagonal and 0 off it.  With p = e^a / (e^a + 1):
  row 0 weights (p, 1-p)  -> O_0 = p*(1,2) + (1-p)*(3,4) = (3-2p, 4-2p)
  row 1 weights (1-p, p)  -> O_1 = (1+2p, 2+2p)
  LSE_q = log(e^a + e^0)
  causal: row 0 sees key 0 only -> (1,2); row 1 unchanged.
Uses only the math module (no oracle, no CUDA path)."""
import json
import math
import os

a = 1 / math.sqrt(2)
p = math.exp(a) / (math.exp(a) + 1)
g = {
    "cite": "PAPER.md P:L186-189 Eq.3; P:L227-242 Listing 1 (mask True = -inf)",
    "Q": [[1, 0], [0, 1]], "K": [[1, 0], [0, 1]], "V": [[1, 2], [3, 4]],
    "O": [[3 - 2 * p, 4 - 2 * p], [1 + 2 * p, 2 + 2 * p]],
    "LSE": [math.log(math.exp(a) + 1)] * 2,
    "O_causal": [[1, 2], [1 + 2 * p, 2 + 2 * p]],
}
json.dump(g, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "hand_2x2.json"), "w"), indent=1)
