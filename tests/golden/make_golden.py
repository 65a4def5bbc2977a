"""Writes tests/golden/reference_known_answers.json.

The reference (/root/reference/proj, C++20 + Eigen) cannot be compiled in
this image (Eigen3 and vendor/ are absent), so its golden
vectors are the known answers its own test suite asserts.  Each entry below
is transcribed from the cited test line; nothing here is computed by this
repository's code.  Re-run to regenerate the JSON:

    python tests/golden/make_golden.py
"""
import json
import os

I = "proj/tests/"
CASES = {
    "fft_delta": {
        "cite": I + "test_fft.cpp:8-16",
        "dims": [8], "input_re": [1, 0, 0, 0, 0, 0, 0, 0],
        "want_re": [1] * 8, "want_im": [0] * 8, "tol": 1e-12,
    },
    "fft_ones": {
        "cite": I + "test_fft.cpp:18-24",
        "dims": [4], "input_re": [1, 1, 1, 1],
        "want_re": [4, 0, 0, 0], "want_im": [0, 0, 0, 0], "tol": 1e-12,
    },
    "identity_spectrum": {
        "cite": I + "test_spectral.cpp:29-36",
        "dims": [4, 6], "fields": 1, "offsets": [[0, 0]], "values": [1.0],
        "want_all": [1.0, 0.0], "tol": 1e-12,
    },
    "appendix_generator": {
        "cite": I + "test_spectral.cpp:38-46 (generator [1,-2,0,3], Lambda[0] = 2)",
        "dims": [4], "fields": 1, "offsets": [[-1], [0], [1]], "values": [-2.0, 1.0, 3.0],
        "want_lambda0": [2.0, 0.0], "tol": 1e-12,
    },
    "shift_spectrum": {
        "cite": I + "test_spectral.cpp:48-57 (fixes the sign convention)",
        "dims": [4], "fields": 1, "offsets": [[1]], "values": [1.0],
        "want_re": [1, 0, -1, 0], "want_im": [0, 1, 0, -1], "tol": 1e-12,
    },
    "pow_scalar": {
        "cite": I + "test_spectral.cpp:99-113",
        "lambda": [[2.0, 0.0], [0.0, 1.0]],
        "checks": [
            {"T": 10, "index": 0, "want": [1024.0, 0.0], "tol": 1e-9},
            {"T": 4, "index": 1, "want": [1.0, 0.0], "tol": 1e-12},
            {"T": 0, "index": 0, "want": [1.0, 0.0], "tol": 0.0},
            {"T": 0, "index": 1, "want": [1.0, 0.0], "tol": 0.0},
        ],
    },
    "pinv": {
        "cite": I + "test_spectral.cpp:149-174",
        "lambda": [[2.0, 0.0], [0.0, 0.0], [0.0, -1.0]],
        "want": [[0.5, 0.0], [0.0, 0.0], [0.0, 1.0]], "tol": 1e-15,
    },
    "appendix_matrix": {
        "cite": I + "acceptance.cpp:168-188 (dense step matrix, exact)",
        "dims": [4], "fields": 1, "offsets": [[-1], [0], [1]], "values": [-2.0, 1.0, 3.0],
        "want": [[1, 3, 0, -2], [-2, 1, 3, 0], [0, -2, 1, 3], [3, 0, -2, 1]], "tol": 0.0,
    },
    "appendix_one_step": {
        "cite": I + "test_periodic.cpp:39-46 and acceptance.cpp:177-183",
        "dims": [4], "fields": 1, "offsets": [[-1], [0], [1]], "values": [-2.0, 1.0, 3.0],
        "a0": [1, 2, 3, 4], "T": 1, "want": [-1, 9, 11, 1], "tol": 1e-12,
    },
    "blowup_numeric_error": {
        "cite": I + "test_periodic.cpp:230-239 (k={+1:1e8, 0:1e8}, T=2^20 -> NumericError)",
        "dims": [16], "fields": 1, "offsets": [[0], [1]], "values": [1e8, 1e8],
        "T": 1048576, "seed": 101, "raises": "NumericError",
    },
    "vector_rejects_scalar": {
        "cite": I + "test_periodic.cpp:241-246",
        "dims": [8], "fields": 1, "offsets": [[0]], "values": [1.0], "T": 1, "raises": "SpecError",
    },
    "splitmix_seed7": {
        "cite": I + "test_io_cli.cpp:157-163 and proj/src/problem.cpp:222-247",
        "seed": 7, "n": 16, "formula": "2*((splitmix64(state)>>11)*2^-53)-1",
    },
    "cli_verify_heat1d": {
        "cite": I + "data/verify_heat1d.json + proj/src/runner.cpp:87-88 (pass iff max_abs <= 1e-8*(1+max|oracle|))",
        "dims": [256], "fields": 1, "offsets": [[-1], [0], [1]], "values": [0.125, 0.75, 0.125],
        "builtin": "heat1d (proj/src/stencils.cpp:9-24, alpha = 0.125)",
        "T": 100, "seed": 42, "tol_rel1p": 1e-8,
    },
    "cli_solve_delta": {
        "cite": I + "data/solve_delta.json (heat1d, delta init, T=500)",
        "dims": [64], "fields": 1, "offsets": [[-1], [0], [1]], "values": [0.125, 0.75, 0.125],
        "T": 500, "init": "delta", "tol_rel1p": 1e-8,
    },
}

if __name__ == "__main__":
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_known_answers.json")
    with open(path, "w") as f:
        json.dump(CASES, f, indent=1, sort_keys=True)
    print("wrote", path)
