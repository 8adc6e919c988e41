"""Text-format cases for tests/test_textio.py: a tiny valid problem (n = m = 2)
and mutations of it covering every error path of io.hpp / validate()."""

BASE = """2 2
2 2 3
0 0 4
0 1 1
1 1 2
1
1
2 2 3
0 0 1
0 1 1
1 1 1
1
0
2
inf
"""


def _lines(text):
    return text.split("\n")


def _set(text, i, new):
    ls = _lines(text)
    ls[i] = new
    return "\n".join(ls)


TEXTIO_CASES = {
    "ok_base": BASE,
    "ok_one_line": " ".join(BASE.split()),
    "ok_crlf": BASE.replace("\n", "\r\n"),
    "ok_tabs_and_blank_lines": BASE.replace(" ", "\t").replace("\n", "\n\n"),
    "ok_hex_value": _set(BASE, 2, "0 0 0x1p+2"),
    "ok_value_prefix": _set(BASE, 2, "0 0 4abc"),
    "ok_neg_inf_lower": _set(BASE, 11, "-inf"),
    "ok_infinity_spelled": _set(BASE, 14, "Infinity"),
    "ok_plus_sign_index": _set(BASE, 2, "+0 0 4"),
    "ok_trailing_tokens": BASE + "5 6 7\n",
    "ok_two_entries_per_line": BASE.replace("0 0 4\n0 1 1\n", "0 0 4 0 1 1\n"),
    "err_empty": "",
    "err_truncated": "\n".join(_lines(BASE)[:14]) + "\n",
    "err_negative_index": _set(BASE, 2, "-1 0 4"),
    "err_alpha_index": _set(BASE, 2, "x 0 4"),
    "err_index_glued": _set(BASE, 2, "0 0x 4"),
    "err_alpha_value": _set(BASE, 2, "0 0 abc"),
    "err_subnormal_value": _set(BASE, 2, "0 0 1e-320"),
    "err_subnormal_f32": _set(BASE, 2, "0 0 1e-40"),  # (valid as double)
    "err_overflow_value": _set(BASE, 2, "0 0 1e400"),
    "err_overflow_f32": _set(BASE, 2, "0 0 1e39"),  # (valid as double)
    "err_unsorted": BASE.replace("0 0 4\n0 1 1\n", "0 1 1\n0 0 4\n"),
    "err_duplicate": BASE.replace("0 1 1\n1 1 2\n", "0 1 1\n0 1 2\n"),
    "err_col_out_of_bounds": _set(BASE, 3, "0 5 1"),
    "err_row_out_of_bounds": _set(BASE, 4, "7 1 2"),
    "err_header_n": _set(BASE, 0, "3 2"),
    "err_header_m": _set(BASE, 0, "2 1"),
    "err_below_diagonal": BASE.replace("1 1 2\n1\n1\n", "1 0 1\n1 1 2\n1\n1\n").replace(
        "2 2 3\n0 0 4", "2 2 4\n0 0 4", 1),
    "err_p_not_square": _set(BASE, 1, "2 3 3"),
    "err_a_cols": _set(BASE, 7, "2 3 3"),
    "err_nan_bound": _set(BASE, 11, "nan"),
    "err_l_gt_u": _set(BASE, 11, "3"),
    "err_l_plus_inf": _set(BASE, 11, "inf"),
    "err_u_minus_inf": _set(BASE, 14, "-inf"),
    "err_inf_in_a": _set(BASE, 8, "0 0 inf"),
    "err_nan_in_p": _set(BASE, 2, "0 0 nan"),
    "err_inf_in_q": _set(BASE, 5, "-inf"),
    "err_zero_vars": "0 0\n0 0 0\n0 0 0\n",
}
