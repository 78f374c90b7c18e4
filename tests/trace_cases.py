"""Trace CSV fixtures for load_trace / save_trace_csv parity (trace.cpp:56-145): the edge
cases the reference's loader distinguishes (line endings, empty lines, trailing commas,
from_chars corner cases, int truncation, class column checks, error precedence)."""
H3 = b"arrival_ms,prompt_tokens,output_tokens"
H4 = b"arrival_ms,prompt_tokens,output_tokens,class"


def _rows(*r):
    return b"\n".join(r) + b"\n"


# (name, bytes, class_threshold)
CASES = [
    ("valid3_lf", _rows(H3, b"0,10,5", b"5,2000,3", b"5,1024,1"), 1024),
    ("valid4_crlf", H4 + b"\r\n0,10,5,SM\r\n7,2000,3,L\r\n9,1024,2,SM\r\n", 1024),
    ("no_trailing_newline", H3 + b"\n0,10,5\n3,11,6", 1024),
    ("no_trailing_newline_cr", H3 + b"\n0,10,5\n3,11,6\r", 1024),
    ("empty_lines", H3 + b"\n\n0,10,5\n\r\n\n4,12,7\n\n\n", 1024),
    ("trailing_comma", _rows(H3, b"0,10,5,", b"1,11,6,"), 1024),
    ("trailing_comma_4col", _rows(H4, b"0,10,5,SM,"), 1024),
    ("leading_zeros", _rows(H3, b"0007,00010,0005", b"00000000000000000000008,1,1"), 1024),
    ("int_truncation_ok", _rows(H3, b"0,4294967297,5"), 1024),  # static_cast<int> -> 1
    ("int_truncation_neg", _rows(H3, b"0,4294967296,5"), 1024),  # -> 0: out of range
    ("max_i64", _rows(H3, b"9223372036854775807,1,1"), 1024),
    ("overflow_i64", _rows(H3, b"9223372036854775808,1,1"), 1024),
    ("min_i64", _rows(H3, b"-9223372036854775808,1,1"), 1024),
    ("neg_zero", _rows(H3, b"-0,1,1", b"0,2,2"), 1024),
    ("threshold_boundary", _rows(H4, b"0,100,5,SM", b"1,101,5,L"), 100),
    ("header_only", H3 + b"\n", 1024),
    ("header_only_no_nl", H4, 1024),
    ("empty_file", b"", 1024),
    ("newline_only", b"\n", 1024),
    ("bad_header_space", _rows(H3 + b" ", b"0,1,1"), 1024),
    ("bad_header_order", _rows(b"prompt_tokens,arrival_ms,output_tokens", b"0,1,1"), 1024),
    ("header_crlf_cr", H3 + b"\r\r\n0,1,1\n", 1024),
    ("cols_2", _rows(H3, b"0,10,5", b"1,2"), 1024),
    ("cols_5", _rows(H4, b"0,10,5,SM,x"), 1024),
    ("cols_comma_only", _rows(H3, b","), 1024),
    ("cr_only_line", H3 + b"\n\r\r\n0,1,1\n", 1024),
    ("bad_arrival_alpha", _rows(H3, b"abc,1,1"), 1024),
    ("bad_arrival_plus", _rows(H3, b"+5,1,1"), 1024),
    ("bad_arrival_space", _rows(H3, b" 5,1,1"), 1024),
    ("bad_arrival_trailing_space", _rows(H3, b"5 ,1,1"), 1024),
    ("bad_arrival_empty", _rows(H3, b",1,1"), 1024),
    ("bad_arrival_minus", _rows(H3, b"-,1,1"), 1024),
    ("bad_prompt_float", _rows(H3, b"0,1.5,1"), 1024),
    ("bad_output_hex", _rows(H3, b"0,1,0x1"), 1024),
    ("range_arrival", _rows(H3, b"-1,1,1"), 1024),
    ("range_prompt", _rows(H3, b"0,0,1"), 1024),
    ("range_output", _rows(H3, b"0,1,-3"), 1024),
    ("non_monotone", _rows(H3, b"5,1,1", b"6,1,1", b"4,1,1"), 1024),
    ("bad_class", _rows(H4, b"0,1,1,S"), 1024),
    ("bad_class_lower", _rows(H4, b"0,1,1,sm"), 1024),
    ("class_mismatch", _rows(H4, b"0,2000,1,SM"), 1024),
    ("class_mismatch_l", _rows(H4, b"0,20,1,L"), 1024),
    ("first_error_wins", _rows(H4, b"0,1,1,SM", b"1,1,1,X", b"2,1,1,SM", b"abc,1,1,SM"), 1024),
    ("monotone_before_class", _rows(H4, b"5,1,1,SM", b"4,1,1,X"), 1024),
    ("range_before_monotone", _rows(H3, b"5,1,1", b"4,0,1"), 1024),
    ("columns_before_fields", _rows(H3, b"x,y"), 1024),
    ("long_field", _rows(H3, b"0,1,1", b"1," + b"9" * 3000 + b",1"), 1024),
    ("long_header", b"x" * 2000 + b"\n0,1,1\n", 1024),
    ("nul_byte", _rows(H3, b"0,1\x00,1"), 1024),
]


def tile_straddle_case(n_rows: int = 3000, crlf: bool = False) -> bytes:
    """> 4 KB so lines straddle the GPU's 4 KB tiles; a few long and empty lines."""
    out = [H4]
    for i in range(n_rows):
        p = 1 + (i * 7919) % 3000
        c = b"SM" if p <= 1024 else b"L"
        if i % 997 == 5:
            out.append(b"")
        if i % 1499 == 7:
            out.append(b"%d,%s,%d,%s" % (i * 3, b"0" * 400 + str(p).encode(), 1 + i % 9, c))
        else:
            out.append(b"%d,%d,%d,%s" % (i * 3, p, 1 + i % 9, c))
    sep = b"\r\n" if crlf else b"\n"
    return sep.join(out) + sep
