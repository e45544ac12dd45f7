"""MPS texts exercising every rule of the reference reader
(proj/core/src/mps_reader.cpp) and of its tests (proj/tests/test_mps.cpp):
sections in either spelling, RANGES on E/G/L rows with both signs, OBJSENSE
MAX (header token and section line), objective RHS offset, secondary N rows,
MARKER lines, RHS/RANGES/BOUNDS with and without set names, every bound type,
comments, blank lines, CRLF, duplicate coefficients, zero coefficients, fixed
format, and the reference's error paths. Shared by tests/test_mps.py and
tests/golden/make_mps_golden.py."""

GOOD = {
    "basic": """NAME          BASIC
ROWS
 N  COST
 L  LIM1
 G  LIM2
 E  MYEQN
COLUMNS
    XONE      COST         1.0   LIM1         1.0
    XONE      LIM2         1.0
    YTWO      COST         2.0   LIM1         1.0
    YTWO      MYEQN       -1.0
    ZTHREE    COST        -1.0   MYEQN        1.0
RHS
    RHS       LIM1         4.0   LIM2         1.0
    RHS       MYEQN        7.0
BOUNDS
 UP BND       XONE         4.0
 LO BND       YTWO        -1.0
 UP BND       YTWO         1.0
ENDATA
""",
    "ranges_all": """NAME RANGED
ROWS
 N obj
 E e_pos
 E e_neg
 G g_r
 L l_r
 G plain
COLUMNS
 x obj 1 e_pos 1
 x e_neg 2 g_r 3
 y obj 2 l_r 1
 y plain 4 e_pos -1
 z obj -3 e_neg 1
 z g_r 1 l_r 2
RHS
 rhs e_pos 1 e_neg 2
 rhs g_r 3 l_r 4
 rhs plain 5
RANGES
 rng e_pos 2 e_neg -3
 rng g_r -4 l_r 5
BOUNDS
 UP bnd x 10
 UP bnd y 10
 UP bnd z 10
ENDATA
""",
    "objsense_header": """NAME MAXI
OBJSENSE MAX
ROWS
 N obj
 L c1
COLUMNS
 x obj 3 c1 1
 y obj 2 c1 1
RHS
 RHS c1 4
 RHS obj -7
BOUNDS
 UP B x 3
ENDATA
""",
    "objsense_section": """NAME MAXI2
OBJSENSE
    MAXIMIZE
ROWS
 N obj
 G c1
COLUMNS
 x obj 1 c1 1
RHS
 obj 2.5
 c1 1
ENDATA
""",
    "objsense_min": """NAME
OBJSENSE
 MIN
ROWS
 N obj
 G c1
COLUMNS
 x obj 1 c1 1
RHS
 RHS c1 1
ENDATA
""",
    "secondary_n_marker": """* comment line
NAME SEC
ROWS
 N obj
 N other
 E e1
COLUMNS
    MARKER                 'MARKER'                 'INTORG'
 x obj 1 other 5
 x e1 1
    MARKER                 'MARKER'                 'INTEND'
 y e1 1 other 7
RHS
 RHS e1 3 other 9
ENDATA
""",
    "bounds_all": """NAME BOUNDS
ROWS
 N obj
 G c
COLUMNS
 a obj 1 c 1
 b obj 1 c 1
 c obj 1 c 1
 d obj 1 c 1
 e obj 1 c 1
 f obj 1 c 1
 g obj 1 c 1
 h obj 1 c 1
 i obj 1 c 1
RHS
 c 1
BOUNDS
 LO BND a -2
 UP BND b 3
 FX BND c 1.5
 FR BND d
 MI BND e
 PL f
 BV BND g
 LI BND h 2
 UI i 7
 MI BND i
ENDATA
""",
    "crlf_blank_dupes": "NAME CRLF\r\nROWS\r\n N obj\r\n G c1\r\n\r\n E c2\r\n"
                        "COLUMNS\r\n x obj 1 c1 1\r\n x c1 2 c2 0\r\n y c2 1 obj 0.5\r\n x c2 3\r\n"
                        "RHS\r\n RHS c1 1 c2 2\r\nENDATA\r\n",
    "unsorted_columns": """NAME UNSORTED
ROWS
 N obj
 G r1
 G r2
COLUMNS
 b obj 1 r1 2
 a obj 1 r2 1
 b r2 3
 c r1 1
 a r1 -1
RHS
 RHS r1 1 r2 1
ENDATA
""",
    "numbers": """NAME NUMS
ROWS
 N obj
 G r
COLUMNS
 x obj +1.25 r 1e-3
 y obj -0.1 r 3.14159265358979323846
 z obj 1E+2 r .5
 w obj 0x1.8p1 r 1e-320
RHS
 RHS r 123456789012345678901234567890
ENDATA
""",
    "no_rhs_no_bounds": """NAME
ROWS
 N obj
 E r
COLUMNS
 x obj 1 r 1
ENDATA
""",
    "lowercase_sections": """name lower
rows
 n obj
 g r
columns
 x obj 1 r 1
rhs
 rhs r 2
bounds
 up bnd x 5
endata
""",
}

def fixed_line(*fields):
    """A data line with the fixed-format fields at their MPS columns
    (1-based 2-3, 5-12, 15-22, 25-36, 40-47, 50-61)."""
    starts = [1, 4, 14, 24, 39, 49]
    line = ""
    for st, f in zip(starts, fields):
        line = line.ljust(st) + f
    return line


FIXED = {
    # Names without blanks (the reference splits ROWS lines on whitespace even
    # in fixed mode), text past column 61 that only fixed mode ignores.
    "fixed_basic": "\n".join([
        "NAME          FIXED",
        "ROWS",
        fixed_line("N", "COST"),
        fixed_line("L", "LIM1"),
        fixed_line("G", "LIM2"),
        fixed_line("E", "MYEQN"),
        "COLUMNS",
        fixed_line("", "X1", "COST", "1.0", "LIM1", "1.0").ljust(61) + "  trailing junk",
        fixed_line("", "X1", "LIM2", "1.0"),
        fixed_line("", "Y2", "COST", "2.0", "LIM1", "1.0"),
        fixed_line("", "Y2", "MYEQN", "-1.0"),
        "RHS",
        fixed_line("", "RHS", "LIM1", "4.0", "LIM2", "1.0"),
        fixed_line("", "", "MYEQN", "7.0"),
        "RANGES",
        fixed_line("", "RNG", "LIM2", "2.5"),
        "BOUNDS",
        fixed_line("UP", "BND", "X1", "4.0"),
        fixed_line("MI", "BND", "Y2"),
        "ENDATA", ""]),
    # Blanks inside names: rejected by the reference's ROWS handling.
    "fixed_blank_names": "\n".join([
        "NAME",
        "ROWS",
        fixed_line("N", "COST"),
        fixed_line("L", "LIM 1"),
        "ENDATA", ""]),
}

BAD = {
    "unknown_section": "NAME x\nROWZ\n",
    "out_of_order": "NAME x\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nROWS\n",
    "data_outside": " x y\n",
    "dup_row": "NAME\nROWS\n N o\n G r\n L r\n",
    "bad_row_type": "NAME\nROWS\n N o\n Q r\n",
    "row_line_tokens": "NAME\nROWS\n N o extra\n",
    "unknown_row": "NAME\nROWS\n N o\nCOLUMNS\n x o 1 nope 2\n",
    "column_pairs": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r\n",
    "bad_number": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1.5x\n",
    "nan_value": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r nan\n",
    "rhs_malformed": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nRHS\n RHS r\n",
    "range_on_objective": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nRANGES\n RNG o 1\n",
    "bound_type": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nBOUNDS\n XX B x 1\n",
    "bound_malformed": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nBOUNDS\n UP\n",
    "bound_column": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nBOUNDS\n UP B y 1\n",
    "bound_conflict": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nBOUNDS\n LO B x 5\n UP B x 1\n",
    "missing_columns": "NAME\nROWS\n N o\n G r\n",
    "no_variables": "NAME\nROWS\n N o\nCOLUMNS\nENDATA\n",
    "objsense_bad": "NAME\nOBJSENSE\n SIDEWAYS\n",
    "dup_rows_section": "NAME\nROWS\n N o\nROWS\n",
    "infinite_cost": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o inf r 1\n",
    "empty_rhs_line": "NAME\nROWS\n N o\n G r\nCOLUMNS\n x o 1 r 1\nRHS\n RHS r 1 r\n",
}
