"""The four bundled network descriptions of the reference (proj/nets/*.net),
in the canonical grammar that format_network_spec (netspec.cpp:133-151)
emits -- the GPU box has no /root/reference, so the bench and tests load
them from here.  Any .net file parses with voxin.parse_network_spec."""

NETS = {
    "n337": (
        "input 1\n"
        "conv 80 2 relu\n"
        "pool 2\n"
        "conv 80 3 relu\n"
        "pool 2\n"
        "conv 80 3 relu\n"
        "pool 2\n"
        "conv 80 3 relu\n"
        "conv 80 3 relu\n"
        "conv 80 3 relu\n"
        "conv 3 3 relu\n"
    ),
    "n537": (
        "input 1\n"
        "conv 80 4 relu\n"
        "pool 2\n"
        "conv 80 5 relu\n"
        "pool 2\n"
        "conv 80 5 relu\n"
        "pool 2\n"
        "conv 80 5 relu\n"
        "conv 80 5 relu\n"
        "conv 80 5 relu\n"
        "conv 3 5 relu\n"
    ),
    "n726": (
        "input 1\n"
        "conv 80 6 relu\n"
        "pool 2\n"
        "conv 80 7 relu\n"
        "pool 2\n"
        "conv 80 7 relu\n"
        "conv 80 7 relu\n"
        "conv 80 7 relu\n"
        "conv 80 7 relu\n"
    ),
    "n926": (
        "input 1\n"
        "conv 80 8 relu\n"
        "pool 2\n"
        "conv 80 9 relu\n"
        "pool 2\n"
        "conv 80 9 relu\n"
        "conv 80 9 relu\n"
        "conv 80 9 relu\n"
        "conv 80 9 relu\n"
    ),
}

# field of view of each (cost.cpp:107-122; cli_test.cpp:137-159 pins 85/163/117/155)
FOV = {"n337": 85, "n537": 163, "n726": 117, "n926": 155}
