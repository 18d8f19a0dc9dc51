"""FD known answers from the reference's own unit tests
(/root/reference/proj/tests/test_table.cpp:166-227), restated as data."""
import paper_2403_05821_b200 as po


def known_fd_cases():
    """(name, check(api)) pairs; `api` has validate_fds / discover_fds."""
    T = po.Table

    def validate_witness(api):
        t = T([b"title", b"info", b"review"], [[b"m1", b"i1", b"ra"], [b"m1", b"i1", b"rb"],
                                               [b"m2", b"i2", b"rc"]])
        assert api.validate_fds(t, [[b"title", b"info"]]).all_satisfied()
        bad = T([b"k", b"v"], [[b"k1", b"v1"], [b"k1", b"v2"]])
        rep = api.validate_fds(bad, [[b"k", b"v"]])
        assert not rep.all_satisfied()
        w = rep.groups[0].witness
        assert w is not None and (w.row_a, w.row_b) == (0, 1)
        assert (w.agree_field, w.differ_field) == (b"k", b"v")
        assert api.validate_fds(bad, []).all_satisfied()

    def validate_errors(api):
        t = T([b"a", b"b"], [[b"1", b"2"]])
        for groups in ([[b"a", b"zzz"]], [[b"a", b"b"], [b"b"]]):
            try:
                api.validate_fds(t, groups)
            except po.SchemaError:
                continue
            raise AssertionError(f"no schema_error for {groups}")

    def discover(api):
        copies = T([b"A", b"B", b"C"], [[b"x", b"x", b"1"], [b"y", b"y", b"2"], [b"x", b"x", b"3"]])
        assert api.discover_fds(copies, 100).groups == [[b"A", b"B"]]
        id_const = T([b"id", b"k"], [[b"1", b"c"], [b"2", b"c"], [b"3", b"c"]])
        assert api.discover_fds(id_const, 100).groups == []
        one = T([b"a", b"b", b"c"], [[b"1", b"2", b"3"]])
        assert api.discover_fds(one, 100).groups == [[b"a", b"b", b"c"]]

    def oversized(api):
        t = T([b"a"], [[b"1"], [b"2"], [b"3"]])
        try:
            api.discover_fds(t, 2)
        except po.SizeError:
            return
        raise AssertionError("no size_error")

    return [("validate_witness", validate_witness), ("validate_errors", validate_errors),
            ("discover", discover), ("oversized", oversized)]
