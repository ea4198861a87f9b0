"""ctypes front end of integration/_build/libcvm_refshim.so: the reference side
of the boundary (the reference's own alu / Machine compiled from
/root/reference in the build container; the built library travels to the GPU
box).  Used by tests/, bench.py and smoke() to obtain recorded circuits for
the B200 library and to run the reference API end to end on the GPU.

    record_fu("add", 16)              -> paper_2101_03403_b200.Dag
    record_program(insns, n_mem, 16)  -> Dag (outputs: registers, then NZCV)
    add_batch_gpu(ctx, ks, a, b, 16)  -> sums, carries, stats  (reference API)
    run_program_gpu(ctx, ks, insns, mem, 16) -> regs, nzcv, stats, branch queries
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libcvm_refshim.so")

FU_OPS = ["add", "add_cin", "sub", "addsub", "cmp", "and", "orr", "eor", "orn", "lsl",
          "lsr", "asr", "umul", "smul", "udiv", "udiv_exact", "mul_lo"]


class RefDag(ctypes.Structure):
    _fields_ = [("nodes", ctypes.c_void_p), ("n_nodes", ctypes.c_uint64),
                ("outputs", ctypes.POINTER(ctypes.c_uint64)), ("n_outputs", ctypes.c_uint64),
                ("n_inputs", ctypes.c_uint64), ("regions", ctypes.POINTER(ctypes.c_char_p)),
                ("n_regions", ctypes.c_uint64)]


class RefInsn(ctypes.Structure):
    _fields_ = [("op", ctypes.c_char * 8), ("cond", ctypes.c_char * 4),
                ("rd", ctypes.c_int32), ("rn", ctypes.c_int32), ("rm", ctypes.c_int32),
                ("sets_flags", ctypes.c_int32), ("has_imm", ctypes.c_int32),
                ("has_imm2", ctypes.c_int32), ("has_target", ctypes.c_int32),
                ("target", ctypes.c_uint32), ("imm", ctypes.c_uint64), ("imm2", ctypes.c_uint64)]


_LIB = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: build it with `make -C integration` "
                               "(needs the reference tree, build container only)")
        import paper_2101_03403_b200  # noqa: F401  (libcvm_b200.so first, same process)
        L = ctypes.CDLL(LIB_PATH)
        p, u64, u32, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        L.cvmref_last_error.restype = ctypes.c_char_p
        L.cvmref_record_fu.argtypes = [ctypes.c_char_p, u32, ctypes.POINTER(RefDag)]
        L.cvmref_record_program.argtypes = [u32, u32, u64, p, u64, ctypes.POINTER(RefDag)]
        L.cvmref_dag_free.argtypes = [ctypes.POINTER(RefDag)]
        L.cvmref_dag_free.restype = None
        L.cvmref_sim_fu_batch.argtypes = [ctypes.c_char_p, u32, u64, p, p, p, p,
                                          ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_uint64)]
        L.cvmref_sim_program.argtypes = [u32, u32, p, u64, p, u64, u64, p, p]
        L.cvmref_add_batch_gpu.argtypes = [p, p, u32, u64, p, p, p, p, p]
        L.cvmref_run_program_gpu.argtypes = [p, p, u32, u32, p, u64, p, u64, u64, p, p, p, p]
        for f in ("cvmref_record_fu", "cvmref_record_program", "cvmref_add_batch_gpu",
                  "cvmref_sim_fu_batch", "cvmref_sim_program",
                  "cvmref_run_program_gpu"):
            getattr(L, f).restype = i
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        import paper_2101_03403_b200._native as N
        msg = (lib().cvmref_last_error() or b"").decode(errors="replace")
        raise {-1: N.CvmInputError, -2: N.CvmDeviceError}.get(rc, N.CvmError)(msg)


def _to_dag(d, name):
    import paper_2101_03403_b200 as P
    nodes = np.frombuffer(ctypes.string_at(d.nodes, d.n_nodes * P.DAG_DTYPE.itemsize),
                          dtype=P.DAG_DTYPE).copy()
    outs = np.ctypeslib.as_array(d.outputs, shape=(d.n_outputs,)).copy() \
        if d.n_outputs else np.zeros(0, np.uint64)
    regions = [d.regions[k].decode() for k in range(d.n_regions)]
    lib().cvmref_dag_free(ctypes.byref(d))
    return P.Dag(nodes, outs, name, regions)


def record_fu(op, width):
    """The functional unit as the reference's alu records it (inputs a, b[, c])."""
    d = RefDag()
    _check(lib().cvmref_record_fu(op.encode(), width, ctypes.byref(d)))
    return _to_dag(d, f"{op}{width}")


def _insns(program):
    """program: tuples (op, rd, rn, rm, imm, sets_flags[, imm2]) with -1 = absent
    (tests/golden/programs.json), or dicts with the RefInsn field names."""
    arr = (RefInsn * max(1, len(program)))()
    for x, ins in zip(arr, program):
        if isinstance(ins, dict):
            for k, v in ins.items():
                setattr(x, k, v.encode() if isinstance(v, str) else v)
            continue
        op, rd, rn, rm, imm, sf = ins[:6]
        x.op = op.encode()
        x.rd, x.rn, x.rm, x.sets_flags = rd, rn, rm, int(sf)
        if imm is not None and imm >= 0:
            x.has_imm, x.imm = 1, imm
        if len(ins) > 6 and ins[6] is not None and ins[6] >= 0:
            x.has_imm2, x.imm2 = 1, ins[6]
    return arr


def record_program(program, n_mem, word_size=16, register_count=8):
    d = RefDag()
    _check(lib().cvmref_record_program(word_size, register_count, n_mem, _insns(program),
                                       len(program), ctypes.byref(d)))
    return _to_dag(d, "program")


def sim_program(program, mem, word_size=16, register_count=8, max_steps=None):
    """The reference Machine on SimBackend: (final registers, NZCV)."""
    mem = np.ascontiguousarray(mem, np.uint64)
    regs = np.zeros(register_count, np.uint64)
    nzcv = np.zeros(4, np.uint8)
    steps = max_steps if max_steps is not None else 10 * len(program) + 1
    _check(lib().cvmref_sim_program(word_size, register_count, mem.ctypes.data, len(mem),
                                    _insns(program), len(program), steps, regs.ctypes.data,
                                    nzcv.ctypes.data))
    return regs, nzcv


def random_program(rng, width, count=16, n_mem=4, n_regs=8):
    """A seeded straight-line program over the whole data-path ISA (isa.hpp:
    MOV/LOAD/STORE, ADD(S)/SUB(S) with register or immediate operands,
    MUL/SMULS/UDIV, shifts by register or immediate, the bitwise ops, NOT,
    BFC/BFI/RBIT/REV, CMP) -- the shape of the reference's random-program
    cross-check (emulator_test.cc:486-640), generated here."""
    mask = (1 << width) - 1
    reg = lambda: int(rng.integers(n_regs))  # noqa: E731
    out = []
    for _ in range(count):
        k = int(rng.integers(16))
        x = dict(rd=-1, rn=-1, rm=-1)
        if k == 0:
            x.update(op="MOV", rd=reg(), has_imm=1, imm=int(rng.integers(mask + 1)))
        elif k == 1:
            x.update(op="LOAD", rd=reg(), has_imm=1, imm=int(rng.integers(n_mem)))
        elif k == 2:
            x.update(op="STORE", rn=reg(), has_imm=1, imm=int(rng.integers(n_mem)))
        elif k in (3, 4):
            x.update(op=["ADDS", "SUBS"][k - 3], rd=reg(), rn=reg(), sets_flags=1)
            if rng.integers(2):
                x.update(has_imm=1, imm=int(rng.integers(mask + 1)))
            else:
                x.update(rm=reg())
        elif k == 5:
            x.update(op=["MUL", "SMULS"][int(rng.integers(2))], rd=reg(), rn=reg(), rm=reg())
            x["sets_flags"] = int(x["op"] == "SMULS")
        elif k == 6:
            x.update(op="UDIV", rd=reg(), rn=reg(), rm=reg())
        elif k == 7:
            x.update(op=["LLS", "LRS", "ARS"][int(rng.integers(3))], rd=reg(), rn=reg())
            if rng.integers(2):
                x.update(has_imm=1, imm=int(rng.integers(width + 1)))
            else:
                x.update(rm=reg())
        elif k in (8, 9, 10, 11):
            x.update(op=["AND", "OR", "XOR", "ORN"][k - 8], rd=reg(), rn=reg(), rm=reg())
        elif k == 12:
            x.update(op="NOT", rd=reg(), rn=reg())
        elif k == 13:
            lsb = int(rng.integers(width))
            wd = 1 + int(rng.integers(width - lsb))
            x.update(op=["BFC", "BFI"][int(rng.integers(2))], rd=reg(), has_imm=1, imm=lsb,
                     has_imm2=1, imm2=wd)
            if x["op"] == "BFI":
                x["rn"] = reg()
        elif k == 14:
            x.update(op=["RBIT", "REV"][int(rng.integers(2))], rd=reg(), rn=reg())
        else:
            x.update(op="CMP", rn=reg(), rm=reg(), sets_flags=1)
        out.append(x)
    return out


def sim_fu_batch(op, width, a, b, c=None):
    """The reference SimBackend (cleartext) on `len(a)` instances of the unit:
    returns (results as ints, seconds, DAG nodes)."""
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    cc = np.ascontiguousarray(c if c is not None else np.zeros(len(a)), np.uint64)
    out = np.zeros(len(a), np.uint64)
    sec, nodes = ctypes.c_double(), ctypes.c_uint64()
    _check(lib().cvmref_sim_fu_batch(op.encode(), width, len(a), a.ctypes.data, b.ctypes.data,
                                     cc.ctypes.data, out.ctypes.data, ctypes.byref(sec),
                                     ctypes.byref(nodes)))
    return out, sec.value, nodes.value


def add_batch_gpu(ctx, ks, a, b, width=16):
    """batch x alu::add through the reference API on cryptovm::GpuBackend."""
    import paper_2101_03403_b200._native as N
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    sums = np.zeros(len(a), np.uint64)
    carries = np.zeros(len(a), np.uint8)
    st = N.BackendStats()
    _check(lib().cvmref_add_batch_gpu(ctx.handle, ks.handle, width, len(a), a.ctypes.data,
                                      b.ctypes.data, sums.ctypes.data, carries.ctypes.data,
                                      ctypes.byref(st)))
    return sums, carries, st.as_dict()


def run_program_gpu(ctx, ks, program, mem, word_size=16, register_count=8, max_steps=None):
    """The reference Machine on the B200 (branches via LocalBranchOracle)."""
    import paper_2101_03403_b200._native as N
    mem = np.ascontiguousarray(mem, np.uint64)
    regs = np.zeros(register_count, np.uint64)
    nzcv = np.zeros(4, np.uint8)
    st = N.BackendStats()
    bq = ctypes.c_uint64()
    steps = max_steps if max_steps is not None else 10 * len(program) + 1
    _check(lib().cvmref_run_program_gpu(ctx.handle, ks.handle, word_size, register_count,
                                        mem.ctypes.data, len(mem), _insns(program),
                                        len(program), steps, regs.ctypes.data,
                                        nzcv.ctypes.data, ctypes.byref(st), ctypes.byref(bq)))
    return regs, nzcv, st.as_dict(), bq.value
