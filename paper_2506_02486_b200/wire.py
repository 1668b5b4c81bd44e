"""Status vocabulary of the data plane (reference/pkg/src/diomp/wire.py:46-52).

The reference carries these codes in ACK / GET_RESP frames of its TCP/shm
transport; here they are the return values of libdiomp_b200.so
(include/diomp_b200.h: DIOMP_OK .. DIOMP_INTERNAL) and map to the same
exceptions.  The 40-byte frame codec (Opcode, WireMessage, encode/decode)
belongs to the reference's TCP transport, which NVLink loads/stores replace
(DESIGN.md section 7), so it is not provided.
"""

import enum


class Status(enum.IntEnum):
    OK = 0
    INVALID_ADDRESS = 1
    BAD_REQUEST = 2
    INTERNAL = 3
